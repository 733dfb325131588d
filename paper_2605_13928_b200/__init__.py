"""B200-native (sm_100a) single-cell hot path: QC -> normalize -> log1p -> HVG -> scale -> PCA -> kNN.

Scanpy-shaped step functions (``pp``) over hand-written CUDA kernels behind a C ABI
(``include/scb.h``, ``libscb_b200.so``); see DESIGN.md.  No CPU fallback.
"""
from . import _lib  # noqa: F401
from .pp import (DeviceCSR, calculate_qc_metrics, filter_masks, subset, normalize_log1p,  # noqa: F401
                 highly_variable_genes, scale, regress_out_scale, Scaled, pca, neighbors, PCAResult)

qc_metrics = calculate_qc_metrics  # SURVEY.md §8(b2) name of the same step

__all__ = ["DeviceCSR", "calculate_qc_metrics", "qc_metrics", "filter_masks", "subset", "normalize_log1p",
           "highly_variable_genes", "scale", "regress_out_scale", "Scaled", "pca", "neighbors", "PCAResult"]
