"""Scanpy's float path for highly_variable_genes(flavor="seurat") -- TEST INFRASTRUCTURE.

A literal transcription of Scanpy's ``_highly_variable_genes_single_batch`` for
``flavor="seurat"`` (scanpy 1.9/1.10, ``scanpy/preprocessing/_highly_variable_genes.py``;
Scanpy is third-party and absent here):

    X = np.expm1(X_log)                       # float32 data of the log-normalised matrix
    mean, var = _get_mean_var(X)              # float64 accumulators, var with ddof = 1
    mean[mean == 0] = 1e-12
    dispersion = var / mean
    dispersion[dispersion == 0] = np.nan
    dispersion = np.log(dispersion); mean = np.log1p(mean)
    df["mean_bin"] = pd.cut(df["means"], bins=n_bins)
    disp_mean_bin / disp_std_bin = groupby(mean_bin).mean() / .std(ddof=1)
    one-gene bins: std := mean, mean := 0
    dispersions_norm = (disp - disp_mean_bin[bin]) / disp_std_bin[bin]
    cutoff = n_top_genes-th largest finite dispersions_norm;
    highly_variable = nan_to_num(dispersions_norm, nan=-inf) >= cutoff

``_get_mean_var`` for a sparse matrix is Scanpy's ``sparse_mean_variance_axis`` (numba,
float64): mean = sum(x)/N, var = (sum((x - mean)^2 over nonzeros) + (N - nnz) mean^2)/N,
then var *= N/(N-1).  This is the "float64, expm1-based" statistic the product's
fixed-point integer sums (oracle/pipeline.py, csrc/csr_kernels.cu) must agree with at the
level of the selected gene SET: tests compare the two selections.
"""
from __future__ import annotations

import numpy as np


def sparse_mean_var(indices, data32, n_rows: int, n_cols: int):
    """Scanpy's sparse mean / variance over rows (float64 accumulation, two-pass, ddof=1)."""
    x = np.asarray(data32).astype(np.float64)
    idx = np.asarray(indices)
    N = float(n_rows)
    mean = np.bincount(idx, weights=x, minlength=n_cols) / N
    nnz = np.bincount(idx, minlength=n_cols).astype(np.float64)
    dev = x - mean[idx]
    ss = np.bincount(idx, weights=dev * dev, minlength=n_cols) + (N - nnz) * mean * mean
    var = ss / N * (N / (N - 1.0))
    return mean, var


def seurat_from_mean_var(mean, var, n_top: int, n_bins: int = 20):
    """Returns (highly_variable bool[G], dispersions_norm f64[G]) exactly as Scanpy's pandas code."""
    import pandas as pd
    mean = np.array(mean, dtype=np.float64, copy=True)
    mean[mean == 0] = 1e-12
    disp = var / mean
    disp[disp == 0] = np.nan
    with np.errstate(divide="ignore", invalid="ignore"):
        disp = np.log(disp)
    mean = np.log1p(mean)
    df = pd.DataFrame({"means": mean, "dispersions": disp})
    df["mean_bin"] = pd.cut(df["means"], bins=n_bins)
    g = df.groupby("mean_bin", observed=False)["dispersions"]
    bmean, bstd = g.mean(), g.std(ddof=1)
    one = bstd.isnull()
    bstd[one.values] = bmean[one.values].values
    bmean[one.values] = 0
    dn = (df["dispersions"].values - bmean[df["mean_bin"]].values) / bstd[df["mean_bin"]].values
    finite = dn[~np.isnan(dn)]
    n = min(n_top, finite.size)
    if n == 0:
        return np.zeros(len(dn), bool), dn
    cut = np.sort(finite)[::-1][n - 1]
    return np.nan_to_num(dn, nan=-np.inf) >= cut, dn


def hvg_seurat_expm1(indices, log_data32, n_rows: int, n_cols: int, n_top: int, n_bins: int = 20):
    """Scanpy's seurat HVG on a log1p-normalised CSR (its data array and column indices)."""
    x = np.expm1(np.asarray(log_data32, dtype=np.float32))  # float32, as Scanpy's X.expm1()
    mean, var = sparse_mean_var(indices, x, n_rows, n_cols)
    return seurat_from_mean_var(mean, var, n_top, n_bins)
