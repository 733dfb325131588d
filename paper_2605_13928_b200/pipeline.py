"""Fused QC -> normalize -> log1p -> HVG -> scale -> PCA -> kNN pipeline (one call per step).

This is what the paper's pipeline script runs between its CudaMon markers
(reference PAPER.md:44-52 cm_timestamp; marker labels ``qc, norm_hvg, regress, pca, knn``
as in the reference fixtures pkg/tests/helpers.py:31-36).  Each step is a short sequence of
C-ABI calls on one CUDA stream; per-step device time comes from CUDA events (the
reference's 1 ms marker resolution and zero-length-step drop, trace.py:270-274, cannot
resolve B200 stage times), and an optional ``mark(label)`` callback -- e.g. a gputrace
``SamplerHandle.mark`` or ``paper_2605_13928_b200.trace`` handle -- is invoked at each
step boundary so NVML samples are attributed to steps exactly as in the reference.

Multi-GPU: cells (rows) are sharded across ranks; the only collectives are the
all-reduces of per-gene integer sums / gene counts and of the partial Gram matrix, a
broadcast of the eigenvectors, and the all-gather of the embedding for kNN
(SURVEY.md §8(e)).  ``comm`` is any object with the small interface of ``dist.Comm``.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Optional

import torch

from . import pp

STEPS = ("qc", "norm_hvg", "regress", "pca", "knn")


@dataclasses.dataclass(frozen=True)
class Params:
    min_genes: int = 200
    max_genes: Optional[int] = None
    max_pct_mt: float = 20.0
    min_cells: int = 3
    target_sum: float = 1e4
    n_top_genes: int = 2000
    n_bins: int = 20
    hvg_ties: str = "cutoff"  # Scanpy's ">= n-th largest" rule; "rank" = exactly n_top_genes
    max_value: float = 10.0
    clip: str = "symmetric"  # [-max_value, max_value] (Scanpy >= 1.10, rapids-singlecell); "upper" = Scanpy <= 1.9
    n_comps: int = 50
    n_neighbors: int = 15
    regress_out: bool = False  # sc.pp.regress_out(["total_counts", "pct_counts_mt"]) before scale
    connectivities: bool = False  # also sc.pp.neighbors' distances/connectivities (umap fuzzy graph)
    umap: bool = False  # also sc.tl.umap (layout from X_pca[:, :2]; implies connectivities)
    cluster: bool = False  # also community detection on connectivities (sc.tl.leiden / sc.tl.louvain)
    cluster_method: str = "leiden"
    resolution: float = 1.0
    rank_genes: bool = False  # also sc.tl.rank_genes_groups(t-test vs rest) over the clusters
    umap_epochs: Optional[int] = None


@dataclasses.dataclass
class Result:
    qc: dict
    cell_mask: torch.Tensor
    gene_mask: torch.Tensor
    X_log: pp.DeviceCSR
    hvg_mask: torch.Tensor
    hvg_index: torch.Tensor
    hvg_stats: dict
    scaled: pp.Scaled
    pca: pp.PCAResult
    knn_index: torch.Tensor
    knn_dist: torch.Tensor
    n_cells_total: int
    step_ms: dict
    graph: Optional[pp.NeighborsGraph] = None
    umap: Optional[torch.Tensor] = None
    clusters: Optional[torch.Tensor] = None
    modularity: Optional[float] = None
    rank_genes: Optional[dict] = None


class _Timer:
    def __init__(self, enabled: bool, mark: Optional[Callable[[str], None]]):
        self.enabled = enabled
        self.mark = mark
        self.events = []

    def step(self, label: str):
        if self.mark is not None:
            if self.enabled:
                torch.cuda.current_stream().synchronize()  # align host markers with device work
            self.mark(label)
        if self.enabled:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.events.append((label, ev))

    def finish(self):
        if not self.enabled:
            return {}
        end = torch.cuda.Event(enable_timing=True)
        end.record()
        end.synchronize()
        out = {}
        evs = self.events + [("end", end)]
        for (lab, a), (_, b) in zip(evs[:-1], evs[1:]):
            out[lab] = a.elapsed_time(b)
        return out


def run(X: pp.DeviceCSR, mt_mask: torch.Tensor, params: Params = Params(), *, comm=None,
        mark: Optional[Callable[[str], None]] = None, timing: bool = True, with_knn: bool = True,
        knn_timer=None, qc: Optional[dict] = None) -> Result:
    """Run the whole hot path on the device-resident count matrix ``X`` (this rank's rows).
    ``qc``: QC metrics already computed while the matrix was uploaded (``ingest.upload_qc``)."""
    p = params
    tm = _Timer(timing, mark)
    dev = X.device

    # ------------------------------------------------------------------ qc
    tm.step("qc")
    if qc is None:
        qc = pp.calculate_qc_metrics(X, mt_mask, row_splits=True, defer_check=True)
    if comm is not None:
        comm.allreduce_(qc["n_cells_by_counts"])
        comm.allreduce_(qc["gene_total_counts"])
    # one host round trip: kept counts, kept-row nonzeros and QC's deferred data check
    cm, gm, (nk_local, gk), kept_nnz = pp.filter_masks_ex(qc, min_genes=p.min_genes, max_genes=p.max_genes,
                                                          max_pct_mt=p.max_pct_mt, min_cells=p.min_cells,
                                                          indptr=X.indptr)
    n_total = nk_local if comm is None else comm.allreduce_int(nk_local)

    # ------------------------------------------------------------------ norm_hvg
    tm.step("norm_hvg")
    # subset + normalize: pass 1 (kept counts, row factors); the HVG statistics come straight
    # from the raw matrix (remapped genes, per-original-row factors); pass 2 writes the kept
    # log1p matrix and, for the plain scale path, accumulates the scale step's gene sums of
    # the selected HVG columns on the way (no second read of the kept matrix)
    if gk == X.n_cols:  # every gene kept: row factors from QC's totals, no count pass (no host sync)
        remap, new_indptr, row_scale, row_scale_orig = pp.subset_rows_all_genes(X, cm, qc["total_counts"], nk_local,
                                                                                p.target_sum)
        nnz = kept_nnz
    else:
        remap, new_indptr, row_scale, row_scale_orig, nnz = pp.subset_count_scale(X, cm, gm, (nk_local, gk),
                                                                                 p.target_sum)
    sums = pp.hvg_gene_sums(X, counts=X.data, row_scale=row_scale_orig, gene_remap=remap, n_out=gk,
                            row_splits=qc["hvg_row_splits"])
    if comm is not None:
        comm.allreduce_(sums)
    hvg_mask, hvg_index, st = pp.hvg_select(sums, n_total, p.n_top_genes, p.n_bins, p.hvg_ties)
    H = int(hvg_index.numel())
    slot = pp.gene_slots(hvg_index, gk)
    ssum = None
    if p.regress_out:
        X_log = pp.subset_fill_log(X, cm, remap, new_indptr, row_scale, nnz, gk)
    else:
        X_log, ssum = pp.subset_fill_log_scale_sums(X, cm, remap, new_indptr, row_scale, nnz, gk, slot, H,
                                                    all_kept=(nk_local == X.n_rows and gk == X.n_cols))

    # ------------------------------------------------------------------ regress (scale)
    tm.step("regress")
    if p.regress_out:
        s6 = pp.regress_cov_sums(qc, cm)
        if comm is not None:
            comm.allreduce_(s6)
        design = pp.regress_design(qc, cm, s6, nk_local)
        sc = pp.regress_dense_log(X_log, slot, H)
        xty = pp.regress_xty(sc, design)
        if comm is not None:
            comm.allreduce_(xty)
        beta, inv = pp.regress_finalize(xty, s6)
        sc = pp.regress_apply(sc, design, beta, inv, p.max_value, p.clip)
    else:
        if ssum is None:
            ssum = pp.scale_gene_sums(X_log, slot, H)
        if comm is not None:
            comm.allreduce_(ssum)
        mean, inv = pp.scale_finalize(ssum, n_total)
        # written directly as the Gram's / projection's BF16 planes (no float32 matrix, no split pass)
        sc = pp.scale_dense(X_log, slot, H, mean, inv, p.max_value, clip=p.clip, planes=True)

    # ------------------------------------------------------------------ pca
    tm.step("pca")
    C = pp.gram(sc)
    if comm is not None:
        comm.allreduce_(C)
    npad = 64 if p.n_comps <= 64 else 128
    if comm is None or comm.rank == 0:
        lam, comp_t, cmean, tr = pp.pca_from_gram(sc, C, n_total, p.n_comps)
    else:
        lam = torch.empty(p.n_comps, dtype=torch.float64, device=dev)
        comp_t = torch.empty((npad, sc.ld), dtype=torch.float32, device=dev)
        cmean = torch.empty(sc.ld, dtype=torch.float32, device=dev)
        tr = torch.empty(1, dtype=torch.float64, device=dev)
    if comm is not None:
        for t in (lam, comp_t, cmean, tr):
            comm.broadcast_(t, 0)
    Xp = pp.project(sc, comp_t, cmean, p.n_comps)
    res_pca = pp.PCAResult(Xp, comp_t[: p.n_comps, :H], lam, lam / tr, cmean, p.n_comps)

    # ------------------------------------------------------------------ knn
    tm.step("knn")
    if with_knn:
        keys = Xp if comm is None else comm.allgather_rows(Xp)
        ki, kd = pp.neighbors(Xp, p.n_neighbors, n_comps=p.n_comps, keys=keys, timer=knn_timer)
    else:
        ki = kd = None
    graph = emb = labels = None
    q = None
    n_c = 0
    if with_knn and (p.connectivities or p.umap or p.cluster):
        tm.step("graph")
        graph = pp.neighbors_graph(ki, kd, comm=comm)
    if with_knn and p.umap:
        if comm is not None:
            raise NotImplementedError("umap layout is single-GPU (the layout SGD needs the whole graph)")
        tm.step("umap")
        emb = pp.umap_layout(graph.connectivities, Xp[:, :2], n_epochs=p.umap_epochs)
    if with_knn and p.cluster:
        if comm is not None:
            raise NotImplementedError("clustering is single-GPU (it contracts the whole graph)")
        tm.step("cluster")
        fn = pp.leiden if p.cluster_method == "leiden" else pp.louvain
        labels, n_c, q = fn(graph.connectivities, resolution=p.resolution)
    de = None
    if with_knn and p.cluster and p.rank_genes and n_c >= 2:
        tm.step("rank_genes")
        de = pp.rank_genes_groups(X_log, labels, n_c)
    ms = tm.finish()
    return Result(qc, cm, gm, X_log, hvg_mask, hvg_index, st, sc, res_pca, ki, kd, n_total, ms, graph, emb, labels, q,
                  de)
