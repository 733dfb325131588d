"""Row-chunked, multi-process driver of the CPU oracle for full-size matrices (C3: 1M x 25k,
1.75e9 nonzeros) -- TEST INFRASTRUCTURE (imported only by tests/ and tools/).

Runs exactly the arithmetic of ``oracle/pipeline.py`` stage by stage on contiguous row chunks
(each chunk a sub-CSR handed to the same functions), in worker processes forked from the
caller (the CSR is inherited copy-on-write, results come back pickled):

* QC metrics per chunk; per-gene integer counts / float64 sums of integer counts add
  exactly across chunks.
* filter masks on the combined metrics (``pipeline.filter_masks``).
* subset + normalize_total + log1p per chunk (row factors are per row, so chunking is exact);
  the HVG fixed-point sums are 128-bit integers per gene, combined with carries, so the
  statistics and the selected set are those of the unchunked oracle bit for bit.
* scale: fixed-point sums of the kept log values over the HVG columns (same), then
  ``mean_var``; the dense z-scores of each chunk (float32, ``clip_z``) feed a float64 Gram
  ``Z^T Z`` and column sums, combined by summation (fp64 rounding order differs from the
  unchunked oracle only at the 1e-16 level, far below the 1e-3 subspace-angle tolerance).
* PCA: ``eigh`` of the combined covariance, sign-canonical components, and the projection of
  every chunk.
* kNN of a query subset against all keys with ``pipeline.knn`` (float64 brute force), query
  blocks spread over the workers.
"""
from __future__ import annotations

import multiprocessing as mp
import os
from typing import Optional

import numpy as np

from . import pipeline as op

_G = {}  # inherited by forked workers


def _pool(workers):
    return mp.get_context("fork").Pool(workers)


def _limit_blas():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:  # pragma: no cover
        pass


def _sub(r0, r1):
    ip, ix, d, G = _G["indptr"], _G["indices"], _G["data"], _G["n_cols"]
    a, b = int(ip[r0]), int(ip[r1])
    return op.CSR((ip[r0:r1 + 1] - a).astype(np.int64), ix[a:b], d[a:b], G)


def _add128(a, b):
    lo = a[0] + b[0]
    carry = (lo < a[0]).astype(np.uint64)
    return lo, a[1] + b[1] + carry


# ----------------------------------------------------------------------------- workers
def _w_qc(rng):
    _limit_blas()
    return rng, op.qc_metrics(_sub(*rng), _G["mt"])


def _w_norm(rng):
    """HVG fixed-point limbs of y = float32(x * scale) over the kept rows/genes of this chunk."""
    _limit_blas()
    r0, r1 = rng
    X = _sub(r0, r1)
    cm = _G["cell_mask"][r0:r1]
    Xs = op.subset(X, cm, _G["gene_mask"])
    Xl, y32, s = op.normalize_log1p(Xs, _G["target_sum"])
    v = y32.astype(np.float64)
    q1 = np.rint(v * 2.0 ** op.FX1).astype(np.uint64)
    q2 = np.rint((v * v) * 2.0 ** op.FX2).astype(np.uint64)
    return rng, op._fx_sum(Xs.indices, q1, Xs.n_cols), op._fx_sum(Xs.indices, q2, Xs.n_cols)


def _chunk_log(r0, r1):
    X = _sub(r0, r1)
    Xs = op.subset(X, _G["cell_mask"][r0:r1], _G["gene_mask"])
    Xl, _, _ = op.normalize_log1p(Xs, _G["target_sum"])
    return Xl


def _w_scale_sums(rng):
    _limit_blas()
    Xl = _chunk_log(*rng)
    slot = _G["slot"]
    j = slot[Xl.indices]
    k = j >= 0
    v = Xl.data[k].astype(np.float64)
    q1 = np.rint(v * 2.0 ** op.FX1).astype(np.uint64)
    q2 = np.rint((v * v) * 2.0 ** op.FX2).astype(np.uint64)
    H = _G["H"]
    return rng, op._fx_sum(j[k], q1, H), op._fx_sum(j[k], q2, H)


def _dense_z(r0, r1):
    Xl = _chunk_log(r0, r1)
    H, slot, mean, inv = _G["H"], _G["slot"], _G["mean"], _G["inv"]
    Z = np.empty((Xl.n_rows, H), dtype=np.float32)
    Z[:] = op.clip_z((0.0 - mean) * inv, _G["max_value"], _G["clip"]).astype(np.float32)[None, :]
    rows = Xl.row_ids()
    j = slot[Xl.indices]
    k = j >= 0
    Z[rows[k], j[k]] = op.clip_z((Xl.data[k].astype(np.float64) - mean[j[k]]) * inv[j[k]], _G["max_value"],
                                 _G["clip"]).astype(np.float32)
    return Z


def _w_gram(rng):
    _limit_blas()
    Z = _dense_z(*rng).astype(np.float64)
    return rng, Z.T @ Z, Z.sum(0), Z.shape[0]


def _w_project(rng):
    _limit_blas()
    Z = _dense_z(*rng).astype(np.float64)
    return rng, ((Z - _G["m"]) @ _G["V"]).astype(np.float32)


def _w_knn(qblock):
    _limit_blas()
    return qblock[0], op.knn(_G["E"], _G["k"], queries=qblock, block=64)


# ----------------------------------------------------------------------------- driver
def _chunks(n, rows):
    return [(a, min(n, a + rows)) for a in range(0, n, rows)]


def run(indptr, indices, data, n_cols: int, mt_mask, p: op.Params, workers: Optional[int] = None,
        chunk_rows: int = 32768, knn_queries=None, with_pca: bool = True):
    """Oracle stage outputs for the full matrix.  ``knn_queries``: kept-row indices whose exact
    neighbours (among all kept rows) are computed.  Returns a dict like ``pipeline.run``'s
    (``qc``, ``cell_mask``, ``gene_mask``, ``hvg_mask``, ``hvg_stats``, ``scale_mean``,
    ``scale_inv_std``, ``components``, ``variance``, ``variance_ratio``, ``X_pca``, ``knn_idx``)."""
    workers = workers or max(1, min(32, len(os.sched_getaffinity(0))))
    N = len(indptr) - 1
    _G.update(indptr=indptr, indices=indices, data=data, n_cols=n_cols, mt=np.asarray(mt_mask),
              target_sum=p.target_sum, max_value=p.max_value, clip=p.clip)
    out = {}
    ch = _chunks(N, chunk_rows)
    with _pool(workers) as pool:
        res = sorted(pool.map(_w_qc, ch), key=lambda t: t[0])
    qc = {}
    for key in ("n_genes_by_counts", "total_counts", "total_counts_mt", "pct_counts_mt"):
        qc[key] = np.concatenate([r[1][key] for r in res])
    qc["n_cells_by_counts"] = np.sum([r[1]["n_cells_by_counts"].astype(np.int64) for r in res], 0).astype(np.int32)
    qc["gene_total_counts"] = np.sum([r[1]["gene_total_counts"] for r in res], 0)
    out["qc"] = qc
    cm, gm = op.filter_masks(qc, p)
    out["cell_mask"], out["gene_mask"] = cm, gm
    _G.update(cell_mask=cm, gene_mask=gm)
    with _pool(workers) as pool:
        res = sorted(pool.map(_w_norm, ch), key=lambda t: t[0])
    a1 = res[0][1]
    a2 = res[0][2]
    for r in res[1:]:
        a1 = _add128(a1, r[1])
        a2 = _add128(a2, r[2])
    s1 = op.fx_to_double(*a1) * 2.0 ** -op.FX1
    s2 = op.fx_to_double(*a2) * 2.0 ** -op.FX2
    n_kept = int(cm.astype(bool).sum())
    out["n_kept"] = n_kept
    out["hvg_sums"] = (s1, s2)
    hvg, st = op.hvg_seurat_from_sums(s1, s2, n_kept, p.n_top_genes, p.n_bins, p.hvg_ties)
    out["hvg_mask"], out["hvg_stats"] = hvg, st
    hv = np.nonzero(hvg)[0]
    H = len(hv)
    slot = np.full(int(gm.astype(bool).sum()), -1, dtype=np.int64)
    slot[hv] = np.arange(H)
    _G.update(slot=slot, H=H)
    kept_rows = np.nonzero(cm.astype(bool))[0]
    ch_k = _chunks(N, chunk_rows)  # chunks over the ORIGINAL rows; each yields its kept rows in order
    with _pool(workers) as pool:
        res = sorted(pool.map(_w_scale_sums, ch_k), key=lambda t: t[0])
    b1, b2 = res[0][1], res[0][2]
    for r in res[1:]:
        b1 = _add128(b1, r[1])
        b2 = _add128(b2, r[2])
    t1 = op.fx_to_double(*b1) * 2.0 ** -op.FX1
    t2 = op.fx_to_double(*b2) * 2.0 ** -op.FX2
    mean, var = op.mean_var(t1, t2, float(n_kept))
    with np.errstate(invalid="ignore"):
        std = np.sqrt(var)
    std = np.where((std == 0) | np.isnan(std), 1.0, std)
    inv = 1.0 / std
    out["scale_mean"], out["scale_inv_std"] = mean, inv
    _G.update(mean=mean, inv=inv)
    if not with_pca:
        return out
    with _pool(workers) as pool:
        res = pool.map(_w_gram, ch_k)
    ZtZ = np.sum([r[1] for r in res], 0)
    colsum = np.sum([r[2] for r in res], 0)
    assert sum(r[3] for r in res) == n_kept == len(kept_rows)
    m = colsum / n_kept
    C = (ZtZ - n_kept * np.outer(m, m)) / (n_kept - 1.0)
    w, V = np.linalg.eigh(C)
    order = np.argsort(w)[::-1][:p.n_comps]
    lam = w[order]
    V = op.sign_canonical(V[:, order])
    out.update(components=V, variance=lam, variance_ratio=lam / np.trace(C), col_mean=m)
    _G.update(m=m, V=V)
    with _pool(workers) as pool:
        res = sorted(pool.map(_w_project, ch_k), key=lambda t: t[0])
    E = np.concatenate([r[1] for r in res])
    out["X_pca"] = E
    if knn_queries is not None:
        q = np.asarray(knn_queries)
        _G.update(E=E, k=p.n_neighbors)
        blocks = [q[i:i + 64] for i in range(0, len(q), 64)]
        with _pool(workers) as pool:
            res = pool.map(_w_knn, blocks)
        out["knn_idx"] = np.concatenate([r[1][0] for r in res])
        out["knn_dist"] = np.concatenate([r[1][1] for r in res])
        out["knn_queries"] = q
    _G.clear()
    return out


def knn_queries(E, k: int, queries, workers: Optional[int] = None, block: int = 64):
    """Exact kNN (pipeline.knn, float64 brute force) of ``queries`` against all rows of E, query
    blocks spread over forked workers.  Returns (idx, dist)."""
    workers = workers or max(1, min(32, len(os.sched_getaffinity(0))))
    q = np.asarray(queries)
    _G.update(E=E, k=k)
    blocks = [q[i:i + block] for i in range(0, len(q), block)]
    with _pool(workers) as pool:
        res = pool.map(_w_knn, blocks)
    _G.clear()
    return np.concatenate([r[1][0] for r in res]), np.concatenate([r[1][1] for r in res])
