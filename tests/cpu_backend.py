"""TEST-ONLY stand-in for paper_2605_13928_b200.pp on CPU tensors, built from the oracle.

It mirrors the device functions' interfaces and partial-result semantics (integer fixed-point
gene-sum limbs, partial Gram, per-shard kNN against all-gathered keys) so that the multi-rank
orchestration in paper_2605_13928_b200.pipeline can be exercised with gloo on CPU.  It is never
used by the product (the product raises when the CUDA library is missing)."""
import numpy as np
import torch

from oracle import pipeline as op
from paper_2605_13928_b200 import pp as real_pp

DeviceCSR = real_pp.DeviceCSR
Scaled = real_pp.Scaled
PCAResult = real_pp.PCAResult
gene_slots = real_pp.gene_slots
padded_width = real_pp.padded_width


def _np(t):
    return t.detach().cpu().numpy()


def _csr(X):
    return op.CSR(_np(X.indptr), _np(X.indices), _np(X.data), X.n_cols)


def calculate_qc_metrics(X, mt_mask, row_splits=False, defer_check=False):
    q = op.qc_metrics(_csr(X), _np(mt_mask))
    out = {k: torch.as_tensor(v) for k, v in q.items()}
    out["hvg_row_splits"] = None
    return out


def filter_masks(qc, gene=None, *, min_genes=200, max_genes=None, max_pct_mt=20.0, min_cells=3):
    p = op.Params(min_genes=min_genes, max_genes=max_genes, max_pct_mt=max_pct_mt, min_cells=min_cells)
    cm, gm = op.filter_masks({k: _np(v) for k, v in qc.items() if v is not None}, p)
    return torch.as_tensor(cm), torch.as_tensor(gm), (int(cm.sum()), int(gm.sum()))


def filter_masks_ex(qc, gene=None, *, min_genes=200, max_genes=None, max_pct_mt=20.0, min_cells=3, indptr=None):
    cm, gm, kept = filter_masks(qc, min_genes=min_genes, max_genes=max_genes, max_pct_mt=max_pct_mt,
                                min_cells=min_cells)
    nnz = 0
    if indptr is not None:
        ip = _np(indptr)
        nnz = int(np.diff(ip)[_np(cm).astype(bool)].sum())
    return cm, gm, kept, nnz


def subset_rows_all_genes(X, cm, total_counts, n_kept, target_sum=1e4):
    gm = torch.ones(X.n_cols, dtype=torch.uint8)
    remap, new_indptr, row_scale, rso, _ = subset_count_scale(X, cm, gm, (n_kept, X.n_cols), target_sum)
    return remap, new_indptr, row_scale, rso


def subset_normalize(X, cm, gm, n_kept, target_sum=1e4):
    S = op.subset(_csr(X), _np(cm), _np(gm))
    Xl, y32, s = op.normalize_log1p(S, target_sum)
    remap = np.full(X.n_cols, -1, np.int32)
    remap[_np(gm).astype(bool)] = np.arange(int(_np(gm).sum()), dtype=np.int32)
    rso = np.zeros(X.n_rows, np.float32)
    rso[_np(cm).astype(bool)] = s
    out = DeviceCSR(torch.as_tensor(Xl.indptr), torch.as_tensor(Xl.indices), torch.as_tensor(Xl.data), Xl.n_cols,
                    row_scale=torch.as_tensor(s))
    return out, torch.as_tensor(remap), torch.as_tensor(rso)


def subset_count_scale(X, cm, gm, n_kept, target_sum=1e4):
    """First pass (CPU stand-in): returns (remap, new_indptr, row_scale, row_scale_orig, nnz); the
    second pass below recomputes the kept matrix from the same inputs."""
    Xl, remap, rso = subset_normalize(X, cm, gm, n_kept, target_sum)
    _PASS[id(X)] = Xl
    return remap, Xl.indptr, Xl.row_scale, rso, int(Xl.nnz)


_PASS = {}


def subset_fill_log(X, cm, remap, new_indptr, row_scale, nnz, n_genes_kept):
    return _PASS.pop(id(X))


def subset_fill_log_scale_sums(X, cm, remap, new_indptr, row_scale, nnz, n_genes_kept, slot, H, sums=None, all_kept=False):
    Xl = subset_fill_log(X, cm, remap, new_indptr, row_scale, nnz, n_genes_kept)
    return Xl, scale_gene_sums(Xl, slot, H)


def _limbs(idx, v32, n, f1, f2):
    v64 = v32.astype(np.float64)
    out = np.zeros((2, 2, n), dtype=np.int64)
    for st, q in enumerate((np.rint(v64 * 2.0 ** f1), np.rint(v64 * v64 * 2.0 ** f2))):
        q = q.astype(np.uint64)
        lo = np.bincount(idx, weights=(q & np.uint64(0xFFFFFFFF)).astype(np.float64), minlength=n)
        hi = np.bincount(idx, weights=(q >> np.uint64(32)).astype(np.float64), minlength=n)
        out[st, 0], out[st, 1] = lo.astype(np.int64), hi.astype(np.int64)
    return torch.as_tensor(out)


def _limb_values(sums, f1, f2):
    s = _np(sums).astype(np.uint64)
    vals = []
    for st, f in ((0, f1), (1, f2)):
        l0, l1 = s[st, 0], s[st, 1]
        lo = l0 + (l1 << np.uint64(32))
        hi = (l1 >> np.uint64(32)) + (lo < l0).astype(np.uint64)
        vals.append(op.fx_to_double(lo, hi) * 2.0 ** -f)
    return vals


def hvg_gene_sums(X, counts=None, row_scale=None, gene_remap=None, n_out=None, sums=None, row_splits=None):
    A = _csr(X)
    rows = A.row_ids()
    s = _np(row_scale)[rows]
    g = _np(gene_remap)[A.indices] if gene_remap is not None else A.indices
    keep = (s != 0) & (g >= 0)
    y32 = (_np(counts)[keep] * s[keep]).astype(np.float32)
    return _limbs(g[keep], y32, n_out, op.FX1, op.FX2)


def hvg_select(sums, n_cells, n_top_genes, n_bins=20, ties="cutoff"):
    s1, s2 = _limb_values(sums, op.FX1, op.FX2)
    mask, st = op.hvg_seurat_from_sums(s1, s2, n_cells, n_top_genes, n_bins, ties)
    idx = np.nonzero(mask)[0].astype(np.int32)
    st = {k: torch.as_tensor(v) for k, v in st.items()}
    st["n_selected"] = len(idx)
    return torch.as_tensor(mask), torch.as_tensor(idx), st


def scale_gene_sums(X_log, slot, H, sums=None):
    A = _csr(X_log)
    j = _np(slot)[A.indices]
    keep = j >= 0
    return _limbs(j[keep], A.data[keep], H, op.FX1, op.FX2)


def scale_finalize(sums, n_cells):
    s1, s2 = _limb_values(sums, op.FX1, op.FX2)
    mean, var = op.mean_var(s1, s2, float(n_cells))
    with np.errstate(invalid="ignore"):
        std = np.sqrt(var)
    std = np.where((std == 0) | np.isnan(std), 1.0, std)
    return torch.as_tensor(mean), torch.as_tensor(1.0 / std)


def scale_dense(X_log, slot, H, mean, inv, max_value=10.0, out=None, clip="symmetric", planes=False):  # noqa: ARG001
    A = _csr(X_log)
    ld = padded_width(H)
    m, iv = _np(mean), _np(inv)
    Z = np.zeros((A.n_rows, ld), np.float32)
    Z[:, :H] = op.clip_z((0.0 - m) * iv, max_value, clip).astype(np.float32)[None, :]
    Z[:, H] = 1.0
    rows = A.row_ids()
    j = _np(slot)[A.indices]
    k = j >= 0
    Z[rows[k], j[k]] = op.clip_z((A.data[k].astype(np.float64) - m[j[k]]) * iv[j[k]], max_value,
                                 clip).astype(np.float32)
    return Scaled(torch.as_tensor(Z), H, H, mean, inv)


def regress_cov_sums(qc, cell_mask):
    k = _np(cell_mask).astype(bool)
    return torch.as_tensor(op.regress_cov_sums(_np(qc["total_counts"])[k], _np(qc["pct_counts_mt"])[k]))


def regress_design(qc, cell_mask, sums6, n_kept):
    k = _np(cell_mask).astype(bool)
    a1, a2, _ = op.regress_design(_np(qc["total_counts"])[k], _np(qc["pct_counts_mt"])[k], _np(sums6))
    assert len(a1) == n_kept
    return torch.as_tensor(np.stack([a1, a2]))


def regress_dense_log(X_log, slot, H):
    return scale_dense(X_log, slot, H, torch.zeros(H, dtype=torch.float64), torch.ones(H, dtype=torch.float64),
                       float("inf"), clip="upper")


def regress_xty(L, design, xty=None):
    Lh = _np(L.Z)[:, :L.H].astype(np.float64)
    a = _np(design)
    v = np.stack([Lh.sum(0), a[0] @ Lh, a[1] @ Lh, (Lh * Lh).sum(0)])
    return torch.as_tensor(v) if xty is None else xty + torch.as_tensor(v)


def regress_finalize(xty, sums6):
    S0, S1, S2, Q = _np(xty)
    s6 = _np(sums6)
    n = s6[0]
    m1, m2 = s6[1] / n, s6[3] / n
    v1, v2 = max(s6[2] / n - m1 * m1, 0.0), max(s6[4] / n - m2 * m2, 0.0)
    s1, s2 = (np.sqrt(v1) if v1 > 0 else 1.0), (np.sqrt(v2) if v2 > 0 else 1.0)
    c = (s6[5] - n * m1 * m2) / (s1 * s2)
    b0 = S0 / n
    det = n * n - c * c
    b1, b2 = ((n * S1 - c * S2) / det, (n * S2 - c * S1) / det) if det > 1e-12 * n * n else (S1 / n, 0 * S1)
    var = (Q - (b0 * S0 + b1 * S1 + b2 * S2)) / (n - 1.0)
    std = np.sqrt(np.where(var > 0, var, 0.0))
    std = np.where(std == 0, 1.0, std)
    return torch.as_tensor(np.stack([b0, b1, b2])), torch.as_tensor(1.0 / std)


def regress_apply(L, design, beta, inv, max_value=10.0, clip="symmetric"):
    Z = _np(L.Z).copy()
    a, b, iv = _np(design), _np(beta), _np(inv)
    fit = b[0][None, :] + a[0][:, None] * b[1][None, :] + a[1][:, None] * b[2][None, :]
    Z[:, :L.H] = op.clip_z((Z[:, :L.H].astype(np.float64) - fit) * iv[None, :], max_value, clip).astype(np.float32)
    return Scaled(torch.as_tensor(Z), L.H, L.ones_col, torch.zeros(L.H, dtype=torch.float64), inv)


def gram(sc, out=None, planes=True):  # noqa: ARG001 (no BF16 planes on the CPU)
    Z = _np(sc.Z).astype(np.float64)
    return torch.as_tensor(Z.T @ Z)


def pca_from_gram(sc, C, n_cells, n_comps=50):
    C = _np(C)
    H, ld = sc.H, sc.ld
    m = C[sc.ones_col, :H] / n_cells
    cov = (C[:H, :H] - n_cells * np.outer(m, m)) / (n_cells - 1.0)
    w, V = np.linalg.eigh(cov)
    o = np.argsort(w)[::-1][:n_comps]
    V = op.sign_canonical(V[:, o])
    npad = 64 if n_comps <= 64 else 128
    comp_t = np.zeros((npad, ld), np.float32)
    comp_t[:n_comps, :H] = V.T
    mean = np.zeros(ld, np.float32)
    mean[:H] = m
    return (torch.as_tensor(w[o]), torch.as_tensor(comp_t), torch.as_tensor(mean),
            torch.as_tensor([np.trace(cov)]))


def project(sc, comp_t, mean, n_comps, ld_out=64):
    Z = _np(sc.Z).astype(np.float64)
    V = _np(comp_t).astype(np.float64)[:n_comps].T
    X = np.zeros((Z.shape[0], max(ld_out, comp_t.shape[0])), np.float32)
    X[:, :n_comps] = ((Z - _np(mean).astype(np.float64)) @ V).astype(np.float32)
    return torch.as_tensor(X)


def neighbors(X_pca, n_neighbors=15, n_comps=None, keys=None, timer=None):
    keys = X_pca if keys is None else keys
    d = n_comps or X_pca.shape[1]
    Q = _np(X_pca)[:, :d].astype(np.float64)
    K = _np(keys)[:, :d].astype(np.float64)
    d2 = ((Q[:, None, :] - K[None, :, :]) ** 2).sum(-1)
    idx = np.empty((len(Q), n_neighbors), np.int32)
    dist = np.empty((len(Q), n_neighbors), np.float32)
    cand = np.arange(len(K))
    for r in range(len(Q)):
        o = np.lexsort((cand, d2[r]))[:n_neighbors]
        idx[r] = o
        dist[r] = np.sqrt(d2[r][o])
    return torch.as_tensor(idx), torch.as_tensor(dist)
