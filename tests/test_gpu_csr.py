"""GPU parity of the CSR stages (QC, masks, subset, normalize+log1p, HVG, scale) vs the oracle."""
import functools

import numpy as np
import pytest

from oracle.synth import SynthSpec, generate_csr, mt_mask
from tests.gpu_fixtures import C1, c1_inputs, c1_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev_state():
    import torch
    import paper_2605_13928_b200 as scb
    from paper_2605_13928_b200 import pp
    X, mt = c1_inputs()
    p = C1["params"]
    Xd = scb.DeviceCSR.from_host(X.indptr, X.indices, X.data, X.n_cols)
    qc = scb.calculate_qc_metrics(Xd, torch.as_tensor(mt))
    cm, gm, kept = scb.filter_masks(qc, min_genes=p.min_genes, max_genes=p.max_genes, max_pct_mt=p.max_pct_mt, min_cells=p.min_cells)
    Xs = scb.subset(Xd, cm, gm, kept)
    Xl = scb.normalize_log1p(Xs, p.target_sum)
    hvg_mask, hvg_index, st = scb.highly_variable_genes(Xl, p.n_top_genes, p.n_bins)
    sc = scb.scale(Xl, hvg_index, p.max_value)
    torch.cuda.synchronize()
    return dict(qc=qc, cm=cm, gm=gm, Xs=Xs, Xl=Xl, hvg=hvg_mask, hvg_index=hvg_index, st=st, sc=sc)


def test_qc_bit_exact(dev_state):
    o = c1_oracle(False)["qc"]
    qc = dev_state["qc"]
    for k in ["n_genes_by_counts", "total_counts", "total_counts_mt", "n_cells_by_counts", "gene_total_counts"]:
        np.testing.assert_array_equal(qc[k].cpu().numpy(), o[k], err_msg=k)
    np.testing.assert_array_equal(qc["pct_counts_mt"].cpu().numpy(), o["pct_counts_mt"])


def test_masks_bit_exact(dev_state):
    o = c1_oracle(False)
    np.testing.assert_array_equal(dev_state["cm"].cpu().numpy(), o["cell_mask"])
    np.testing.assert_array_equal(dev_state["gm"].cpu().numpy(), o["gene_mask"])


def test_subset_bit_exact(dev_state):
    o = c1_oracle(False)["X_sub"]
    ip, ix, d, g = dev_state["Xs"].to_host()
    assert g == o.n_cols
    np.testing.assert_array_equal(ip, o.indptr)
    np.testing.assert_array_equal(ix, o.indices)
    np.testing.assert_array_equal(d, o.data)


def test_normalize_log1p(dev_state):
    o = c1_oracle(False)
    Xl = dev_state["Xl"]
    np.testing.assert_array_equal(Xl.row_scale.cpu().numpy(), o["row_scale"])
    got = Xl.data.cpu().numpy()
    ref = o["X_log"].data
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=0)


def test_hvg_set_bit_exact(dev_state):
    o = c1_oracle(False)
    np.testing.assert_array_equal(dev_state["hvg"].cpu().numpy(), o["hvg_mask"])
    st, ost = dev_state["st"], o["hvg_stats"]
    np.testing.assert_array_equal(st["means"].cpu().numpy(), ost["means"])
    np.testing.assert_array_equal(st["variances"].cpu().numpy(), ost["variances"])
    np.testing.assert_array_equal(st["mean_bin"].cpu().numpy(), ost["mean_bin"])
    np.testing.assert_allclose(st["dispersions_norm"].cpu().numpy(), ost["dispersions_norm"], rtol=1e-12, atol=1e-12)


def test_scale(dev_state):
    o = c1_oracle(False)
    sc = dev_state["sc"]
    Z = sc.values().cpu().numpy()
    ref = o["Z"]
    assert Z.shape == ref.shape
    # relative error w.r.t. the magnitude before centring: log1p differs from numpy's by
    # <= 1 ulp, and (l - mean) cancels when l ~ mean, so |ref| alone is not a fair scale.
    mag = np.maximum(np.abs(ref), np.abs(o["scale_mean"] * o["scale_inv_std"])[None, :])
    err = np.abs(Z - ref) / np.maximum(mag, 1e-30)
    assert err.max() < 1e-5, err.max()
    np.testing.assert_allclose(sc.mean.cpu().numpy(), o["scale_mean"], rtol=1e-7)
    np.testing.assert_allclose(sc.inv_std.cpu().numpy(), o["scale_inv_std"], rtol=1e-7)
    full = sc.Z.cpu().numpy()
    assert np.all(full[:, sc.ones_col] == 1.0)
    assert np.all(full[:, sc.H + 1:] == 0.0)


def test_qc_large_counts_exact():
    """Counts >= 2^12 take the global high-part path of the gene totals; up to 2^24 - 1."""
    import torch
    import paper_2605_13928_b200 as scb
    from oracle import pipeline as op
    rng = np.random.default_rng(11)
    n, g = 3000, 700
    dense = (rng.random((n, g)) < 0.2) * rng.integers(1, 50, (n, g))
    big = rng.random((n, g)) < 0.01
    dense = np.where(big, rng.integers(4096, 1 << 24, (n, g)), dense).astype(np.float32)
    dense[:, 5] = np.where(dense[:, 5] > 0, (1 << 24) - 1, 0)      # a gene of maximal counts
    import scipy.sparse as sp
    A = sp.csr_matrix(dense)
    X = op.CSR(A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.astype(np.float32), g)
    mt = np.zeros(g, np.uint8)
    mt[:7] = 1
    ref = op.qc_metrics(X, mt)
    Xd = scb.DeviceCSR.from_host(X.indptr, X.indices, X.data, g)
    qc = scb.calculate_qc_metrics(Xd, torch.as_tensor(mt))
    for k in ["n_genes_by_counts", "total_counts", "total_counts_mt", "n_cells_by_counts", "gene_total_counts"]:
        np.testing.assert_array_equal(qc[k].cpu().numpy(), ref[k], err_msg=k)


def test_cpm_normalization_hvg_and_scale_exact():
    """target_sum = 1e6 (CPM): normalized values beyond 2^15 take the global-limb path of the
    HVG sums; the statistics stay bit-exact and the scaled values within tolerance."""
    import dataclasses
    import torch
    import paper_2605_13928_b200 as scb
    from oracle import pipeline as op
    X, mt = c1_inputs()
    p = dataclasses.replace(C1["params"], target_sum=1e6)
    o = op.run(X, mt, p, with_knn=False)
    Xd = scb.DeviceCSR.from_host(X.indptr, X.indices, X.data, X.n_cols)
    qc = scb.calculate_qc_metrics(Xd, torch.as_tensor(mt))
    cm, gm, kept = scb.filter_masks(qc, min_genes=p.min_genes, max_genes=p.max_genes, max_pct_mt=p.max_pct_mt, min_cells=p.min_cells)
    Xl = scb.normalize_log1p(scb.subset(Xd, cm, gm, kept), p.target_sum)
    hvg_mask, hvg_index, st = scb.highly_variable_genes(Xl, p.n_top_genes, p.n_bins)
    np.testing.assert_array_equal(hvg_mask.cpu().numpy(), o["hvg_mask"])
    np.testing.assert_array_equal(st["means"].cpu().numpy(), o["hvg_stats"]["means"])
    np.testing.assert_array_equal(st["variances"].cpu().numpy(), o["hvg_stats"]["variances"])
    sc = scb.scale(Xl, hvg_index, p.max_value)
    np.testing.assert_allclose(sc.mean.cpu().numpy(), o["scale_mean"], rtol=1e-7)
    np.testing.assert_allclose(sc.inv_std.cpu().numpy(), o["scale_inv_std"], rtol=1e-7)


@functools.lru_cache(maxsize=1)
def _wide_case():
    from oracle import pipeline as op
    spec = SynthSpec(3000, 20000, seed=7)
    ip, ix, d = generate_csr(spec)
    X = op.CSR(ip, ix, d, spec.n_genes)
    mt = mt_mask(spec)
    p = op.Params(min_genes=50, max_pct_mt=20.0, n_top_genes=1000, n_neighbors=15)
    return spec, ip, ix, d, mt, p, op.run(X, mt, p, with_knn=False)


@pytest.mark.parametrize("shuffle", [False, True])
def test_hvg_row_splits_sorted_and_unsorted_rows(shuffle):
    """> 1 HVG gene tile (20k genes): QC's per-row tile splits let each tile stream only its
    sub-range of a row.  With the column indices of every row shuffled (non-canonical CSR) the
    split pass detects entries outside its tile and is redone unsplit; the HVG statistics stay
    bit-exact against the oracle either way."""
    import torch
    from paper_2605_13928_b200 import _lib, pipeline, pp
    spec, ip, ix, d, mt, p, o = _wide_case()
    if shuffle:
        rng = np.random.default_rng(3)
        ix = ix.copy()
        d = d.copy()
        for r in range(len(ip) - 1):
            perm = ip[r] + rng.permutation(ip[r + 1] - ip[r])
            ix[ip[r]:ip[r + 1]] = ix[perm]
            d[ip[r]:ip[r + 1]] = d[perm]
    assert int(_lib.call("scb_hvg_tiles", spec.n_genes)) > 1
    Xd = pp.DeviceCSR.from_host(ip, ix, d, spec.n_genes)
    pp_ = pipeline.Params(min_genes=p.min_genes, max_pct_mt=p.max_pct_mt, min_cells=p.min_cells,
                          n_top_genes=p.n_top_genes)
    r = pipeline.run(Xd, torch.as_tensor(mt, device="cuda"), pp_, with_knn=False, timing=False)
    np.testing.assert_array_equal(r.hvg_mask.cpu().numpy(), o["hvg_mask"])
    np.testing.assert_array_equal(r.hvg_stats["means"].cpu().numpy(), o["hvg_stats"]["means"])
    np.testing.assert_array_equal(r.hvg_stats["variances"].cpu().numpy(), o["hvg_stats"]["variances"])


def test_pipeline_40k_genes_bitmap_map_and_three_hvg_tiles():
    """G > 32767 takes the bit/prefix kept-gene map in subset and three HVG gene tiles; masks,
    kept matrix and HVG statistics stay bit-exact."""
    import torch
    from paper_2605_13928_b200 import pipeline, pp
    from oracle import pipeline as op
    spec = SynthSpec(1500, 40000, seed=9)
    ip, ix, d = generate_csr(spec)
    mt = mt_mask(spec)
    p = op.Params(min_genes=50, max_pct_mt=20.0, n_top_genes=1000, n_neighbors=15)
    o = op.run(op.CSR(ip, ix, d, spec.n_genes), mt, p, with_knn=False)
    Xd = pp.DeviceCSR.from_host(ip, ix, d, spec.n_genes)
    pp_ = pipeline.Params(min_genes=p.min_genes, max_pct_mt=p.max_pct_mt, min_cells=p.min_cells,
                          n_top_genes=p.n_top_genes)
    r = pipeline.run(Xd, torch.as_tensor(mt, device="cuda"), pp_, with_knn=False, timing=False)
    np.testing.assert_array_equal(r.cell_mask.cpu().numpy(), o["cell_mask"])
    np.testing.assert_array_equal(r.gene_mask.cpu().numpy(), o["gene_mask"])
    lip, lix, _, _ = r.X_log.to_host()
    np.testing.assert_array_equal(lip, o["X_log"].indptr)
    np.testing.assert_array_equal(lix, o["X_log"].indices)
    np.testing.assert_array_equal(r.hvg_mask.cpu().numpy(), o["hvg_mask"])
    np.testing.assert_array_equal(r.hvg_stats["variances"].cpu().numpy(), o["hvg_stats"]["variances"])


def test_fused_fill_scale_sums_equal_separate_pass():
    """The fill pass's fused HVG scale sums are the same integers scale_gene_sums computes
    from the written log matrix, and the written matrix is unchanged."""
    import torch
    import paper_2605_13928_b200 as scb
    from paper_2605_13928_b200 import pp
    X, mt = c1_inputs()
    p = C1["params"]
    Xd = scb.DeviceCSR.from_host(X.indptr, X.indices, X.data, X.n_cols)
    qc = scb.calculate_qc_metrics(Xd, torch.as_tensor(mt))
    cm, gm, kept = scb.filter_masks(qc, min_genes=p.min_genes, max_genes=p.max_genes, max_pct_mt=p.max_pct_mt, min_cells=p.min_cells)
    _, hvg_index, _ = scb.highly_variable_genes(scb.normalize_log1p(scb.subset(Xd, cm, gm, kept), p.target_sum),
                                                p.n_top_genes, p.n_bins)
    remap, nip, rs, rso, nnz = pp.subset_count_scale(Xd, cm, gm, kept, p.target_sum)
    ref = pp.subset_fill_log(Xd, cm, remap, nip, rs, nnz, kept[1])
    H = int(hvg_index.numel())
    slot = pp.gene_slots(hvg_index, kept[1])
    fused, sums = pp.subset_fill_log_scale_sums(Xd, cm, remap, nip, rs, nnz, kept[1], slot, H)
    assert sums is not None
    assert torch.equal(fused.indices, ref.indices) and torch.equal(fused.data, ref.data)
    sep = pp.scale_gene_sums(ref, slot, H)

    def canonical(t):  # exact integer limb0 + limb1 * 2^32 (the limb split depends on the row blocks)
        a = t.cpu().numpy().astype(object)
        return a[:, 0] + a[:, 1] * (1 << 32)

    assert (canonical(sums) == canonical(sep)).all()
    n = int(kept[0])
    m1, i1 = pp.scale_finalize(sums, n)
    m2, i2 = pp.scale_finalize(sep, n)
    assert torch.equal(m1, m2) and torch.equal(i1, i2)


def test_hvg_tie_rules_gpu_match_oracle():
    """Both selection rules on the device equal the oracle's, on sums with planted exact ties
    (every gene has a twin, so the cutoff falls on a tie)."""
    import torch
    from oracle import pipeline as op
    from paper_2605_13928_b200 import pp
    rng = np.random.default_rng(3)
    G, N = 600, 1000
    y = rng.gamma(0.5, 2.0, (N, G // 2)).astype(np.float32) * (rng.random((N, G // 2)) < 0.3)
    y = np.concatenate([y, y], axis=1)                     # exact twins -> tied statistics
    import scipy.sparse as sp
    A = sp.csr_matrix(y)
    q1 = np.rint(A.data.astype(np.float64) * 2.0 ** op.FX1).astype(np.uint64)
    q2 = np.rint(A.data.astype(np.float64) ** 2 * 2.0 ** op.FX2).astype(np.uint64)
    lo1, hi1 = op._fx_sum(A.indices, q1, G)
    lo2, hi2 = op._fx_sum(A.indices, q2, G)
    sums = torch.as_tensor(np.stack([np.stack([lo1, hi1]), np.stack([lo2, hi2])]).view(np.int64)).cuda()
    s1, s2 = op.fx_gene_sums(A.indices, A.data, G)
    _, st = op.hvg_seurat_from_sums(s1, s2, N, 10)
    key = np.sort(np.where(np.isnan(st["dispersions_norm"]), -np.inf, st["dispersions_norm"]))[::-1]
    n = int(np.nonzero(key[:-1] == key[1:])[0][3]) + 1
    for ties in ("cutoff", "rank"):
        ref, _ = op.hvg_seurat_from_sums(s1, s2, N, n, ties=ties)
        mask, idx, dst = pp.hvg_select(sums, N, n, 20, ties)
        np.testing.assert_array_equal(mask.cpu().numpy(), ref, err_msg=ties)
        assert dst["n_selected"] == int(ref.sum()) == idx.numel()
        np.testing.assert_array_equal(idx.cpu().numpy(), np.nonzero(ref)[0])
    assert int(op.hvg_seurat_from_sums(s1, s2, N, n, ties="cutoff")[0].sum()) > n


@pytest.mark.parametrize("clip", ["symmetric", "upper"])
def test_scale_clip_modes_gpu(dev_state, clip):
    """scale_dense with both clip modes vs the oracle, at a max_value (1.0) that clips both sides."""
    import torch
    from oracle import pipeline as op
    from paper_2605_13928_b200 import pp
    o = c1_oracle(False)
    Xl = dev_state["Xl"]
    sc = pp.scale(Xl, dev_state["hvg"], 1.0, clip=clip)
    torch.cuda.synchronize()
    oXl = o["X_log"]
    ref, mean, inv = op.scale(oXl, o["hvg_mask"], 1.0, clip=clip)
    Z = sc.values().cpu().numpy()
    mag = np.maximum(np.abs(ref), np.abs(mean * inv)[None, :])
    assert (np.abs(Z - ref) / np.maximum(mag, 1e-30)).max() < 1e-5
    assert Z.max() <= 1.0
    if clip == "symmetric":
        assert Z.min() >= -1.0
    else:
        assert Z.min() < -1.0

def test_fused_fill_all_kept_shares_indices():
    """Every row and gene kept: the fill pass writes only the log values and the kept matrix
    shares the input's indices; values and fused sums equal the copying path's."""
    import torch
    import paper_2605_13928_b200 as scb
    from paper_2605_13928_b200 import pp
    X, mt = c1_inputs()
    Xd = scb.DeviceCSR.from_host(X.indptr, X.indices, X.data, X.n_cols)
    qc = scb.calculate_qc_metrics(Xd, torch.as_tensor(mt))
    cm, gm, kept = scb.filter_masks(qc, min_genes=0, max_genes=None, max_pct_mt=101.0, min_cells=0)
    assert (int(kept[0]), int(kept[1])) == (Xd.n_rows, Xd.n_cols)
    remap, nip, rs, rso, nnz = pp.subset_count_scale(Xd, cm, gm, kept, 1e4)
    H = 300
    slot = pp.gene_slots(torch.arange(0, 3 * H, 3, dtype=torch.int32, device=Xd.indices.device), kept[1])
    ref, s_ref = pp.subset_fill_log_scale_sums(Xd, cm, remap, nip, rs, nnz, kept[1], slot, H)
    got, s_got = pp.subset_fill_log_scale_sums(Xd, cm, remap, nip, rs, nnz, kept[1], slot, H, all_kept=True)
    assert got.indices.data_ptr() == Xd.indices.data_ptr() and ref.indices.data_ptr() != Xd.indices.data_ptr()
    assert torch.equal(got.indices, ref.indices) and torch.equal(got.data, ref.data)
    assert torch.equal(got.indptr, Xd.indptr)
    assert torch.equal(s_got, s_ref)


def test_pipeline_all_kept_shared_indices_matches_copy(monkeypatch):
    """Whole pipeline with filters that keep every cell and gene: the shared-indices fill path
    gives bit-identical HVG set, scale statistics, PCA and kNN to the copying path, and leaves
    the input matrix untouched."""
    import torch
    import paper_2605_13928_b200 as scb
    from paper_2605_13928_b200 import pipeline, pp
    X, mt = c1_inputs()
    Xd = scb.DeviceCSR.from_host(X.indptr, X.indices, X.data, X.n_cols)
    ind0, dat0 = Xd.indices.clone(), Xd.data.clone()
    prm = pipeline.Params(min_genes=0, max_pct_mt=101.0, min_cells=0, n_top_genes=500, n_neighbors=10)
    mtd = torch.as_tensor(mt, device="cuda")
    shared = pipeline.run(Xd, mtd, prm, timing=False)
    assert shared.X_log.indices.data_ptr() == Xd.indices.data_ptr()
    orig = pp.subset_fill_log_scale_sums
    monkeypatch.setattr(pp, "subset_fill_log_scale_sums",
                        lambda *a, **k: orig(*a, **{**k, "all_kept": False}))
    copied = pipeline.run(Xd, mtd, prm, timing=False)
    assert copied.X_log.indices.data_ptr() != Xd.indices.data_ptr()
    assert torch.equal(shared.hvg_index, copied.hvg_index)
    assert torch.equal(shared.X_log.data, copied.X_log.data)
    assert torch.equal(shared.pca.X_pca, copied.pca.X_pca)
    assert torch.equal(shared.knn_index, copied.knn_index)
    assert torch.equal(Xd.indices, ind0) and torch.equal(Xd.data, dat0)
