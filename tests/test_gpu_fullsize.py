"""Full-size (C3: 1M cells x 25k genes, BASELINE.json's headline config) checks of the whole
path through size-independent properties (the stage-by-stage comparison with the CPU oracle at
this size is tests/test_gpu_parity_scale.py); each stage is checked against an identity that
holds at any size:

* QC: checksum of checksums -- sum over cells of total_counts == sum over genes of total_counts ==
  sum of the stored counts, and likewise for the nonzero counts (exact: integer counts in f64);
* masks: recomputed from the GPU metrics with torch integer/float compares, bit-identical;
* HVG: exactly n_top genes, every selected gene's normalized dispersion >= every unselected one's;
* scale: |z| <= max_value, finite;
* PCA: orthonormal components, non-increasing variances, X_pca == (Z - mean) V^T on sampled rows
  (float64 recomputation);
* kNN: self at distance 0 first, distances non-decreasing, and 512 random queries against an
  exact float64 brute force over all 1M rows (recall >= 0.999, distances within 1e-4);
* the compact u16 input at full size: every stage bit-identical to the 32-bit input;
* kNN with k = 30 (config C5's k) on the C3 embedding: recall >= 0.999 on 1000 random queries
  against the CPU oracle's exact float64 neighbours.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, G = 1_000_000, 25_000


@pytest.fixture(scope="module")
def c3():
    import torch
    from paper_2605_13928_b200 import pipeline, synth
    spec = synth.Spec(N, G, seed=0)
    X = synth.generate(spec)
    mt = synth.mt_mask(spec)
    data_sum = X.data.double().sum().item()
    nnz_pos = int((X.data > 0).sum().item())
    p = pipeline.Params()
    r = pipeline.run(X, mt, p)
    torch.cuda.synchronize()
    Xu = X.to_u16()
    del X
    return dict(r=r, p=p, data_sum=data_sum, nnz_pos=nnz_pos, Xu=Xu, mt=mt)


def test_c3_qc_checksums_and_masks(c3):
    import torch
    r, p = c3["r"], c3["p"]
    qc = r.qc
    assert qc["total_counts"].double().sum().item() == c3["data_sum"]
    assert qc["gene_total_counts"].double().sum().item() == c3["data_sum"]
    assert int(qc["n_genes_by_counts"].long().sum().item()) == c3["nnz_pos"]
    assert int(qc["n_cells_by_counts"].long().sum().item()) == c3["nnz_pos"]
    cell = (qc["n_genes_by_counts"] >= p.min_genes) & (qc["pct_counts_mt"] < p.max_pct_mt)
    gene = qc["n_cells_by_counts"] >= p.min_cells
    assert torch.equal(r.cell_mask.bool(), cell)
    assert torch.equal(r.gene_mask.bool(), gene)
    assert 0.9 * N < int(cell.sum()) <= N


def test_c3_hvg_selection_is_a_top_set(c3):
    import torch
    r, p = c3["r"], c3["p"]
    sel = r.hvg_mask.bool()
    assert int(sel.sum()) == p.n_top_genes == r.hvg_index.numel()
    dn = r.hvg_stats["dispersions_norm"]
    fin = torch.isfinite(dn)
    assert bool(fin[sel].all())
    assert dn[sel].min().item() >= dn[~sel & fin].max().item()


def test_c3_scale_clip(c3):
    import torch
    Z = c3["r"].scaled.values()
    assert bool(torch.isfinite(Z).all())
    assert Z.abs().max().item() <= c3["p"].max_value


def test_c3_pca_orthonormal_and_projection(c3):
    import torch
    r = c3["r"]
    V = r.pca.components.double()                       # [n_comps][H]
    eye = torch.eye(V.shape[0], dtype=torch.float64, device=V.device)
    assert (V @ V.T - eye).abs().max().item() < 1e-4
    lam = r.pca.variance
    assert bool((lam[1:] <= lam[:-1] * (1 + 1e-12)).all())
    assert 0 < r.pca.variance_ratio.sum().item() <= 1 + 1e-9
    g = torch.Generator(device="cpu").manual_seed(3)
    rows = torch.randint(0, r.pca.X_pca.shape[0], (2048,), generator=g).to(V.device)
    H = r.scaled.H
    Zs = r.scaled.dense()[rows, :H].double() - r.pca.col_mean[:H].double()
    ref = Zs @ V.T
    got = r.pca.X_pca[rows, : r.pca.n_comps].double()
    scale = ref.abs().max().item()
    assert (got - ref).abs().max().item() <= 1e-4 * scale


def test_c3_knn_sampled_exact(c3):
    import torch
    r, p = c3["r"], c3["p"]
    idx, dist = r.knn_index, r.knn_dist
    k = p.n_neighbors
    assert idx.shape[1] == k
    assert bool((dist[:, 0] == 0).all())
    assert bool((dist[:, 1:] >= dist[:, :-1]).all())
    E = r.pca.X_pca[:, : r.pca.n_comps].double()
    g = torch.Generator(device="cpu").manual_seed(11)
    q = torch.randint(0, E.shape[0], (512,), generator=g).to(E.device)
    d2 = (E[q] * E[q]).sum(1, keepdim=True) - 2.0 * (E[q] @ E.T) + (E * E).sum(1)[None, :]
    ref_d, ref_i = torch.topk(d2.clamp_min(0), k, dim=1, largest=False)
    got = idx[q].long()
    hits = sum(len(set(a.tolist()) & set(b.tolist())) for a, b in zip(got.cpu(), ref_i.cpu()))
    assert hits / (512 * k) >= 0.999
    np.testing.assert_allclose(dist[q].double().cpu().numpy(), ref_d.sqrt().cpu().numpy(), rtol=1e-4, atol=1e-4)


def test_c3_u16_input_bit_identical(c3):
    """The compact u16 CSR (292 escaped counts >= 65535 at C3) through every raw-matrix pass
    gives exactly the 32-bit input's results at full size."""
    import torch
    from paper_2605_13928_b200 import pipeline
    r, Xu = c3["r"], c3["Xu"]
    assert Xu.esc_pos.numel() > 0
    ru = pipeline.run(Xu, c3["mt"], c3["p"], timing=False)
    torch.cuda.synchronize()
    for k in ("n_genes_by_counts", "total_counts", "n_cells_by_counts", "gene_total_counts"):
        assert torch.equal(ru.qc[k], r.qc[k]), k
    assert torch.equal(ru.cell_mask, r.cell_mask) and torch.equal(ru.hvg_mask, r.hvg_mask)
    assert torch.equal(ru.X_log.data, r.X_log.data)
    assert torch.equal(ru.scaled.Z_hi, r.scaled.Z_hi) and torch.equal(ru.scaled.Z_lo, r.scaled.Z_lo)
    assert torch.equal(ru.pca.X_pca, r.pca.X_pca) and torch.equal(ru.knn_index, r.knn_index)


def test_c3_knn_k30_recall_vs_oracle(c3):
    """k = 30 (config C5) on the C3 embedding against the CPU oracle's float64 brute force."""
    import os
    import torch
    from oracle import chunked
    from oracle import pipeline as op
    from paper_2605_13928_b200 import pp
    E = c3["r"].pca.X_pca[:, :50].contiguous()
    idx, dist = pp.neighbors(E, 30)
    torch.cuda.synchronize()
    q = np.sort(np.random.default_rng(7).choice(E.shape[0], 1000, replace=False))
    ref_i, ref_d = chunked.knn_queries(E.cpu().numpy(), 30, q, workers=max(1, min(32, len(os.sched_getaffinity(0)))))
    got = idx.cpu().numpy()[q]
    assert op.knn_recall(got, ref_i) >= 0.999
    np.testing.assert_allclose(dist.cpu().numpy()[q][:, -1], ref_d[:, -1], rtol=1e-4, atol=1e-5)
