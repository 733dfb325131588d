"""CPU tests of the oracle (oracle/): hand known-answer tests, the committed golden fixtures,
and cross-checks against independent restatements (scipy.sparse, pandas -- the library Scanpy's
seurat-flavour HVG code is written in --, sklearn PCA / NearestNeighbors).  No GPU needed."""
import numpy as np
import pandas as pd
import pytest
import scipy.sparse as sp

from oracle import pipeline as op
from oracle.synth import SynthSpec, generate_csr, mt_mask
from tests.golden import make_golden as mg

GOLDEN = "tests/golden/g600x300.npz"


# ----------------------------------------------------------------------------- known answers
def micro():
    # 4 cells x 5 genes, gene 0 mitochondrial; row 1 has an explicit zero, row 2 is empty
    indptr = np.array([0, 3, 5, 5, 10], dtype=np.int64)
    indices = np.array([0, 2, 3, 1, 4, 0, 1, 2, 3, 4], dtype=np.int32)
    data = np.array([1, 2, 3, 5, 0, 1, 1, 1, 1, 6], dtype=np.float32)
    return op.CSR(indptr, indices, data, 5), np.array([1, 0, 0, 0, 0], dtype=np.uint8)


def test_qc_known_answers():
    X, mt = micro()
    q = op.qc_metrics(X, mt)
    np.testing.assert_array_equal(q["n_genes_by_counts"], [3, 1, 0, 5])
    np.testing.assert_array_equal(q["total_counts"], [6, 5, 0, 10])
    np.testing.assert_array_equal(q["total_counts_mt"], [1, 0, 0, 1])
    np.testing.assert_allclose(q["pct_counts_mt"][[0, 1, 3]], [100 / 6, 0, 10])
    assert np.isnan(q["pct_counts_mt"][2])
    np.testing.assert_array_equal(q["n_cells_by_counts"], [2, 2, 2, 2, 1])
    np.testing.assert_array_equal(q["gene_total_counts"], [2, 6, 3, 4, 6])


def test_filter_and_subset_known_answers():
    X, mt = micro()
    q = op.qc_metrics(X, mt)
    cm, gm = op.filter_masks(q, op.Params(min_genes=1, max_genes=None, max_pct_mt=20.0, min_cells=2))
    np.testing.assert_array_equal(cm, [1, 1, 0, 1])        # row 2 empty (NaN pct fails)
    np.testing.assert_array_equal(gm, [1, 1, 1, 1, 0])     # gene 4 in one cell only
    S = op.subset(X, cm, gm)
    np.testing.assert_array_equal(S.indptr, [0, 3, 4, 8])
    np.testing.assert_array_equal(S.indices, [0, 2, 3, 1, 0, 1, 2, 3])
    np.testing.assert_array_equal(S.data, [1, 2, 3, 5, 1, 1, 1, 1])
    assert S.n_cols == 4


def test_filter_mask_max_genes():
    X, mt = micro()
    q = op.qc_metrics(X, mt)
    cm, _ = op.filter_masks(q, op.Params(min_genes=1, max_genes=4, max_pct_mt=50.0, min_cells=2))
    # row0: 3 genes, 16.7% mt -> kept; row1 kept; row2 empty; row3 has 5 genes > 4
    np.testing.assert_array_equal(cm, [1, 1, 0, 0])


def test_normalize_log1p_known_answers():
    X, mt = micro()
    Xl, y32, s = op.normalize_log1p(X, target_sum=10.0)
    np.testing.assert_array_equal(s, np.array([10 / 6, 10 / 5, 1.0, 1.0], dtype=np.float32))
    np.testing.assert_array_equal(y32[:3], (np.array([1, 2, 3], np.float32) * np.float32(10 / 6)))
    np.testing.assert_allclose(Xl.data[:3], np.log1p(np.array([1, 2, 3]) * 10 / 6), rtol=1e-6)
    assert Xl.data[4] == 0.0  # explicit zero stays zero


def test_fixed_point_sums_match_float64():
    rng = np.random.default_rng(0)
    idx = rng.integers(0, 50, 20000).astype(np.int32)
    v = (rng.integers(1, 30, 20000) * rng.uniform(0.1, 5, 20000)).astype(np.float32)
    s1, s2 = op.fx_gene_sums(idx, v, 50)
    r1, r2 = op.gene_sums(idx, v.astype(np.float64), 50)
    np.testing.assert_allclose(s1, r1, rtol=1e-12)
    np.testing.assert_allclose(s2, r2, rtol=1e-9)
    # order independence: any permutation gives the identical (integer) result
    perm = rng.permutation(len(idx))
    t1, t2 = op.fx_gene_sums(idx[perm], v[perm], 50)
    np.testing.assert_array_equal(s1, t1)
    np.testing.assert_array_equal(s2, t2)


def test_scale_constant_gene_std_one():
    # a gene with the same log value in every cell (incl. zeros?) -> std 0 -> 1, z = l - mean
    indptr = np.array([0, 2, 4, 6], np.int64)
    indices = np.array([0, 1, 0, 1, 0, 1], np.int32)
    data = np.array([2.0, 1.0, 2.0, 3.0, 2.0, 5.0], np.float32)
    X = op.CSR(indptr, indices, data, 2)
    Z, mean, inv = op.scale(X, np.array([1, 1], np.uint8), max_value=10.0)
    assert inv[0] == 1.0
    np.testing.assert_allclose(Z[:, 0], 0.0, atol=1e-6)


def test_scale_clip_upper_only():
    rng = np.random.default_rng(1)
    n = 400
    rows = np.arange(n)
    data = np.zeros(n, np.float32)
    data[0] = 50.0   # one huge outlier, everything else zero -> z0 slightly negative, outlier clipped to 10
    X = op.CSR(np.arange(n + 1, dtype=np.int64), np.zeros(n, np.int32), np.maximum(data, 1e-3).astype(np.float32), 1)
    Z, _, _ = op.scale(X, np.array([1], np.uint8), max_value=10.0)
    assert Z.max() == 10.0 and Z.min() > -10.0
    del rows, rng


def _regress_case(seed=5, n=600, g=60, h=12):
    rng = np.random.default_rng(seed)
    M = sp.random(n, g, density=0.3, random_state=seed, format="csr", dtype=np.float64)
    M.data = np.floor(M.data * 20) + 1
    M.sort_indices()
    X = op.CSR(M.indptr.astype(np.int64), M.indices.astype(np.int32), M.data.astype(np.float32), g)
    Xl, _, _ = op.normalize_log1p(X, 1e4)
    hvg = np.zeros(g, np.uint8)
    hvg[rng.choice(g, h, replace=False)] = 1
    tk = rng.integers(500, 5000, n).astype(np.float64)
    pk = rng.uniform(0, 15, n)
    return Xl, hvg, tk, pk


def test_regress_out_matches_lstsq_residuals():
    """The standardised-design normal-equation fit equals OLS on [1, total_counts, pct_mt]
    (numpy lstsq) and the residual scaling equals np.std(ddof=1) of the explicit residuals."""
    Xl, hvg, tk, pk = _regress_case()
    Z, beta, inv = op.regress_out_scale(Xl, hvg, tk, pk, max_value=1e30)
    cols = np.nonzero(hvg)[0]
    L = np.asarray(sp.csr_matrix((Xl.data, Xl.indices, Xl.indptr), shape=(Xl.n_rows, Xl.n_cols)).todense(),
                   np.float64)[:, cols]
    A = np.stack([np.ones_like(tk), tk, pk], 1)
    B, *_ = np.linalg.lstsq(A, L, rcond=None)
    R = L - A @ B
    assert np.abs(R.mean(0)).max() < 1e-10
    Zref = (R - R.mean(0)) / R.std(0, ddof=1)
    np.testing.assert_allclose(Z, Zref, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(1.0 / inv, R.std(0, ddof=1), rtol=1e-9)


def test_regress_out_clip_and_constant_gene():
    Xl, hvg, tk, pk = _regress_case(seed=9)
    Z, _, inv = op.regress_out_scale(Xl, hvg, tk, pk, max_value=1.5)
    assert Z.max() <= 1.5
    # a covariate that is constant -> std 0 -> 1 and the fit still works (collinear with 1)
    Z2, _, _ = op.regress_out_scale(Xl, hvg, tk, np.full_like(pk, 3.0), max_value=1e30)
    assert np.isfinite(Z2).all()


# ----------------------------------------------------------------------------- golden fixtures
@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def test_generator_reproduces_golden_input(golden):
    ip, ix, d = generate_csr(mg.SPEC)
    np.testing.assert_array_equal(ip, golden["indptr"])
    np.testing.assert_array_equal(ix, golden["indices"])
    np.testing.assert_array_equal(d, golden["data"])


def test_generator_chunking_independent():
    spec = SynthSpec(300, 120, seed=3)
    a = generate_csr(spec, chunk_cells=64)
    b = generate_csr(spec, chunk_cells=1000)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_oracle_reproduces_golden(golden):
    out = mg.compute()
    for k in golden.files:
        a, b = out[k], golden[k]
        if a.dtype.kind in "iub":
            np.testing.assert_array_equal(a, b, err_msg=k)
        else:
            np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12, equal_nan=True, err_msg=k)


# ----------------------------------------------------------------------------- cross-checks
def _sp(X):
    return sp.csr_matrix((X.data.astype(np.float64), X.indices, X.indptr), shape=(X.n_rows, X.n_cols))


def test_qc_vs_scipy(golden):
    X = op.CSR(golden["indptr"], golden["indices"], golden["data"], 300)
    q = op.qc_metrics(X, golden["mt_mask"])
    A = _sp(X)
    np.testing.assert_array_equal(q["total_counts"], np.asarray(A.sum(1)).ravel())
    np.testing.assert_array_equal(q["gene_total_counts"], np.asarray(A.sum(0)).ravel())
    np.testing.assert_array_equal(q["n_genes_by_counts"], np.asarray((A > 0).sum(1)).ravel())
    np.testing.assert_array_equal(q["n_cells_by_counts"], np.asarray((A > 0).sum(0)).ravel())


def scanpy_seurat_pandas(mean, var, n_top, n_bins=20):
    """Transcription of Scanpy's seurat-flavour normalised dispersion (pandas cut/groupby)."""
    mean = mean.copy()
    mean[mean == 0] = 1e-12
    disp = var / mean
    disp[disp == 0] = np.nan
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
    srt = np.sort(dn[~np.isnan(dn)])[::-1]
    cut = srt[n_top - 1]
    return np.nan_to_num(dn) >= cut, dn


def test_hvg_vs_pandas_scanpy_transcription(golden):
    sub = op.CSR(golden["sub_indptr"], golden["sub_indices"], golden["sub_data"], int(golden["gene_mask"].sum()))
    Xl, y32, _ = op.normalize_log1p(sub, 1e4)
    s1, s2 = op.fx_gene_sums(Xl.indices, y32, Xl.n_cols)
    mean, var = op.mean_var(s1, s2, float(sub.n_rows))
    sel_pd, dn_pd = scanpy_seurat_pandas(mean, var, 100)
    mask, st = op.hvg_seurat_from_sums(s1, s2, sub.n_rows, 100)
    np.testing.assert_allclose(st["dispersions_norm"], dn_pd, rtol=1e-10, atol=1e-12, equal_nan=True)
    assert sel_pd.sum() == 100  # no ties at the cutoff here, so Scanpy's >= rule picks exactly n
    np.testing.assert_array_equal(mask.astype(bool), sel_pd)


def test_pandas_cut_edges_match_pandas():
    rng = np.random.default_rng(5)
    x = rng.normal(size=1000)
    e = op.pandas_cut_edges(float(x.min()), float(x.max()), 20)
    _, bins = pd.cut(x, 20, retbins=True)
    np.testing.assert_array_equal(e, bins)


def test_pca_vs_sklearn(golden):
    from sklearn.decomposition import PCA
    Z = golden["Z"].astype(np.float64)
    k = golden["components"].shape[1]
    skp = PCA(n_components=k, svd_solver="full").fit(Z)
    assert op.subspace_angle(skp.components_.T, golden["components"]) < 1e-6  # arccos resolution ~1e-8
    np.testing.assert_allclose(skp.explained_variance_, golden["variance"], rtol=1e-9)
    np.testing.assert_allclose(skp.explained_variance_ratio_, golden["variance_ratio"], rtol=1e-9)


def test_knn_vs_sklearn(golden):
    from sklearn.neighbors import NearestNeighbors
    X = golden["X_pca"].astype(np.float64)
    k = golden["knn_idx"].shape[1]
    d, i = NearestNeighbors(n_neighbors=k, algorithm="brute").fit(X).kneighbors(X)
    np.testing.assert_allclose(golden["knn_dist"], d, rtol=1e-5, atol=1e-5)
    assert op.knn_recall(golden["knn_idx"], i) > 0.999
    assert np.all(golden["knn_idx"][:, 0] == np.arange(len(X)))  # self first


def test_knn_tie_order_by_index():
    X = np.array([[0.0, 0.0], [1.0, 0.0], [-1.0, 0.0], [0.0, 1.0], [0.0, -1.0], [1.0, 0.0]])
    i, d = op.knn(X, 6)
    # all four unit-distance points (and the duplicate of point 1) tie: ascending index order
    np.testing.assert_array_equal(i[0], [0, 1, 2, 3, 4, 5])
    np.testing.assert_array_equal(i[1], [1, 5, 0, 3, 4, 2])
    np.testing.assert_allclose(d[1][:2], [0.0, 0.0])


def _smooth_knn_dist_loop(distances, k, n_iter=64):
    """Literal transcription of umap-learn 0.5 smooth_knn_dist (local_connectivity 1,
    bandwidth 1) -- the loop the vectorised oracle restates."""
    target = np.log2(k)
    n = distances.shape[0]
    rho = np.zeros(n, np.float32)
    result = np.zeros(n, np.float32)
    mean_distances = np.mean(distances)
    for i in range(n):
        lo, hi, mid = 0.0, np.inf, 1.0
        ith = distances[i]
        nz = ith[ith > 0.0]
        if nz.shape[0] >= 1:
            rho[i] = nz[0]
        for _ in range(n_iter):
            psum = 0.0
            for j in range(1, distances.shape[1]):
                d = distances[i, j] - rho[i]
                psum += np.exp(-(float(d) / mid)) if d > 0 else 1.0  # numba: f32 / f64 -> f64
            if np.fabs(psum - target) < 1e-5:
                break
            if psum > target:
                hi = mid
                mid = (lo + hi) / 2.0
            else:
                lo = mid
                mid = mid * 2 if hi == np.inf else (lo + hi) / 2.0
        result[i] = mid
        if rho[i] > 0.0:
            if result[i] < 1e-3 * np.mean(ith):
                result[i] = 1e-3 * np.mean(ith)
        elif result[i] < 1e-3 * mean_distances:
            result[i] = 1e-3 * mean_distances
    return result, rho


def test_umap_graph_oracle_vs_literal_loop_and_properties():
    rng = np.random.default_rng(2)
    E = rng.standard_normal((400, 6)).astype(np.float32)
    E[7] = E[3]  # an exact duplicate -> a zero non-self distance
    ki, kd = op.knn(E, 12)
    sig, rho = op.smooth_knn_dist(kd, 12)
    sig_l, rho_l = _smooth_knn_dist_loop(kd, 12)
    np.testing.assert_array_equal(rho, rho_l)
    np.testing.assert_allclose(sig, sig_l, rtol=1e-6)
    C, Dm, _, _ = op.umap_connectivities(ki, kd, 400)
    assert abs(C - C.T).max() == 0 and C.data.min() > 0 and C.data.max() <= 1.0
    assert C.has_sorted_indices and Dm.nnz == (kd > 0).sum()
    # each row's membership strengths (self 0, nearest non-self neighbour 1) sum to log2(k)
    W = op.membership_strengths(ki, kd, sig, rho)
    excess = W.sum(1) - np.log2(12)
    assert np.abs(excess[rho > 0]).max() < 1e-3


def test_louvain_oracle_quality_vs_networkx():
    """The deterministic bucketed-synchronous modularity optimisation (the algorithm csrc/cluster.cu
    implements) reaches the modularity of networkx's sequential Louvain on a weakly clustered
    single-cell-like graph (independent implementation as the quality reference)."""
    nx = pytest.importorskip("networkx")
    rng = np.random.default_rng(4)
    centers = rng.standard_normal((6, 8)) * 1.2
    lab = rng.integers(0, 6, 1500)
    E = (centers[lab] + rng.standard_normal((1500, 8))).astype(np.float32)
    ki, kd = op.knn(E, 15)
    C, _, _, _ = op.umap_connectivities(ki, kd, 1500)
    _, nc, q = op.louvain(C, seed=3)
    G = nx.from_scipy_sparse_array(C)
    qs = [nx.community.modularity(G, nx.community.louvain_communities(G, weight="weight", seed=s), weight="weight")
          for s in (0, 1, 2)]
    assert q >= min(qs) - 0.01, (q, qs)
    # modularity reported by the oracle equals networkx's formula on its own partition
    labels, _, q2 = op.louvain(C, seed=3)
    comms = [set(np.nonzero(labels == c)[0].tolist()) for c in range(labels.max() + 1)]
    assert abs(nx.community.modularity(G, comms, weight="weight") - q2) < 1e-6


def test_leiden_oracle_quality_and_connectivity():
    """The deterministic Leiden restatement: modularity at least networkx's sequential Louvain
    (minus 0.01) on a weakly clustered graph, and every community connected."""
    nx = pytest.importorskip("networkx")
    import scipy.sparse.csgraph as cg
    rng = np.random.default_rng(4)
    centers = rng.standard_normal((6, 8)) * 1.2
    lab = rng.integers(0, 6, 1500)
    E = (centers[lab] + rng.standard_normal((1500, 8))).astype(np.float32)
    ki, kd = op.knn(E, 15)
    C, _, _, _ = op.umap_connectivities(ki, kd, 1500)
    labels, nc, q = op.leiden(C, seed=3)
    G = nx.from_scipy_sparse_array(C)
    qs = [nx.community.modularity(G, nx.community.louvain_communities(G, weight="weight", seed=s), weight="weight")
          for s in (0, 1, 2)]
    assert q >= min(qs) - 0.01, (q, qs)
    comms = [set(np.nonzero(labels == c)[0].tolist()) for c in range(nc)]
    assert abs(nx.community.modularity(G, comms, weight="weight") - q) < 1e-6
    for c in range(nc):
        idx = np.nonzero(labels == c)[0]
        assert cg.connected_components(C[idx][:, idx], directed=False)[0] == 1


# ----------------------------------------------------------------------------- Scanpy float pin
def _c1_scanpy_vs_fixed_point(spec, n_top, min_genes, max_pct_mt):
    from oracle import scanpy_float as sf
    ip, ix, d = generate_csr(spec, threads=8)
    X = op.CSR(ip, ix, d, spec.n_genes)
    p = op.Params(min_genes=min_genes, max_pct_mt=max_pct_mt, n_top_genes=n_top)
    o = op.run(X, mt_mask(spec), p, with_knn=False)
    Xl = o["X_log"]
    sel, dn = sf.hvg_seurat_expm1(Xl.indices, Xl.data, Xl.n_rows, Xl.n_cols, n_top)
    return o, sel, dn


def test_hvg_fixed_point_set_equals_scanpy_float64_expm1_c1():
    """The fixed-point HVG statistics (device arithmetic) select exactly the gene set that
    Scanpy's float64 mean/var of expm1(X_log) selects, at C1 (10k x 2k, H = 1000)."""
    o, sel, dn = _c1_scanpy_vs_fixed_point(SynthSpec(10000, 2000, seed=1), 1000, 50, 15.0)
    flips = np.nonzero(o["hvg_mask"].astype(bool) != sel)[0]
    assert flips.size == 0, f"HVG set differs from Scanpy's float path at genes {flips.tolist()}"
    # the normalised dispersions agree to ~1e-6 relative (expm1(log1p(y)) vs y rounding)
    st = o["hvg_stats"]["dispersions_norm"]
    ok = ~np.isnan(st)
    np.testing.assert_allclose(st[ok], dn[ok], rtol=1e-5, atol=1e-6)


def test_hvg_tie_rules():
    """'cutoff' (Scanpy) keeps every gene tied at the n-th value; 'rank' keeps exactly n by index."""
    rng = np.random.default_rng(3)
    G = 400
    mean = rng.uniform(0.1, 2.0, G)
    var = mean * np.exp(rng.normal(0, 0.5, G))
    s1, s2 = mean * 1000.0, (var * 999.0 / 1000.0 + mean * mean) * 1000.0
    s1[200:], s2[200:] = s1[:200], s2[:200]          # every gene has an exact twin
    _, st = op.hvg_seurat_from_sums(s1, s2, 1000, 10)
    key = np.where(np.isnan(st["dispersions_norm"]), -np.inf, st["dispersions_norm"])
    srt = np.sort(key)[::-1]
    i = int(np.nonzero(srt[:-1] == srt[1:])[0][5])     # a tie inside the ranking
    n = i + 1                                           # n-th largest value is tied with the (n+1)-th
    m_cut, _ = op.hvg_seurat_from_sums(s1, s2, 1000, n, ties="cutoff")
    m_rank, _ = op.hvg_seurat_from_sums(s1, s2, 1000, n, ties="rank")
    assert m_rank.sum() == n
    assert m_cut.sum() == int((key >= srt[n - 1]).sum()) > n
    assert np.all(m_cut >= m_rank)
    tied = np.nonzero(key == srt[n - 1])[0]
    assert m_rank[tied].sum() == n - int((key > srt[n - 1]).sum()) and m_rank[tied.min()]


def test_scale_clip_modes():
    ip = np.array([0, 2, 3, 3], np.int64)
    ix = np.array([0, 1, 0], np.int32)
    l = np.array([5.0, 0.1, 0.2], np.float32)
    Xl = op.CSR(ip, ix, l, 2)
    mask = np.array([1, 1], np.uint8)
    Zs, mean, inv = op.scale(Xl, mask, max_value=0.5, clip="symmetric")
    Zu, _, _ = op.scale(Xl, mask, max_value=0.5, clip="upper")
    assert Zs.max() <= 0.5 and Zs.min() >= -0.5
    assert Zu.max() <= 0.5 and Zu.min() < -0.5
    np.testing.assert_array_equal(Zs, np.maximum(Zu, np.float32(-0.5)))


def test_chunked_oracle_equals_unchunked():
    """oracle/chunked.py (row chunks in forked workers, 128-bit limb sums) reproduces
    pipeline.run stage by stage: the driver of the full-size (C3) parity test."""
    from oracle import chunked
    spec = SynthSpec(3000, 800, seed=9)
    ip, ix, d = generate_csr(spec)
    p = op.Params(min_genes=20, max_pct_mt=15.0, n_top_genes=300, n_comps=20, n_neighbors=10)
    ref = op.run(op.CSR(ip, ix, d, spec.n_genes), mt_mask(spec), p)
    q = np.arange(0, ref["X_pca"].shape[0], 7)
    got = chunked.run(ip, ix, d, spec.n_genes, mt_mask(spec), p, workers=3, chunk_rows=700, knn_queries=q)
    for k, v in ref["qc"].items():
        np.testing.assert_array_equal(got["qc"][k], v, err_msg=k)
    for k in ("cell_mask", "gene_mask", "hvg_mask", "scale_mean", "scale_inv_std"):
        np.testing.assert_array_equal(got[k], ref[k], err_msg=k)
    assert op.subspace_angle(got["components"], ref["components"]) < 1e-7
    np.testing.assert_allclose(got["variance"], ref["variance"], rtol=1e-10)
    np.testing.assert_array_equal(got["knn_idx"], ref["knn_idx"][q])


def _oracle_native():
    import subprocess
    from oracle import synth as osynth
    if osynth.native_lib() is None:
        subprocess.run(["make", "-C", "oracle"], check=True, capture_output=True)
    return osynth


def test_c_generator_equals_numpy_generator():
    """oracle/csynth.c (pthreads) reproduces oracle/synth.py bit for bit (row windows, two specs)."""
    osynth = _oracle_native()
    for spec, rows in ((SynthSpec(3000, 700, seed=5), None), (SynthSpec(1_000_000, 25_000, seed=0), (123_456, 123_800))):
        a = generate_csr(spec, rows=rows)
        b = osynth.generate_csr_native(spec, rows=rows, threads=4)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
