"""GPU parity of the kNN graph (tcgen05 TF32 candidates + exact FP32 re-rank) vs the oracle."""
import numpy as np
import pytest

from oracle import pipeline as op
from tests.gpu_fixtures import C1, c1_oracle

pytestmark = pytest.mark.gpu


def _pad(X, ld=64):
    P = np.zeros((X.shape[0], ld), dtype=np.float32)
    P[:, : X.shape[1]] = X
    return P


def test_knn_matches_oracle_c1():
    import torch
    from paper_2605_13928_b200 import pp
    o = c1_oracle(True)
    X = o["X_pca"]
    k = C1["params"].n_neighbors
    Xd = torch.as_tensor(_pad(X)).cuda()
    idx, dist = pp.neighbors(Xd, k, n_comps=X.shape[1])
    idx, dist = idx.cpu().numpy(), dist.cpu().numpy()
    assert np.all(idx[:, 0] == np.arange(len(X)))          # self first (distance 0)
    rec = op.knn_recall(idx, o["knn_idx"])
    assert rec >= 0.999, rec
    np.testing.assert_allclose(dist, o["knn_dist"], rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("n,d,k", [(1000, 50, 15), (3001, 50, 30), (517, 20, 8), (900, 40, 48)])
def test_knn_random_exact(n, d, k):
    import torch
    from paper_2605_13928_b200 import pp
    rng = np.random.default_rng(n + d + k)
    X = rng.standard_normal((n, d)).astype(np.float32) * rng.uniform(0.5, 3.0, d).astype(np.float32)
    ref_i, ref_d = op.knn(X, k)
    idx, dist = pp.neighbors(torch.as_tensor(_pad(X)).cuda(), k, n_comps=d)
    idx, dist = idx.cpu().numpy(), dist.cpu().numpy()
    assert op.knn_recall(idx, ref_i) >= 0.999
    np.testing.assert_allclose(dist, ref_d, rtol=1e-4, atol=1e-4)


def test_knn_ties_and_duplicates():
    """Duplicated embeddings give exact ties; order must be (distance, index)."""
    import torch
    from paper_2605_13928_b200 import pp
    rng = np.random.default_rng(7)
    base = rng.integers(-3, 4, size=(200, 8)).astype(np.float32)   # lattice points
    X = np.concatenate([base, base, base[:50]])                     # duplicates
    k = 10
    ref_i, ref_d = op.knn(X, k)
    idx, dist = pp.neighbors(torch.as_tensor(_pad(X)).cuda(), k, n_comps=8)
    idx, dist = idx.cpu().numpy(), dist.cpu().numpy()
    np.testing.assert_allclose(dist, ref_d, atol=1e-5)
    np.testing.assert_array_equal(idx, ref_i)


def test_knn_sharded_queries():
    """Queries = a shard of the rows, keys = all rows (the multi-GPU layout)."""
    import torch
    from paper_2605_13928_b200 import pp
    rng = np.random.default_rng(3)
    X = rng.standard_normal((2500, 50)).astype(np.float32)
    Xd = torch.as_tensor(_pad(X)).cuda()
    full_i, _ = pp.neighbors(Xd, 15, n_comps=50)
    part_i, _ = pp.neighbors(Xd[1000:1700], 15, n_comps=50, keys=Xd)
    np.testing.assert_array_equal(part_i.cpu().numpy(), full_i.cpu().numpy()[1000:1700])


@pytest.mark.parametrize("n,d,k", [(15, 1, 15), (128, 62, 15), (129, 3, 15), (255, 50, 15), (256, 50, 15),
                                   (257, 50, 15), (384, 62, 64)])
def test_knn_tile_boundaries_and_widths(n, d, k):
    """Row counts around the 128-row query/key tiles and the 256-row query pairs (padding keys in
    the last tile, a pair whose second tile is empty), the narrowest and widest embeddings
    (d = 1, d = 62 = 64 - 2 augmented columns), k = n and the largest k."""
    import torch
    from paper_2605_13928_b200 import pp
    rng = np.random.default_rng(1000 * n + d)
    X = rng.standard_normal((n, d)).astype(np.float32)
    ref_i, ref_d = op.knn(X, k)
    idx, dist = pp.neighbors(torch.as_tensor(_pad(X)).cuda(), k, n_comps=d)
    idx, dist = idx.cpu().numpy(), dist.cpu().numpy()
    assert op.knn_recall(idx, ref_i) >= 0.999
    np.testing.assert_allclose(dist, ref_d, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("n", [256 * 158 - 37, 256 * 149 + 5, 256 * 147 - 3])
def test_knn_tail_split_units_and_ragged_last_tile(n):
    """Query pairs beyond one grid round: 158 pairs = 79 two-CTA cluster units on 74 co-resident
    clusters (the final partial round is split into half-scan units whose two lists per row are
    re-ranked together), 150 pairs = 75 units (one split unit), 147 pairs (odd: the last
    cluster's second CTA has no queries but still loads and releases its half of every key
    tile); the last key tile is ragged (padding keys in the second column half only).  Checked
    against the float64 oracle on random rows."""
    import torch
    from paper_2605_13928_b200 import pp
    d, k = 50, 15
    rng = np.random.default_rng(11)
    centers = rng.standard_normal((40, d)) * np.linspace(3.0, 0.5, d)
    X = (centers[rng.integers(0, 40, n)] + rng.standard_normal((n, d)) * np.linspace(1.0, 0.2, d)).astype(np.float32)
    idx, dist = pp.neighbors(torch.as_tensor(_pad(X)).cuda(), k, n_comps=d)
    idx, dist = idx.cpu().numpy(), dist.cpu().numpy()
    # rows are re-ordered along the Morton curve inside the kernel, so the split pairs' rows are
    # not a contiguous range of input rows: check a large random sample instead
    q = np.sort(rng.choice(n, 4000, replace=False))
    ref_i, ref_d = op.knn(X, k, queries=q)
    assert op.knn_recall(idx[q], ref_i) >= 0.999
    np.testing.assert_allclose(dist[q], ref_d, rtol=1e-4, atol=1e-4)
    assert np.all(idx[:, 0] == np.arange(n))
