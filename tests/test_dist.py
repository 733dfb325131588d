"""World-size-2 gloo test of the cell-sharded pipeline orchestration (collectives, shard
bookkeeping, rank-0 eigenvector broadcast, kNN key all-gather).  Device kernels are replaced
by the oracle-backed tests/cpu_backend.py; the assertion is that 2-way sharded results equal
the single-process results (bit-exact for masks/HVG/scale statistics/kNN)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp

from tests.golden import make_golden as mg


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _params(regress_out=False):
    from paper_2605_13928_b200.pipeline import Params
    P = mg.PARAMS
    return Params(min_genes=P.min_genes, max_genes=P.max_genes, max_pct_mt=P.max_pct_mt, min_cells=P.min_cells,
                  target_sum=P.target_sum, n_top_genes=P.n_top_genes, n_bins=P.n_bins, max_value=P.max_value,
                  n_comps=P.n_comps, n_neighbors=P.n_neighbors, regress_out=regress_out)


def _run(rank, world, port, out_dir, regress_out=False):
    import tests.cpu_backend as cb
    from paper_2605_13928_b200 import pipeline
    from paper_2605_13928_b200.dist import Comm, shard_rows_by_nnz
    from paper_2605_13928_b200.pp import DeviceCSR
    pipeline.pp = cb  # test-only substitution of the device step functions
    comm = None
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        td.init_process_group("gloo", rank=rank, world_size=world)
        comm = Comm()
    g = np.load("tests/golden/g600x300.npz")
    r0, r1 = shard_rows_by_nnz(g["indptr"], rank, world)
    ip = g["indptr"][r0:r1 + 1] - g["indptr"][r0]
    sl = slice(int(g["indptr"][r0]), int(g["indptr"][r1]))
    X = DeviceCSR(torch.as_tensor(ip), torch.as_tensor(g["indices"][sl]), torch.as_tensor(g["data"][sl]), 300)
    res = pipeline.run(X, torch.as_tensor(g["mt_mask"]), _params(regress_out), comm=comm, timing=False)
    np.savez(os.path.join(out_dir, f"r{rank}_w{world}.npz"), cell_mask=res.cell_mask.numpy(), Z=res.scaled.values().numpy(),
             gene_mask=res.gene_mask.numpy(), hvg=res.hvg_mask.numpy(), mean=res.scaled.mean.numpy(),
             inv=res.scaled.inv_std.numpy(), comps=res.pca.components.numpy(), var=res.pca.variance.numpy(),
             xpca=res.pca.X_pca.numpy()[:, :res.pca.n_comps], knn=res.knn_index.numpy(), n=res.n_cells_total)
    if comm is not None:
        td.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_matches_single_process(tmp_path):
    _run(0, 1, 0, str(tmp_path))
    mp.spawn(_run, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    one = np.load(tmp_path / "r0_w1.npz")
    parts = [np.load(tmp_path / f"r{r}_w2.npz") for r in range(2)]
    np.testing.assert_array_equal(np.concatenate([p["cell_mask"] for p in parts]), one["cell_mask"])
    for p in parts:
        assert int(p["n"]) == int(one["n"])
        np.testing.assert_array_equal(p["gene_mask"], one["gene_mask"])
        np.testing.assert_array_equal(p["hvg"], one["hvg"])          # integer gene sums: exact
        np.testing.assert_array_equal(p["mean"], one["mean"])
        np.testing.assert_array_equal(p["inv"], one["inv"])
        np.testing.assert_allclose(p["var"], one["var"], rtol=1e-12)
        np.testing.assert_allclose(p["comps"], one["comps"], atol=1e-10)
    np.testing.assert_allclose(np.concatenate([p["xpca"] for p in parts]), one["xpca"], atol=1e-5)
    np.testing.assert_array_equal(np.concatenate([p["knn"] for p in parts]), one["knn"])
    # and the single-process orchestration reproduces the oracle's golden outputs
    g = np.load("tests/golden/g600x300.npz")
    np.testing.assert_array_equal(one["hvg"], g["hvg_mask"])
    np.testing.assert_array_equal(one["knn"], g["knn_idx"])


@pytest.mark.timeout(300)
def test_two_rank_gloo_regress_out_matches_single_process_and_oracle(tmp_path):
    """regress_out path: all-reduced covariate sums and Aᵀl partials give the single-process
    residual scaling (float64 sums in a different order: tolerance, not bit-exact), and the
    single-process result equals the oracle's regress_out_scale."""
    from oracle import pipeline as op
    _run(0, 1, 0, str(tmp_path), True)
    mp.spawn(_run, args=(2, _port(), str(tmp_path), True), nprocs=2, join=True)
    one = np.load(tmp_path / "r0_w1.npz")
    parts = [np.load(tmp_path / f"r{r}_w2.npz") for r in range(2)]
    for p in parts:
        np.testing.assert_allclose(p["inv"], one["inv"], rtol=1e-10)
    np.testing.assert_allclose(np.concatenate([p["Z"] for p in parts]), one["Z"], rtol=1e-5, atol=1e-5)
    g = np.load("tests/golden/g600x300.npz")
    X = op.CSR(g["indptr"], g["indices"], g["data"], 300)
    P = mg.PARAMS
    import dataclasses
    o = op.run(X, g["mt_mask"], dataclasses.replace(P, regress_out=True), with_knn=False)
    np.testing.assert_allclose(one["Z"], o["Z"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(one["inv"], o["scale_inv_std"], rtol=1e-10)


def test_shard_rows_by_nnz_balances_nonzeros():
    from paper_2605_13928_b200.dist import row_shards_from_counts, shard_rows_by_nnz
    rng = np.random.default_rng(0)
    nnz = rng.integers(0, 500, 10001)
    nnz[:100] = 5000  # a dense head: equal row counts would unbalance the shards
    ip = np.r_[0, np.cumsum(nnz)]
    for world in (1, 2, 3, 8):
        sh = row_shards_from_counts(nnz, world)
        assert sh[0][0] == 0 and sh[-1][1] == len(nnz)
        assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
        z = [int(ip[e] - ip[b]) for b, e in sh]
        assert max(z) - min(z) <= 2 * 5000
        assert sh == [shard_rows_by_nnz(ip, r, world) for r in range(world)]
    assert shard_rows_by_nnz(np.zeros(5, np.int64), 1, 2) == (2, 4)  # no nonzeros: balanced row counts
