"""Two ranks running the REAL sm_100a kernels (both on cuda:0, gloo collectives through host
memory -- a functional check of the multi-rank path, not a timing configuration): cells
sharded by nonzeros (dist.shard_rows_by_nnz), integer gene-sum / Gram all-reduces, rank-0
eigenvector broadcast and the embedding all-gather for the kNN keys.  The sharded results must
equal the single-rank run: masks, HVG set and scale statistics bit-identical (integer sums are
order independent), Gram / PCA within fp64 reduction-order rounding, kNN indices identical up
to FP rounding of near-ties (recall >= 0.9999), and the neighbors graph consistent."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N, G = 24000, 3000


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _params(regress_out=False):
    from paper_2605_13928_b200.pipeline import Params
    return Params(min_genes=100, max_pct_mt=20.0, n_top_genes=1000, n_neighbors=15, regress_out=regress_out,
                  connectivities=not regress_out)


def _run(rank, world, port, out_dir, regress_out):
    from paper_2605_13928_b200 import pipeline, synth
    from paper_2605_13928_b200.dist import Comm, row_shards_from_counts
    torch.cuda.set_device(0)
    comm = None
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        td.init_process_group("gloo", rank=rank, world_size=world)
        comm = Comm()
    spec = synth.Spec(N, G, seed=11)
    r0, r1 = row_shards_from_counts(synth.row_nnz(spec).cpu().numpy(), world)[rank]
    X = synth.generate_rows(spec, r0, r1)
    res = pipeline.run(X, synth.mt_mask(spec), _params(regress_out), comm=comm, timing=False)
    torch.cuda.synchronize()
    out = dict(rows=np.array([r0, r1, X.nnz]), cell_mask=res.cell_mask.cpu().numpy(),
               gene_mask=res.gene_mask.cpu().numpy(), hvg=res.hvg_mask.cpu().numpy(),
               mean=res.scaled.mean.cpu().numpy(), inv=res.scaled.inv_std.cpu().numpy(),
               Z=res.scaled.values().cpu().numpy(), comps=res.pca.components.cpu().numpy(),
               var=res.pca.variance.cpu().numpy(), xpca=res.pca.X_pca[:, :res.pca.n_comps].cpu().numpy(),
               knn=res.knn_index.cpu().numpy(), n=np.array(res.n_cells_total))
    if res.graph is not None:
        out["conn_indptr"] = res.graph.connectivities.indptr.cpu().numpy()
        out["conn_nnz"] = np.array(res.graph.connectivities.nnz)
    np.savez(os.path.join(out_dir, f"r{rank}_w{world}.npz"), **out)
    if comm is not None:
        td.destroy_process_group()


def _spawn(tmp_path, regress_out):
    ctx = mp.get_context("spawn")
    p1 = ctx.Process(target=_run, args=(0, 1, 0, str(tmp_path), regress_out))
    p1.start()
    p1.join()
    assert p1.exitcode == 0
    mp.spawn(_run, args=(2, _port(), str(tmp_path), regress_out), nprocs=2, join=True)
    return np.load(tmp_path / "r0_w1.npz"), [np.load(tmp_path / f"r{r}_w2.npz") for r in range(2)]


@pytest.mark.timeout(600)
def test_two_ranks_real_kernels_match_single_rank(tmp_path):
    one, parts = _spawn(tmp_path, False)
    # nnz-balanced, contiguous shards
    (a0, a1, z0), (b0, b1, z1) = parts[0]["rows"], parts[1]["rows"]
    assert a0 == 0 and a1 == b0 and b1 == N
    assert abs(int(z0) - int(z1)) <= 2 * G
    np.testing.assert_array_equal(np.concatenate([p["cell_mask"] for p in parts]), one["cell_mask"])
    for p in parts:
        assert int(p["n"]) == int(one["n"])
        np.testing.assert_array_equal(p["gene_mask"], one["gene_mask"])
        np.testing.assert_array_equal(p["hvg"], one["hvg"])
        np.testing.assert_array_equal(p["mean"], one["mean"])
        np.testing.assert_array_equal(p["inv"], one["inv"])
        # the Gram is fp32-accumulated per shard (different partial-sum boundaries): ~1e-7 relative
        np.testing.assert_allclose(p["var"], one["var"], rtol=1e-6)
        c = np.abs(np.sum(p["comps"].astype(np.float64) * one["comps"], axis=1))
        assert c.min() > 1 - 1e-6, c.min()
    np.testing.assert_array_equal(np.concatenate([p["Z"] for p in parts]), one["Z"])  # row-local kernel
    np.testing.assert_allclose(np.concatenate([p["xpca"] for p in parts]), one["xpca"], atol=1e-4)
    knn2 = np.concatenate([p["knn"] for p in parts])
    hit = sum(len(np.intersect1d(a, b)) for a, b in zip(knn2, one["knn"]))
    assert hit / one["knn"].size >= 0.9999
    assert abs(int(parts[0]["conn_nnz"]) + int(parts[1]["conn_nnz"]) - int(one["conn_nnz"])) <= 0.001 * int(one["conn_nnz"])


@pytest.mark.timeout(600)
def test_two_ranks_real_kernels_regress_out(tmp_path):
    one, parts = _spawn(tmp_path, True)
    for p in parts:
        np.testing.assert_allclose(p["inv"], one["inv"], rtol=1e-10)
    np.testing.assert_allclose(np.concatenate([p["Z"] for p in parts]), one["Z"], rtol=1e-5, atol=1e-5)
