"""The C ABI's own NCCL communicator (scb_ctx_create_comm + scb_comm_*; one GPU in this test
pool, so world size 1 -- NCCL refuses two ranks on one device): the collectives are the
world-1 identities, and the pipeline run through NcclComm equals the run without a comm."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_nccl_comm_world1_collectives_and_pipeline():
    from paper_2605_13928_b200 import pipeline, synth
    from paper_2605_13928_b200.dist import NcclComm
    nid = NcclComm.unique_id()
    assert len(nid) == 128
    comm = NcclComm(0, 0, 1, nid)
    a = torch.arange(10, dtype=torch.float64, device="cuda")
    comm.allreduce_(a)
    assert torch.equal(a, torch.arange(10, dtype=torch.float64, device="cuda"))
    b = torch.tensor([3, -4], dtype=torch.int64, device="cuda")
    comm.allreduce_(b)
    assert b.tolist() == [3, -4]
    assert comm.allreduce_int(7) == 7 and comm.allreduce_max(2.5) == 2.5
    c = torch.randn(5, 3, device="cuda")
    c0 = c.clone()
    comm.broadcast_(c, 0)
    assert torch.equal(c, c0)
    g = comm.allgather_rows(torch.randn(17, 64, device="cuda"))
    assert g.shape == (17, 64)
    spec = synth.Spec(4000, 1500, seed=6)
    X = synth.generate(spec)
    p = pipeline.Params(min_genes=30, max_pct_mt=25.0, n_top_genes=400, n_neighbors=10)
    r0 = pipeline.run(X, synth.mt_mask(spec), p, timing=False)
    r1 = pipeline.run(X, synth.mt_mask(spec), p, timing=False, comm=comm)
    torch.cuda.synchronize()
    assert torch.equal(r0.hvg_mask, r1.hvg_mask)
    assert torch.equal(r0.scaled.Z_hi, r1.scaled.Z_hi) and torch.equal(r0.scaled.Z_lo, r1.scaled.Z_lo)
    np.testing.assert_allclose(r0.pca.components.cpu().numpy(), r1.pca.components.cpu().numpy(), atol=1e-6)
    assert (r0.knn_index == r1.knn_index).float().mean().item() > 0.999
