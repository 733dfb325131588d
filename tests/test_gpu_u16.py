"""The compact u16 CSR input (uint16 gene indices + uint16 counts, DeviceCSR.to_u16) gives
bit-identical results to the 32-bit input through every raw-matrix pass: QC, masks, subset,
normalize + log1p, HVG sums / selection, fused scale sums, and downstream PCA / kNN."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(X, mt, p):
    from paper_2605_13928_b200 import pipeline
    r = pipeline.run(X, mt, p, timing=False)
    torch.cuda.synchronize()
    out = {k: v.cpu().numpy() for k, v in r.qc.items() if v is not None}
    out.update(cell_mask=r.cell_mask.cpu().numpy(), gene_mask=r.gene_mask.cpu().numpy(),
               hvg=r.hvg_mask.cpu().numpy(), log_ip=r.X_log.indptr.cpu().numpy(), log_ix=r.X_log.indices.cpu().numpy(),
               log=r.X_log.data.cpu().numpy(), Z=r.scaled.dense().cpu().numpy(), mean=r.scaled.mean.cpu().numpy(),
               xpca=r.pca.X_pca.cpu().numpy(), knn=r.knn_index.cpu().numpy(), dist=r.knn_dist.cpu().numpy())
    return out


@pytest.mark.parametrize("n,g,seed", [(6000, 2000, 3), (5000, 40000, 4)])
def test_u16_input_bit_identical_to_f32(n, g, seed):
    from paper_2605_13928_b200 import pipeline, synth
    spec = synth.Spec(n, g, seed=seed)
    X = synth.generate(spec)
    # plant counts beyond the u16 range (escape entries), including a run of neighbours in one quad
    sel = torch.arange(5, X.nnz, 7919, device=X.data.device)
    X.data[sel] = 65535.0 + (sel % 50000).float()
    X.data[100:104] = torch.tensor([65535.0, 65536.0, 70000.0, 65534.0], device=X.data.device)
    mt = synth.mt_mask(spec)
    p = pipeline.Params(min_genes=30, max_pct_mt=25.0, n_top_genes=500, n_neighbors=10)
    Xu = X.to_u16()
    assert Xu.esc_pos.numel() == int((X.data >= 65535).sum())
    assert Xu.indices.dtype == torch.uint16 and Xu.data.dtype == torch.uint16
    assert Xu.indices.element_size() + Xu.data.element_size() == 4
    a, b = _run(X, mt, p), _run(Xu, mt, p)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    np.testing.assert_array_equal(Xu.to_f32().data.cpu().numpy(), X.data.cpu().numpy())


def test_u16_conversion_refuses_lossy_inputs():
    from paper_2605_13928_b200.pp import DeviceCSR
    ip = np.array([0, 2, 3], np.int64)
    ix = np.array([0, 5, 1], np.int32)
    for bad in ([1.0, 2.0 ** 24, 2.0], [1.0, 2.5, 2.0], [1.0, -1.0, 2.0]):
        X = DeviceCSR.from_host(ip, ix, np.array(bad, np.float32), 10)
        with pytest.raises(ValueError):
            X.to_u16()
    with pytest.raises(ValueError):
        DeviceCSR.from_host(ip, ix, np.array([1.0, 2.0, 3.0], np.float32), 70000).to_u16()
    ok = DeviceCSR.from_host(ip, ix, np.array([1.0, 65535.0, 0.0], np.float32), 65536).to_u16()
    assert ok.data.to(torch.int32).cpu().tolist() == [1, 65535, 0]
    assert ok.esc_pos.cpu().tolist() == [1] and ok.esc_val.cpu().tolist() == [65535.0]
    big = DeviceCSR.from_host(ip, ix, np.array([1.0, 100000.0, 7.0], np.float32), 65536).to_u16()
    assert big.to_f32().data.cpu().tolist() == [1.0, 100000.0, 7.0]


def test_u16_wire_decode_matches_f32():
    """scb_csr_u16_decode (the e2e wire format's device decode) restores the 32-bit CSR exactly,
    including escaped counts and a tail that is not a multiple of 8."""
    from paper_2605_13928_b200 import synth
    X = synth.generate(synth.Spec(3001, 1700, seed=8))
    X.data[7::1000] = 65535.0 + torch.arange(X.data[7::1000].numel(), device=X.data.device, dtype=torch.float32)
    Xu = X.to_u16()
    Y = Xu.to_f32()
    assert torch.equal(Y.indices, X.indices) and torch.equal(Y.data, X.data)
    n = X.nnz - 5  # odd length: exercises the tail kernel
    from paper_2605_13928_b200.pp import DeviceCSR
    part = DeviceCSR(X.indptr, Xu.indices[:n], Xu.data[:n], X.n_cols, esc_pos=Xu.esc_pos[Xu.esc_pos < n],
                     esc_val=Xu.esc_val[Xu.esc_pos < n]).to_f32()
    assert torch.equal(part.data, X.data[:n]) and torch.equal(part.indices, X.indices[:n])
