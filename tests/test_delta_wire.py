"""Byte-delta CSR wire form (pp.DeltaCSR): the torch encoder on CPU tensors against a plain numpy
decode -- escapes for large gene gaps and large counts, explicit zeros, empty rows, chunk seams."""
import numpy as np
import pytest
import torch

from paper_2605_13928_b200.pp import DeltaCSR, DeviceCSR


def _decode_np(D):
    ip = D.indptr.numpy()
    dg, dc = D.dgene.numpy().astype(np.int64), D.dcount.numpy().astype(np.float32)
    gd = dg.copy()
    gd[D.gesc_pos.numpy()] = D.gesc_val.numpy()
    dc[D.cesc_pos.numpy()] = D.cesc_val.numpy()
    ind = np.empty(len(dg), np.int64)
    for r in range(len(ip) - 1):
        b, e = ip[r], ip[r + 1]
        ind[b:e] = np.cumsum(gd[b:e] + 1) - 1
    return ind, dc


def _random_csr(rng, n, G, density, big_every=0):
    rows = []
    for r in range(n):
        if r % 7 == 3:
            rows.append(np.empty(0, np.int64))  # empty rows
            continue
        m = rng.binomial(G, density)
        rows.append(np.sort(rng.choice(G, m, replace=False)))
    ip = np.zeros(n + 1, np.int64)
    ip[1:] = np.cumsum([len(x) for x in rows])
    ind = np.concatenate(rows) if ip[-1] else np.empty(0, np.int64)
    data = rng.negative_binomial(1, 0.05, ip[-1]).astype(np.float32)  # includes explicit zeros
    if big_every:
        data[::big_every] = rng.integers(255, 1 << 24, len(data[::big_every]))
    return ip, ind.astype(np.int32), data


@pytest.mark.parametrize("G,density,chunk", [(2000, 0.05, 1 << 28), (70000, 0.002, 997), (300, 0.5, 64)])
def test_delta_roundtrip(G, density, chunk):
    rng = np.random.default_rng(G)
    ip, ind, data = _random_csr(rng, 400, G, density, big_every=53)
    X = DeviceCSR(torch.as_tensor(ip), torch.as_tensor(ind), torch.as_tensor(data), G)
    D = DeltaCSR.from_csr(X, chunk=chunk)
    assert D.dgene.dtype == torch.uint8 and D.dcount.dtype == torch.uint8
    gi, dv = _decode_np(D)
    np.testing.assert_array_equal(gi, ind)
    np.testing.assert_array_equal(dv, data)
    if G == 70000:
        assert D.gesc_pos.numel() > 0  # gaps > 254 genes escaped
    assert D.cesc_pos.numel() >= len(data[::53])


def test_delta_rejects_unsorted_and_fractional():
    ip = torch.tensor([0, 3], dtype=torch.int64)
    X = DeviceCSR(ip, torch.tensor([5, 2, 9], dtype=torch.int32), torch.ones(3), 10)
    with pytest.raises(ValueError):
        DeltaCSR.from_csr(X)
    X = DeviceCSR(ip, torch.tensor([1, 2, 9], dtype=torch.int32), torch.tensor([1.0, 0.5, 2.0]), 10)
    with pytest.raises(ValueError):
        DeltaCSR.from_csr(X)
