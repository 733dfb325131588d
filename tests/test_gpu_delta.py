"""GPU decode of the byte-delta CSR wire form (scb_csr_delta8_decode) is bit-identical to the
32-bit CSR it was encoded from: random matrices with escapes / empty rows / explicit zeros, and
a 16k-row window of the C3 matrix (device generator)."""
import numpy as np
import pytest

from tests.test_delta_wire import _random_csr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G,density", [(2000, 0.05), (70000, 0.002), (25000, 0.08)])
def test_delta8_decode_matches_source(G, density):
    import torch
    from paper_2605_13928_b200.pp import DeltaCSR, DeviceCSR
    rng = np.random.default_rng(G + 1)
    ip, ind, data = _random_csr(rng, 3000, G, density, big_every=101)
    X = DeviceCSR.from_host(ip, ind, data, G)
    D = DeltaCSR.from_csr(X)
    Y = D.to_f32()
    torch.cuda.synchronize()
    assert torch.equal(Y.indices, X.indices)
    assert torch.equal(Y.data, X.data)


def test_delta8_c3_window_and_pipeline_input():
    import torch
    from paper_2605_13928_b200 import synth
    from paper_2605_13928_b200.pp import DeltaCSR
    spec = synth.Spec(1_000_000, 25_000, seed=0)
    X = synth.generate_rows(spec, 400_000, 416_384)
    D = DeltaCSR.from_csr(X)
    Y = D.to_f32()
    torch.cuda.synchronize()
    assert torch.equal(Y.indices, X.indices) and torch.equal(Y.data, X.data)
    # 2 bytes per nonzero plus the escape tables
    wire = sum(t.numel() * t.element_size() for t in D.tensors())
    assert wire < 2.2 * X.nnz + 8 * (X.n_rows + 1) + 64
    print(f"C3 window: {X.nnz} nonzeros, {D.gesc_pos.numel()} gene-gap and {D.cesc_pos.numel()} count escapes, "
          f"{wire / X.nnz:.3f} B per nonzero on the wire")


@pytest.mark.parametrize("seed", [0, 1])
def test_delta8_decode_tiny_rows_and_edge_escapes(seed):
    """Rows of 0-9 entries (every window partial, row starts at every offset mod 4), gene gaps
    > 254 at a row's first entry and across its last entries, counts >= 255 on first and last
    entries, total nnz not a multiple of 4 (the byte-load tail at the end of the streams)."""
    import torch
    from paper_2605_13928_b200.pp import DeltaCSR, DeviceCSR
    rng = np.random.default_rng(seed)
    G, n = 40000, 5001
    lens = rng.integers(0, 10, n)
    rows = [np.sort(rng.choice(G, m, replace=False)) for m in lens]
    ip = np.zeros(n + 1, np.int64)
    ip[1:] = np.cumsum(lens)
    if ip[-1] % 4 == 0:  # make the stream length ragged
        rows[-1] = np.sort(np.append(rows[-1][:0], rng.choice(G, 1)))
        lens[-1] = 1
        ip[1:] = np.cumsum(lens)
    ind = np.concatenate(rows).astype(np.int32)
    data = rng.integers(1, 5, ip[-1]).astype(np.float32)
    first, last = ip[:-1][lens > 0], ip[1:][lens > 0] - 1
    data[first[::3]] = rng.integers(255, 1 << 20, len(first[::3]))
    data[last[1::3]] = rng.integers(255, 1 << 20, len(last[1::3]))
    X = DeviceCSR.from_host(ip, ind, data, G)
    D = DeltaCSR.from_csr(X)
    assert D.gesc_pos.numel() > 0 and D.cesc_pos.numel() > 0
    Y = D.to_f32()
    torch.cuda.synchronize()
    assert torch.equal(Y.indices, X.indices)
    assert torch.equal(Y.data, X.data)
