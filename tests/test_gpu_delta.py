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
