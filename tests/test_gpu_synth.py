"""The device generator (csrc/synth.cu via paper_2605_13928_b200.synth) and the CPU generator
(oracle/synth.py) produce the same CSR entry for entry: at C1 (10k x 2k) and on a 16k-row
window of the C3 matrix (1M x 25k, seed 0) that the bench runs on.  This ties the benched
device-generated input to the oracle's model (bench.py's cpu_baseline and the C3 parity tests
take their inputs from the device generator)."""
import os

import numpy as np
import pytest

from oracle.synth import SynthSpec, generate_csr

pytestmark = pytest.mark.gpu


def _device_rows(n, g, seed, r0, r1):
    from paper_2605_13928_b200 import synth
    X = synth.generate_rows(synth.Spec(n, g, seed=seed), r0, r1)
    ip, ix, d, _ = X.to_host()
    return ip, ix, d


def _check(n, g, seed, r0, r1):
    ip, ix, d = _device_rows(n, g, seed, r0, r1)
    threads = max(1, min(32, len(os.sched_getaffinity(0))))
    oip, oix, od = generate_csr(SynthSpec(n, g, seed=seed), rows=(r0, r1), threads=threads)
    assert np.array_equal(ip, oip), "row nnz differ"
    assert np.array_equal(ix, oix), "gene indices differ"
    assert np.array_equal(d, od), "counts differ"
    return len(d)


def test_synth_c1_identical():
    z = _check(10000, 2000, 1, 0, 10000)
    assert 0.05 < z / 2e7 < 0.12


def test_synth_c3_window_identical():
    z = _check(1_000_000, 25_000, 0, 500_000, 516_384)
    assert 0.05 < z / (16384 * 25000) < 0.12


def test_synth_c3_windows_identical_to_c_oracle():
    """Four more 16k-row windows spread over the C3 matrix (first, last and two inside) against
    the C restatement of the generator (oracle/csynth.c, itself == numpy in test_oracle.py)."""
    import subprocess
    from oracle import synth as osynth
    if osynth.native_lib() is None:
        subprocess.run(["make", "-C", "oracle"], check=True, capture_output=True)
    spec = SynthSpec(1_000_000, 25_000, seed=0)
    for r0 in (0, 250_000, 750_000, 1_000_000 - 16384):
        ip, ix, d = _device_rows(1_000_000, 25_000, 0, r0, r0 + 16384)
        oip, oix, od = osynth.generate_csr_native(spec, rows=(r0, r0 + 16384))
        assert np.array_equal(ip, oip) and np.array_equal(ix, oix) and np.array_equal(d, od), r0


def test_synth_row_windows_compose():
    """Shards generated separately concatenate to the whole matrix (cell sharding)."""
    from paper_2605_13928_b200 import synth
    spec = synth.Spec(5000, 1500, seed=4)
    whole = synth.generate(spec).to_host()
    a = synth.generate_rows(spec, 0, 2100).to_host()
    b = synth.generate_rows(spec, 2100, 5000).to_host()
    assert np.array_equal(whole[1], np.concatenate([a[1], b[1]]))
    assert np.array_equal(whole[2], np.concatenate([a[2], b[2]]))
    assert np.array_equal(whole[0], np.concatenate([a[0][:-1], b[0] + a[0][-1]]))
