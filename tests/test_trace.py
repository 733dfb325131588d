"""The NVML sampler writes sessions the reference's own gputrace parser accepts (when the
reference is importable in this container), with a deterministic fake backend."""
import os
import sys
import time

import pytest

from paper_2605_13928_b200 import trace

REF = "/root/reference/pkg/src"


class FakeBackend:
    def __init__(self):
        self.n = 0

    def enumerate_devices(self):
        return [dict(index=0, name="SIM-B200", memory_total=183_359 * 2**20)]

    def read_instant(self, i):
        self.n += 1
        if self.n == 3:
            raise trace.ReadFailure("flaky")
        return dict(gpu_util_pct=50.0, mem_used_bytes=10 * 2**30, mem_total_bytes=183_359 * 2**20,
                    temperature_c=40.0, power_mw=500_000)

    def close(self):
        pass


def test_session_roundtrip(tmp_path):
    h = trace.start(trace.SamplerConfig(str(tmp_path), period=0.05), backend=FakeBackend())
    for lab in ("qc", "norm_hvg", "regress", "pca", 'knn, "k=15"'):
        time.sleep(0.06)
        h.mark(lab)
    time.sleep(0.05)
    paths = h.stop()
    assert h.stop() == paths  # idempotent
    with pytest.raises(RuntimeError):
        h.mark("late")
    lines = open(paths["metrics"]).read().splitlines()
    assert lines[0] == "elapsed_ms,device_index,gpu_util_pct,mem_used_bytes,mem_total_bytes,temperature_c,power_mw"
    ms = [int(l.split(",")[0]) for l in lines[1:]]
    assert ms == sorted(ms) and len(set(ms)) == len(ms) and len(ms) >= 5
    assert any(l.endswith(",,,,,") for l in lines[1:])  # gap row for the failed read
    meta = open(paths["meta"]).read()
    assert meta.startswith("schema_version=1\n") and "diagnostic=read_failures=1" in meta
    trace.write_device_steps(str(tmp_path), {"qc": 6.1, "knn": 187.0})
    assert open(os.path.join(tmp_path, "steps_device.csv")).read().startswith("step,device_ms\nqc,6.1000")
    if os.path.isdir(REF):
        sys.path.insert(0, REF)
        try:
            import gputrace
        finally:
            sys.path.remove(REF)
        s = gputrace.parse_session(str(tmp_path))
        steps = gputrace.summarize_steps(s)
        labels = [st.label for st in steps]
        assert labels[-5:] == ["qc", "norm_hvg", "regress", "pca", 'knn, "k=15"']
        assert gputrace.peak_gpu_memory(s) == 10 * 2**30
