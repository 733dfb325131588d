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


class FakeMulti(FakeBackend):
    def enumerate_devices(self):
        return [dict(index=i, name=f"SIM-B200-{i}", memory_total=183_359 * 2**20) for i in range(3)]

    def read_instant(self, i):
        self.n += 1
        return dict(gpu_util_pct=10.0 * (i + 1), mem_used_bytes=(i + 1) * 2**30 + self.n, mem_total_bytes=183_359 * 2**20,
                    temperature_c=40.0, power_mw=400_000 + i)


def _ref():
    if not os.path.isdir(REF):
        return None
    sys.path.insert(0, REF)
    try:
        import gputrace
    finally:
        sys.path.remove(REF)
    return gputrace


def _same_as_reference(gputrace, d, ours):
    ref = gputrace.summarize_steps(gputrace.parse_session(str(d)))
    assert [s.label for s in ref] == [o["label"] for o in ours]
    for r, o in zip(ref, ours):
        assert r.runtime_s == o["runtime_s"] and r.sample_count == o["sample_count"]
        assert r.peak_gpu_mem_bytes == o["peak_gpu_mem_bytes"] and r.mean_gpu_util_pct == o["mean_gpu_util_pct"]


def test_multi_device_session_and_us_marks(tmp_path):
    h = trace.start_multi(str(tmp_path), devices=[0, 2], period=0.02, backend=FakeMulti())
    for lab in ("qc", "norm_hvg", "regress", "pca", "knn"):
        time.sleep(0.03)
        h.mark(lab)
    time.sleep(0.03)
    paths = h.stop()
    assert len(paths) == 2
    for dev in (0, 2):
        d = tmp_path / f"dev{dev}"
        ev = open(d / "events.csv").read().splitlines()[1:]
        us = open(d / "events_us.csv").read().splitlines()[1:]
        assert [e.split(",")[1] for e in ev] == ["qc", "norm_hvg", "regress", "pca", "knn"]
        for e, u in zip(ev, us):  # same instant at both resolutions
            assert abs(int(e.split(",")[0]) - int(u.split(",")[0]) / 1000) <= 0.5
        rows = open(d / "metrics.csv").read().splitlines()[1:]
        assert all(r.split(",")[1] == str(dev) for r in rows) and len(rows) >= 5
        trace.write_device_steps(str(d), {"qc": 4.1, "knn": 146.0})
        ours = trace.summarize_session(str(d))
        assert [o["label"] for o in ours][-5:] == ["qc", "norm_hvg", "regress", "pca", "knn"]
        assert ours[-1]["device_ms"] == 146.0
        g = _ref()
        if g is not None:
            _same_as_reference(g, d, ours)
    # the two devices' marks are identical
    assert open(tmp_path / "dev0" / "events_us.csv").read() == open(tmp_path / "dev2" / "events_us.csv").read()


def test_summarize_session_matches_reference_on_a_large_session(tmp_path):
    """100k samples x 1000 markers (with gaps, a pre-marker segment and duplicate-timestamp
    markers): the same per-step numbers as the reference, without its O(steps x samples) scan."""
    import random
    rnd = random.Random(5)
    with open(tmp_path / "metrics.csv", "w") as f:
        f.write("elapsed_ms,device_index,gpu_util_pct,mem_used_bytes,mem_total_bytes,temperature_c,power_mw\n")
        for i in range(100_000):
            if rnd.random() < 0.01:
                f.write(f"{10 * i},0,,,,,\n")
            else:
                f.write(f"{10 * i},0,{rnd.randint(0, 100)},{rnd.randint(1, 1 << 36)},{1 << 37},40,500000\n")
    marks = sorted(rnd.randint(500, 999_000) for _ in range(1000))
    marks[10] = marks[11]  # zero-length step
    with open(tmp_path / "events.csv", "w") as f:
        f.write("elapsed_ms,label\n" + "".join(f"{m},step{i}\n" for i, m in enumerate(marks)))
    with open(tmp_path / "meta.txt", "w") as f:
        f.write("schema_version=1\nstart_wall_utc=2026-01-01T00:00:00+00:00\nstop_wall_utc=2026-01-01T00:16:40.5+00:00\n"
                "period_s=0.01\ndevice_index=0\ndevice_name=SIM\ndevice_mem_total_bytes=137438953472\n")
    t0 = time.perf_counter()
    ours = trace.summarize_session(str(tmp_path))
    dt = time.perf_counter() - t0
    assert ours[0]["label"] == "(pre)" and len(ours) == 1000  # 1000 marks + pre - 1 zero-length
    assert dt < 5.0
    g = _ref()
    if g is not None:
        _same_as_reference(g, tmp_path, ours)
