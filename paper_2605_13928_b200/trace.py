"""CudaMon-style NVML sampler that writes gputrace-compatible sessions.

The reference's harness (``/root/reference/pkg/src/gputrace``) is the pipeline-facing API the
paper's script calls between steps (cm_start / cm_timestamp / cm_stop).  This
module keeps that contract so the same session directory can be analysed with the reference's
own ``parse_session`` / ``summarize_steps`` / ``fit_linear``:

* ``start(SamplerConfig(output_dir, period, device_index))`` -> handle; ``handle.mark(label)``;
  ``handle.stop()`` (idempotent) -- as gputrace ``sampler.py:228-257, 129-155``;
* files ``metrics.csv`` (header ``elapsed_ms,device_index,gpu_util_pct,mem_used_bytes,
  mem_total_bytes,temperature_c,power_mw``), ``events.csv`` (``elapsed_ms,label``),
  ``meta.txt`` (``key=value``, schema 1) and ``marks.txt`` -- as ``traceio.py:35-65``;
* samples on the absolute grid t0 + k*period, one at t0, strictly increasing integer ms
  (+1 ms nudge), a failed read becomes a gap row -- as ``sampler.py:180-225``.

Extensions, all in extra files the reference parser ignores:
* B200 stages take 0.2-20 ms, below the 1 ms marker resolution, and the reference drops
  zero-length steps (``trace.py:270-274``): every mark is also written with microsecond
  resolution (``events_us.csv``), and ``write_device_steps`` records the CUDA-event per-step
  device times (``steps_device.csv``);
* multi-device sessions (a reference non-goal, ``SPEC.md:174``): ``start_multi`` samples
  several GPUs from ONE poller on one time grid and writes one reference-format session per
  device (``<dir>/dev<i>/``) with the same markers;
* ``summarize_session``: the reference's ``attribute_steps`` + ``summarize_steps`` semantics
  (``trace.py:250-309``) in O((S + M) log S) instead of O(steps x samples), merged with the
  device step times when present.
"""
from __future__ import annotations

import bisect
import csv
import dataclasses
import os
import threading
import time
from datetime import datetime, timezone

METRICS_HEADER = ["elapsed_ms", "device_index", "gpu_util_pct", "mem_used_bytes", "mem_total_bytes",
                  "temperature_c", "power_mw"]
EVENTS_HEADER = ["elapsed_ms", "label"]
META_ORDER = ["schema_version", "start_wall_utc", "stop_wall_utc", "period_s", "device_index", "device_name",
              "device_mem_total_bytes", "child_exit_status"]


class ReadFailure(RuntimeError):
    """Transient backend failure: the tick becomes a gap row."""


@dataclasses.dataclass(frozen=True)
class SamplerConfig:
    output_dir: str
    period: float = 1.0
    device_index: int = 0

    def __post_init__(self):
        if not self.period > 0:
            raise ValueError("period must be > 0")


class NvmlBackend:
    """NVML readings through nvidia-ml-py (pynvml)."""

    def __init__(self):
        import pynvml
        self._n = pynvml
        pynvml.nvmlInit()

    def enumerate_devices(self):
        n = self._n
        out = []
        for i in range(n.nvmlDeviceGetCount()):
            h = n.nvmlDeviceGetHandleByIndex(i)
            name = n.nvmlDeviceGetName(h)
            out.append(dict(index=i, name=name.decode() if isinstance(name, bytes) else name,
                            memory_total=int(n.nvmlDeviceGetMemoryInfo(h).total)))
        return out

    def read_instant(self, i):
        n = self._n
        try:
            h = n.nvmlDeviceGetHandleByIndex(i)
            mem = n.nvmlDeviceGetMemoryInfo(h)
            util = n.nvmlDeviceGetUtilizationRates(h)
            return dict(gpu_util_pct=float(util.gpu), mem_used_bytes=int(mem.used), mem_total_bytes=int(mem.total),
                        temperature_c=float(n.nvmlDeviceGetTemperature(h, 0)), power_mw=int(n.nvmlDeviceGetPowerUsage(h)))
        except n.NVMLError as e:  # transient -> gap row
            raise ReadFailure(str(e)) from e

    def close(self):
        try:
            self._n.nvmlShutdown()
        except Exception:
            pass


class SamplerHandle:
    def __init__(self, config: SamplerConfig, backend, device: dict, autostart: bool = True, t0: float | None = None):
        self.config = config
        self.backend = backend
        self.device = device
        os.makedirs(config.output_dir, exist_ok=True)
        self.paths = {k: os.path.join(config.output_dir, f) for k, f in
                      (("metrics", "metrics.csv"), ("events", "events.csv"), ("meta", "meta.txt"),
                       ("marks", "marks.txt"), ("events_us", "events_us.csv"))}
        self._lock = threading.Lock()
        self._stop = threading.Event()
        self._diag = []
        self._state = "running"
        self._last_ms = -1
        self._read_failures = 0
        self.start_wall = datetime.now(timezone.utc)
        self.t0 = time.monotonic() if t0 is None else t0
        self._mf = open(self.paths["metrics"], "w", newline="")
        self._ef = open(self.paths["events"], "w", newline="")
        self._uf = open(self.paths["events_us"], "w", newline="")
        self._mw, self._ew = csv.writer(self._mf, lineterminator="\n"), csv.writer(self._ef, lineterminator="\n")
        self._uw = csv.writer(self._uf, lineterminator="\n")
        self._mw.writerow(METRICS_HEADER)
        self._ew.writerow(EVENTS_HEADER)
        self._uw.writerow(["elapsed_us", "label"])
        self._mf.flush()
        self._ef.flush()
        self._uf.flush()
        open(self.paths["marks"], "a").close()
        self._write_meta(stopped=False)
        self._thread = None
        if autostart:
            self._thread = threading.Thread(target=self._poll, name="scb-trace-poller", daemon=True)
            self._thread.start()

    def _elapsed_ms(self):
        return int(round((time.monotonic() - self.t0) * 1000.0))

    def _poll(self):
        k = 0
        while not self._stop.is_set():
            self._sample()
            k += 1
            delay = self.t0 + k * self.config.period - time.monotonic()
            if delay > 0 and self._stop.wait(delay):
                break

    def _sample(self):
        idx = self.config.device_index
        try:
            r = self.backend.read_instant(idx)
            row = [r["gpu_util_pct"], r["mem_used_bytes"], r["mem_total_bytes"], r["temperature_c"], r["power_mw"]]
        except ReadFailure:
            self._read_failures += 1
            row = ["", "", "", "", ""]
        except Exception as e:  # backend bug: record and stop polling
            self._diag.append(f"poller stopped: {e!r}")
            self._stop.set()
            return
        with self._lock:
            ms = max(self._elapsed_ms(), self._last_ms + 1)
            self._last_ms = ms
            self._mw.writerow([ms, idx] + row)
            self._mf.flush()

    def mark(self, label: str, t: float | None = None):
        if not label:
            raise ValueError("label must be non-empty")
        t = time.monotonic() if t is None else t
        with self._lock:
            if self._state != "running":
                raise RuntimeError("sampler stopped")
            self._ew.writerow([int(round((t - self.t0) * 1000.0)), label])
            self._uw.writerow([int(round((t - self.t0) * 1e6)), label])
            self._ef.flush()
            self._uf.flush()

    def stop(self):
        with self._lock:
            if self._state == "stopped":
                return dict(self.paths)
            self._state = "stopped"
        self._stop.set()
        if self._thread is not None:
            self._thread.join()
        if self._read_failures:
            self._diag.append(f"read_failures={self._read_failures}")
        self._write_meta(stopped=True)
        self._mf.close()
        self._ef.close()
        self._uf.close()
        return dict(self.paths)

    def _write_meta(self, stopped: bool):
        meta = {"schema_version": "1", "start_wall_utc": self.start_wall.isoformat(),
                "period_s": str(self.config.period), "device_index": str(self.config.device_index),
                "device_name": self.device["name"], "device_mem_total_bytes": str(self.device["memory_total"])}
        if stopped:
            meta["stop_wall_utc"] = datetime.now(timezone.utc).isoformat()
        lines = [f"{k}={meta[k]}" for k in META_ORDER if k in meta] + [f"diagnostic={d}" for d in self._diag]
        with open(self.paths["meta"], "w") as f:
            f.write("".join(x + "\n" for x in lines))


def start(config: SamplerConfig, backend=None) -> SamplerHandle:
    backend = backend if backend is not None else NvmlBackend()
    devs = {d["index"]: d for d in backend.enumerate_devices()}
    if config.device_index not in devs:
        raise ValueError(f"unknown device {config.device_index}")
    return SamplerHandle(config, backend, devs[config.device_index])


def write_device_steps(session_dir: str, step_ms: dict, extra: dict | None = None):
    """steps_device.csv: CUDA-event device time per pipeline step (max over ranks)."""
    path = os.path.join(session_dir, "steps_device.csv")
    with open(path, "w", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(["step", "device_ms"])
        for k, v in step_ms.items():
            w.writerow([k, f"{v:.4f}"])
    if extra:
        with open(os.path.join(session_dir, "meta_pipeline.txt"), "w") as f:
            f.write("".join(f"{k}={v}\n" for k, v in extra.items()))
    return path


class MultiSamplerHandle:
    """One poller thread sampling several devices on one absolute grid; one reference-format
    session per device under ``<output_dir>/dev<i>/``; marks go to every device's session with
    the same timestamp."""

    def __init__(self, output_dir: str, devices, period: float, backend, infos: dict):
        self.t0 = time.monotonic()
        self.period = period
        self.handles = [SamplerHandle(SamplerConfig(os.path.join(output_dir, f"dev{d}"), period, d), backend, infos[d],
                                      autostart=False, t0=self.t0) for d in devices]
        self._stop = threading.Event()
        self._thread = threading.Thread(target=self._poll, name="scb-trace-multi", daemon=True)
        self._thread.start()

    def _poll(self):
        k = 0
        while not self._stop.is_set():
            for h in self.handles:
                h._sample()
            k += 1
            delay = self.t0 + k * self.period - time.monotonic()
            if delay > 0 and self._stop.wait(delay):
                break

    def mark(self, label: str):
        t = time.monotonic()
        for h in self.handles:
            h.mark(label, t)

    def stop(self):
        self._stop.set()
        self._thread.join()
        return [h.stop() for h in self.handles]


def start_multi(output_dir: str, devices=None, period: float = 1.0, backend=None) -> MultiSamplerHandle:
    if not period > 0:
        raise ValueError("period must be > 0")
    backend = backend if backend is not None else NvmlBackend()
    infos = {d["index"]: d for d in backend.enumerate_devices()}
    devices = sorted(infos) if devices is None else list(devices)
    for d in devices:
        if d not in infos:
            raise ValueError(f"unknown device {d}")
    return MultiSamplerHandle(output_dir, devices, period, backend, infos)


def _wall_ms(meta: dict):
    try:
        a = datetime.fromisoformat(meta["start_wall_utc"])
        b = datetime.fromisoformat(meta["stop_wall_utc"])
        return int(round((b - a).total_seconds() * 1000))
    except (KeyError, ValueError):
        return None


def summarize_session(session_dir: str):
    """Per-step summary with the reference's semantics (gputrace trace.py:250-309: half-open
    tiling from the first marker to the session end, a "(pre)" step only when samples precede
    the first marker, zero-length steps dropped, per-step peak memory / mean utilisation over
    non-gap samples, sample_count including gap rows, duration = max(wall span, last sample,
    last marker)) computed with binary searches -- O((S + M) log S) instead of O(steps x S).
    Adds ``device_ms`` from steps_device.csv when that file exists."""
    with open(os.path.join(session_dir, "metrics.csv")) as f:
        rows = list(csv.reader(f))[1:]
    t = [int(r[0]) for r in rows]
    mem = [int(r[3]) if r[3] != "" else None for r in rows]
    util = [float(r[2]) if r[2] != "" else None for r in rows]
    with open(os.path.join(session_dir, "events.csv")) as f:
        marks = [(int(r[0]), r[1]) for r in list(csv.reader(f))[1:]]
    meta = {}
    with open(os.path.join(session_dir, "meta.txt")) as f:
        for line in f:
            if "=" in line:
                k, v = line.rstrip("\n").split("=", 1)
                meta.setdefault(k, v)
    if not marks:
        raise ValueError("session has no event markers")
    cands = [c for c in (_wall_ms(meta), t[-1] if t else None, marks[-1][0]) if c is not None]
    duration = max(cands)
    steps = []
    if t and t[0] < marks[0][0]:
        steps.append(("(pre)", 0, marks[0][0]))
    for i, (m, lab) in enumerate(marks):
        end = marks[i + 1][0] if i + 1 < len(marks) else duration
        if m != end:
            steps.append((lab, m, end))
    dev = {}
    p = os.path.join(session_dir, "steps_device.csv")
    if os.path.exists(p):
        with open(p) as f:
            dev = {r[0]: float(r[1]) for r in list(csv.reader(f))[1:]}
    out = []
    for lab, a, b in steps:
        i0, i1 = bisect.bisect_left(t, a), bisect.bisect_left(t, b)
        ms = [v for v in mem[i0:i1] if v is not None]
        us = [v for v in util[i0:i1] if v is not None]
        out.append(dict(label=lab, start_ms=a, end_ms=b, runtime_s=(b - a) / 1000, peak_gpu_mem_bytes=max(ms) if ms else None,
                        mean_gpu_util_pct=sum(us) / len(us) if us else None, sample_count=i1 - i0,
                        device_ms=dev.get(lab)))
    return out
