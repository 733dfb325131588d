"""Build the committed profile summaries from one measurement call's raw ncu outputs
(tools/gpu_call_final.sh): <dir>/tensor_pipe.csv -> tensor_pipe.json, <dir>/knn_full.ncu-rep ->
knn_traffic.json, <dir>/launches.csv -> launches_c3_summary.csv (via tools/launch_summary.py).

usage: python tools/make_profile_jsons.py gpurun_out/r02c profiles/r02c "round 2, session 3"
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

src, dst, tag = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
os.makedirs(dst, exist_ok=True)
SCALE = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}

# ---- tensor pipe per kernel (one bench step under ncu --metrics)
rows = list(csv.reader(open(os.path.join(src, "tensor_pipe.csv"))))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ki, mi, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per = collections.defaultdict(dict)
names = {}
for r in rows[start + 1:]:
    if len(r) <= vi or not r[vi]:
        continue
    names[r[ii]] = r[ki].split("(")[0].replace("void ", "").replace("scb::", "").strip()
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        v *= SCALE.get(r[ui], 1.0)
    per[r[ii]][r[mi]] = v
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for lid, m in per.items():
    n = names[lid]
    cnt[n] += 1
    for k, v in m.items():
        agg[n][k] += v
out = {"source": f"ncu --metrics gpu__time_duration, sm__pipe_tensor_cycles_active, sm__pipe_tensor_subpipe_hmma_cycles_active, "
                 f"sm__pipe_fp64_cycles_active, dram bytes; --clock-control none; one C3 bench step (tools/gpu_call_final.sh, {tag}); "
                 f"raw: {dst}/tensor_pipe.csv; values averaged over launches", "kernels": {}}
for n, m in agg.items():
    c = cnt[n]
    out["kernels"][n] = {
        "launches": c,
        "tensor_pipe_pct": round(m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0) / c, 2),
        "hmma_pipe_pct": round(m.get("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed", 0) / c, 2),
        "fp64_pipe_pct": round(m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", 0) / c, 2),
        "ms_ncu": round(m.get("gpu__time_duration.sum", 0) / c, 4),
        "dram_bytes": int((m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / c)}
json.dump(out, open(os.path.join(dst, "tensor_pipe.json"), "w"), indent=1)
subprocess.run(["cp", os.path.join(src, "tensor_pipe.csv"), os.path.join(dst, "tensor_pipe.csv")], check=True)

# ---- kNN candidate kernel, ncu --set full
raw = subprocess.run(["ncu", "-i", os.path.join(src, "knn_full.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True, check=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, units, vals = rr[0], rr[1], rr[2]
BYTES = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}
HZ = {"hz": 1e-6, "khz": 1e-3, "mhz": 1.0, "ghz": 1e3}
def get(name):
    return float(vals[h.index(name)].replace(",", "")), units[h.index(name)]
def nbytes(name):
    v, u = get(name)
    return int(round(v * BYTES[u.lower()]))
dur, du = get("gpu__time_duration.sum")
tr = {"cells": 1000000, "genes": 25000, "kernel": vals[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("scb::", ""),
      "source": f"ncu --set full --clock-control none -k regex:knn_candidates -c 1 (tools/gpu_call_final.sh), {tag}",
      "dram__bytes_read.sum": nbytes("dram__bytes_read.sum"), "dram__bytes_write.sum": nbytes("dram__bytes_write.sum"),
      "gpu__time_duration_ms": dur * SCALE.get(du, 1.0)}
for key, name in (("sm__pipe_tensor_cycles_active_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                  ("alu_pipe_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                  ("issue_active_pct", "sm__issue_active.avg.pct_of_peak_sustained_active"),
                  ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
                  ("sm_mhz", "sm__cycles_elapsed.avg.per_second")):
    try:
        v, u = get(name)
        tr[key] = v * HZ[u.lower()] if key == "sm_mhz" else v
    except (ValueError, IndexError):
        pass
json.dump(tr, open(os.path.join(dst, "knn_traffic.json"), "w"), indent=1)
det = subprocess.run(["ncu", "-i", os.path.join(src, "knn_full.ncu-rep"), "--page", "details"], capture_output=True, text=True).stdout
open(os.path.join(dst, "knn_candidates_c3_ncu_details.txt"), "w").write(det)
summ = subprocess.run([sys.executable, "tools/launch_summary.py", os.path.join(src, "launches.csv"), f"C3 bench step ({tag})",
                       "synth|sgemm"], capture_output=True, text=True).stdout
open(os.path.join(dst, "launches_c3_summary.csv"), "w").write(summ)
print(json.dumps(tr))
print(json.dumps({k: (v["tensor_pipe_pct"], v["ms_ncu"]) for k, v in out["kernels"].items()}))
