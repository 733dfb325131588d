"""Summarise an ncu --csv launch list (gpu__time_duration.sum) into per-kernel totals and shares.

usage: python tools/launch_summary.py launches.csv [title] [exclude_regex] > summary.csv
(exclude_regex drops kernels that are not part of the measured step, e.g. the synthetic-input
generator's GEMM: 'synth|sgemm')
"""
import re
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def main(path, title="", exclude=""):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    mi = hdr.index("Metric Name") if "Metric Name" in hdr else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        if mi is not None and r[mi] != "gpu__time_duration.sum":  # other metrics of a multi-metric list
            continue
        name = r[ki].split("(")[0].replace("void ", "").strip()
        if exclude and re.search(exclude, name):
            continue
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list {title} (gpu__time_duration.sum, --clock-control none; cold-cache serialised"
          " replay: compare SHARES, not absolutes)")
    print("kernel,launches,total_ms,share")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k},{n},{v:.3f},{v / tot:.4f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", sys.argv[3] if len(sys.argv) > 3 else "")
