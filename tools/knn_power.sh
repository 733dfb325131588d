#!/bin/bash
# Board power and SM clock while the kNN candidate kernel runs back to back (C3 embedding):
# nvidia-smi sampled every 100 ms during 24 consecutive pp.neighbors calls.
O=${OUT:-gpurun_out/r02j}
mkdir -p $O
make -C paper_2605_13928_b200/csrc -j16 > /dev/null 2>&1
timeout 300 python tools/knn_time.py warm lists 2 > /dev/null 2>&1   # builds the cached embedding
nvidia-smi --query-gpu=timestamp,power.draw,power.limit,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > $O/knn_power_samples.csv &
P=$!
timeout 300 python tools/knn_time.py sustained lists 24 > $O/knn_power_time.log 2>&1
kill $P
python - "$O" << 'PY'
import sys, statistics
o = sys.argv[1]
rows = [l.strip().split(", ") for l in open(f"{o}/knn_power_samples.csv") if l.strip()]
pw = [float(r[1].split()[0]) for r in rows if r[1].split()[0].replace(".", "").isdigit()]
lim = rows[0][2]
sm = [int(r[3].split()[0]) for r in rows]
busy = [p for p in pw if p > 300]
print(f"samples {len(pw)}; power limit {lim}; loaded samples {len(busy)}: median {statistics.median(busy):.0f} W, "
      f"max {max(busy):.0f} W; SM clock median {statistics.median(sm)} MHz (max {rows[0][4]})")
print(open(f"{o}/knn_power_time.log").read().strip().splitlines()[-1])
PY
