#!/bin/bash
# DRAM bytes / duration / clock of the kNN candidate kernel for library variants (ncu --metrics,
# one launch each): tools/knn_ncu_variants.sh "label:EXTRA flags" ...
mkdir -p /tmp/scb_variants gpurun_out/s3
for v in "$@"; do
  label="${v%%:*}"; flags="${v#*:}"
  (cd paper_2605_13928_b200/csrc && rm -f build/knn.o && make -j16 EXTRA="$flags" > /dev/null 2>&1) || { echo "build failed $label"; continue; }
  cp paper_2605_13928_b200/libscb_b200.so /tmp/scb_variants/$label.so
done
(cd paper_2605_13928_b200/csrc && rm -f build/knn.o && make -j16 > /dev/null 2>&1)
SCB_LIB_PATH=/tmp/scb_variants/${1%%:*}.so timeout 300 python tools/knn_time.py warm lists 1 > /dev/null 2>&1  # cache the embedding
for v in "$@"; do
  label="${v%%:*}"
  SCB_LIB_PATH=/tmp/scb_variants/$label.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:knn_candidates -c 1 --csv python tools/knn_time.py "$label" lists 1 2>/dev/null | \
    python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; print('$label', [(r[h.index('Metric Name')], r[h.index('Metric Value')], r[h.index('Metric Unit')]) for r in rows[1:]])"
done
