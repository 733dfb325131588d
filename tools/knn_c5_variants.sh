#!/bin/bash
# C5 (k given) timing of library variants: tools/knn_c5_variants.sh K "label:flags" ...
k=$1; shift
mkdir -p /tmp/scb_variants
for v in "$@"; do
  label="${v%%:*}"; flags="${v#*:}"
  (cd paper_2605_13928_b200/csrc && rm -f build/knn.o && make -j16 EXTRA="$flags" > /dev/null 2>&1) || { echo "build failed $label"; continue; }
  cp paper_2605_13928_b200/libscb_b200.so /tmp/scb_variants/$label.so
done
(cd paper_2605_13928_b200/csrc && rm -f build/knn.o && make -j16 > /dev/null 2>&1)
for r in 1 2; do for v in "$@"; do label="${v%%:*}"
  echo -n "$label r$r: "; SCB_LIB_PATH=/tmp/scb_variants/$label.so timeout 300 python tools/knn_only_c5.py 1000000 $k 2>&1 | tail -1 | cut -c1-160
done; done
