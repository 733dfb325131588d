#!/bin/bash
# A/B kNN candidate-kernel variants in one session: each "label:EXTRA flags" is built into its
# own copy of the library, then the variants are timed in alternating rounds.
# usage: [KNN_REPS=n] tools/knn_variants.sh ROUNDS "label:flags" ...  (KNN_REPS: back-to-back calls per timing, default 3)
rounds=$1; shift
mkdir -p /tmp/scb_variants
for v in "$@"; do
  label="${v%%:*}"; flags="${v#*:}"
  (cd paper_2605_13928_b200/csrc && rm -f build/knn.o && make -j16 EXTRA="$flags" > /dev/null 2>&1) || { echo "build failed $label"; continue; }
  cp paper_2605_13928_b200/libscb_b200.so /tmp/scb_variants/$label.so
done
(cd paper_2605_13928_b200/csrc && rm -f build/knn.o && make -j16 > /dev/null 2>&1)
for r in $(seq 1 $rounds); do
  for v in "$@"; do
    label="${v%%:*}"
    SCB_LIB_PATH=/tmp/scb_variants/$label.so timeout 300 python tools/knn_time.py "$label r$r" lists ${KNN_REPS:-3} 2>&1 | grep "knn time\|Error" | tail -1
  done
done
