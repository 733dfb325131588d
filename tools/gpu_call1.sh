#!/bin/bash
# round-2 first GPU call: sanitizer logs + tensor-pipe metric names
set -x
mkdir -p gpurun_out/r02
python __graft_entry__.py > gpurun_out/r02/smoke.log 2>&1; echo smoke rc $? >> gpurun_out/r02/smoke.log
python tools/sanitize_run.py > gpurun_out/r02/plain.log 2>&1; echo rc $? >> gpurun_out/r02/plain.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_run.py > gpurun_out/r02/sanitizer_$t.log 2>&1
  echo "exit $?" >> gpurun_out/r02/sanitizer_$t.log
done
ncu --query-metrics 2>&1 | grep -i -E "pipe_tensor|pipe_tc" > gpurun_out/r02/tensor_metrics.txt
