#!/bin/bash
# bench (1M) + ncu launch list of the same command (input generation excluded) + one --set full
# capture of the kNN candidates kernel
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(?!.*(synth|sgemm)).*' -c 1000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
if [ "$1" == "full" ]; then
ncu --set full --import-source on --clock-control none -k regex:knn_candidates -c 1 -o gpurun_out/knn_full_1m \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_knn.log 2>&1
fi
tail -2 gpurun_out/pytest_gpu.log
tail -c 300 gpurun_out/bench.json
if [ "$1" == "gram" ]; then
ncu --set full --import-source on --clock-control none -k 'regex:gram_split|split_bf16' -c 2 -o gpurun_out/gram_full_1m \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gram.log 2>&1
fi
