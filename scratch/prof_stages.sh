#!/bin/bash
# ncu --set full of the non-kNN pipeline kernels at C3 (1 step, no warmup)
ncu --set full --clock-control none -k 'regex:gram_kernel|hvg_sums|subset_fill|qc_kernel|scale_dense|scale_sums|subset_count|project_kernel|jacobi|normalize' \
    -c 12 -o gpurun_out/stages_1m python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_stages.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(?!.*synth)(?!.*cutlass).*' -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/ncu_stages.log
