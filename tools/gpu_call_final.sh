#!/bin/bash
# round-2 measurement call: bench (+cpu_baseline, e2e), reference arm, ncu launch list of one
# bench step, ncu --set full of the kNN candidate kernel, tensor-pipe metrics of the tcgen05 kernels
set -u
O=${OUT:-gpurun_out/r02/final}
mkdir -p $O
make -C paper_2605_13928_b200/csrc -j16 > $O/build.log 2>&1 && make -C oracle >> $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 1200 python bench.py --steps ${STEPS:-10} --warmup ${WARMUP:-3} > $O/bench.json 2> $O/bench.err; echo "bench rc $?" >> $O/bench.err
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc $?" >> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu1 rc $?" >> $O/ncu_launches.log
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"knn_candidates|gram_split|project_planes|dgemm_kernel" --csv --log-file $O/tensor_pipe.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_tensor.log 2>&1; echo "ncu2 rc $?" >> $O/ncu_tensor.log
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:knn_candidates -c 1 -o $O/knn_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu3 rc $?" >> $O/ncu_full.log
tail -c 400 $O/bench.json; tail -c 300 $O/bench_ref.json; for f in $O/ncu_launches.log $O/ncu_tensor.log $O/ncu_full.log; do tail -n 1 $f; done
