#!/bin/bash
# bench + reference arm + 2-rank functional bench + ncu tensor-pipe capture (round 2)
mkdir -p gpurun_out/r02
make -C paper_2605_13928_b200/csrc -j16 > gpurun_out/r02/build.log 2>&1 && make -C oracle >> gpurun_out/r02/build.log 2>&1 || { tail -30 gpurun_out/r02/build.log; exit 1; }
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02/bench.json 2> gpurun_out/r02/bench.err; echo "bench rc $?" >> gpurun_out/r02/bench.err
tail -c 3000 gpurun_out/r02/bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02/bench_ref.json 2> gpurun_out/r02/bench_ref.err; echo "ref rc $?" >> gpurun_out/r02/bench_ref.err
tail -c 1500 gpurun_out/r02/bench_ref.json
SCB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-e2e > gpurun_out/r02/bench_2rank_gloo.json 2> gpurun_out/r02/bench_2rank.err; echo "2rank rc $?" >> gpurun_out/r02/bench_2rank.err
tail -c 1500 gpurun_out/r02/bench_2rank_gloo.json
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"knn_candidates|gram_split|project_kernel" --csv --log-file gpurun_out/r02/tensor_pipe.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r02/ncu_bench.log 2>&1; echo "ncu rc $?" >> gpurun_out/r02/ncu_bench.log
tail -3 gpurun_out/r02/ncu_bench.log
