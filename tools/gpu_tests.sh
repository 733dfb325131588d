#!/bin/bash
# run GPU tests: tools/gpu_tests.sh [pytest args...]   (default: the whole GPU suite)
mkdir -p gpurun_out/r02
make -C paper_2605_13928_b200/csrc -j16 > gpurun_out/r02/build.log 2>&1 || { tail -30 gpurun_out/r02/build.log; exit 1; }
nproc > gpurun_out/r02/host.txt; free -g >> gpurun_out/r02/host.txt; lscpu | grep "Model name" >> gpurun_out/r02/host.txt
args=("$@"); [ ${#args[@]} -eq 0 ] && args=(tests)
timeout 1500 python -m pytest "${args[@]}" -m gpu -x -q -s --durations=15 > gpurun_out/r02/pytest_gpu.log 2>&1
echo "pytest rc $?" >> gpurun_out/r02/pytest_gpu.log
tail -40 gpurun_out/r02/pytest_gpu.log
