#!/bin/bash
# run the GPU test suite (optionally a subset: $1 = pytest -k expression / path)
mkdir -p gpurun_out/r02
make -C paper_2605_13928_b200/csrc -j16 > gpurun_out/r02/build.log 2>&1 || { tail -30 gpurun_out/r02/build.log; exit 1; }
nproc > gpurun_out/r02/host.txt; free -g >> gpurun_out/r02/host.txt; lscpu | grep "Model name" >> gpurun_out/r02/host.txt
timeout 1500 python -m pytest ${1:-tests} -m gpu -x -q -s --durations=15 ${@:2} > gpurun_out/r02/pytest_gpu.log 2>&1
echo "pytest rc $?" >> gpurun_out/r02/pytest_gpu.log
tail -40 gpurun_out/r02/pytest_gpu.log
