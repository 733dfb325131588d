#!/bin/bash
# Synchronisation check without compute-sanitizer (closed on this pool): rebuild the library with
# SCB_MBAR_WATCHDOG (every mbarrier wait in the tcgen05/TMA pipelines bounded at ~2 s; a lost
# arrival prints the block/thread/barrier and traps) and run the GPU suites that drive them.
mkdir -p gpurun_out/r02c
(cd paper_2605_13928_b200/csrc && make clean > /dev/null && make -j16 EXTRA=-DSCB_MBAR_WATCHDOG > /dev/null 2>&1) || { echo build failed; exit 1; }
strings paper_2605_13928_b200/libscb_b200.so | grep -c "mbar watchdog" > gpurun_out/r02c/watchdog_build_check.txt
timeout 1500 python -m pytest tests/test_gpu_knn.py tests/test_gpu_pca.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py \
  tests/test_gpu_golden.py tests/test_gpu_dist.py -m gpu -q -s > gpurun_out/r02c/watchdog_suite.log 2>&1
echo "pytest rc $?" >> gpurun_out/r02c/watchdog_suite.log
grep -c "mbar watchdog" gpurun_out/r02c/watchdog_suite.log >> gpurun_out/r02c/watchdog_build_check.txt
tail -3 gpurun_out/r02c/watchdog_suite.log
(cd paper_2605_13928_b200/csrc && make clean > /dev/null && make -j16 > /dev/null 2>&1)
