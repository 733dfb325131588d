#!/bin/bash
# PCA eigensolver A/B on one B200: PCA/edge/dist GPU tests, per-stage PCA times (C3), eigensolver launch list
mkdir -p gpurun_out/r02
make -C paper_2605_13928_b200/csrc -j16 > gpurun_out/r02/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_pca.py tests/test_gpu_edge.py tests/test_gpu_dist.py -m gpu -x -q 2>&1 | tail -3
SCB_EIG_VERBOSE=1 timeout 300 python tools/time_pca.py 2>&1 | tail -12
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dgemm|jacobi|chol|trsm|splitk|cheb" --csv python tools/time_pca.py > gpurun_out/r02/eig_ncu.csv 2>/dev/null; python tools/launch_summary.py gpurun_out/r02/eig_ncu.csv 2>/dev/null | head -20
