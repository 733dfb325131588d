#!/bin/bash
# CSR-stage A/B on one B200: CSR/QC GPU tests, then a short C3 bench (device step only)
mkdir -p gpurun_out/r02
make -C paper_2605_13928_b200/csrc -j16 > gpurun_out/r02/build.log 2>&1 || { tail -20 gpurun_out/r02/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_csr.py tests/test_gpu_golden.py tests/test_gpu_edge.py tests/test_gpu_u16.py tests/test_gpu_upload.py tests/test_gpu_parity_scale.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/csr_ab.json 2> gpurun_out/r02/csr_ab.err
python -c "import json; d=json.load(open('gpurun_out/r02/csr_ab.json')); print(d['ms_per_step'], d['step_ms'], d['stages']['qc'], d['stages']['norm_hvg'])"
