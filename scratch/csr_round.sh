#!/bin/bash
# CSR-stage iteration: GPU parity tests for the CSR kernels, the 1M bench (no e2e / CPU leg),
# and a launch list + one --set full capture of the CSR kernels
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_csr.json 2> gpurun_out/bench_csr.err
python - <<'PY'
import json
j = json.loads(open("gpurun_out/bench_csr.json").read().strip().splitlines()[-1])
print(j["ms_per_step"], {k: v for k, v in j["stages"].items()})
PY
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k 'regex:qc_kernel|subset|hvg_sums|scale_sums|scale_dense|split_bf16' -c 14 --csv --log-file gpurun_out/csr_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/csr_launches.csv csr
if [ "$1" == "full" ]; then
ncu --set full --import-source on --clock-control none -k 'regex:qc_kernel|subset|hvg_sums|scale_sums' -c 5 -o gpurun_out/csr_full \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_csr.log 2>&1
fi
