#!/bin/bash
# one --set full capture per CSR-stage kernel of the 1M bench step (+ regress_out kernels)
ncu --set full --import-source on --clock-control none -k 'regex:qc_kernel|subset_count|subset_fill_sums|hvg_sums|scale_dense' -c 5 \
    -o gpurun_out/csr_v13_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_csr13.log 2>&1
ncu --set full --clock-control none -k 'regex:regress_xty|regress_apply' -c 2 \
    -o gpurun_out/regress_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --regress-out > gpurun_out/ncu_reg.log 2>&1
for f in csr_v13_full regress_full; do
  ncu -i gpurun_out/$f.ncu-rep --page details 2>&1 | grep -E "^  [a-zA-Z_].*\(|Duration|DRAM Throughput|Memory Throughput|Compute \(SM\) Throughput|Issue Slots Busy|highest-utilized|Achieved Occupancy|L1/TEX Cache Throughput|Registers Per" > gpurun_out/$f.txt
done
ncu -i gpurun_out/csr_v13_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum > gpurun_out/csr_v13_traffic.csv 2>&1
