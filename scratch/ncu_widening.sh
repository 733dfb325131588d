#!/bin/bash
# one --set full capture per widened component's main kernel at 1M cells (bench --umap --de)
for k in umap_epoch_kernel move_decide_kernel refine_decide_kernel de_sums_kernel umap_weights_kernel fuzzy_fill_in_kernel; do
  ncu --set full --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/w_$k \
      python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --umap --de > gpurun_out/ncu_w_$k.log 2>&1
  ncu -i gpurun_out/w_$k.ncu-rep --page details 2>&1 | grep -E "^  [a-zA-Z_].*\(|Duration|DRAM Throughput|Memory Throughput|Compute \(SM\) Throughput|Issue Slots Busy|highest-utilized|Achieved Occupancy|L1/TEX Cache Throughput|L2 Cache Throughput" >> gpurun_out/widening_ncu.txt
done
cat gpurun_out/widening_ncu.txt | cut -c1-120
