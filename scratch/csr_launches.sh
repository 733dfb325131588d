ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:qc_kernel|subset|hvg_sums|scale_sums|scale_dense|gram_kernel|project_kernel' -c 8 --csv --log-file gpurun_out/csr_launches.csv python scratch/time_stages.py 1000000 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/csr_launches.csv csr
