mkdir -p gpurun_out/r02
cd paper_2605_13928_b200/csrc && rm -f build/knn.o && make -j16 EXTRA=-DSCB_KNN_PROF > /dev/null 2>&1 && cd ../..
timeout 200 python tools/knn_only_c5.py > gpurun_out/r02/prof_base.log 2>&1
SCB_KNN_ATM=1 timeout 200 python tools/knn_only_c5.py > gpurun_out/r02/prof_atm.log 2>&1
grep -h "knn prof\|config" gpurun_out/r02/prof_base.log gpurun_out/r02/prof_atm.log | cut -c1-300
