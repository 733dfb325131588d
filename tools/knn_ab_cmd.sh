(cd paper_2605_13928_b200/csrc && rm -f build/knn.o && make -j16 EXTRA="-DSCB_KNN_CL=4 -DSCB_MBAR_WATCHDOG" > /dev/null 2>&1)
SCB_KNN_DEBUG=1 timeout 300 python -m pytest tests/test_gpu_knn.py -m gpu -q -x 2>&1 | tail -2
SCB_KNN_DEBUG=1 timeout 300 python tools/knn_time.py cl4_wd lists 1 2>&1 | tail -2
(cd paper_2605_13928_b200/csrc && rm -f build/knn.o && make -j16 > /dev/null 2>&1)
bash tools/knn_ncu_variants.sh "cl2:" "cl4:-DSCB_KNN_CL=4"
bash tools/knn_variants.sh 3 "cl2:" "cl4:-DSCB_KNN_CL=4"
