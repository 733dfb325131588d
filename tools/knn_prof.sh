#!/bin/bash
# clock64 breakdown of the kNN candidate kernel (C5 embedding): rebuilds knn.o with -DSCB_KNN_PROF
mkdir -p gpurun_out/r02
(cd paper_2605_13928_b200/csrc && rm -f build/knn.o && make -j16 EXTRA=-DSCB_KNN_PROF > /dev/null 2>&1)
timeout 200 python tools/knn_only_c5.py 1000000 15 > gpurun_out/r02/knn_prof.log 2>&1
grep -h "knn prof\|config" gpurun_out/r02/knn_prof.log | cut -c1-300
(cd paper_2605_13928_b200/csrc && rm -f build/knn.o && make -j16 > /dev/null 2>&1)
