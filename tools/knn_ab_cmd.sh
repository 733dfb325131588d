bash tools/knn_variants.sh 3 "base:" "stash8:-DSCB_KNN_STASH -DSCB_KNN_STAGES=8"
SCB_LIB_PATH=/tmp/scb_variants/stash8.so timeout 600 python -m pytest tests/test_gpu_knn.py -m gpu -x -q 2>&1 | tail -2
