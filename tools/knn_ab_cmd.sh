bash tools/knn_variants.sh 3 "base:" "pool:-DSCB_KNN_POOL"
SCB_LIB_PATH=/tmp/scb_variants/pool.so timeout 600 python -m pytest tests/test_gpu_knn.py -m gpu -x -q 2>&1 | tail -2
