timeout 600 python -m pytest tests/test_gpu_knn.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -1
bash tools/knn_variants.sh 2 "new_rerank:"
