KNN_REPS=16 bash tools/knn_variants.sh 3 "base:" "e32:-DSCB_KNN_SLEEP_E=32" "e64:-DSCB_KNN_SLEEP_E=64" "spin:-DSCB_KNN_SLEEP_P=0 -DSCB_KNN_SLEEP_M=0"
