KNN_REPS=16 bash tools/knn_variants.sh 3 "base:" "hint2k:-DSCB_KNN_HINT_E=2000" "hint200:-DSCB_KNN_HINT_E=200"
