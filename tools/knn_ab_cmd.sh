bash tools/knn_ncu_variants.sh "base:" "roundstart:-DSCB_KNN_ROUNDSTART"
bash tools/knn_variants.sh 3 "base:" "roundstart:-DSCB_KNN_ROUNDSTART"
