bash tools/knn_variants.sh 3 "base:" "onevote:-DSCB_KNN_ONEVOTE"
