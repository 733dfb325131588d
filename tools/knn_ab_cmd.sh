bash tools/knn_ncu_variants.sh "base:" "cl2:-DSCB_KNN_CL=2"
bash tools/knn_variants.sh 4 "base:" "cl2:-DSCB_KNN_CL=2"
