#!/bin/bash
# ncu source-level counters of the list-based kNN candidate kernel on the C3 embedding
mkdir -p gpurun_out/s3
make -C paper_2605_13928_b200/csrc -j16 > /dev/null 2>&1 || exit 1
cat > /tmp/knn_lists_once.py << 'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2605_13928_b200 import pipeline, pp, synth
spec = synth.Spec(1000000, 25000, seed=0)
X = synth.generate(spec)
r = pipeline.run(X, synth.mt_mask(spec), pipeline.Params(), with_knn=False)
E = r.pca.X_pca.contiguous(); del X, r; torch.cuda.empty_cache()
idx, dist = pp.neighbors(E, 15, n_comps=50); torch.cuda.synchronize(); print("ok")
PY
timeout 900 ncu --section SourceCounters --section WarpStateStats --section InstructionStats --section ComputeWorkloadAnalysis \
  --import-source on --clock-control none -k regex:knn_candidates -c 1 -o gpurun_out/s3/knn_src4 -f python /tmp/knn_lists_once.py > gpurun_out/s3/knn_src.log 2>&1
echo "ncu rc $?"; tail -3 gpurun_out/s3/knn_src.log
ncu -i gpurun_out/s3/knn_src4.ncu-rep --page details --csv > gpurun_out/s3/knn_src4_details.csv 2>&1
ncu -i gpurun_out/s3/knn_src4.ncu-rep --page source --csv --print-source sass > gpurun_out/s3/knn_src4_sass.csv 2>&1
ls -la gpurun_out/s3/
