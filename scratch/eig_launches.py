# eigensolve only, on the C3-spectrum covariance (pipeline up to the Gram, then 2 eig calls)
import sys, torch
sys.path.insert(0, ".")
from paper_2605_13928_b200 import synth, pipeline, pp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
spec = synth.Spec(n, 25000, seed=0)
X = synth.generate(spec); mt = synth.mt_mask(spec)
r = pipeline.run(X, mt, pipeline.Params(), with_knn=False)
C = pp.gram(r.scaled)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(2):
    pp.pca_from_gram(r.scaled, C, r.scaled.Z.shape[0], 50)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
