# per-kernel device time of the CSR stages at C3 via CUDA events around pipeline steps
import sys, torch
sys.path.insert(0, ".")
from paper_2605_13928_b200 import synth, pipeline
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
spec = synth.Spec(n, 25000, seed=0)
X = synth.generate(spec); mt = synth.mt_mask(spec)
for i in range(3):
    r = pipeline.run(X, mt, pipeline.Params(), timing=True, with_knn=(i == 2))
    print({k: round(v, 2) for k, v in r.step_ms.items()})
