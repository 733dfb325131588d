# per-call wall time of pp.louvain on the 1M-cell neighbors graph (diagnostic)
import time, sys, torch
sys.path.insert(0, ".")
from paper_2605_13928_b200 import pp, pipeline, synth
spec = synth.Spec(1_000_000, 25_000, seed=0)
X = synth.generate(spec)
r = pipeline.run(X, synth.mt_mask(spec), pipeline.Params(connectivities=True), timing=False)
G = r.graph.connectivities
del X
torch.cuda.synchronize()
for i in range(3):
    t = time.perf_counter()
    lab, nc, q = pp.louvain(G)
    torch.cuda.synchronize()
    print(f"call {i}: {1e3 * (time.perf_counter() - t):.1f} ms, {nc} communities, Q {q:.4f}", flush=True)
