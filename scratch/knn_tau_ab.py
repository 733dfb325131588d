# A/B of the list seed (SCB_KNN_TAU=0/1): candidate-stage time at n cells and the kNN result saved
# for an exact comparison between the two processes.
import os, sys, torch
sys.path.insert(0, ".")
from paper_2605_13928_b200 import synth, pipeline, pp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
tag = os.environ.get("SCB_KNN_TAU", "1")
spec = synth.Spec(n, 20000, seed=0)
X = synth.generate(spec); mt = synth.mt_mask(spec)
r = pipeline.run(X, mt, pipeline.Params(), with_knn=False)
E = r.pca.X_pca.contiguous()
del X, r
for i in range(3):
    t = (torch.cuda.Event(True), torch.cuda.Event(True))
    idx, d = pp.neighbors(E, 15, n_comps=50, timer=t); torch.cuda.synchronize()
    print(f"[tau={tag}] n={n} candidate stage {t[0].elapsed_time(t[1]):.2f} ms", flush=True)
os.makedirs("gpurun_out", exist_ok=True)
torch.save({"idx": idx.cpu(), "d": d.cpu()}, f"/tmp/knn_tau{tag}.pt")
