import sys, torch
sys.path.insert(0, ".")
from paper_2605_13928_b200 import synth, pipeline, pp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
spec = synth.Spec(n, 20000, seed=0)
X = synth.generate(spec); mt = synth.mt_mask(spec)
r = pipeline.run(X, mt, pipeline.Params(), with_knn=False)
E = r.pca.X_pca.contiguous()
torch.save(E.cpu(), f"/tmp/emb_{n}.pt")
for i in range(2):
    t = (torch.cuda.Event(True), torch.cuda.Event(True))
    idx, d = pp.neighbors(E, 15, n_comps=50, timer=t); torch.cuda.synchronize()
    ms = t[0].elapsed_time(t[1]); units = (n / 256) * (n / 128)
    print(f"[real] n={n} candidates {ms:.2f} ms ns/unit/SM {ms*1e6*148/units:.1f} TFLOP/s {2*n*n*50/ms/1e9:.1f}")
