"""Candidate-kernel device time of pp.neighbors on the C3 embedding (cached in /tmp for the
call): python tools/knn_time.py [label] [tag] [reps]  (SCB_LIB_PATH selects a library build)"""
import os, sys, torch
sys.path.insert(0, ".")
from paper_2605_13928_b200 import pipeline, pp, synth
label = sys.argv[1] if len(sys.argv) > 1 else ""
method = sys.argv[2] if len(sys.argv) > 2 else "lists"  # tag printed with the label
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
cache = "/tmp/emb_c3_knn.pt"
if os.path.exists(cache):
    E = torch.load(cache).cuda()
else:
    spec = synth.Spec(1000000, 25000, seed=0)
    X = synth.generate(spec)
    r = pipeline.run(X, synth.mt_mask(spec), pipeline.Params(), with_knn=False)
    E = r.pca.X_pca[:, :50].contiguous()
    del X, r
    torch.save(E.cpu(), cache)
torch.cuda.empty_cache()
Ep = torch.zeros((E.shape[0], 64), device="cuda"); Ep[:, :50] = E
ms, tot = [], []
for _ in range(reps):
    t = (torch.cuda.Event(True), torch.cuda.Event(True))
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    idx, dist = pp.neighbors(Ep, 15, n_comps=50, timer=t)
    b.record()
    torch.cuda.synchronize()
    ms.append(round(t[0].elapsed_time(t[1]), 2))
    tot.append(round(a.elapsed_time(b) - t[0].elapsed_time(t[1]), 2))
ref = "/tmp/knn_ref_idx.pt"
if os.path.exists(ref):
    agree = (torch.load(ref).cuda() == idx).float().mean().item()
else:
    torch.save(idx.cpu(), ref); agree = 1.0
print(f"[knn time] {label} {method}: cand ms {ms} rest ms {tot} agree_with_first {agree:.6f}", flush=True)
