# C5-style kNN-only: 1M x 50 embedding, k = 30 (k_cand 64 path) and k = 15, timing + recall on a query subset
import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2605_13928_b200 import pp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
g = torch.Generator(device="cuda"); g.manual_seed(0)
sig = torch.linspace(4.0, 0.6, 50, device="cuda")
centers = torch.randn(30, 50, device="cuda", generator=g) * sig * 1.5
lab = torch.randint(0, 30, (n,), device="cuda", generator=g)
X = (centers[lab] + torch.randn(n, 50, device="cuda", generator=g) * sig * 0.6).contiguous()
for k in (15, 30):
    for rep in range(2):
        t = (torch.cuda.Event(True), torch.cuda.Event(True))
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); idx, dist = pp.neighbors(X, k, timer=t); b.record(); torch.cuda.synchronize()
    # exact check on 2000 random queries (fp64 brute force on the GPU)
    q = torch.randperm(n, device="cuda", generator=g)[:2000]
    D = torch.cdist(X[q].double(), X.double())
    ref = D.topk(k, largest=False).indices
    hit = sum(len(set(ref[i].tolist()) & set(idx[q[i]].tolist())) for i in range(len(q)))
    print(f"k={k}: total {a.elapsed_time(b):.1f} ms, candidates {t[0].elapsed_time(t[1]):.1f} ms, recall {hit / (len(q) * k):.5f}")
