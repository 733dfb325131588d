"""C5 kNN-only stress on one B200: a 1M x 50 Gaussian-mixture embedding (30 clusters, decaying
per-component spread), k = 15 and k = 30, device time of the whole pp.neighbors call and of the
candidate kernel, and recall against an exact fp64 brute force on 2000 random queries.  Prints
one JSON line per k.

usage: python tools/knn_only_c5.py [n]
"""
import json
import sys

import torch
sys.path.insert(0, ".")
from paper_2605_13928_b200 import pp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
g = torch.Generator(device="cuda"); g.manual_seed(0)
sig = torch.linspace(4.0, 0.6, 50, device="cuda")
centers = torch.randn(30, 50, device="cuda", generator=g) * sig * 1.5
lab = torch.randint(0, 30, (n,), device="cuda", generator=g)
X = (centers[lab] + torch.randn(n, 50, device="cuda", generator=g) * sig * 0.6).contiguous()
for k in [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["15", "30"])]:
    for rep in range(2):
        t = (torch.cuda.Event(True), torch.cuda.Event(True))
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); idx, dist = pp.neighbors(X, k, timer=t); b.record(); torch.cuda.synchronize()
    # exact check on 2000 random queries (fp64 brute force on the GPU)
    q = torch.randperm(n, device="cuda", generator=g)[:2000]
    D = torch.cdist(X[q].double(), X.double())
    ref = D.topk(k, largest=False).indices
    hit = sum(len(set(ref[i].tolist()) & set(idx[q[i]].tolist())) for i in range(len(q)))
    print(json.dumps({"config": f"C5 (1 GPU): {n} x 50 embedding, k={k}", "total_ms": round(a.elapsed_time(b), 2),
                      "candidates_kernel_ms": round(t[0].elapsed_time(t[1]), 2),
                      "recall_2000_random_queries": hit / (len(q) * k),
                      "tflops_algorithmic": 2 * n * n * 50 / (t[0].elapsed_time(t[1]) / 1e3) / 1e12}), flush=True)
