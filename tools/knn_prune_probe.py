"""Probe: fraction of (32-query warp, 128-key tile) pairs of the kNN candidate scan whose filter
could be skipped by a bounding-box lower bound over the first m PCs (keys and queries in 4-D
Morton order over PC1-4, as the kernel orders them).  The per-lane threshold is taken as the
exact 32nd-neighbour squared distance (the best a list can reach), so the numbers are upper
bounds on what a box test could skip.

usage: python tools/knn_prune_probe.py [n_warps_sampled]"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_13928_b200 import pipeline, synth

nw = int(sys.argv[1]) if len(sys.argv) > 1 else 512
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
n = E.shape[0]
var = E.var(0)
print("variance share PC1-4 / PC1-8 / PC1-16:", [round((var[:m].sum() / var.sum()).item(), 3) for m in (4, 8, 16)])
# 4-D Morton order over PC1-4 (16 bits per dim)
lo, hi = E[:, :4].min(0).values, E[:, :4].max(0).values
qz = ((E[:, :4] - lo) / (hi - lo) * 65535).clamp(0, 65535).long()
code = torch.zeros(n, dtype=torch.long, device="cuda")
for b in range(16):
    for dd in range(4):
        code |= ((qz[:, dd] >> b) & 1) << (4 * b + dd)
order = torch.argsort(code)
Es = E[order].contiguous()
nt = (n + 127) // 128
pad = nt * 128 - n
Ep = torch.cat([Es, Es[-1:].expand(pad, -1)]) if pad else Es
T = Ep.view(nt, 128, 50)
g = torch.Generator(device="cuda"); g.manual_seed(1)
warps = torch.randint(0, n // 32, (nw,), device="cuda", generator=g)
res = {m: 0 for m in (2, 4, 8, 16, 50)}
tot = 0
for w in warps.tolist():
    Q = Es[32 * w: 32 * w + 32]
    d2 = torch.cdist(Q.double(), Es.double()).pow(2)
    thr = d2.topk(32, largest=False).values[:, -1]  # per lane
    for m in res:
        blo = T[:, :, :m].min(1).values  # [nt, m]
        bhi = T[:, :, :m].max(1).values
        gap = torch.clamp(torch.maximum(blo[None] - Q[:, None, :m], Q[:, None, :m] - bhi[None]), min=0)
        lb = gap.pow(2).sum(-1)  # [32, nt]
        skip = (lb.double() > thr[:, None]).all(0)  # every lane of the warp prunable
        res[m] += int(skip.sum())
    tot += nt
print({f"PC1-{m}": round(res[m] / tot, 4) for m in res}, "of", tot, "warp-tile pairs")
