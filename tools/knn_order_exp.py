"""Experiment: does a better scan order (outward from each query pair's own position) cut the
kNN candidate kernel's insert work?  C3 embedding; orders: built-in Morton-3D, random, k-means
clusters (ordered by centroid PC1), kd-style recursive median splits over the top PCs.
Prints candidate-kernel ms and recall on 2000 random queries (fp64 brute force) per order."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13928_b200 import _lib, pipeline, pp, synth  # noqa: E402
from paper_2605_13928_b200.pp import _ctx, _p, _stream  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
spec = synth.Spec(n, 25_000, seed=0)
X = synth.generate(spec)
r = pipeline.run(X, synth.mt_mask(spec), pipeline.Params(), with_knn=False, timing=False)
E = r.pca.X_pca[:, :50].contiguous()
del X, r
torch.cuda.empty_cache()
N = E.shape[0]
g = torch.Generator(device="cuda")
g.manual_seed(0)
qs = torch.randperm(N, device="cuda", generator=g)[:2000]
D = torch.cdist(E[qs].double(), E.double())
ref = D.topk(15, largest=False).indices
del D


def run(key, label):
    idx = torch.empty((N, 15), dtype=torch.int32, device="cuda")
    dist = torch.empty((N, 15), dtype=torch.float32, device="cuda")
    best = 1e9
    for _ in range(2):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); e1.record()
        if key is None:
            pp.neighbors(E, 15, timer=(e0, e1))
        else:
            _lib.call("scb_knn_ordered", _ctx(E), _p(E), N, 50, E.stride(0), 15, _p(key), _p(idx), _p(dist), _stream(),
                      e0.cuda_event, e1.cuda_event)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    if key is None:
        idx, _ = pp.neighbors(E, 15)
    hit = sum(len(set(ref[i].tolist()) & set(idx[qs[i]].tolist())) for i in range(len(qs)))
    print(json.dumps({"order": label, "candidates_ms": round(best, 2), "recall": hit / (len(qs) * 15)}), flush=True)


def morton_sub(vals, bits):
    """quantile rank of vals within [0, 2^bits)"""
    rk = torch.argsort(torch.argsort(vals))
    return (rk * (1 << bits) // max(1, vals.numel())).clamp_max((1 << bits) - 1)


run(None, "morton3 (built-in)")
run(torch.randint(0, 65536, (N,), device="cuda", generator=g).to(torch.int32).to(torch.uint16), "random")

for C in (16, 64, 256):
    cent = E[torch.randperm(N, device="cuda", generator=g)[:C]].clone()
    for _ in range(10):
        lab = torch.cdist(E, cent).argmin(1)
        s = torch.zeros_like(cent).index_add_(0, lab, E)
        c = torch.bincount(lab, minlength=C).clamp_min(1).unsqueeze(1).float()
        cent = s / c
    lab = torch.cdist(E, cent).argmin(1)
    # order clusters along a greedy nearest-neighbour chain of centroids
    Dc = torch.cdist(cent, cent)
    order, seen = [int(cent[:, 0].argmin())], {int(cent[:, 0].argmin())}
    for _ in range(C - 1):
        d = Dc[order[-1]].clone()
        d[list(seen)] = float("inf")
        nx = int(d.argmin())
        order.append(nx)
        seen.add(nx)
    rank = torch.empty(C, dtype=torch.int64, device="cuda")
    rank[torch.tensor(order, device="cuda")] = torch.arange(C, device="cuda")
    sub_bits = 16 - (C - 1).bit_length()
    key = torch.empty(N, dtype=torch.int64, device="cuda")
    cl = rank[lab]
    for ci in range(C):
        m = cl == ci
        if m.any():
            key[m] = ci * (1 << sub_bits) + morton_sub(E[m, 0], sub_bits)
    run(key.to(torch.int32).to(torch.uint16), f"kmeans{C}+chain+pc1")

for dims in (8, 16):
    grp = torch.zeros(N, dtype=torch.int64, device="cuda")
    for lvl in range(16):
        v = E[:, lvl % dims]
        o = torch.argsort(v, stable=True)
        o = o[torch.argsort(grp[o], stable=True)]          # sorted by (group, value)
        gs = grp[o]
        cnt = torch.bincount(gs, minlength=int(gs.max()) + 1)
        start = torch.cumsum(cnt, 0) - cnt
        rank_in = torch.arange(N, device="cuda") - start[gs]
        bit = (rank_in * 2 >= cnt[gs]).long()
        newg = torch.empty_like(grp)
        newg[o] = gs * 2 + bit
        grp = newg
    run(grp.to(torch.int32).to(torch.uint16), f"kd16 over top-{dims} PCs")
