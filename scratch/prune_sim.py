# CPU estimate: fraction of key tiles a box lower bound could skip (ideal thresholds)
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from oracle import pipeline as op
from oracle.synth import SynthSpec, generate_csr, mt_mask
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
spec = SynthSpec(n, 25000, seed=0)
t = time.time()
import os
cache = f"/tmp/emb_cpu_{n}.npy"
if os.path.exists(cache):
    E = np.load(cache)
else:
    ip, ix, d = generate_csr(spec)
    X = op.CSR(ip, ix, d, 25000)
    r = op.run(X, mt_mask(spec), op.Params(), with_knn=False)
    E = np.asarray(r["X_pca"], np.float32)
    np.save(cache, E)
print("pipeline", time.time() - t, E.shape)
lo, hi = E[:, :3].min(0), E[:, :3].max(0)
q = np.clip(((E[:, :3] - lo) / (hi - lo) * 1024).astype(int), 0, 1023)
def spread(v):
    out = np.zeros_like(v)
    for b in range(10): out |= ((v >> b) & 1) << (3 * b)
    return out
code = (spread(q[:, 0]) << 2) | (spread(q[:, 1]) << 1) | spread(q[:, 2])
E = E[np.argsort(code >> 14, kind="stable")]
T = torch.from_numpy(E)
N = len(E); nt = (N + 127) // 128
klo = np.stack([E[i*128:(i+1)*128].min(0) for i in range(nt)]); khi = np.stack([E[i*128:(i+1)*128].max(0) for i in range(nt)])
kc = torch.stack([T[i*128:(i+1)*128].mean(0) for i in range(nt)])
kr = torch.stack([(T[i*128:(i+1)*128] - kc[i]).norm(dim=1).max() for i in range(nt)])
print("median tile radius", kr.median().item(), "median 16-NN dist", torch.cdist(T[:2000], T).topk(16, largest=False).values[:, -1].median().item())
for KC in (16, 32):
    tot = 0; kept = 0; kept_b = 0; kept_pb = 0
    for p in range(0, nt, 2):
        Q = T[p*128:(p+2)*128]
        dd = torch.cdist(Q, T) ** 2
        thr = dd.topk(KC, largest=False).values[:, -1].max().item()
        qlo = np.minimum(klo[p], klo[min(p+1, nt-1)]); qhi = np.maximum(khi[p], khi[min(p+1, nt-1)])
        gap = np.maximum(0, np.maximum(qlo[None] - khi, klo - qhi[None]))
        lb = (gap ** 2).sum(1)
        kept += (lb <= thr).sum(); tot += nt
        # ball bounds: per-query vs key-tile ball
        thrq = dd.topk(KC, largest=False).values[:, -1]
        dq = torch.cdist(Q, kc).clamp_min(0) - kr[None]
        lbq = dq.clamp_min(0) ** 2
        need = (lbq <= thrq[:, None]).any(0)
        kept_b += need.sum().item()
        # pair ball vs key ball
        qc = Q.mean(0); qr = (Q - qc).norm(dim=1).max()
        lbp = ((kc - qc).norm(dim=1) - qr - kr).clamp_min(0) ** 2
        kept_pb += (lbp <= thr).sum().item()
        # per-query-tile (128) version
    print(f"KC={KC}: tiles kept box {kept/tot:.3f} query-vs-ball {kept_b/tot:.3f} ball-ball {kept_pb/tot:.3f}")
