# CPU simulation: number of top-16 list insertions per row (2 half-lists of 16, as the kernel)
# under the kernel's Morton-outward tile order vs. an order by tile-centroid distance.
import sys, numpy as np, torch
E = np.load(sys.argv[1] if len(sys.argv) > 1 else "/tmp/emb_cpu_40000.npy").astype(np.float32)
n = len(E)
lo, hi = E[:, :3].min(0), E[:, :3].max(0)
q = np.clip(((E[:, :3] - lo) / (hi - lo) * 1024).astype(int), 0, 1023)
def spread(v):
    out = np.zeros_like(v)
    for b in range(10): out |= ((v >> b) & 1) << (3 * b)
    return out
code = (spread(q[:, 0]) << 2) | (spread(q[:, 1]) << 1) | spread(q[:, 2])
E = E[np.argsort(code >> 14, kind="stable")]
T = torch.from_numpy(E)
nt = (n + 127) // 128
cent = torch.stack([T[i*128:(i+1)*128].mean(0) for i in range(nt)])
def outward(st):
    out = [st]
    for d in range(1, nt):
        if st + d < nt: out.append(st + d)
        if st - d >= 0: out.append(st - d)
    return out
def count(order, Q, qi0):
    # simulate per row-half lists: insert count = # times a score beats the current 16th best
    D = torch.cdist(Q, T) ** 2                     # [256, n]
    ins = 0
    thr = torch.full((Q.shape[0], 2), float("inf"))
    lists = [[[] for _ in range(2)] for _ in range(Q.shape[0])]
    for kt in order:
        blk = D[:, kt*128:(kt+1)*128]
        for h in range(2):
            sub = blk[:, h*64:(h+1)*64]
            for r in range(Q.shape[0]):
                vals = sub[r][sub[r] < thr[r, h]]
                if len(vals):
                    L = lists[r][h] + vals.tolist()
                    L.sort()
                    lists[r][h] = L[:16]
                    ins += len(vals)
                    if len(lists[r][h]) == 16: thr[r, h] = lists[r][h][-1]
    return ins
rng = np.random.default_rng(0)
tot_m = tot_c = 0
pairs = rng.choice(nt // 2, 6, replace=False)
for p in pairs:
    Q = T[p*256:(p+1)*256]
    st = 2 * p
    om = outward(st)
    qc = Q.mean(0)
    oc = torch.argsort(((cent - qc) ** 2).sum(1)).tolist()
    m, c = count(om, Q, p*256), count(oc, Q, p*256)
    tot_m += m; tot_c += c
    print(f"pair {p}: inserts morton-outward {m/256:.1f}/row, centroid order {c/256:.1f}/row", flush=True)
print(f"mean: morton {tot_m/len(pairs)/256:.1f}, centroid {tot_c/len(pairs)/256:.1f} inserts per row")
