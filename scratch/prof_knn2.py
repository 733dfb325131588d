import sys, torch
sys.path.insert(0, '.')
from paper_2605_13928_b200 import pp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = torch.Generator(device='cuda'); g.manual_seed(0)
# PCA-like embedding: 30 clusters + decaying per-component spread
sig = torch.linspace(4.0, 0.6, 50, device='cuda')
centers = torch.randn(30, 50, device='cuda', generator=g) * sig * 1.5
lab = torch.randint(0, 30, (n,), device='cuda', generator=g)
X = torch.zeros((n, 64), device='cuda')
X[:, :50] = centers[lab] + torch.randn(n, 50, device='cuda', generator=g) * sig * 0.6
for i in range(reps):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    t = (torch.cuda.Event(True), torch.cuda.Event(True))
    a.record(); idx, d = pp.neighbors(X, 15, n_comps=50, timer=t); b.record(); torch.cuda.synchronize()
    ms = t[0].elapsed_time(t[1])
    units = (n / 256) * (n / 128)
    print(f"[pca-like] n={n} knn total {a.elapsed_time(b):.2f} ms, candidates {ms:.2f} ms, ns/unit/SM {ms*1e6*148/units:.1f}, TFLOP/s {2*n*n*50/ms/1e9:.1f}")
