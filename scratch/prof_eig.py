import sys, torch, time
sys.path.insert(0, '.')
from paper_2605_13928_b200 import pp
import os
os.environ["SCB_EIG_VERBOSE"] = "1"
n = 200000; h = 2000
ld = pp.padded_width(h)
g = torch.Generator(device='cuda'); g.manual_seed(0)
# planted spectrum: low-rank + noise
F = torch.randn(n, 80, device='cuda', generator=g) * torch.linspace(3, 0.5, 80, device='cuda')
W = torch.randn(80, h, device='cuda', generator=g) / 9
Z = torch.zeros((n, ld), device='cuda'); Z[:, :h] = F @ W + torch.randn(n, h, device='cuda', generator=g); Z[:, h] = 1
sc = pp.Scaled(Z, h, h, None, None)
C = pp.gram(sc)
for mode in range(2):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); lam, comp_t, mean, tr = pp.pca_from_gram(sc, C, n, 50); b.record(); torch.cuda.synchronize()
    print("eig total", a.elapsed_time(b), "ms", lam[:3].tolist(), lam[47:50].tolist())
