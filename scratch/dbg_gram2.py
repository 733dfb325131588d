import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2605_13928_b200 import pp
for (n, h) in [(4099, 1000), (70001, 300), (300000, 200)]:
    rng = np.random.default_rng(n)
    Z = rng.standard_normal((n, h)).astype(np.float32)
    ld = pp.padded_width(h)
    Zp = np.zeros((n, ld), np.float32); Zp[:, :h] = Z; Zp[:, h] = 1
    sc = pp.Scaled(torch.as_tensor(Zp).cuda(), h, h, None, None)
    C = pp.gram(sc).cpu().numpy()
    Zt = torch.as_tensor(Zp).cuda().double()
    ref = (Zt.T @ Zt).cpu().numpy()
    d = (np.diag(C) - np.diag(ref)) / np.diag(ref)
    off = (C - ref) / np.sqrt(np.outer(np.diag(ref), np.diag(ref)))
    np.fill_diagonal(off, 0)
    print(n, h, "diag rel err mean %.3e std %.3e min %.3e max %.3e | offdiag max %.3e mean %.3e" % (d[:h].mean(), d[:h].std(), d[:h].min(), d[:h].max(), np.abs(off).max(), off[:h,:h].mean()))
