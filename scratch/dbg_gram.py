import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2605_13928_b200 import pp
np.set_printoptions(precision=3, suppress=True, linewidth=200)
for (n, h) in [(32, 127), (64, 127), (1000, 200)]:
    rng = np.random.default_rng(0)
    Z = rng.standard_normal((n, h)).astype(np.float32)
    ld = pp.padded_width(h)
    Zp = np.zeros((n, ld), np.float32); Zp[:, :h] = Z; Zp[:, h] = 1
    sc = pp.Scaled(torch.as_tensor(Zp).cuda(), h, h, None, None)
    C = pp.gram(sc).cpu().numpy()
    ref = Zp.astype(np.float64).T @ Zp
    print(n, h, ld, "maxabs C", np.abs(C).max(), "ref", np.abs(ref).max())
    print(C[:5, :5]); print(ref[:5, :5])
    print("C[0,:40]", C[0, :40]); print("ref[0,:40]", ref[0, :40])
    d = np.diag(C); dr = np.diag(ref); print("diag ratio", (d / dr)[:40])
    # find permutation-like match: for row 0 of C, which ref entries match
    for j in range(8):
        k = np.argmin(np.abs(ref[0] - C[0, j])); print(j, C[0, j], "closest ref col", k, ref[0, k])
