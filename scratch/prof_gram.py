import sys, torch
sys.path.insert(0, '.')
from paper_2605_13928_b200 import pp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
h = 2000
ld = pp.padded_width(h)
Z = torch.zeros((n, ld), device='cuda'); Z[:, :h] = torch.randn(n, h, device='cuda'); Z[:, h] = 1
sc = pp.Scaled(Z, h, h, None, None)
for i in range(2):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); C = pp.gram(sc); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"gram n={n} {ms:.2f} ms  unique TFLOP/s {n*h*(h+1)/ms/1e9:.1f}  (3xTF32 issued {3*n*72*128*256*2/ms/1e9:.1f})")
    lam, comp_t, mean, tr = pp.pca_from_gram(sc, C, n, 50)
    a.record(); lam, comp_t, mean, tr = pp.pca_from_gram(sc, C, n, 50); b.record(); torch.cuda.synchronize()
    print(f"eig {a.elapsed_time(b):.2f} ms")
    a.record(); X = pp.project(sc, comp_t, mean, 50); b.record(); torch.cuda.synchronize()
    print(f"project {a.elapsed_time(b):.2f} ms  GB/s {(n*ld*4 + n*64*4)/a.elapsed_time(b)/1e6:.0f}")
