# Gram precision at C2 scale: our 3xBF16 tcgen05 Gram vs an fp64 Gram of the same Z, and the
# PCA subspace angle each one gives against the CPU oracle's components
import sys, torch, numpy as np
sys.path.insert(0, ".")
from oracle import pipeline as op
from oracle.synth import SynthSpec, generate_csr, mt_mask
from paper_2605_13928_b200 import pipeline, pp
from paper_2605_13928_b200.pp import DeviceCSR
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
g = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
spec = SynthSpec(n, g, seed=0)
ip, ix, d = generate_csr(spec); mt = mt_mask(spec)
X = DeviceCSR.from_host(ip, ix, d, g)
r = pipeline.run(X, torch.as_tensor(mt).cuda(), pipeline.Params(), with_knn=False)
sc = r.scaled
C = pp.gram(sc)
Z = sc.Z.double()
C64 = Z.T @ Z
rel = ((C - C64).abs().max() / C64.abs().max()).item()
print("gram max abs err / max |C|:", rel, " diag rel err max:", ((C.diagonal() - C64.diagonal()).abs() / C64.diagonal().abs().clamp_min(1e-30)).max().item())
N = Z.shape[0]
lam_a, comp_a, _, _ = pp.pca_from_gram(sc, C, N, 50)
lam_b, comp_b, _, _ = pp.pca_from_gram(sc, C64.contiguous(), N, 50)
H = sc.H
A = comp_a[:50, :H].double().cpu().numpy().T
B = comp_b[:50, :H].double().cpu().numpy().T
print("angle(ours, fp64 Gram):", op.subspace_angle(A, B))
lam = lam_b.cpu().numpy()
print("eigen gaps near 50:", lam[45:50], "ratio lam50/lam49", lam[49] / lam[48])
