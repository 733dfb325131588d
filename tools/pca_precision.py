"""Where does the PCA subspace error come from?  C2 (or given size) on the GPU vs the chunked
CPU oracle: angle of (a) the shipped path, (b) our eigensolver on an fp64 Gram of the GPU's Z,
(c) numpy eigh of our Gram, (d) numpy eigh of the fp64 Gram; plus the Gram's error and the
eigen-gap at n_comps.  Set SCB_GRAM_SLICE_CELLS to vary the Gram's fp32 accumulation length.

usage: python tools/pca_precision.py [cells] [genes]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import chunked  # noqa: E402
from oracle import pipeline as op  # noqa: E402
from paper_2605_13928_b200 import pipeline, pp, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
g = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
spec = synth.Spec(n, g, seed=0)
X = synth.generate(spec)
mt = synth.mt_mask(spec)
p = pipeline.Params()
r = pipeline.run(X, mt, p, with_knn=False, timing=False)
host = X.to_host()
o = chunked.run(*host, mt.cpu().numpy(), op.Params(), workers=16)
V = o["components"]
sc = r.scaled
H = sc.H
N = sc.n_rows
sc = pp.Scaled(sc.dense().contiguous(), sc.H, sc.ones_col, sc.mean, sc.inv_std)  # fp32 copy for the experiments
out = {"cells": n, "genes": g, "slice_cells": os.environ.get("SCB_GRAM_SLICE_CELLS", "default")}
out["angle_shipped"] = op.subspace_angle(r.pca.components.cpu().numpy().T.astype(np.float64), V)
for planes in (True, False):
    C = pp.gram(sc, planes=planes)
    Z64 = sc.Z.double()
    C64 = Z64.T @ Z64
    tag = "planes" if planes else "inkernel"
    out[f"gram_rel_err_{tag}"] = ((C - C64).abs().max() / C64.abs().max()).item()
    out[f"gram_diag_rel_err_{tag}"] = ((C.diagonal() - C64.diagonal()) / C64.diagonal()).abs().max().item()
    lam_a, comp_a, _, _ = pp.pca_from_gram(sc, C, N, 50)
    out[f"angle_oursgram_ourseig_{tag}"] = op.subspace_angle(comp_a[:50, :H].double().cpu().numpy().T, V)
lam_b, comp_b, _, _ = pp.pca_from_gram(sc, C64.contiguous(), N, 50)
out["angle_fp64gram_ourseig"] = op.subspace_angle(comp_b[:50, :H].double().cpu().numpy().T, V)


def np_pca(Cg):
    Cn = Cg.cpu().numpy()[:H + 1, :H + 1]
    s = Cn[:H, H]  # column sums (ones column)
    Cc = (Cn[:H, :H] - np.outer(s, s) / N) / (N - 1.0)
    w, U = np.linalg.eigh(Cc)
    o_ = np.argsort(w)[::-1]
    return w[o_], U[:, o_[:50]]


w1, U1 = np_pca(pp.gram(sc))
w2, U2 = np_pca(C64)
out["angle_oursgram_npeigh"] = op.subspace_angle(U1, V)
out["angle_fp64gram_npeigh"] = op.subspace_angle(U2, V)
out["eig_48_52"] = w2[47:52].tolist()
out["rel_gap_50_51"] = float((w2[49] - w2[50]) / w2[49])
print(json.dumps(out))
