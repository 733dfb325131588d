"""Would a single-pass TF32 Gram keep the PCA subspace angle well under 1e-3?  Emulation on the
GPU: round the scaled matrix Z to TF32 (10-bit mantissa, round to nearest), form the Gram in
float64 from the rounded values (operand rounding only; the tensor-core accumulation would add
to it), solve with the shipped eigensolver and compare with the CPU oracle's components.

usage: python tools/tf32_gram_precision.py [cells] [genes]
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
r = pipeline.run(X, mt, pipeline.Params(), with_knn=False, timing=False)
o = chunked.run(*X.to_host(), mt.cpu().numpy(), op.Params(), workers=16)
V = o["components"]
sc = r.scaled
sc = pp.Scaled(sc.dense().contiguous(), sc.H, sc.ones_col, sc.mean, sc.inv_std)
N, H = sc.n_rows, sc.H


def round_mant(Z, bits):
    u = Z.view(torch.int32)
    drop = 23 - bits
    half = 1 << (drop - 1)
    u = (u + half + ((u >> drop) & 1) - 1) & ~((1 << drop) - 1)  # round to nearest even
    return u.view(torch.float32)


out = {"cells": n, "genes": g, "angle_shipped_3xbf16": op.subspace_angle(r.pca.components.cpu().numpy().T.astype(np.float64), V)}
for name, bits in (("tf32", 10), ("bf16", 7)):
    C = torch.zeros((sc.Z.shape[1], sc.Z.shape[1]), dtype=torch.float64, device=sc.Z.device)
    for a in range(0, N, 65536):
        Zr = round_mant(sc.Z[a:a + 65536].contiguous(), bits).double()
        C += Zr.T @ Zr
    lam, comp, _, _ = pp.pca_from_gram(sc, C.contiguous(), N, 50)
    out[f"angle_{name}_operands_fp64_accum"] = op.subspace_angle(comp[:50, :H].double().cpu().numpy().T, V)
print(json.dumps(out), flush=True)
