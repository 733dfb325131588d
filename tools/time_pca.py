"""Per-kernel-group timing of the PCA step at C3 (split planes, Gram, eigensolve, projection)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13928_b200 import pipeline, pp, synth  # noqa: E402

spec = synth.Spec(1_000_000, 25_000, seed=0)
X = synth.generate(spec)
r = pipeline.run(X, synth.mt_mask(spec), pipeline.Params(), with_knn=False, timing=False)
del X
sc = r.scaled
N = sc.n_rows
out = {}
for rep in range(3):
    ev = [torch.cuda.Event(True) for _ in range(5)]
    ev[0].record()
    pp.split_planes(sc)
    ev[1].record()
    C = torch.empty((sc.ld, sc.ld), dtype=torch.float64, device="cuda")
    from paper_2605_13928_b200 import _lib
    from paper_2605_13928_b200.pp import _ctx, _p, _stream
    _lib.call("scb_gram_split", _ctx(sc.Z_hi), _p(sc.Z_hi), _p(sc.Z_lo), N, sc.ld, _p(C), _stream())
    ev[2].record()
    lam, comp_t, mean, tr = pp.pca_from_gram(sc, C, N, 50)
    ev[3].record()
    Xp = pp.project(sc, comp_t, mean, 50)
    ev[4].record()
    torch.cuda.synchronize()
    out = {k: round(ev[i].elapsed_time(ev[i + 1]), 3) for i, k in enumerate(["split", "gram", "eig", "project"])}
    print(json.dumps(out), flush=True)
