"""Shared inputs for the GPU parity tests (seeded synthetic NB counts + oracle run)."""
import functools

import numpy as np

from oracle import pipeline as op
from oracle.synth import SynthSpec, generate_csr, mt_mask

C1 = dict(spec=SynthSpec(10000, 2000, seed=1),
          params=op.Params(min_genes=50, max_pct_mt=15.0, n_top_genes=1000, n_neighbors=15))


@functools.lru_cache(maxsize=4)
def c1_inputs():
    spec = C1["spec"]
    ip, ix, d = generate_csr(spec)
    return op.CSR(ip, ix, d, spec.n_genes), mt_mask(spec)


@functools.lru_cache(maxsize=2)
def c1_oracle(with_knn=True):
    X, mt = c1_inputs()
    return op.run(X, mt, C1["params"], with_knn=with_knn)
