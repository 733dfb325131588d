"""Regenerate the committed golden fixtures (run from the repo root: python tests/golden/make_golden.py).

The reference repository has no golden vectors for this path; these are
builder-made: a seeded 600 x 300 synthetic NB matrix (oracle/synth.py) and every stage output
of the CPU oracle (oracle/pipeline.py) on it.  Tests check (a) that the generator and the
oracle still reproduce them bit for bit (pinning the oracle against silent drift) and (b)
that the GPU path matches them.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import pipeline as op  # noqa: E402
from oracle.synth import SynthSpec, generate_csr, mt_mask  # noqa: E402

SPEC = SynthSpec(600, 300, seed=7)
PARAMS = op.Params(min_genes=10, max_genes=None, max_pct_mt=25.0, min_cells=3, target_sum=1e4,
                   n_top_genes=100, n_bins=20, max_value=10.0, n_comps=10, n_neighbors=10)


def compute():
    ip, ix, d = generate_csr(SPEC)
    mt = mt_mask(SPEC)
    o = op.run(op.CSR(ip, ix, d, SPEC.n_genes), mt, PARAMS)
    out = dict(indptr=ip, indices=ix, data=d, mt_mask=mt)
    for k, v in o["qc"].items():
        out["qc_" + k] = v
    out.update(cell_mask=o["cell_mask"], gene_mask=o["gene_mask"],
               sub_indptr=o["X_sub"].indptr, sub_indices=o["X_sub"].indices, sub_data=o["X_sub"].data,
               row_scale=o["row_scale"], log_data=o["X_log"].data, hvg_mask=o["hvg_mask"],
               scale_mean=o["scale_mean"], scale_inv_std=o["scale_inv_std"], Z=o["Z"],
               components=o["components"], variance=o["variance"], variance_ratio=o["variance_ratio"],
               spectrum=o["spectrum"], X_pca=o["X_pca"], knn_idx=o["knn_idx"], knn_dist=o["knn_dist"])
    for k in ("means", "variances", "dispersions", "dispersions_norm", "mean_bin"):
        out["hvg_" + k] = o["hvg_stats"][k]
    return out


if __name__ == "__main__":
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "g600x300.npz")
    np.savez_compressed(path, **compute())
    print("wrote", path, os.path.getsize(path), "bytes")
