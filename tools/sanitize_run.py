"""Small end-to-end run of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Test infrastructure: it checks nothing itself beyond "no CUDA error";
the sanitizer logs are the evidence (profiles/r02/sanitizer_*.log).

Covers: device synth, QC / masks / subset / normalize / HVG sums + select / scale (plain and
regress_out), Gram (planes and in-kernel split), eigensolve, projection, kNN (k_cand 32 and 64),
neighbors graph, UMAP layout, Leiden + Louvain, rank_genes_groups, MatrixMarket ingest.

usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py [cells] [genes]
"""
import io
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13928_b200 import ingest, pipeline, pp, synth  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
    g = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
    spec = synth.Spec(n, g, seed=3)
    X = synth.generate(spec)
    mt = synth.mt_mask(spec)
    p = pipeline.Params(min_genes=40, max_pct_mt=15.0, n_top_genes=400, n_neighbors=15, connectivities=True,
                        umap=True, umap_epochs=20, cluster=True, rank_genes=True)
    r = pipeline.run(X, mt, p, timing=False)
    torch.cuda.synchronize()
    # regress_out path + the in-kernel-split Gram + k_cand 64 + Louvain
    p2 = pipeline.Params(min_genes=40, max_pct_mt=15.0, n_top_genes=400, n_neighbors=40, regress_out=True)
    r2 = pipeline.run(X, mt, p2, timing=False)
    pp.gram(r2.scaled, planes=False)
    pp.louvain(r.graph.connectivities)
    # ingest: a small MatrixMarket file of the same matrix (genes x cells, 10x orientation)
    ip, ix, d, G = X.to_host()
    rows = np.repeat(np.arange(n), np.diff(ip))
    buf = io.StringIO()
    buf.write("%%MatrixMarket matrix coordinate integer general\n")
    buf.write(f"{G} {n} {len(d)}\n")
    for gi, ci, v in zip(ix[:20000], rows[:20000], d[:20000]):
        buf.write(f"{gi + 1} {ci + 1} {int(v)}\n")
    raw = buf.getvalue().encode()
    raw = raw.replace(f"{G} {n} {len(d)}".encode(), f"{G} {n} {min(20000, len(d))}".encode(), 1)
    Xm, _ = ingest.parse_mtx_device(np.frombuffer(raw, np.uint8).copy(), transpose=True)
    torch.cuda.synchronize()
    print("sanitize run ok:", r.n_cells_total, int(r.hvg_index.numel()), r2.knn_index.shape,
          Xm.nnz)


if __name__ == "__main__":
    main()
