"""C2 parity + speed: 100k cells x 20k genes (~7 % dense), the full QC->kNN pipeline on one B200
against the CPU oracle (numpy/scipy BLAS on all host cores) on the same synthetic counts.
Checks the §8 tolerances at this scale and records both timings.  Test infrastructure: runs on
the GPU box (the oracle is the checker).

usage: python tools/parity_c2.py [cells] [genes] > gpurun_out/c2_parity.json
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pipeline as op  # noqa: E402
from oracle.synth import SynthSpec, generate_csr, mt_mask  # noqa: E402
from paper_2605_13928_b200 import pipeline  # noqa: E402
from paper_2605_13928_b200.pp import DeviceCSR  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
    g = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000
    spec = SynthSpec(n, g, seed=0)
    t0 = time.time()
    ip, ix, d = generate_csr(spec)
    gen_s = time.time() - t0
    mt = mt_mask(spec)
    p = pipeline.Params()
    X = DeviceCSR.from_host(ip, ix, d, g)
    mtd = torch.as_tensor(mt).cuda()
    for _ in range(3):
        r = pipeline.run(X, mtd, p, timing=True)
    torch.cuda.synchronize()
    gpu_ms = sum(r.step_ms.values())
    t0 = time.time()
    o = op.run(op.CSR(ip, ix, d, g), mt, op.Params())
    cpu_s = time.time() - t0
    qc = {k: bool(np.array_equal(r.qc[k].cpu().numpy(), o["qc"][k]))
          for k in ["n_genes_by_counts", "total_counts", "total_counts_mt", "n_cells_by_counts", "gene_total_counts"]}
    out = {
        "config": f"C2: {n} cells x {g} genes, nnz {len(d)}", "seed": 0,
        "qc_bit_exact": qc,
        "cell_mask_bit_exact": bool(np.array_equal(r.cell_mask.cpu().numpy(), o["cell_mask"])),
        "gene_mask_bit_exact": bool(np.array_equal(r.gene_mask.cpu().numpy(), o["gene_mask"])),
        "hvg_set_bit_exact": bool(np.array_equal(r.hvg_mask.cpu().numpy(), o["hvg_mask"])),
        "pca_subspace_angle": float(op.subspace_angle(r.pca.components.cpu().numpy().T.astype(np.float64),
                                                      o["components"])),
        "pca_variance_ratio_max_rel_err": float(np.max(np.abs(r.pca.variance_ratio.cpu().numpy() - o["variance_ratio"])
                                                       / o["variance_ratio"])),
        "knn_recall": float(op.knn_recall(r.knn_index.cpu().numpy(), o["knn_idx"])),
        "gpu_step_ms": {k: round(v, 3) for k, v in r.step_ms.items()}, "gpu_total_ms": round(gpu_ms, 3),
        "gpu_cells_per_s": n / (gpu_ms / 1e3),
        "cpu_oracle_s": round(cpu_s, 2), "cpu_cells_per_s": n / cpu_s,
        "cpu_cores": len(os.sched_getaffinity(0)), "generator_s": round(gen_s, 1),
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
