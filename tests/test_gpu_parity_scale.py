"""Parity at the benchmark sizes: C2 (100k x 20k) and the headline C3 (1M x 25k), GPU pipeline
vs the CPU oracle on the same matrix, inside ``pytest -m gpu``.

Inputs come from the device generator, which is bit-identical to oracle/synth.py
(tests/test_gpu_synth.py); the matrix is copied to the host and the oracle runs on it row
chunk by row chunk in forked workers (oracle/chunked.py -- the same arithmetic as
oracle/pipeline.py, checked equal to it in tests/test_oracle.py).

Tolerances (BASELINE.json north_star): QC counts, filter masks and the HVG gene set bit-exact;
scale statistics within 1e-6 relative (the log values are within 1e-5); PCA subspace angle < 1e-3 (with a >= 5x margin asserted on the
shipped Gram); kNN recall >= 0.999 on 10k random queries against all cells.  The HVG set is
also checked against Scanpy's float64 expm1 path (oracle/scanpy_float.py) on C2 and on a
100k-cell sample of C3.
"""
import os
import time

import numpy as np
import pytest

from oracle import chunked
from oracle import pipeline as op
from oracle import scanpy_float as sf

pytestmark = pytest.mark.gpu

WORKERS = max(1, min(32, len(os.sched_getaffinity(0))))


def _device_run(n, g, seed, params):
    import torch
    from paper_2605_13928_b200 import pipeline, synth
    spec = synth.Spec(n, g, seed=seed)
    X = synth.generate(spec)
    mt = synth.mt_mask(spec)
    r = pipeline.run(X, mt, params, timing=False)
    torch.cuda.synchronize()
    host = X.to_host()
    gpu = dict(qc={k: v.cpu().numpy() for k, v in r.qc.items() if v is not None and k != "hvg_row_splits"},
               cell_mask=r.cell_mask.cpu().numpy(), gene_mask=r.gene_mask.cpu().numpy(),
               hvg_mask=r.hvg_mask.cpu().numpy(), scale_mean=r.scaled.mean.cpu().numpy(),
               scale_inv_std=r.scaled.inv_std.cpu().numpy(),
               components=r.pca.components.cpu().numpy().T.astype(np.float64),
               variance_ratio=r.pca.variance_ratio.cpu().numpy(), knn_idx=r.knn_index.cpu().numpy())
    del r, X
    torch.cuda.empty_cache()
    return host, mt.cpu().numpy(), gpu


def _oracle_params(params):
    return op.Params(min_genes=params.min_genes, max_genes=params.max_genes, max_pct_mt=params.max_pct_mt,
                     min_cells=params.min_cells, target_sum=params.target_sum, n_top_genes=params.n_top_genes,
                     n_bins=params.n_bins, hvg_ties=params.hvg_ties, max_value=params.max_value, clip=params.clip,
                     n_comps=params.n_comps, n_neighbors=params.n_neighbors)


def _compare(host, mt, gpu, params, n_queries=10000, seed=0):
    ip, ix, d, G = host
    n_kept = int(gpu["cell_mask"].sum())
    rng = np.random.default_rng(seed)
    q = np.sort(rng.choice(n_kept, size=min(n_queries, n_kept), replace=False))
    t0 = time.time()
    o = chunked.run(ip, ix, d, G, mt, _oracle_params(params), workers=WORKERS, knn_queries=q)
    report = {"oracle_s": round(time.time() - t0, 1)}
    for k in ("n_genes_by_counts", "total_counts", "total_counts_mt", "pct_counts_mt", "n_cells_by_counts",
              "gene_total_counts"):
        np.testing.assert_array_equal(gpu["qc"][k], o["qc"][k], err_msg=k)
    np.testing.assert_array_equal(gpu["cell_mask"], o["cell_mask"])
    np.testing.assert_array_equal(gpu["gene_mask"], o["gene_mask"])
    np.testing.assert_array_equal(gpu["hvg_mask"], o["hvg_mask"])
    # log1p values differ from numpy's by <= 1 ulp, so the scale statistics agree to ~1e-8
    np.testing.assert_allclose(gpu["scale_mean"], o["scale_mean"], rtol=1e-6)
    np.testing.assert_allclose(gpu["scale_inv_std"], o["scale_inv_std"], rtol=1e-6)
    ang = op.subspace_angle(gpu["components"], o["components"])
    vr = float(np.max(np.abs(gpu["variance_ratio"] - o["variance_ratio"]) / o["variance_ratio"]))
    rec = op.knn_recall(gpu["knn_idx"][q], o["knn_idx"])
    report.update(angle=ang, variance_ratio_rel=vr, recall=rec, n_queries=len(q), hvg=int(o["hvg_mask"].sum()))
    print("parity", report)
    assert ang < 2e-4, f"subspace angle {ang} (bar 1e-3, 5x margin required)"
    assert vr < 1e-4, vr
    assert rec >= 0.999, rec
    return o, report


def _scanpy_float_set(host, cell_mask, gene_mask, params):
    """Scanpy's float64 expm1 HVG set of the oracle's kept log matrix."""
    ip, ix, d, G = host
    X = op.CSR(ip, ix, d, G)
    Xs = op.subset(X, cell_mask, gene_mask)
    Xl, _, _ = op.normalize_log1p(Xs, params.target_sum)
    sel, _ = sf.hvg_seurat_expm1(Xl.indices, Xl.data, Xl.n_rows, Xl.n_cols, params.n_top_genes, params.n_bins)
    return sel


def test_c2_parity_and_scanpy_float_hvg():
    from paper_2605_13928_b200.pipeline import Params
    p = Params()
    host, mt, gpu = _device_run(100_000, 20_000, 0, p)
    o, _ = _compare(host, mt, gpu, p)
    sel = _scanpy_float_set(host, o["cell_mask"], o["gene_mask"], p)
    flips = np.nonzero(sel != o["hvg_mask"].astype(bool))[0]
    assert flips.size == 0, f"fixed-point HVG set differs from Scanpy's float64 set at {flips.tolist()}"


@pytest.mark.slow
def test_c3_parity_full_size():
    """The headline config, 1M x 25k (1.75e9 nonzeros): every stage vs the chunked oracle."""
    from paper_2605_13928_b200.pipeline import Params
    p = Params()
    host, mt, gpu = _device_run(1_000_000, 25_000, 0, p)
    _compare(host, mt, gpu, p)


def test_c3_sample_scanpy_float_hvg():
    """Fixed-point (device) vs Scanpy float64 HVG set on the first 100k cells of C3."""
    import torch
    from paper_2605_13928_b200 import pipeline, synth
    p = pipeline.Params()
    spec = synth.Spec(1_000_000, 25_000, seed=0)
    X = synth.generate_rows(spec, 0, 100_000)
    r = pipeline.run(X, synth.mt_mask(spec), p, timing=False, with_knn=False)
    torch.cuda.synchronize()
    host = X.to_host()
    sel = _scanpy_float_set(host, r.cell_mask.cpu().numpy(), r.gene_mask.cpu().numpy(), p)
    got = r.hvg_mask.cpu().numpy().astype(bool)
    flips = np.nonzero(sel != got)[0]
    assert flips.size == 0, f"device HVG set differs from Scanpy's float64 set at {flips.tolist()}"


def test_c2_regress_out_parity():
    """regress_out + scale (paper Table 1 step 4) at C2 vs the oracle's OLS restatement."""
    import torch
    from paper_2605_13928_b200 import pipeline, synth
    p = pipeline.Params(regress_out=True)
    spec = synth.Spec(100_000, 20_000, seed=0)
    X = synth.generate(spec)
    r = pipeline.run(X, synth.mt_mask(spec), p, timing=False, with_knn=False)
    torch.cuda.synchronize()
    ip, ix, d, G = X.to_host()
    o = op.run(op.CSR(ip, ix, d, G), synth.mt_mask(spec).cpu().numpy(),
               op.Params(regress_out=True, hvg_ties=p.hvg_ties, clip=p.clip), with_knn=False)
    np.testing.assert_array_equal(r.hvg_mask.cpu().numpy(), o["hvg_mask"])
    Z = r.scaled.values().cpu().numpy()
    np.testing.assert_allclose(Z, o["Z"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(r.scaled.inv_std.cpu().numpy(), o["scale_inv_std"], rtol=1e-7)
    ang = op.subspace_angle(r.pca.components.cpu().numpy().T.astype(np.float64), o["components"])
    assert ang < 2e-4, ang
