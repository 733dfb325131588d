"""GPU parity of the optional regress_out + scale step (paper Table 1 step 4) vs the oracle."""
import dataclasses

import numpy as np
import pytest

from tests.gpu_fixtures import C1, c1_inputs

pytestmark = pytest.mark.gpu


def _oracle():
    from oracle import pipeline as op
    X, mt = c1_inputs()
    return op.run(X, mt, dataclasses.replace(C1["params"], regress_out=True), with_knn=False)


def test_regress_out_scale_matches_oracle():
    import torch
    import paper_2605_13928_b200 as scb
    from paper_2605_13928_b200 import pipeline
    X, mt = c1_inputs()
    o = _oracle()
    P = C1["params"]
    p = pipeline.Params(min_genes=P.min_genes, max_genes=P.max_genes, max_pct_mt=P.max_pct_mt, min_cells=P.min_cells,
                        target_sum=P.target_sum, n_top_genes=P.n_top_genes, n_bins=P.n_bins, max_value=P.max_value,
                        n_comps=P.n_comps, n_neighbors=P.n_neighbors, regress_out=True)
    Xd = scb.DeviceCSR.from_host(X.indptr, X.indices, X.data, X.n_cols)
    r = pipeline.run(Xd, torch.as_tensor(mt, device="cuda"), p, with_knn=False, timing=False)
    np.testing.assert_array_equal(r.hvg_mask.cpu().numpy(), o["hvg_mask"])
    Z = r.scaled.values().cpu().numpy()
    ref = o["Z"]
    assert Z.shape == ref.shape
    err = np.abs(Z.astype(np.float64) - ref) / np.maximum(np.abs(ref), 1.0)
    assert err.max() < 1e-5, err.max()
    np.testing.assert_allclose(r.scaled.inv_std.cpu().numpy(), o["scale_inv_std"], rtol=1e-7)
    full = r.scaled.Z.cpu().numpy()
    assert np.all(full[:, r.scaled.ones_col] == 1.0) and np.all(full[:, r.scaled.H + 1:] == 0.0)
    # the residual columns have zero mean and unit variance before clipping
    assert np.abs(Z.astype(np.float64).mean(0)).max() < 0.05


def test_regress_out_scale_step_api_matches_pipeline():
    import torch
    import paper_2605_13928_b200 as scb
    X, mt = c1_inputs()
    o = _oracle()
    P = C1["params"]
    Xd = scb.DeviceCSR.from_host(X.indptr, X.indices, X.data, X.n_cols)
    qc = scb.calculate_qc_metrics(Xd, torch.as_tensor(mt))
    cm, gm, kept = scb.filter_masks(qc, min_genes=P.min_genes, max_genes=P.max_genes, max_pct_mt=P.max_pct_mt, min_cells=P.min_cells)
    Xl = scb.normalize_log1p(scb.subset(Xd, cm, gm, kept), P.target_sum)
    _, hvg_index, _ = scb.highly_variable_genes(Xl, P.n_top_genes, P.n_bins)
    sc = scb.regress_out_scale(Xl, hvg_index, qc, cm, P.max_value)
    Z = sc.values().cpu().numpy()
    err = np.abs(Z.astype(np.float64) - o["Z"]) / np.maximum(np.abs(o["Z"]), 1.0)
    assert err.max() < 1e-5, err.max()
