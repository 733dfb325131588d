"""GPU pipeline vs the committed golden fixtures (tests/golden/g600x300.npz), end to end
through paper_2605_13928_b200.pipeline.run (the fused path the bench times)."""
import numpy as np
import pytest

from oracle import pipeline as op

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def run():
    import torch
    from paper_2605_13928_b200 import pipeline
    from paper_2605_13928_b200.pp import DeviceCSR
    from tests.test_dist import _params
    g = np.load("tests/golden/g600x300.npz")
    X = DeviceCSR.from_host(g["indptr"], g["indices"], g["data"], 300)
    r = pipeline.run(X, torch.as_tensor(g["mt_mask"]).cuda(), _params())
    torch.cuda.synchronize()
    return g, r


def test_golden_qc_masks_hvg_exact(run):
    g, r = run
    for k in ("n_genes_by_counts", "total_counts", "n_cells_by_counts", "gene_total_counts"):
        np.testing.assert_array_equal(r.qc[k].cpu().numpy(), g["qc_" + k])
    np.testing.assert_array_equal(r.cell_mask.cpu().numpy(), g["cell_mask"])
    np.testing.assert_array_equal(r.gene_mask.cpu().numpy(), g["gene_mask"])
    np.testing.assert_array_equal(r.hvg_mask.cpu().numpy(), g["hvg_mask"])
    np.testing.assert_array_equal(r.hvg_stats["means"].cpu().numpy(), g["hvg_means"])
    np.testing.assert_array_equal(r.hvg_stats["variances"].cpu().numpy(), g["hvg_variances"])
    np.testing.assert_array_equal(r.X_log.row_scale.cpu().numpy(), g["row_scale"])


def test_golden_log_and_scale(run):
    g, r = run
    np.testing.assert_array_equal(r.X_log.indptr.cpu().numpy(), g["sub_indptr"])
    np.testing.assert_array_equal(r.X_log.indices.cpu().numpy(), g["sub_indices"])
    np.testing.assert_allclose(r.X_log.data.cpu().numpy(), g["log_data"], rtol=1e-5)
    Z = r.scaled.values().cpu().numpy()
    mag = np.maximum(np.abs(g["Z"]), np.abs(g["scale_mean"] * g["scale_inv_std"])[None, :])
    assert (np.abs(Z - g["Z"]) / mag).max() < 1e-5


def test_golden_pca_and_knn(run):
    g, r = run
    V = r.pca.components.cpu().numpy().T.astype(np.float64)
    assert op.subspace_angle(V, g["components"]) < 1e-3
    np.testing.assert_allclose(r.pca.variance.cpu().numpy(), g["variance"], rtol=1e-4)
    assert op.knn_recall(r.knn_index.cpu().numpy(), g["knn_idx"]) >= 0.999
