"""GPU edge cases of the whole path vs the oracle: tiny inputs (fewer cells/genes than one tile),
empty rows, never-expressed genes, explicit zeros, every cell filtered but a few, k close to the
number of cells, and a cell count that is not a multiple of any tile size."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import pipeline as op

pytestmark = pytest.mark.gpu


def _csr(dense):
    A = sp.csr_matrix(dense.astype(np.float32))
    return op.CSR(A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.astype(np.float32), dense.shape[1])


def _run(X, mt, p):
    import torch
    from paper_2605_13928_b200 import pipeline
    from paper_2605_13928_b200.pp import DeviceCSR
    Xd = DeviceCSR.from_host(X.indptr, X.indices, X.data, X.n_cols)
    r = pipeline.run(Xd, torch.as_tensor(mt).cuda(), pipeline.Params(**p.__dict__))
    torch.cuda.synchronize()
    return r


def _check(r, o, k):
    np.testing.assert_array_equal(r.cell_mask.cpu().numpy(), o["cell_mask"])
    np.testing.assert_array_equal(r.gene_mask.cpu().numpy(), o["gene_mask"])
    np.testing.assert_array_equal(r.hvg_mask.cpu().numpy(), o["hvg_mask"])
    ang = op.subspace_angle(r.pca.components.cpu().numpy().T.astype(np.float64), o["components"])
    assert ang < 1e-3, ang
    idx = r.knn_index.cpu().numpy()
    assert idx.shape == (o["knn_idx"].shape[0], k)
    assert op.knn_recall(idx, o["knn_idx"]) >= 0.999


def _random_counts(rng, n, g, density, scale=20):
    dense = (rng.random((n, g)) < density) * rng.integers(1, scale, (n, g))
    return dense


def test_tiny_matrix_below_one_tile():
    rng = np.random.default_rng(21)
    dense = _random_counts(rng, 150, 300, 0.3)
    X = _csr(dense)
    mt = np.zeros(300, np.uint8)
    mt[:5] = 1
    p = op.Params(min_genes=20, max_pct_mt=60.0, min_cells=3, n_top_genes=120, n_comps=20, n_neighbors=10)
    o = op.run(X, mt, p)
    _check(_run(X, mt, p), o, 10)


def test_empty_rows_dead_genes_explicit_zeros_ragged_n():
    rng = np.random.default_rng(22)
    n, g = 1037, 611                       # not a multiple of 32/128/256
    dense = _random_counts(rng, n, g, 0.15)
    dense[::17] = 0                        # empty cells (NaN pct_mt -> filtered)
    dense[:, 100:140] = 0                  # never-expressed genes (removed by min_cells)
    dense[:, 200] = 0
    dense[3, 200] = 1                      # a gene in fewer than min_cells cells
    X = _csr(dense)
    # explicit zeros stored in the CSR (kept by subset, ignored by the counts)
    A = sp.csr_matrix(dense.astype(np.float32))
    A.data[::97] = 0.0
    X = op.CSR(A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.astype(np.float32), g)
    mt = np.zeros(g, np.uint8)
    mt[:9] = 1
    p = op.Params(min_genes=30, max_pct_mt=25.0, min_cells=3, n_top_genes=200, n_comps=30, n_neighbors=15)
    o = op.run(X, mt, p)
    _check(_run(X, mt, p), o, 15)


def test_k_close_to_cell_count():
    rng = np.random.default_rng(23)
    dense = _random_counts(rng, 70, 400, 0.4)
    X = _csr(dense)
    mt = np.zeros(400, np.uint8)
    p = op.Params(min_genes=10, max_pct_mt=100.0, min_cells=1, n_top_genes=200, n_comps=20, n_neighbors=60)
    o = op.run(X, mt, p)
    _check(_run(X, mt, p), o, 60)


def test_pipeline_reports_invalid_counts_through_deferred_qc_check():
    """pipeline.run defers QC's data-validity check to the filter round trip: non-integral
    counts still raise (SCB_ERR_DATA), and the ctx is back in synchronous-check mode after."""
    import numpy as np
    import pytest
    import torch
    from paper_2605_13928_b200 import _lib, pipeline, pp
    ip = np.array([0, 2, 4, 6], np.int64)
    ix = np.array([0, 1, 1, 2, 0, 2], np.int32)
    d = np.array([1.0, 2.5, 3.0, 1.0, 4.0, 2.0], np.float32)
    X = pp.DeviceCSR.from_host(ip, ix, d, 3)
    with pytest.raises(_lib.ScbError, match="deferred"):
        pipeline.run(X, torch.zeros(3, dtype=torch.uint8), pipeline.Params(min_genes=0, min_cells=0), timing=False)
    with pytest.raises(_lib.ScbError):
        pp.calculate_qc_metrics(X, torch.zeros(3, dtype=torch.uint8))
