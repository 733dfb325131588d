"""GPU parity of the ingest path (MatrixMarket text parsed on the device, COO -> CSR) against
scipy.io.mmread (the checker; scipy >= 1.12 reads through fast_matrix_market)."""
import io
import os

import numpy as np
import pytest
import scipy.io as sio
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


def _mm_bytes(M, field):
    b = io.BytesIO()
    sio.mmwrite(b, M, field=field)
    return b.getvalue()


def _check(X, ref):
    ref = ref.tocsr()
    ref.sort_indices()
    ip, ix, d, ncol = X.to_host()
    assert ncol == ref.shape[1] and len(ip) - 1 == ref.shape[0]
    np.testing.assert_array_equal(ip, ref.indptr)
    np.testing.assert_array_equal(ix, ref.indices)
    np.testing.assert_array_equal(d, ref.data.astype(np.float32))


@pytest.mark.parametrize("field", ["integer", "real", "pattern"])
@pytest.mark.parametrize("transpose", [False, True])
def test_mtx_parse_matches_scipy_unsorted_file_order(field, transpose):
    from paper_2605_13928_b200.ingest import parse_mtx_device
    M = sp.random(700, 300, density=0.05, format="coo", random_state=3)
    M.data = (np.round(M.data * 50) + 1 if field == "integer"
              else M.data * 10.0 ** np.random.default_rng(0).integers(-3, 4, M.nnz))
    raw = np.frombuffer(_mm_bytes(M, field), np.uint8)
    X, h = parse_mtx_device(raw, transpose=transpose)
    ref = sio.mmread(io.BytesIO(raw.tobytes()))
    _check(X, ref.T if transpose else ref)


def test_mtx_sorted_10x_order_fast_path_and_empty_cells():
    """10x writes column-major (by barcode) with ascending genes; empty cells in between."""
    from paper_2605_13928_b200.ingest import parse_mtx_device
    rng = np.random.default_rng(5)
    n_genes, n_cells = 400, 900
    C = sp.random(n_cells, n_genes, density=0.04, format="csr", random_state=5)
    C.data = np.floor(C.data * 30) + 1
    C[::7] = 0
    C.eliminate_zeros()
    C.sort_indices()
    lines = ["%%MatrixMarket matrix coordinate integer general", "%metadata_json: {}",
             f"{n_genes} {n_cells} {C.nnz}"]
    for c in range(n_cells):
        for k in range(C.indptr[c], C.indptr[c + 1]):
            lines.append(f"{C.indices[k] + 1} {c + 1} {int(C.data[k])}")
    raw = np.frombuffer(("\n".join(lines) + "\n").encode(), np.uint8)
    X, _ = parse_mtx_device(raw, transpose=True)
    _check(X, C)
    del rng


@pytest.mark.parametrize("bad, err", [
    ("1 1 3\n2 x 4\n", "malformed"),
    ("1 1 3\n", "data lines"),
    ("1 1 3\n1 1 4\n", "duplicate"),
    ("1 1 3\n9 1 4\n", "malformed"),
])
def test_mtx_errors(bad, err):
    from paper_2605_13928_b200.ingest import parse_mtx_device
    text = "%%MatrixMarket matrix coordinate integer general\n3 3 2\n" + bad
    with pytest.raises(RuntimeError, match=err):
        parse_mtx_device(np.frombuffer(text.encode(), np.uint8), transpose=False)


def test_read_10x_mtx_qc_matches_oracle(tmp_path):
    """A 10x directory (matrix.mtx genes x cells, features.tsv with MT- genes, barcodes) read
    on the device gives the oracle's QC metrics for the same counts."""
    import torch
    import paper_2605_13928_b200 as scb
    from paper_2605_13928_b200.ingest import read_10x_mtx
    from oracle import pipeline as op
    from oracle.synth import SynthSpec, generate_csr
    spec = SynthSpec(1500, 800, seed=11)
    ip, ix, d = generate_csr(spec)
    C = sp.csr_matrix((d, ix, ip), shape=(spec.n_cells, spec.n_genes))
    names = [f"MT-{i}" if i < 13 else f"GENE{i}" for i in range(spec.n_genes)]
    with open(os.path.join(tmp_path, "matrix.mtx"), "wb") as f:
        f.write(_mm_bytes(C.T.tocoo(), "integer"))
    with open(os.path.join(tmp_path, "features.tsv"), "w") as f:
        f.writelines(f"ENSG{i}\t{g}\tGene Expression\n" for i, g in enumerate(names))
    with open(os.path.join(tmp_path, "barcodes.tsv"), "w") as f:
        f.writelines(f"CELL{i}-1\n" for i in range(spec.n_cells))
    X, mt, genes, bcs = read_10x_mtx(str(tmp_path))
    assert genes == names and len(bcs) == spec.n_cells
    assert mt.cpu().numpy().sum() == 13
    C.sort_indices()
    _check(X, C)
    qc = scb.calculate_qc_metrics(X, mt)
    o = op.qc_metrics(op.CSR(C.indptr.astype(np.int64), C.indices.astype(np.int32), C.data.astype(np.float32),
                             spec.n_genes), mt.cpu().numpy())
    np.testing.assert_array_equal(qc["n_genes_by_counts"].cpu().numpy(), o["n_genes_by_counts"])
    np.testing.assert_array_equal(qc["total_counts_mt"].cpu().numpy(), o["total_counts_mt"])
    del torch
