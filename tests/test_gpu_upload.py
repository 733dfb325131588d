"""ingest.upload_qc: chunked pinned H2D overlapped with per-chunk QC gives the
same device CSR and QC metrics as a plain upload + calculate_qc_metrics, for the 32-bit and the
compact u16 wire formats (escaped counts included), and the pipeline run from it equals the
plain run."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("wire", ["f32", "u16"])
def test_upload_qc_matches_plain_path(wire):
    from paper_2605_13928_b200 import ingest, pipeline, pp, synth
    spec = synth.Spec(9000, 1800, seed=21)
    X = synth.generate(spec)
    X.data[5::9973] = 70000.0  # escaped counts in the u16 wire format
    mt = synth.mt_mask(spec)
    H = ingest.HostCSR.from_device(X.to_u16() if wire == "u16" else X)
    Xd, qc = ingest.upload_qc(H, mt, chunk_rows=1000)  # 9 chunks, unaligned chunk starts
    torch.cuda.synchronize()
    assert torch.equal(Xd.indptr, X.indptr) and torch.equal(Xd.indices, X.indices) and torch.equal(Xd.data, X.data)
    ref = pp.calculate_qc_metrics(X, mt, row_splits=True)
    for k, v in ref.items():
        if v is not None:
            assert torch.equal(qc[k], v), k
    p = pipeline.Params(min_genes=30, max_pct_mt=25.0, n_top_genes=400, n_neighbors=10)
    r0 = pipeline.run(X, mt, p, timing=False)
    r1 = pipeline.run(Xd, mt, p, timing=False, qc=qc)
    torch.cuda.synchronize()
    assert torch.equal(r0.hvg_mask, r1.hvg_mask) and torch.equal(r0.knn_index, r1.knn_index)


def test_upload_qc_reports_invalid_counts():
    import numpy as np
    from paper_2605_13928_b200 import _lib, ingest
    ip = torch.tensor([0, 2, 3], dtype=torch.int64)
    H = ingest.HostCSR(ip, torch.tensor([0, 1, 1], dtype=torch.int32), torch.tensor([1.0, 0.5, 2.0]), 3)
    with pytest.raises(_lib.ScbError):
        ingest.upload_qc(H, torch.zeros(3, dtype=torch.uint8), chunk_rows=1)
    del np
