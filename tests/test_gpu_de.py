"""GPU sc.tl.rank_genes_groups (t-test vs rest, csrc/de.cu) against the oracle restatement:
scores / logfoldchanges bit-identical (exact fixed-point sums, explicit-rounding formulas),
gene ranking identical, p-values and BH-adjusted p-values vs scipy's t distribution."""
import numpy as np
import pytest

from tests.gpu_fixtures import C1, c1_inputs

pytestmark = pytest.mark.gpu


def test_rank_genes_groups_matches_oracle():
    import torch
    import paper_2605_13928_b200 as scb
    from oracle import pipeline as op
    from paper_2605_13928_b200 import pp
    X, mt = c1_inputs()
    P = C1["params"]
    Xd = scb.DeviceCSR.from_host(X.indptr, X.indices, X.data, X.n_cols)
    qc = scb.calculate_qc_metrics(Xd, torch.as_tensor(mt))
    cm, gm, kept = scb.filter_masks(qc, min_genes=P.min_genes, max_genes=P.max_genes, max_pct_mt=P.max_pct_mt, min_cells=P.min_cells)
    Xl = scb.normalize_log1p(scb.subset(Xd, cm, gm, kept), P.target_sum)
    rng = np.random.default_rng(0)
    labels = rng.integers(0, 5, Xl.n_rows).astype(np.int32)
    labels[: Xl.n_rows // 5] = 4  # unequal group sizes
    r = pp.rank_genes_groups(Xl, torch.as_tensor(labels, device="cuda"), 5)
    ip, ix, d, G = Xl.to_host()
    o = op.rank_genes_groups(op.CSR(ip, ix, d, G), labels, 5)
    np.testing.assert_array_equal(r["scores"].cpu().numpy(), o["scores"])
    np.testing.assert_array_equal(r["order"].cpu().numpy(), o["order"])
    np.testing.assert_allclose(r["logfoldchanges"].cpu().numpy(), o["logfoldchanges"], rtol=1e-12, atol=1e-12)
    pv, opv = r["pvals"].cpu().numpy(), o["pvals"]
    ok = opv > 1e-250
    np.testing.assert_allclose(pv[ok], opv[ok], rtol=1e-8)
    np.testing.assert_allclose(r["pvals_adj"].cpu().numpy()[ok], o["pvals_adj"][ok], rtol=1e-8)
