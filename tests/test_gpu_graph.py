"""GPU parity of sc.pp.neighbors' graph outputs (umap fuzzy_simplicial_set connectivities and
the distances matrix) against the oracle restatement (oracle/pipeline.py umap_connectivities)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _graph_case(n, d, k, seed, dup=False):
    import torch
    from oracle import pipeline as op
    rng = np.random.default_rng(seed)
    E = rng.standard_normal((n, d)).astype(np.float32)
    E[: n // 10] *= 0.2  # denser core: hub cells with long rows
    if dup:
        E[5] = E[4]  # exact duplicate: a zero non-self distance
    ki, kd = op.knn(E, k)
    return torch.as_tensor(ki, device="cuda"), torch.as_tensor(kd, device="cuda"), op.umap_connectivities(ki, kd, n)


@pytest.mark.parametrize("n,d,k,dup", [(3000, 12, 15, False), (2500, 8, 30, True)])
def test_neighbors_graph_matches_oracle(n, d, k, dup):
    from paper_2605_13928_b200 import pp
    ki, kd, (C, Dm, sig, rho) = _graph_case(n, d, k, 7, dup)
    g = pp.neighbors_graph(ki, kd)
    np.testing.assert_allclose(g.rho.cpu().numpy(), rho, rtol=0, atol=0)
    np.testing.assert_allclose(g.sigma.cpu().numpy(), sig, rtol=1e-4)
    ip, ix, v, ncol = g.connectivities.to_host()
    assert ncol == n
    np.testing.assert_array_equal(ip, C.indptr)
    np.testing.assert_array_equal(ix, C.indices)
    np.testing.assert_allclose(v, C.data, rtol=1e-4, atol=1e-7)
    # symmetric with values in (0, 1]
    assert v.min() > 0 and v.max() <= 1.0
    dp, dx, dv, _ = g.distances.to_host()
    np.testing.assert_array_equal(dp, Dm.indptr)
    np.testing.assert_array_equal(dx, Dm.indices)
    np.testing.assert_array_equal(dv, Dm.data)
