"""GPU community detection (csrc/cluster.cu) equals the oracle's restatement of the same
deterministic algorithm (labels, community count, modularity), and recovers planted clusters."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _graph(n=1500, k=6, seed=4):
    import torch
    from paper_2605_13928_b200 import pp
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((k, 8)) * 5.0
    lab = rng.integers(0, k, n)
    X = (centers[lab] + rng.standard_normal((n, 8))).astype(np.float32)
    Xd = torch.as_tensor(X, device="cuda")
    ki, kd = pp.neighbors(Xd, 15)
    return pp.neighbors_graph(ki, kd).connectivities, lab


@pytest.mark.parametrize("resolution", [1.0, 0.5])
def test_louvain_matches_oracle_and_recovers_clusters(resolution):
    import scipy.sparse as sp
    from sklearn.metrics import adjusted_rand_score
    from oracle import pipeline as op
    from paper_2605_13928_b200 import pp
    G, truth = _graph()
    lab, nc, q = pp.louvain(G, resolution=resolution, seed=3)
    ip, ix, w, n = G.to_host()
    C = sp.csr_matrix((w, ix, ip), shape=(n, n))
    olab, onc, oq = op.louvain(C, resolution=resolution, seed=3)
    np.testing.assert_array_equal(lab.cpu().numpy(), olab)
    assert nc == onc
    assert abs(q - oq) <= 1e-12 * max(1.0, abs(oq))
    assert q > 0.5
    if resolution == 1.0:
        assert adjusted_rand_score(truth, olab) > 0.9


@pytest.mark.parametrize("resolution", [1.0, 0.5])
def test_leiden_matches_oracle(resolution):
    import scipy.sparse as sp
    import scipy.sparse.csgraph as cg
    from sklearn.metrics import adjusted_rand_score
    from oracle import pipeline as op
    from paper_2605_13928_b200 import pp
    G, truth = _graph(n=1500, k=6, seed=11)
    lab, nc, q = pp.leiden(G, resolution=resolution, seed=3)
    ip, ix, w, n = G.to_host()
    C = sp.csr_matrix((w, ix, ip), shape=(n, n))
    olab, onc, oq = op.leiden(C, resolution=resolution, seed=3)
    np.testing.assert_array_equal(lab.cpu().numpy(), olab)
    assert nc == onc and abs(q - oq) <= 1e-12 * max(1.0, abs(oq))
    for c in range(nc):  # Leiden's guarantee: every community is connected
        idx = np.nonzero(olab == c)[0]
        assert cg.connected_components(C[idx][:, idx], directed=False)[0] == 1
    if resolution == 1.0:
        assert adjusted_rand_score(truth, olab) > 0.9
