"""sc.tl.umap layout on the device vs the oracle's sequential restatement of umap-learn's
optimize_layout_euclidean (fixture tests/golden/umap600.npz, made by make_umap_golden.py).
The GPU applies the SGD updates edge-parallel (racing on the embedding), so parity is on layout
quality: trustworthiness of the 2-D embedding w.r.t. the input space and separation of the
planted clusters, each within tolerance of the oracle's on the same fuzzy graph."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_umap_layout_quality_matches_oracle():
    import torch
    from sklearn.manifold import trustworthiness
    from sklearn.metrics import silhouette_score
    from paper_2605_13928_b200 import pp
    g = np.load("tests/golden/umap600.npz")
    X, lab = g["X"], g["lab"]
    Xd = torch.as_tensor(X, device="cuda")
    ki, kd = pp.neighbors(Xd, 15)
    graph = pp.neighbors_graph(ki, kd)
    a, b = pp.umap_ab(0.5, 1.0)
    assert abs(a - float(g["a"])) < 1e-3 and abs(b - float(g["b"])) < 1e-3
    emb = pp.umap_layout(graph.connectivities, Xd[:, :2].contiguous(), n_epochs=int(g["epochs"]), seed=1).cpu().numpy()
    assert emb.shape == (len(X), 2) and np.isfinite(emb).all()
    t = trustworthiness(X, emb, n_neighbors=15)
    s = silhouette_score(emb, lab)
    assert float(g["trust_init"]) < 0.6          # the overlapping start is poor ...
    assert abs(t - float(g["trust"])) < 0.03, (t, float(g["trust"]))   # ... and both layouts fix it
    assert s > float(g["sil"]) - 0.1, (s, float(g["sil"]))


def test_umap_layout_quality_stable_across_seeds():
    """The racing SGD is not bit-reproducible, but its quality is: different seeds (negative
    samples) all reach the oracle's trustworthiness."""
    import torch
    from sklearn.manifold import trustworthiness
    from paper_2605_13928_b200 import pp
    g = np.load("tests/golden/umap600.npz")
    X = g["X"]
    Xd = torch.as_tensor(X, device="cuda")
    ki, kd = pp.neighbors(Xd, 15)
    graph = pp.neighbors_graph(ki, kd)
    for seed in (2, 3):
        emb = pp.umap_layout(graph.connectivities, Xd[:, :2].contiguous(), n_epochs=int(g["epochs"]),
                             seed=seed).cpu().numpy()
        assert trustworthiness(X, emb, n_neighbors=15) > float(g["trust"]) - 0.03
