"""Generates tests/golden/umap600.npz: planted clusters whose first two coordinates overlap
(so the initial layout is poor), the oracle's sequential umap layout of their exact-kNN fuzzy
graph, and its quality (trustworthiness, silhouette).  python tests/golden/make_umap_golden.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import pipeline as op  # noqa: E402

N, D, K, EPOCHS, SEED = 600, 10, 5, 120, 1
A, B = 0.5830300199, 1.3341669992  # umap find_ab_params(spread=1, min_dist=0.5)


def blobs(n=N, d=D, k=K, seed=3):
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((k, d)) * 6.0
    centers[:, :2] = 0.0  # clusters overlap in the initial 2-D layout
    lab = rng.integers(0, k, n)
    return (centers[lab] + rng.standard_normal((n, d))).astype(np.float32), lab


def main():
    from sklearn.manifold import trustworthiness
    from sklearn.metrics import silhouette_score
    X, lab = blobs()
    ki, kd = op.knn(X, 15)
    C, _, _, _ = op.umap_connectivities(ki, kd, len(X))
    emb = op.umap_layout(C, X[:, :2], EPOCHS, A, B, seed=SEED)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "umap600.npz")
    np.savez_compressed(out, X=X, lab=lab, emb=emb, trust=trustworthiness(X, emb, n_neighbors=15),
                        sil=silhouette_score(emb, lab), trust_init=trustworthiness(X, X[:, :2], n_neighbors=15),
                        epochs=EPOCHS, a=A, b=B)
    print(out, trustworthiness(X, emb, n_neighbors=15), silhouette_score(emb, lab))


if __name__ == "__main__":
    main()
