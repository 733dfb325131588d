"""GPU parity of PCA: tcgen05 Gram (3xBF16, fp32-fed and pre-split-plane-fed), float64 eigensolve,
tcgen05 projection."""
import numpy as np
import pytest

from oracle import pipeline as op
from tests.gpu_fixtures import C1, c1_oracle

pytestmark = pytest.mark.gpu


def _scaled_from_host(Z, H):
    import torch
    from paper_2605_13928_b200 import pp
    ld = pp.padded_width(H)
    Zp = np.zeros((Z.shape[0], ld), dtype=np.float32)
    Zp[:, :H] = Z
    Zp[:, H] = 1.0
    return pp.Scaled(torch.as_tensor(Zp).cuda(), H, H, None, None)


@pytest.mark.parametrize("n,h", [(1000, 200), (4099, 1000), (70001, 300)])
def test_gram_matches_fp64(n, h):
    import torch
    from paper_2605_13928_b200 import pp
    rng = np.random.default_rng(n)
    Z = rng.standard_normal((n, h)).astype(np.float32)
    sc = _scaled_from_host(Z, h)
    C = pp.gram(sc).cpu().numpy()
    Zp = sc.Z.cpu().numpy().astype(np.float64)
    ref = Zp.T @ Zp
    scale = np.sqrt(np.outer(np.diag(ref), np.diag(ref)))
    err = np.abs(C - ref) / np.maximum(scale, 1e-30)
    # tcgen05 FP32 accumulation rounds toward zero: a systematic relative bias on monotone sums
    # (the diagonal) within one K-slice; slices are <= 8k cells.
    assert err.max() < 1e-3, err.max()
    off = err.copy()
    np.fill_diagonal(off, 0)
    assert off.max() < 2e-6, off.max()
    np.testing.assert_array_equal(C, C.T)


def test_pca_matches_oracle():
    from paper_2605_13928_b200 import pp
    o = c1_oracle(False)
    Z = o["Z"]
    H = Z.shape[1]
    sc = _scaled_from_host(Z, H)
    r = pp.pca(sc, C1["params"].n_comps)
    V = r.components.cpu().numpy().T.astype(np.float64)   # [H][k]
    Vo = o["components"]
    ang = op.subspace_angle(V, Vo)
    assert ang < 1e-3, ang
    lam = r.variance.cpu().numpy()
    np.testing.assert_allclose(lam, o["variance"], rtol=1e-4)
    np.testing.assert_allclose(r.variance_ratio.cpu().numpy(), o["variance_ratio"], rtol=1e-4)
    # per-component agreement (sign-canonical) where the eigen-gap is not tiny
    spec = o["spectrum"]
    k = V.shape[1]
    gaps = np.minimum(np.abs(spec[:k] - np.r_[np.inf, spec[:k - 1]]), np.abs(spec[:k] - spec[1:k + 1])) / spec[:k]
    for j in range(k):
        if gaps[j] > 1e-2:
            c = abs(float(V[:, j] @ Vo[:, j]))
            assert c > 1 - 1e-6, (j, c, gaps[j])
            np.testing.assert_allclose(V[:, j], Vo[:, j], atol=1e-4)
    X = r.X_pca.cpu().numpy()[:, :k]
    # embedding in the oracle's basis (rotation within near-degenerate pairs allowed)
    Xo = o["X_pca"].astype(np.float64)
    resid = X - Xo @ (Vo.T @ V)
    assert np.abs(resid).max() < 1e-3 * np.abs(Xo).max(), np.abs(resid).max()
    assert np.all(r.X_pca.cpu().numpy()[:, k:] == 0)


@pytest.mark.parametrize("n,h", [(3001, 200), (20011, 1000)])
def test_gram_split_planes_match_converter_path(n, h):
    """scb_split_bf16's planes are bit-exact round-to-nearest BF16 (hi) and BF16(Z - hi) (lo); fed
    to gram_split_kernel they give the operands of the in-kernel-converter path.  The planes
    kernel restarts its TMEM accumulators every 256 cells (fp32 running sums), so it is at least
    as close to the fp64 Gram as the converter path (8k-cell accumulations), and both agree."""
    import torch
    from paper_2605_13928_b200 import pp
    rng = np.random.default_rng(n + h)
    Z = rng.standard_normal((n, h)).astype(np.float32)
    sc = _scaled_from_host(Z, h)
    C1 = pp.gram(sc, planes=False).cpu().numpy()
    C2 = pp.gram(sc, keep_planes=True).cpu().numpy()
    from paper_2605_13928_b200 import _lib
    dt = _lib.plane_dtype()
    hi = sc.Z.to(dt)
    lo = (sc.Z - hi.float()).to(dt)
    assert torch.equal(sc.Z_hi.view(torch.int16), hi.view(torch.int16))
    assert torch.equal(sc.Z_lo.view(torch.int16), lo.view(torch.int16))
    scale = np.sqrt(np.outer(np.diag(C1), np.diag(C1)))
    Z64 = Z.astype(np.float64)
    C64 = Z64.T @ Z64
    e1 = (np.abs(C1[:h, :h] - C64) / np.maximum(scale[:h, :h], 1e-30)).max()
    e2 = (np.abs(C2[:h, :h] - C64) / np.maximum(scale[:h, :h], 1e-30)).max()
    if int(_lib.load().scb_plane_format()) == 1:
        # one-product (hi x hi) planes Gram: fp16 operand rounding (2^-12 per operand, unbiased),
        # against the converter path's three products
        assert e2 < 2e-4, e2
        assert (np.abs(C1 - C2) / np.maximum(scale, 1e-30)).max() < 2e-4
    else:
        assert e2 <= e1 * 1.01 + 1e-7, (e1, e2)
        assert e2 < 1e-5, e2
        assert (np.abs(C1 - C2) / np.maximum(scale, 1e-30)).max() < 2e-5


def test_pca_rank_deficient_uses_cgs2_fallback():
    """60 distinct cells repeated (covariance rank <= 59 < the 96-wide block): Cholesky-QR breaks
    down and the solve is redone with CGS2; the leading components still match numpy's eigh."""
    import torch
    from oracle import pipeline as op
    from paper_2605_13928_b200 import pp
    rng = np.random.default_rng(2)
    base = rng.standard_normal((60, 200)) * np.linspace(3.0, 0.2, 200)[None, :]
    Z = np.repeat(base, 50, axis=0).astype(np.float32)
    sc = _scaled_from_host(Z, 200)
    r = pp.pca(sc, n_comps=10)
    torch.cuda.synchronize()
    C, m = op.covariance(Z)
    w, V = np.linalg.eigh(C)
    V = V[:, np.argsort(w)[::-1][:10]]
    got = r.components.cpu().numpy().T.astype(np.float64)
    assert op.subspace_angle(got, V) < 1e-4  # 3xBF16 Gram (fp32 accumulation) vs an fp64 covariance
    np.testing.assert_allclose(r.variance.cpu().numpy(), np.sort(w)[::-1][:10], rtol=1e-5)


def test_scale_planes_bit_identical_to_split_and_projection_close():
    """scale_dense(planes=True) writes exactly split_bf16(scale_dense fp32); the planes projection
    (3xBF16) matches the fp32 (3xTF32) projection to ~1e-5 of the embedding's scale."""
    import torch
    from paper_2605_13928_b200 import pipeline, pp, synth
    spec = synth.Spec(6000, 2000, seed=12)
    X = synth.generate(spec)
    r = pipeline.run(X, synth.mt_mask(spec), pipeline.Params(min_genes=30, n_top_genes=600), timing=False,
                     with_knn=False)
    Xl = r.X_log
    slot = pp.gene_slots(r.hvg_index, Xl.n_cols)
    H = int(r.hvg_index.numel())
    mean, inv = r.scaled.mean, r.scaled.inv_std
    f32 = pp.scale_dense(Xl, slot, H, mean, inv, 10.0)
    pl = pp.scale_dense(Xl, slot, H, mean, inv, 10.0, planes=True)
    pp.split_planes(f32)
    torch.cuda.synchronize()
    assert pl.Z is None
    assert torch.equal(pl.Z_hi.view(torch.int16), f32.Z_hi.view(torch.int16))
    assert torch.equal(pl.Z_lo.view(torch.int16), f32.Z_lo.view(torch.int16))
    rel = ((pl.dense() - f32.Z).abs() / f32.Z.abs().clamp_min(1e-3)).max().item()
    assert rel < 2e-5
    comp_t, cmean = r.pca.components, r.pca.col_mean
    npad = 64
    ct = torch.zeros((npad, pl.ld), dtype=torch.float32, device="cuda")
    ct[: comp_t.shape[0], : comp_t.shape[1]] = comp_t
    a = pp.project(f32, ct, cmean, 50)
    b = pp.project(pl, ct, cmean, 50)
    torch.cuda.synchronize()
    err = (a - b).abs().max().item() / a.abs().max().item()
    assert err < 1e-4, err
    assert torch.all(b[:, 50:] == 0)
