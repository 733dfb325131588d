"""Synthetic negative-binomial single-cell counts -- CPU restatement (TEST INFRASTRUCTURE).

This module is test/bench infrastructure: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline leg may import it.  The product path generates the
same matrix on the GPU (``paper_2605_13928_b200/csrc/synth.cu``); both follow the
one specification below, so a C1-sized matrix generated here and on the device is
identical entry for entry (fp64 arithmetic, no FMA contraction in the sampler).

The reference (``/root/reference``) ships no data generator: the paper's workload is
the 1M-cell 10x mouse-brain dataset, which is out of scope
(SPEC.md:13).  The synthetic model follows SURVEY.md §8(d):

* gene log-means      log mu_g ~ N(-4.1, 1.7) (density ~7% after the planted
                      structure); the first ``n_mt`` genes are mitochondrial with
                      log mu_g ~ N(0.5 + ln(G/2000), 0.5) (~3-4% of counts);
* cell size factors   log s_c ~ N(0, 0.5);
* planted structure   log-fold-change L_cg = A[type(c), g] + sum_r u_cr B_rg, with
                      ``n_types`` cell types (skewed frequencies; each type
                      up-regulates ~2% of genes) and ``n_factors`` continuous
                      factors with decaying weights -- this makes the top-50 PCA
                      subspace well separated from the Marchenko-Pastur bulk;
* counts              x_cg ~ NB(mean = s_c mu_g exp(L_cg), theta = 0.5), sampled by
                      inverse CDF from one counter-based uniform per (c, g).

Every random number is a pure function of (seed, stream, i, j) through the
splitmix64 finaliser, so the matrix is independent of chunking and thread count.
"""
from __future__ import annotations

import dataclasses

import numpy as np

U64 = np.uint64
GOLDEN = U64(0x9E3779B97F4A7C15)
M1 = U64(0xBF58476D1CE4E5B9)
M2 = U64(0x94D049BB133111EB)
THETA = 0.5
TWO_PI = 6.283185307179586
MAX_COUNT = 100000  # inverse-CDF cap (never reached for these means)

# streams
S_GENE_MU, S_TYPE_MARK, S_TYPE_LFC, S_FACTOR_B, S_CELL_TYPE, S_CELL_SIZE, S_CELL_U, S_COUNT = range(1, 9)


@dataclasses.dataclass(frozen=True)
class SynthSpec:
    n_cells: int
    n_genes: int
    seed: int = 0
    n_types: int = 32
    n_factors: int = 64
    marker_frac: float = 0.02
    n_mt: int = 13

    def __post_init__(self):
        if self.n_cells <= 0 or self.n_genes <= 0:
            raise ValueError("n_cells and n_genes must be positive")
        if self.n_mt >= self.n_genes:
            raise ValueError("n_mt must be < n_genes")


def _mix(z):
    z = (z + GOLDEN)
    z = (z ^ (z >> U64(30))) * M1
    z = (z ^ (z >> U64(27))) * M2
    return z ^ (z >> U64(31))


def hash4(seed, stream, i, j):
    """splitmix64(splitmix64(splitmix64(seed*2^8 + stream) + i) + j) as uint64 arrays."""
    with np.errstate(over="ignore"):
        s = _mix(U64(seed) * U64(256) + U64(stream))
        h = _mix(s + np.asarray(i, dtype=U64))
        return _mix(h + np.asarray(j, dtype=U64))


def uniform(seed, stream, i, j):
    """U[0,1) with 53 random bits."""
    return (hash4(seed, stream, i, j) >> U64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def normal(seed, stream, i, j):
    """Box-Muller normal from two counter uniforms (j and j + 2^32)."""
    j = np.asarray(j, dtype=U64)
    u1 = uniform(seed, stream, i, j)
    u2 = uniform(seed, stream, i, j + U64(1 << 32))
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(TWO_PI * u2)


def gene_tables(spec: SynthSpec):
    """Per-gene log means (f64[G]), type LFC table A (f64[T,G]), factor loadings B (f64[R,G]),
    and the cumulative type-frequency table (f64[T])."""
    G, T, R, seed = spec.n_genes, spec.n_types, spec.n_factors, spec.seed
    g = np.arange(G, dtype=np.uint64)
    log_mu = -4.1 + 1.7 * normal(seed, S_GENE_MU, g, 0)
    mt = g < U64(spec.n_mt)
    mt_center = 0.5 + np.log(G / 2000.0)
    log_mu = np.where(mt, mt_center + 0.5 * normal(seed, S_GENE_MU, g, 1), log_mu)
    t = np.arange(T, dtype=np.uint64)[:, None]
    mark = uniform(seed, S_TYPE_MARK, t, g[None, :]) < spec.marker_frac
    lfc = 1.0 + 1.5 * uniform(seed, S_TYPE_LFC, t, g[None, :])
    A = np.where(mark & ~mt[None, :], lfc, 0.0)
    r = np.arange(R, dtype=np.uint64)[:, None]
    w = 0.30 * np.power(0.985, np.arange(R, dtype=np.float64))[:, None]
    B = w * normal(seed, S_FACTOR_B, r, g[None, :])
    B = np.where(mt[None, :], 0.0, B)
    freq = 1.0 / np.power(np.arange(1, T + 1, dtype=np.float64), 0.6)
    cum = np.cumsum(freq / freq.sum())
    cum[-1] = 1.0
    return log_mu, A, B, cum


def cell_tables(spec: SynthSpec, c0: int, c1: int, cum):
    """Per-cell type index (i32), log size factor (f64), factor scores (f64[n, R])."""
    c = np.arange(c0, c1, dtype=np.uint64)
    u = uniform(spec.seed, S_CELL_TYPE, c, 0)
    ctype = np.searchsorted(cum, u, side="right").astype(np.int32)
    ctype = np.minimum(ctype, spec.n_types - 1)
    log_s = 0.5 * normal(spec.seed, S_CELL_SIZE, c, 0)
    r = np.arange(spec.n_factors, dtype=np.uint64)[None, :]
    U = normal(spec.seed, S_CELL_U, c[:, None], r)
    return ctype, log_s, U


def nb_inverse_cdf(mu, u):
    """Smallest k with F_NB(k; mu, theta) > u, evaluated with the same fp64 recurrence the
    CUDA sampler uses (pk *= (k + theta) / (k + 1) * q; F += pk)."""
    theta = THETA
    p0 = np.exp(theta * np.log(theta / (theta + mu)))
    q = mu / (theta + mu)
    k = np.zeros(mu.shape, dtype=np.int64)
    pk = p0.copy()
    F = p0.copy()
    active = F <= u
    idx = np.nonzero(active)[0]
    while idx.size:
        kk = k[idx].astype(np.float64)
        pk[idx] = pk[idx] * ((kk + theta) / (kk + 1.0) * q[idx])
        k[idx] += 1
        F[idx] = F[idx] + pk[idx]
        still = (F[idx] <= u[idx]) & (k[idx] < MAX_COUNT) & (pk[idx] > 0.0)
        idx = idx[still]
    return k


def generate_csr(spec: SynthSpec, chunk_cells: int = 2048):
    """Generate the full CSR (indptr i64[N+1], indices i32[Z], data f32[Z]) on the CPU.

    Practical up to a few times 1e8 dense entries; larger matrices are generated on the
    device by the product's ``synth`` kernels."""
    N, G = spec.n_cells, spec.n_genes
    log_mu, A, B, cum = gene_tables(spec)
    g = np.arange(G, dtype=np.uint64)
    ind_parts, dat_parts, nnz = [], [], np.zeros(N, dtype=np.int64)
    for c0 in range(0, N, chunk_cells):
        c1 = min(N, c0 + chunk_cells)
        ctype, log_s, U = cell_tables(spec, c0, c1, cum)
        L = A[ctype] + U @ B                          # (n, G)
        mu = np.exp(log_s[:, None] + log_mu[None, :] + L)
        c = np.arange(c0, c1, dtype=np.uint64)
        u = uniform(spec.seed, S_COUNT, c[:, None], g[None, :])
        theta = THETA
        p0 = np.exp(theta * np.log(theta / (theta + mu)))
        nzmask = u >= p0
        rows, cols = np.nonzero(nzmask)
        vals = nb_inverse_cdf(mu[rows, cols], u[rows, cols])
        nnz[c0:c1] = np.bincount(rows, minlength=c1 - c0)
        ind_parts.append(cols.astype(np.int32))
        dat_parts.append(vals.astype(np.float32))
    indptr = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(nnz, out=indptr[1:])
    indices = np.concatenate(ind_parts) if ind_parts else np.zeros(0, np.int32)
    data = np.concatenate(dat_parts) if dat_parts else np.zeros(0, np.float32)
    return indptr, indices, data


def mt_mask(spec: SynthSpec):
    m = np.zeros(spec.n_genes, dtype=np.uint8)
    m[: spec.n_mt] = 1
    return m
