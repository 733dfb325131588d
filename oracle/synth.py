"""Synthetic negative-binomial single-cell counts -- CPU restatement (TEST INFRASTRUCTURE).

This module is test/bench infrastructure: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline leg may import it.  The product path generates the
same matrix on the GPU (``paper_2605_13928_b200/csrc/synth.cu``); both follow the
one specification below and use only correctly rounded IEEE-754 fp64 operations
(+, -, *, /, sqrt, rint, ldexp) in a fixed order for every per-entry quantity, so a
matrix generated here and on the device is identical entry for entry.  This is
checked on the GPU at C1 and on a 16k-row window of the C3 matrix
(``tests/test_gpu_synth.py``).

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

Per-entry arithmetic (generator version 2, identical on both sides):
  L  = A[t, g]; L = L + U[c, r] * B[r, g] for r = 0..R-1 (each product and sum rounded);
  x  = (log_s[c] + log_mu[g]) + L;  mu = det_exp(x) (below: Cody-Waite reduction,
  degree-13 Taylor polynomial by Horner, exact ldexp);
  p0 = sqrt(theta / (theta + mu))  (= (theta/(theta+mu))^theta for theta = 1/2);
  nonzero iff u >= p0; value = inverse-CDF recurrence (``nb_inverse_cdf``).
The per-gene and per-cell tables (log_mu, A, B, type, log_s, U) are computed on the
host with numpy by both paths from the same formulas.

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


# det_exp: exp(x) from correctly rounded fp64 operations only (same sequence in csrc/synth.cu)
_INV_LN2 = float.fromhex("0x1.71547652b82fep+0")
_LN2_HI = float.fromhex("0x1.62e42fee00000p-1")
_LN2_LO = float.fromhex("0x1.a39ef35793c76p-33")
_EXP_C = [float.fromhex(h) for h in (
    "0x1.0000000000000p+0", "0x1.0000000000000p+0", "0x1.0000000000000p-1", "0x1.5555555555555p-3",
    "0x1.5555555555555p-5", "0x1.1111111111111p-7", "0x1.6c16c16c16c17p-10", "0x1.a01a01a01a01ap-13",
    "0x1.a01a01a01a01ap-16", "0x1.71de3a556c734p-19", "0x1.27e4fb7789f5cp-22", "0x1.ae64567f544e4p-26",
    "0x1.1eed8eff8d898p-29", "0x1.6124613a86d09p-33")]


def det_exp(x):
    """exp(x) for |x| < 700: k = rint(x/ln2), r = (x - k ln2_hi) - k ln2_lo, Taylor-13 Horner, ldexp(p, k).
    Relative error ~1 ulp; bit-identical to the device's ``det_exp`` (no FMA contraction there)."""
    x = np.asarray(x, dtype=np.float64)
    k = np.rint(x * _INV_LN2)
    r = x - k * _LN2_HI
    r -= k * _LN2_LO
    p = np.full_like(r, _EXP_C[13])
    for c in _EXP_C[12::-1]:   # in place: each product and sum still rounded separately
        np.multiply(p, r, out=p)
        np.add(p, c, out=p)
    return np.ldexp(p, k.astype(np.int32))


def log_means(A_rows, U, B, log_s, log_mu):
    """x[c, g] = (log_s[c] + log_mu[g]) + (A[t,g] + sum_r U[c,r] B[r,g]) in the fixed order."""
    L = np.array(A_rows, dtype=np.float64, copy=True)
    n, G = L.shape
    gb = 512  # gene blocks that stay in cache across the R passes
    tmp = np.empty((n, gb), dtype=np.float64)
    for g0 in range(0, G, gb):
        g1 = min(G, g0 + gb)
        Lb, t = L[:, g0:g1], tmp[:, :g1 - g0]
        for r in range(U.shape[1]):
            np.multiply(U[:, r:r + 1], B[r, g0:g1][None, :], out=t)
            np.add(Lb, t, out=Lb)
    return (log_s[:, None] + log_mu[None, :]) + L


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


def _chunk_entries(spec: SynthSpec, c0: int, c1: int, tables):
    log_mu, A, B, cum = tables
    G = spec.n_genes
    g = np.arange(G, dtype=np.uint64)
    ctype, log_s, U = cell_tables(spec, c0, c1, cum)
    mu = det_exp(log_means(A[ctype], U, B, log_s, log_mu))
    c = np.arange(c0, c1, dtype=np.uint64)
    u = uniform(spec.seed, S_COUNT, c[:, None], g[None, :])
    p0 = np.sqrt(THETA / (THETA + mu))
    rows, cols = np.nonzero(u >= p0)
    vals = nb_inverse_cdf(mu[rows, cols], u[rows, cols])
    return np.bincount(rows, minlength=c1 - c0), cols.astype(np.int32), vals.astype(np.float32)


_POOL_ARGS = {}
_NATIVE = None


def native_lib():
    """ctypes handle of oracle/build/libscb_oracle.so (oracle/csynth.c), or None if not built."""
    global _NATIVE
    if _NATIVE is None:
        import ctypes
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "build", "libscb_oracle.so")
        if not os.path.exists(path):
            return None
        lib = ctypes.CDLL(path)
        P = ctypes.c_void_p
        lib.scb_oracle_synth_rows.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                              ctypes.c_int32, P, P, P, P, P, P, P, P, P, P, ctypes.c_int32]
        lib.scb_oracle_synth_rows.restype = ctypes.c_int
        _NATIVE = lib
    return _NATIVE


def generate_csr_native(spec: SynthSpec, rows=None, threads: int = 0):
    """generate_csr through the C restatement (oracle/csynth.c, OpenMP over rows): the same
    matrix, bit for bit; ~100x faster than numpy for >= 1e8 entries."""
    import os
    threads = threads or len(os.sched_getaffinity(0))
    lib = native_lib()
    if lib is None:
        raise RuntimeError("oracle/build/libscb_oracle.so not built (make -C oracle)")
    r0, r1 = (0, spec.n_cells) if rows is None else rows
    n, G, R = r1 - r0, spec.n_genes, spec.n_factors
    log_mu, A, B, cum = gene_tables(spec)
    ctype, log_s, U = cell_tables(spec, r0, r1, cum)
    arrs = [np.ascontiguousarray(a) for a in (log_mu, A, ctype.astype(np.int32), log_s, U, B)]
    ptr = [a.ctypes.data for a in arrs]
    nnz = np.zeros(n, dtype=np.int64)
    rc = lib.scb_oracle_synth_rows(spec.seed, r0, n, G, R, *ptr, None, nnz.ctypes.data, None, None, threads)
    if rc:
        raise MemoryError("scb_oracle_synth_rows failed")
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(nnz, out=indptr[1:])
    indices = np.empty(int(indptr[-1]), dtype=np.int32)
    data = np.empty(int(indptr[-1]), dtype=np.float32)
    rc = lib.scb_oracle_synth_rows(spec.seed, r0, n, G, R, *ptr, indptr.ctypes.data, None, indices.ctypes.data,
                                   data.ctypes.data, threads)
    if rc:
        raise MemoryError("scb_oracle_synth_rows failed")
    return indptr, indices, data


def _pool_chunk(w):
    return _chunk_entries(_POOL_ARGS["spec"], w[0], w[1], _POOL_ARGS["tables"])


def generate_csr(spec: SynthSpec, chunk_cells: int = 2048, rows=None, threads: int = 1):
    """Generate the CSR (indptr i64[n+1], indices i32[Z], data f32[Z]) of rows [r0, r1) (default:
    all cells) on the CPU; ``threads`` > 1 runs row chunks in that many forked worker processes.

    Practical up to a few times 1e8 dense entries; larger matrices are generated on the
    device by the product's ``synth`` kernels."""
    r0, r1 = (0, spec.n_cells) if rows is None else rows
    tables = gene_tables(spec)
    starts = list(range(r0, r1, chunk_cells))
    work = [(c0, min(r1, c0 + chunk_cells)) for c0 in starts]
    if threads > 1 and len(work) > 1:
        import multiprocessing as mp
        _POOL_ARGS.update(spec=spec, tables=tables)
        with mp.get_context("fork").Pool(threads) as pool:
            parts = pool.map(_pool_chunk, work)
        _POOL_ARGS.clear()
    else:
        parts = [_chunk_entries(spec, a, b, tables) for a, b in work]
    n = r1 - r0
    nnz = np.concatenate([p[0] for p in parts]) if parts else np.zeros(0, np.int64)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(nnz, out=indptr[1:])
    indices = np.concatenate([p[1] for p in parts]) if parts else np.zeros(0, np.int32)
    data = np.concatenate([p[2] for p in parts]) if parts else np.zeros(0, np.float32)
    return indptr, indices, data


def mt_mask(spec: SynthSpec):
    m = np.zeros(spec.n_genes, dtype=np.uint8)
    m[: spec.n_mt] = 1
    return m
