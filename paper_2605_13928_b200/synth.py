"""Synthetic negative-binomial count matrices generated ON THE DEVICE (bench/test inputs).

Same model and counter-based randomness as ``oracle/synth.py``: gene
log-means N(-4.1, 1.7) (13 mitochondrial genes raised), cell size factors LogNormal(0, 0.5),
planted low-rank log-fold-changes (cell types + decaying continuous factors) and NB(theta=0.5)
counts drawn by inverse CDF from one splitmix64 uniform per (cell, gene).  The per-gene and
per-cell tables are a few MB and built on the host with numpy; the O(N*G) work is two kernels
per row chunk: ``scb_synth_logmean`` (fixed-order fp64 log means, including the rank-64 factor
term) and ``scb_synth_rows`` (sampling).  Generator v2: bit-identical to oracle/synth.py
(tests/test_gpu_synth.py).  Generation is input synthesis, never part of a timed region.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np
import torch

from . import _lib
from .pp import DeviceCSR, _ctx, _p, _stream

U64 = np.uint64
_GOLDEN, _M1, _M2 = U64(0x9E3779B97F4A7C15), U64(0xBF58476D1CE4E5B9), U64(0x94D049BB133111EB)
S_GENE_MU, S_TYPE_MARK, S_TYPE_LFC, S_FACTOR_B, S_CELL_TYPE, S_CELL_SIZE, S_CELL_U, S_COUNT = range(1, 9)


@dataclasses.dataclass(frozen=True)
class Spec:
    n_cells: int
    n_genes: int
    seed: int = 0
    n_types: int = 32
    n_factors: int = 64
    marker_frac: float = 0.02
    n_mt: int = 13


def _mix(z):
    z = z + _GOLDEN
    z = (z ^ (z >> U64(30))) * _M1
    z = (z ^ (z >> U64(27))) * _M2
    return z ^ (z >> U64(31))


def _uniform(seed, stream, i, j):
    with np.errstate(over="ignore"):
        s = _mix(U64(seed) * U64(256) + U64(stream))
        h = _mix(_mix(s + np.asarray(i, dtype=U64)) + np.asarray(j, dtype=U64))
    return (h >> U64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def _normal(seed, stream, i, j):
    j = np.asarray(j, dtype=U64)
    u1 = _uniform(seed, stream, i, j)
    u2 = _uniform(seed, stream, i, j + U64(1 << 32))
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(6.283185307179586 * u2)


def gene_tables(spec: Spec):
    G, T, R, seed = spec.n_genes, spec.n_types, spec.n_factors, spec.seed
    g = np.arange(G, dtype=U64)
    log_mu = -4.1 + 1.7 * _normal(seed, S_GENE_MU, g, 0)
    mt = g < U64(spec.n_mt)
    log_mu = np.where(mt, 0.5 + np.log(G / 2000.0) + 0.5 * _normal(seed, S_GENE_MU, g, 1), log_mu)
    t = np.arange(T, dtype=U64)[:, None]
    mark = _uniform(seed, S_TYPE_MARK, t, g[None, :]) < spec.marker_frac
    A = np.where(mark & ~mt[None, :], 1.0 + 1.5 * _uniform(seed, S_TYPE_LFC, t, g[None, :]), 0.0)
    r = np.arange(R, dtype=U64)[:, None]
    B = 0.30 * np.power(0.985, np.arange(R, dtype=np.float64))[:, None] * _normal(seed, S_FACTOR_B, r, g[None, :])
    B = np.where(mt[None, :], 0.0, B)
    freq = 1.0 / np.power(np.arange(1, T + 1, dtype=np.float64), 0.6)
    cum = np.cumsum(freq / freq.sum())
    cum[-1] = 1.0
    return log_mu, A, B, cum


def cell_tables(spec: Spec, c0: int, c1: int, cum):
    c = np.arange(c0, c1, dtype=U64)
    ctype = np.minimum(np.searchsorted(cum, _uniform(spec.seed, S_CELL_TYPE, c, 0), side="right"),
                       spec.n_types - 1).astype(np.int32)
    log_s = 0.5 * _normal(spec.seed, S_CELL_SIZE, c, 0)
    U = _normal(spec.seed, S_CELL_U, c[:, None], np.arange(spec.n_factors, dtype=U64)[None, :])
    return ctype, log_s, U


def mt_mask(spec: Spec, device="cuda"):
    m = torch.zeros(spec.n_genes, dtype=torch.uint8, device=device)
    m[: spec.n_mt] = 1
    return m


def row_nnz(spec: Spec, r0: int = 0, r1: Optional[int] = None, device="cuda", chunk: int = 16384) -> torch.Tensor:
    """Nonzeros per row of rows [r0, r1) (the generator's count pass only; e.g. to cut
    nnz-balanced cell shards before generating them)."""
    r1 = spec.n_cells if r1 is None else r1
    dev = torch.device(device)
    G = spec.n_genes
    log_mu, A, B, cum = gene_tables(spec)
    d_log_mu = torch.as_tensor(log_mu, device=dev)
    d_A = torch.as_tensor(A, device=dev).contiguous()
    d_B = torch.as_tensor(B, device=dev).contiguous()
    ctx, s = _ctx(d_log_mu), _stream(dev)
    nnz = torch.empty(r1 - r0, dtype=torch.int64, device=dev)
    xbuf = torch.empty((min(chunk, max(r1 - r0, 1)), G), dtype=torch.float64, device=dev)
    for c0 in range(r0, r1, chunk):
        c1 = min(r1, c0 + chunk)
        ct, ls, U = cell_tables(spec, c0, c1, cum)
        ct, ls, U = (torch.as_tensor(ct, device=dev), torch.as_tensor(ls, device=dev),
                     torch.as_tensor(U, device=dev).contiguous())
        _lib.call("scb_synth_logmean", ctx, c1 - c0, G, spec.n_factors, _p(d_log_mu), _p(d_A), _p(ct), _p(ls), _p(U),
                  _p(d_B), _p(xbuf), s)
        _lib.call("scb_synth_rows", ctx, spec.seed, c0, c1 - c0, G, _p(xbuf), 0, _p(nnz[c0 - r0:c1 - r0]), 0, 0, s)
    return nnz


def generate(spec: Spec, device="cuda", chunk: int = 16384) -> DeviceCSR:
    """Generate the whole CSR on ``device`` (two passes: count, fill)."""
    return generate_rows(spec, 0, spec.n_cells, device, chunk)


def generate_rows(spec: Spec, r0: int, r1: int, device="cuda", chunk: int = 16384) -> DeviceCSR:
    """Rows [r0, r1) of the global matrix (a cell shard), generated on ``device``."""
    dev = torch.device(device)
    G = spec.n_genes
    log_mu, A, B, cum = gene_tables(spec)
    d_log_mu = torch.as_tensor(log_mu, device=dev)
    d_A = torch.as_tensor(A, device=dev).contiguous()
    d_B = torch.as_tensor(B, device=dev).contiguous()
    ctx, s = _ctx(d_log_mu), _stream(dev)
    n = r1 - r0
    nnz = torch.empty(n, dtype=torch.int64, device=dev)
    tables = []
    for c0 in range(r0, r1, chunk):
        c1 = min(r1, c0 + chunk)
        ct, ls, U = cell_tables(spec, c0, c1, cum)
        tables.append((c0, c1, torch.as_tensor(ct, device=dev), torch.as_tensor(ls, device=dev),
                       torch.as_tensor(U, device=dev).contiguous()))
    xbuf = torch.empty((min(chunk, max(n, 1)), G), dtype=torch.float64, device=dev)

    def logmean(c0, c1, ct, ls, U):
        _lib.call("scb_synth_logmean", ctx, c1 - c0, G, spec.n_factors, _p(d_log_mu), _p(d_A), _p(ct), _p(ls), _p(U),
                  _p(d_B), _p(xbuf), s)
        return xbuf

    for (c0, c1, ct, ls, U) in tables:
        x = logmean(c0, c1, ct, ls, U)
        _lib.call("scb_synth_rows", ctx, spec.seed, c0, c1 - c0, G, _p(x), 0, _p(nnz[c0 - r0:c1 - r0]), 0, 0, s)
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(nnz, 0, out=indptr[1:])
    Z = int(indptr[-1].item())
    indices = torch.empty(Z, dtype=torch.int32, device=dev)
    data = torch.empty(Z, dtype=torch.float32, device=dev)
    for (c0, c1, ct, ls, U) in tables:
        x = logmean(c0, c1, ct, ls, U)
        _lib.call("scb_synth_rows", ctx, spec.seed, c0, c1 - c0, G, _p(x), _p(indptr[c0 - r0:c1 - r0]), 0,
                  _p(indices), _p(data), s)
    del xbuf
    return DeviceCSR(indptr, indices, data, G)
