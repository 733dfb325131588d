"""Ingest: MatrixMarket / 10x Genomics ``matrix.mtx`` -> device CSR.

The host reads the file bytes and parses only the MatrixMarket banner, comments and size line
(``mtx_header``); the data lines are parsed on the GPU (``scb_mtx_parse``) and the CSR over cells
is built there (``scb_coo_to_csr``).  ``read_10x_mtx`` mirrors ``sc.read_10x_mtx``: a 10x
directory holds ``matrix.mtx`` (genes x cells), ``features.tsv`` (or ``genes.tsv``; gene symbol in
column 2) and ``barcodes.tsv``; the returned matrix is cells x genes, and the mitochondrial mask
marks gene symbols starting with ``MT-`` (Scanpy's ``var_names.str.startswith("MT-")``).
Gzipped files are decompressed on the host.  No CPU fallback: parsing requires the CUDA library.
"""
from __future__ import annotations

import dataclasses
import gzip
import os
import warnings
from typing import List, Optional, Tuple

import numpy as np
import torch

from . import _lib
from .pp import DeviceCSR, _ctx, _p, _stream

FIELDS = {"integer": 0, "real": 1, "double": 1, "pattern": 2}


@dataclasses.dataclass
class MtxHeader:
    field: int          # 0 integer, 1 real, 2 pattern
    n_rows: int         # file rows (genes for 10x)
    n_cols: int         # file columns (cells for 10x)
    nnz: int
    data_offset: int    # byte offset of the first data line


def mtx_header(buf: np.ndarray) -> MtxHeader:
    """Parse the MatrixMarket banner, comment lines and size line of ``buf`` (uint8)."""
    def line_at(pos):
        end = int(np.argmax(buf[pos:pos + (1 << 20)] == 10)) if pos < buf.size else 0
        if pos + end >= buf.size or buf[pos + end] != 10:
            end = buf.size - pos
        return bytes(buf[pos:pos + end]).decode("ascii", "replace"), pos + end + 1

    banner, pos = line_at(0)
    parts = banner.strip().split()
    if len(parts) < 5 or parts[0].lower() != "%%matrixmarket" or parts[1].lower() != "matrix":
        raise ValueError(f"not a MatrixMarket matrix file: {banner[:80]!r}")
    if parts[2].lower() != "coordinate":
        raise ValueError("only the sparse 'coordinate' format is supported")
    field = parts[3].lower()
    if field not in FIELDS:
        raise ValueError(f"unsupported MatrixMarket field {field!r}")
    if parts[4].lower() != "general":
        raise ValueError(f"unsupported MatrixMarket symmetry {parts[4]!r} (only 'general')")
    while True:
        line, nxt = line_at(pos)
        s = line.strip()
        if s and not s.startswith("%"):
            break
        if nxt > buf.size:
            raise ValueError("MatrixMarket size line missing")
        pos = nxt
    dims = s.split()
    if len(dims) != 3:
        raise ValueError(f"bad MatrixMarket size line {s!r}")
    m, n, nnz = (int(x) for x in dims)
    return MtxHeader(FIELDS[field], m, n, nnz, min(nxt, buf.size))


def _read_bytes(path: str) -> np.ndarray:
    if path.endswith(".gz"):
        with gzip.open(path, "rb") as f:
            return np.frombuffer(f.read(), dtype=np.uint8)
    return np.fromfile(path, dtype=np.uint8)


def parse_mtx_device(buf: np.ndarray, transpose: bool = True, device=None) -> Tuple[DeviceCSR, MtxHeader]:
    """MatrixMarket bytes (host) -> device CSR.  ``transpose`` (10x convention) makes the CSR
    rows the file's columns (cells) and its columns the file's rows (genes)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    h = mtx_header(buf)
    n = int(buf.size)
    text = torch.empty(n + 16, dtype=torch.uint8, device=dev)  # 16 B of padding for the vector loads
    with warnings.catch_warnings():  # read-only numpy buffers are only read here
        warnings.simplefilter("ignore", UserWarning)
        host = torch.from_numpy(np.ascontiguousarray(buf))
    if n:
        text[:n].copy_(host.pin_memory() if n >= (64 << 20) else host, non_blocking=False)
    nnz = h.nnz
    row = torch.empty(nnz, dtype=torch.int32, device=dev)
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=torch.float32, device=dev)
    ctx, s = _ctx(text), _stream(dev)
    _lib.call("scb_mtx_parse", ctx, _p(text), h.data_offset, n, h.field, nnz, h.n_rows, h.n_cols,
              _p(row), _p(col), _p(val), s)
    major, minor = (col, row) if transpose else (row, col)
    n_major, n_minor = (h.n_cols, h.n_rows) if transpose else (h.n_rows, h.n_cols)
    del text
    indptr = torch.empty(n_major + 1, dtype=torch.int64, device=dev)
    indices = torch.empty(nnz, dtype=torch.int32, device=dev)
    data = torch.empty(nnz, dtype=torch.float32, device=dev)
    _lib.call("scb_coo_to_csr", ctx, _p(major), _p(minor), _p(val), nnz, n_major, _p(indptr), _p(indices),
              _p(data), s)
    return DeviceCSR(indptr, indices, data, n_minor), h


def read_mtx(path: str, transpose: bool = False, device=None) -> DeviceCSR:
    """sc.read_mtx: the file's rows become CSR rows unless ``transpose``."""
    X, _ = parse_mtx_device(_read_bytes(path), transpose=transpose, device=device)
    return X


def _find(d: str, names: List[str]) -> Optional[str]:
    for nm in names:
        for ext in ("", ".gz"):
            p = os.path.join(d, nm + ext)
            if os.path.exists(p):
                return p
    return None


def read_10x_mtx(path: str, device=None):
    """sc.read_10x_mtx(path): returns (X cells x genes DeviceCSR, mt_mask uint8[genes] on the
    device, gene symbols, barcodes)."""
    mtx = _find(path, ["matrix.mtx"])
    if mtx is None:
        raise FileNotFoundError(f"no matrix.mtx[.gz] in {path}")
    X, h = parse_mtx_device(_read_bytes(mtx), transpose=True, device=device)
    feat = _find(path, ["features.tsv", "genes.tsv"])
    genes: List[str] = []
    if feat is not None:
        opener = gzip.open if feat.endswith(".gz") else open
        with opener(feat, "rt") as f:
            for line in f:
                cols = line.rstrip("\n").split("\t")
                genes.append(cols[1] if len(cols) > 1 else cols[0])
        if len(genes) != h.n_rows:
            raise ValueError(f"{feat}: {len(genes)} genes, matrix has {h.n_rows}")
    else:
        genes = [str(i) for i in range(h.n_rows)]
    bc = _find(path, ["barcodes.tsv"])
    barcodes: List[str] = []
    if bc is not None:
        opener = gzip.open if bc.endswith(".gz") else open
        with opener(bc, "rt") as f:
            barcodes = [ln.rstrip("\n").split("\t")[0] for ln in f]
    mt = np.array([g.upper().startswith("MT-") for g in genes], dtype=np.uint8)
    return X, torch.as_tensor(mt, device=X.device), genes, barcodes


# ----------------------------------------------------------------------------- host -> device with QC overlap
@dataclasses.dataclass
class HostCSR:
    """A count matrix in pinned host memory, in the 32-bit layout (int32 indices, float32 counts)
    or the compact u16 wire layout (uint16 indices and counts, counts >= 65535 escaped to the
    sorted (esc_pos, esc_val) table) -- see ``DeviceCSR.to_u16``."""
    indptr: torch.Tensor
    indices: torch.Tensor
    data: torch.Tensor
    n_cols: int
    esc_pos: Optional[torch.Tensor] = None
    esc_val: Optional[torch.Tensor] = None

    @staticmethod
    def from_device(X: DeviceCSR) -> "HostCSR":
        def pin(t):
            return None if t is None else t.cpu().pin_memory()
        return HostCSR(pin(X.indptr), pin(X.indices), pin(X.data), X.n_cols, pin(X.esc_pos), pin(X.esc_val))

    @property
    def is_u16(self) -> bool:
        return self.indices.dtype in (torch.uint16, torch.int16)


def upload_qc(H: HostCSR, mt_mask: torch.Tensor, device=None, chunk_rows: int = 1 << 17):
    """Copy a host count matrix to the device in row chunks and run QC on every chunk as soon as
    it has landed (the pinned, chunked H2D overlapped with QC).  Chunks go
    host -> device on a copy stream; u16-wire chunks are decoded into the 32-bit CSR on the
    compute stream, and QC of rows [r0, r1) runs there while the next chunks are in flight (the
    per-chunk data checks are deferred and read once at the end: no host round trip per chunk).
    Returns (X 32-bit DeviceCSR, qc dict equal to ``pp.calculate_qc_metrics(X, mt,
    row_splits=True)``) -- pass ``qc`` to ``pipeline.run`` to skip its QC pass."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    N = H.indptr.numel() - 1
    G = int(H.n_cols)
    ip_np = H.indptr.numpy()
    Z = int(ip_np[-1]) if N >= 0 else 0
    u16 = H.is_u16
    comp = torch.cuda.current_stream(dev)
    cs = torch.cuda.Stream(dev)
    indptr = torch.empty(N + 1, dtype=torch.int64, device=dev)
    ind = torch.empty(Z, dtype=torch.int32, device=dev)
    dat = torch.empty(Z, dtype=torch.float32, device=dev)
    T = int(_lib.call("scb_hvg_tiles", G))
    out = dict(n_genes_by_counts=torch.empty(N, dtype=torch.int32, device=dev),
               total_counts=torch.empty(N, dtype=torch.float64, device=dev),
               total_counts_mt=torch.empty(N, dtype=torch.float64, device=dev),
               pct_counts_mt=torch.empty(N, dtype=torch.float64, device=dev),
               n_cells_by_counts=torch.zeros(G, dtype=torch.int32, device=dev),
               gene_total_counts=torch.zeros(G, dtype=torch.float64, device=dev))
    splits = torch.empty((N, T - 1), dtype=torch.int32, device=dev) if T > 1 else None
    g_cells = torch.empty(G, dtype=torch.int32, device=dev)
    g_total = torch.empty(G, dtype=torch.float64, device=dev)
    mt = mt_mask.to(device=dev, dtype=torch.uint8).contiguous()
    chunks = [(r0, min(N, r0 + chunk_rows)) for r0 in range(0, N, chunk_rows)]
    flags = torch.zeros(max(1, len(chunks)), dtype=torch.int32, device=dev)
    ctx = _ctx(dat)
    if u16:
        esc_np = H.esc_pos.numpy() if H.esc_pos is not None else np.zeros(0, np.int64)
        esc_pos = H.esc_pos.to(dev) if H.esc_pos is not None else None
        esc_val = H.esc_val.to(dev) if H.esc_val is not None else None
        cap = max([int(ip_np[r1]) - (int(ip_np[r0]) & ~7) for r0, r1 in chunks] + [8])
        st_ind = [torch.empty(cap, dtype=H.indices.dtype, device=dev) for _ in range(2)]
        st_dat = [torch.empty(cap, dtype=H.data.dtype, device=dev) for _ in range(2)]
    cs.wait_stream(comp)
    with torch.cuda.stream(cs):
        indptr.copy_(H.indptr, non_blocking=True)
    copied = [torch.cuda.Event() for _ in chunks]
    freed = [torch.cuda.Event() for _ in chunks]
    _lib.call("scb_ctx_set_deferred_checks", ctx, 1)
    try:
        for ci, (r0, r1) in enumerate(chunks):
            a, b = int(ip_np[r0]), int(ip_np[r1])
            a8 = a & ~7  # u16 decode writes 16-byte aligned output: start at the aligned-down entry
            with torch.cuda.stream(cs):
                if u16:
                    if ci >= 2:
                        cs.wait_event(freed[ci - 2])  # recorded below, before this iteration
                    st_ind[ci % 2][: b - a8].copy_(H.indices[a8:b], non_blocking=True)
                    st_dat[ci % 2][: b - a8].copy_(H.data[a8:b], non_blocking=True)
                else:
                    ind[a:b].copy_(H.indices[a:b], non_blocking=True)
                    dat[a:b].copy_(H.data[a:b], non_blocking=True)
                copied[ci].record(cs)
            comp.wait_event(copied[ci])
            if u16:
                e0, e1 = (int(x) for x in np.searchsorted(esc_np, [a8, b]))
                ep = (esc_pos[e0:e1] - a8) if e1 > e0 else None
                ev = esc_val[e0:e1] if e1 > e0 else None
                # entries [a8, a) belong to the previous chunk: rewritten with the same values
                _lib.call("scb_csr_u16_decode", ctx, _p(st_ind[ci % 2]), _p(st_dat[ci % 2]), b - a8, _p(ep), _p(ev),
                          0 if ep is None else ep.numel(), _p(ind) + 4 * a8, _p(dat) + 4 * a8, _stream(dev))
                freed[ci].record(comp)
            # QC of rows [r0, r1): the row pointers are absolute offsets into the full arrays
            _lib.call("scb_qc_metrics", ctx, _p(indptr) + 8 * r0, _p(ind), _p(dat), r1 - r0, G, _p(mt),
                      _p(out["n_genes_by_counts"]) + 4 * r0, _p(out["total_counts"]) + 8 * r0,
                      _p(out["total_counts_mt"]) + 8 * r0, _p(out["pct_counts_mt"]) + 8 * r0, _p(g_cells),
                      _p(g_total), 0 if splits is None else _p(splits) + 4 * (T - 1) * r0, _stream(dev))
            _lib.call("scb_ctx_copy_data_flag", ctx, _p(flags) + 4 * ci, _stream(dev))  # keep this chunk's check
            out["n_cells_by_counts"] += g_cells
            out["gene_total_counts"] += g_total
    finally:
        _lib.call("scb_ctx_set_deferred_checks", ctx, 0)
    comp.wait_stream(cs)
    if int(flags.max().item()):
        raise _lib.ScbError("scb_qc_metrics", -4, "counts must be non-negative integers < 2^24 with column indices "
                                                  "in range")
    out["hvg_row_splits"] = splits
    return DeviceCSR(indptr, ind, dat, G), out
