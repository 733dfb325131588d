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
