"""Scanpy-shaped step functions backed by the sm_100a kernels of libscb_b200.so.

Each function is a thin host wrapper around one or more C-ABI calls (include/scb.h);
device memory, streams and collectives are PyTorch plumbing.  Semantics are fixed in
oracle/pipeline.py (the CPU restatement used as the parity checker) and DESIGN.md.

Reference anchor: the paper's Table 1 steps (reference PAPER.md:84-89) and the marker
labels the reference's tests use for them (pkg/tests/helpers.py:31-36): ``qc`` ->
calculate_qc_metrics / filter / subset, ``norm_hvg`` -> normalize_total + log1p +
highly_variable_genes, ``regress`` -> scale, ``pca`` -> pca, ``knn`` -> neighbors.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np
import torch

from . import _lib

ONES_PAD = 128  # dense scaled matrix row stride multiple (tcgen05 tile size)


def _p(t):
    return 0 if t is None else t.data_ptr()


def _stream(device=None):
    return torch.cuda.current_stream(device).cuda_stream


def _ctx(t: torch.Tensor):
    if not t.is_cuda:
        raise ValueError("step functions take CUDA tensors (no CPU fallback)")
    return _lib.context(t.device.index if t.device.index is not None else torch.cuda.current_device())


_U16 = (torch.uint16, torch.int16)


def _fmt(indices: torch.Tensor, data: torch.Tensor) -> str:
    """C-ABI suffix of a raw-matrix entry point for these array types: "" for the 32-bit CSR
    (int32 indices, float32 counts), "_u16" for the compact u16 CSR (uint16 indices and counts)."""
    if indices.dtype == torch.int32 and data.dtype == torch.float32:
        return ""
    if indices.dtype in _U16 and data.dtype in _U16:
        return "_u16"
    raise TypeError(f"unsupported CSR array types {indices.dtype}/{data.dtype}: use int32/float32 or the compact "
                    "uint16/uint16 format (DeviceCSR.to_u16)")


def _esc(X, values=None) -> tuple:
    """Escape-table arguments of the _u16 entry points (empty for the 32-bit format)."""
    values = X.data if values is None else values
    if values.dtype not in _U16:
        return ()
    if X.esc_pos is None or X.esc_pos.numel() == 0:
        return (0, 0, 0)
    return (_p(X.esc_pos), _p(X.esc_val), int(X.esc_pos.numel()))


@dataclasses.dataclass
class DeviceCSR:
    """CSR count matrix resident in HBM: indptr int64[N+1], indices int32[nnz], data float32[nnz]
    -- or the lossless compact form (``to_u16``): uint16 indices and uint16 counts, accepted by
    every step that reads the raw matrix (half the bytes per nonzero)."""

    indptr: torch.Tensor
    indices: torch.Tensor
    data: torch.Tensor
    n_cols: int
    # set by normalize_log1p: (raw counts data, per-row scale) of the same sparsity pattern
    counts: Optional[torch.Tensor] = None
    row_scale: Optional[torch.Tensor] = None
    # u16 form: sorted positions (int64) and true values (float32) of counts >= 65535 (stored as 65535)
    esc_pos: Optional[torch.Tensor] = None
    esc_val: Optional[torch.Tensor] = None

    @property
    def n_rows(self) -> int:
        return self.indptr.numel() - 1

    @property
    def nnz(self) -> int:
        return self.indices.numel()

    @property
    def device(self):
        return self.data.device

    @staticmethod
    def from_host(indptr, indices, data, n_cols, device="cuda"):
        def t(a, dt):
            return torch.as_tensor(a).to(dtype=dt).to(device, non_blocking=False)
        return DeviceCSR(t(indptr, torch.int64), t(indices, torch.int32), t(data, torch.float32), int(n_cols))

    def to_host(self):
        return (self.indptr.cpu().numpy(), self.indices.cpu().numpy(), self.data.cpu().numpy(), self.n_cols)

    @property
    def is_u16(self) -> bool:
        return self.indices.dtype in _U16

    def to_u16(self) -> "DeviceCSR":
        """The compact u16 form: uint16 gene indices (n_cols <= 65536) and uint16 counts, the rare
        counts >= 65535 stored as the escape 65535 plus (position, value) in esc_pos/esc_val.
        Needs non-negative integer counts < 2^24 (raises ValueError otherwise: lossless or refused)."""
        if self.is_u16:
            return self
        if self.n_cols > 65536:
            raise ValueError(f"u16 CSR needs n_cols <= 65536 (got {self.n_cols})")
        d = self.data
        if d.numel():
            bad = torch.stack([(d < 0).any(), (d >= 16777216).any(), (d != torch.round(d)).any()]).cpu()
            if bool(bad.any()):
                raise ValueError("u16 CSR needs non-negative integer counts < 2^24")
        big = d >= 65535
        pos = torch.nonzero(big).view(-1).to(torch.int64)
        val = d[pos].contiguous()
        d16 = torch.clamp(d, max=65535.0).to(torch.int32).to(torch.uint16)
        return DeviceCSR(self.indptr, self.indices.to(torch.uint16), d16, self.n_cols, esc_pos=pos, esc_val=val)

    def to_f32(self, out: Optional["DeviceCSR"] = None) -> "DeviceCSR":
        """The 32-bit form (int32 indices, float32 counts), decoded by ``scb_csr_u16_decode``
        (one HBM pass, 12 B per nonzero); ``out`` = preallocated 32-bit arrays to decode into."""
        if not self.is_u16:
            return self
        nnz = self.indices.numel()
        ind = out.indices if out is not None else torch.empty(nnz, dtype=torch.int32, device=self.device)
        dat = out.data if out is not None else torch.empty(nnz, dtype=torch.float32, device=self.device)
        esc = _esc(self)
        _lib.call("scb_csr_u16_decode", _ctx(self.data), _p(self.indices), _p(self.data), nnz, *esc, _p(ind), _p(dat),
                  _stream(self.device))
        return DeviceCSR(self.indptr, ind, dat, self.n_cols)


@dataclasses.dataclass
class DeltaCSR:
    """Byte-delta CSR, the densest lossless host->device wire form: per nonzero one byte ``dgene``
    = g - g_prev - 1 (g_prev = -1 at a row start) and one byte ``dcount`` = the count, each 255
    meaning "escaped" with the true delta / count in a sorted (position, value) table.  2 B per
    nonzero (u16: 4 B, int32 + float32: 8 B); ``to_f32`` decodes it in HBM (scb_csr_delta8_decode)."""

    indptr: torch.Tensor
    dgene: torch.Tensor
    dcount: torch.Tensor
    gesc_pos: torch.Tensor
    gesc_val: torch.Tensor
    cesc_pos: torch.Tensor
    cesc_val: torch.Tensor
    n_cols: int

    @property
    def n_rows(self) -> int:
        return self.indptr.numel() - 1

    @property
    def nnz(self) -> int:
        return self.dgene.numel()

    def tensors(self):
        return [self.indptr, self.dgene, self.dcount, self.gesc_pos, self.gesc_val, self.cesc_pos, self.cesc_val]

    @staticmethod
    def from_tensors(ts, n_cols: int) -> "DeltaCSR":
        return DeltaCSR(*ts, n_cols=n_cols)

    @staticmethod
    def from_csr(X: "DeviceCSR", chunk: int = 1 << 28) -> "DeltaCSR":
        """Encode a 32-bit (or u16) CSR (any device; torch ops).  Needs sorted, unique gene indices
        within each row and non-negative integer counts < 2^24 (ValueError otherwise)."""
        if X.is_u16:
            X = X.to_f32()
        dev, Z = X.indices.device, X.nnz
        ip = X.indptr
        row_start = torch.zeros(Z + 1, dtype=torch.bool, device=dev)
        row_start[ip[:-1]] = True  # (empty rows point at the next row's start: also a start)
        dg = torch.empty(Z, dtype=torch.uint8, device=dev)
        dc = torch.empty(Z, dtype=torch.uint8, device=dev)
        gpos, gval, cpos, cval = [], [], [], []
        for a in range(0, Z, chunk):
            b = min(Z, a + chunk)
            g = X.indices[a:b].to(torch.int32)
            prev = torch.empty_like(g)
            prev[1:] = g[:-1]
            prev[0] = X.indices[a - 1] if a > 0 else -1
            prev = torch.where(row_start[a:b], torch.full_like(g, -1), prev)
            delta = g - prev - 1
            if bool((delta < 0).any()):
                raise ValueError("delta CSR needs sorted, unique gene indices within each row")
            esc = delta > 254
            dg[a:b] = torch.where(esc, torch.full_like(delta, 255), delta).to(torch.uint8)
            idx = torch.nonzero(esc).view(-1)
            gpos.append(idx.to(torch.int64) + a)
            gval.append(delta[idx].to(torch.int32))
            d = X.data[a:b]
            bad = torch.stack([(d < 0).any(), (d >= 16777216).any(), (d != torch.round(d)).any()])
            if bool(bad.any()):
                raise ValueError("delta CSR needs non-negative integer counts < 2^24")
            cesc = d >= 255
            dc[a:b] = torch.clamp(d, max=255.0).to(torch.int32).to(torch.uint8)
            idx = torch.nonzero(cesc).view(-1)
            cpos.append(idx.to(torch.int64) + a)
            cval.append(d[idx].to(torch.float32))
        cat = lambda xs, dt: torch.cat(xs) if xs else torch.empty(0, dtype=dt, device=dev)  # noqa: E731
        return DeltaCSR(ip, dg, dc, cat(gpos, torch.int64), cat(gval, torch.int32), cat(cpos, torch.int64),
                        cat(cval, torch.float32), X.n_cols)

    def to_f32(self, out: Optional["DeviceCSR"] = None) -> "DeviceCSR":
        """The 32-bit CSR in HBM (one pass: 2 B read + 8 B written per nonzero); ``out`` =
        preallocated 32-bit arrays to decode into."""
        nnz = self.nnz
        dev = self.dgene.device
        ind = out.indices if out is not None else torch.empty(nnz, dtype=torch.int32, device=dev)
        dat = out.data if out is not None else torch.empty(nnz, dtype=torch.float32, device=dev)
        _lib.call("scb_csr_delta8_decode", _ctx(self.dgene), _p(self.indptr), self.n_rows, _p(self.dgene),
                  _p(self.dcount), nnz, _p(self.gesc_pos), _p(self.gesc_val), int(self.gesc_pos.numel()),
                  _p(self.cesc_pos), _p(self.cesc_val), int(self.cesc_pos.numel()), _p(ind), _p(dat), _stream(dev))
        return DeviceCSR(self.indptr, ind, dat, self.n_cols)


# ----------------------------------------------------------------------------- qc
def calculate_qc_metrics(X: DeviceCSR, mt_mask: torch.Tensor, row_splits: bool = False, defer_check: bool = False):
    """sc.pp.calculate_qc_metrics(qc_vars=['mt'], percent_top=None, log1p=False).

    With ``row_splits`` the result also holds ``hvg_row_splits`` (per-row gene-tile split
    counts that let the HVG column pass read every nonzero exactly once).  With ``defer_check``
    the data-validity check (non-negative integer counts < 2^24, column indices in range) does
    not wait for the device: ``filter_masks_ex`` raises it instead (one host round trip fewer)."""
    dev = X.device
    N, G = X.n_rows, X.n_cols
    out = dict(
        n_genes_by_counts=torch.empty(N, dtype=torch.int32, device=dev),
        total_counts=torch.empty(N, dtype=torch.float64, device=dev),
        total_counts_mt=torch.empty(N, dtype=torch.float64, device=dev),
        pct_counts_mt=torch.empty(N, dtype=torch.float64, device=dev),
        n_cells_by_counts=torch.empty(G, dtype=torch.int32, device=dev),
        gene_total_counts=torch.empty(G, dtype=torch.float64, device=dev),
    )
    mt = mt_mask.to(device=dev, dtype=torch.uint8).contiguous()
    splits = None
    if row_splits:
        T = int(_lib.call("scb_hvg_tiles", G))
        if T > 1:
            splits = torch.empty((N, T - 1), dtype=torch.int32, device=dev)
    ctx = _ctx(X.data)
    _lib.call("scb_ctx_set_deferred_checks", ctx, 1 if defer_check else 0)
    _lib.call("scb_qc_metrics" + _fmt(X.indices, X.data), ctx, _p(X.indptr), _p(X.indices), _p(X.data), N, G,
              _p(mt),
              _p(out["n_genes_by_counts"]), _p(out["total_counts"]), _p(out["total_counts_mt"]),
              _p(out["pct_counts_mt"]), _p(out["n_cells_by_counts"]), _p(out["gene_total_counts"]),
              _p(splits), *_esc(X), _stream(dev))
    _lib.call("scb_ctx_set_deferred_checks", ctx, 0)
    out["hvg_row_splits"] = splits
    return out


def qc_metrics(X: DeviceCSR, mt_mask: torch.Tensor):
    """SURVEY §8(b2) form of calculate_qc_metrics: returns (cell, gene) -- Scanpy's obs / var
    metric tables as dicts of device tensors."""
    q = calculate_qc_metrics(X, mt_mask)
    cell = {k: q[k] for k in ("n_genes_by_counts", "total_counts", "total_counts_mt", "pct_counts_mt")}
    gene = {"n_cells_by_counts": q["n_cells_by_counts"], "total_counts": q["gene_total_counts"]}
    return cell, gene


def filter_masks_ex(cell, gene=None, *, min_genes=200, max_genes=None, max_pct_mt=20.0, min_cells=3, indptr=None):
    """filter_masks plus, in the same host round trip, the nonzeros of the kept rows (when the
    raw ``indptr`` is given; else 0).  Raises ScbError if a deferred QC data check failed.
    Returns (cell_mask, gene_mask, (n_kept_cells, n_kept_genes), kept_row_nnz)."""
    if gene is not None:
        qc = {"n_genes_by_counts": cell["n_genes_by_counts"], "pct_counts_mt": cell["pct_counts_mt"],
              "n_cells_by_counts": gene["n_cells_by_counts"]}
    else:
        qc = cell
    ng = qc["n_genes_by_counts"]
    dev = ng.device
    N, G = ng.numel(), qc["n_cells_by_counts"].numel()
    cm = torch.empty(N, dtype=torch.uint8, device=dev)
    gm = torch.empty(G, dtype=torch.uint8, device=dev)
    kept = torch.empty(4, dtype=torch.int64, device=dev)
    _lib.call("scb_filter_masks", _ctx(ng), _p(ng), _p(qc["pct_counts_mt"]), N, _p(qc["n_cells_by_counts"]), G,
              int(min_genes), -1 if max_genes is None else int(max_genes), float(max_pct_mt), int(min_cells),
              _p(indptr), _p(cm), _p(gm), _p(kept), _stream(dev))
    k = kept.cpu().tolist()
    if k[3]:
        raise _lib.ScbError("scb_qc_metrics", -4, "counts must be non-negative integers < 2^24 with column indices "
                                                  "in range (deferred check)")
    return cm, gm, (int(k[0]), int(k[1])), int(k[2])


def filter_masks(cell, gene=None, *, min_genes=200, max_genes=None, max_pct_mt=20.0, min_cells=3):
    """sc.pp.filter_cells(min_genes, max_genes) & pct_counts_mt < max_pct_mt; sc.pp.filter_genes(min_cells).
    ``filter_masks(cell, gene, ...)`` takes the two tables of ``qc_metrics``; with ``gene`` omitted,
    ``cell`` is the combined dict of ``calculate_qc_metrics``.
    Returns (cell_mask u8[N], gene_mask u8[G], (n_kept_cells, n_kept_genes))."""
    cm, gm, kept, _ = filter_masks_ex(cell, gene, min_genes=min_genes, max_genes=max_genes, max_pct_mt=max_pct_mt,
                                      min_cells=min_cells)
    return cm, gm, kept


def subset(X: DeviceCSR, cell_mask, gene_mask, n_kept=None, target_sum=None):
    """adata[cell_mask, gene_mask] (rows/columns kept in order, columns renumbered).

    With ``target_sum`` set, the values are normalize_total + log1p'd in the same pass
    (fused pipeline form) and the returned matrix carries ``counts``=None and
    ``row_scale`` (per kept row)."""
    dev = X.device
    if n_kept is None:
        n_kept = (int(cell_mask.sum().item()), int(gene_mask.sum().item()))
    nk, gk = n_kept
    remap = torch.empty(X.n_cols, dtype=torch.int32, device=dev)
    new_indptr = torch.empty(nk + 1, dtype=torch.int64, device=dev)
    row_scale = torch.empty(nk, dtype=torch.float32, device=dev) if target_sum is not None else None
    ctx, s = _ctx(X.data), _stream(dev)
    fmt = _fmt(X.indices, X.data)
    _lib.call("scb_subset_count" + fmt, ctx, _p(X.indptr), _p(X.indices), _p(X.data), X.n_rows, X.n_cols,
              _p(cell_mask), _p(gene_mask), _p(remap), _p(new_indptr), float(target_sum or 0.0),
              _p(row_scale), 0, *_esc(X), s)
    nnz = int(new_indptr[nk].item())
    ind = torch.empty(nnz, dtype=torch.int32, device=dev)
    dat = torch.empty(nnz, dtype=torch.float32, device=dev)
    _lib.call("scb_subset_fill" + fmt, ctx, _p(X.indptr), _p(X.indices), _p(X.data), X.n_rows, X.n_cols,
              _p(cell_mask), _p(remap), _p(new_indptr), _p(row_scale), _p(ind), _p(dat), *_esc(X), s)
    out = DeviceCSR(new_indptr, ind, dat, gk)
    out.row_scale = row_scale
    return out


def subset_count_scale(X: DeviceCSR, cell_mask, gene_mask, n_kept, target_sum: float = 1e4):
    """First pass of the fused subset + normalize: gene remap, kept-row offsets, per-kept-row and
    per-ORIGINAL-row normalization factors (0 for dropped rows).  One host sync (kept nnz)."""
    dev = X.device
    nk, gk = n_kept
    remap = torch.empty(X.n_cols, dtype=torch.int32, device=dev)
    new_indptr = torch.empty(nk + 1, dtype=torch.int64, device=dev)
    row_scale = torch.empty(nk, dtype=torch.float32, device=dev)
    row_scale_orig = torch.empty(X.n_rows, dtype=torch.float32, device=dev)
    ctx, s = _ctx(X.data), _stream(dev)
    _lib.call("scb_subset_count" + _fmt(X.indices, X.data), ctx, _p(X.indptr), _p(X.indices), _p(X.data), X.n_rows,
              X.n_cols, _p(cell_mask), _p(gene_mask), _p(remap), _p(new_indptr), float(target_sum), _p(row_scale),
              _p(row_scale_orig), *_esc(X), s)
    nnz = int(new_indptr[nk].item())
    return remap, new_indptr, row_scale, row_scale_orig, nnz


def subset_rows_all_genes(X: DeviceCSR, cell_mask, total_counts, n_kept: int, target_sum: float = 1e4):
    """subset_count_scale when every gene is kept: the same (remap, new_indptr, row_scale,
    row_scale_orig) from the row lengths and QC's exact totals, without reading the nonzeros."""
    dev = X.device
    remap = torch.empty(X.n_cols, dtype=torch.int32, device=dev)
    new_indptr = torch.empty(n_kept + 1, dtype=torch.int64, device=dev)
    row_scale = torch.empty(n_kept, dtype=torch.float32, device=dev)
    row_scale_orig = torch.empty(X.n_rows, dtype=torch.float32, device=dev)
    _lib.call("scb_subset_rows_all_genes", _ctx(X.indptr), _p(X.indptr), X.n_rows, X.n_cols, _p(cell_mask),
              _p(total_counts), float(target_sum), _p(remap), _p(new_indptr), _p(row_scale), _p(row_scale_orig),
              _stream(dev))
    return remap, new_indptr, row_scale, row_scale_orig


def subset_fill_log(X: DeviceCSR, cell_mask, remap, new_indptr, row_scale, nnz: int, n_genes_kept: int) -> DeviceCSR:
    """Second pass: compacted kept matrix with log1p(x * row_scale) values."""
    dev = X.device
    ind = torch.empty(nnz, dtype=torch.int32, device=dev)
    logv = torch.empty(nnz, dtype=torch.float32, device=dev)
    _lib.call("scb_subset_fill" + _fmt(X.indices, X.data), _ctx(X.data), _p(X.indptr), _p(X.indices), _p(X.data),
              X.n_rows, X.n_cols, _p(cell_mask), _p(remap), _p(new_indptr), _p(row_scale), _p(ind), _p(logv),
              *_esc(X), _stream(dev))
    return DeviceCSR(new_indptr, ind, logv, n_genes_kept, row_scale=row_scale)


def subset_normalize(X: DeviceCSR, cell_mask, gene_mask, n_kept, target_sum: float = 1e4):
    """Fused subset + normalize_total + log1p (two streaming passes over X).  Returns the
    log-normalized kept matrix, the gene remap (new column or -1) and the per-ORIGINAL-row
    normalization factor (0 for dropped rows) used by hvg_gene_sums on X itself."""
    remap, new_indptr, row_scale, row_scale_orig, nnz = subset_count_scale(X, cell_mask, gene_mask, n_kept, target_sum)
    X_log = subset_fill_log(X, cell_mask, remap, new_indptr, row_scale, nnz, n_kept[1])
    return X_log, remap, row_scale_orig


def subset_fill_log_scale_sums(X: DeviceCSR, cell_mask, remap, new_indptr, row_scale, nnz: int, n_genes_kept: int,
                               slot: torch.Tensor, H: int, sums=None, all_kept: bool = False):
    """subset_fill_log fused with the scale step's gene sums of the HVG columns (``slot``: int32
    per kept gene, -1 = not an HVG).  Returns (X_log, sums u64[2][2][H]) or (X_log, None) when
    the fused kernel does not apply (more than 32767 input genes) -- then use scale_gene_sums.
    ``all_kept``: every row and gene of X is kept (the caller's QC counts say so): X_log shares
    X's int32 indices instead of copying them (the kernel traps if that is not true)."""
    if X.n_cols > 32767:
        return subset_fill_log(X, cell_mask, remap, new_indptr, row_scale, nnz, n_genes_kept), None
    dev = X.device
    share = all_kept and X.indices.dtype == torch.int32 and nnz == X.nnz
    ind = X.indices if share else torch.empty(nnz, dtype=torch.int32, device=dev)
    logv = torch.empty(nnz, dtype=torch.float32, device=dev)
    if sums is None:
        sums = torch.zeros((2, 2, H), dtype=torch.int64, device=dev)
    _lib.call("scb_subset_fill_scale_sums" + _fmt(X.indices, X.data), _ctx(X.data), _p(X.indptr), _p(X.indices),
              _p(X.data), X.n_rows, X.n_cols, _p(cell_mask), _p(remap), _p(new_indptr), _p(row_scale), _p(slot), H,
              _p(None if share else ind), _p(logv), _p(sums), *_esc(X), _stream(dev))
    return DeviceCSR(new_indptr, ind, logv, n_genes_kept, row_scale=row_scale), sums


# ----------------------------------------------------------------------------- norm_hvg
def normalize_log1p(X: DeviceCSR, target_sum: float = 1e4) -> DeviceCSR:
    """sc.pp.normalize_total(target_sum) followed by sc.pp.log1p (out of place).  The result
    keeps a reference to the raw counts and the per-row factor for highly_variable_genes."""
    X = X.to_f32()  # the standalone (unfused) step writes float values in the input's layout
    dev = X.device
    out = torch.empty_like(X.data)
    scale = torch.empty(X.n_rows, dtype=torch.float32, device=dev)
    _lib.call("scb_normalize_log1p", _ctx(X.data), _p(X.indptr), _p(X.data), X.n_rows, float(target_sum),
              _p(out), _p(scale), _stream(dev))
    return DeviceCSR(X.indptr, X.indices, out, X.n_cols, counts=X.data, row_scale=scale)


def hvg_gene_sums(X: DeviceCSR, counts=None, row_scale=None, gene_remap=None, n_out=None, sums=None,
                  row_splits=None):
    """Fixed-point per-gene sums of the normalized counts (u64[2][2][G]); additive across shards."""
    counts = X.counts if counts is None else counts
    row_scale = X.row_scale if row_scale is None else row_scale
    if counts is None or row_scale is None:
        raise ValueError("highly_variable_genes needs the output of normalize_log1p (raw counts + row scale)")
    n_out = X.n_cols if n_out is None else n_out
    if sums is None:
        sums = torch.zeros((2, 2, n_out), dtype=torch.int64, device=X.device)
    _lib.call("scb_hvg_gene_sums" + _fmt(X.indices, counts), _ctx(X.data), _p(X.indptr), _p(X.indices), _p(counts),
              _p(row_scale), X.n_rows, X.n_cols, _p(gene_remap), n_out, _p(row_splits), _p(sums), *_esc(X, counts),
              _stream(X.device))
    return sums


HVG_TIES = {"rank": 0, "cutoff": 1}


def hvg_select(sums, n_cells: int, n_top_genes: int, n_bins: int = 20, ties: str = "cutoff"):
    """Seurat selection from the (all-reduced) gene sums.  ``ties="cutoff"`` is Scanpy's rule
    (every gene with dispersions_norm >= the n-th largest); ``"rank"`` returns exactly n."""
    if ties not in HVG_TIES:
        raise ValueError(f"ties must be one of {sorted(HVG_TIES)}")
    dev = sums.device
    G = sums.shape[-1]
    st = dict(means=torch.empty(G, dtype=torch.float64, device=dev),
              variances=torch.empty(G, dtype=torch.float64, device=dev),
              dispersions=torch.empty(G, dtype=torch.float64, device=dev),
              dispersions_norm=torch.empty(G, dtype=torch.float64, device=dev),
              mean_bin=torch.empty(G, dtype=torch.int32, device=dev))
    mask = torch.empty(G, dtype=torch.uint8, device=dev)
    index = torch.empty(max(1, G), dtype=torch.int32, device=dev)
    nsel = torch.empty(1, dtype=torch.int32, device=dev)
    _lib.call("scb_hvg_select", _ctx(sums), _p(sums), G, int(n_cells), int(n_top_genes), int(n_bins), HVG_TIES[ties],
              _p(st["means"]), _p(st["variances"]), _p(st["dispersions"]), _p(st["dispersions_norm"]),
              _p(st["mean_bin"]), _p(mask), _p(index), _p(nsel), _stream(dev))
    n = int(nsel.item())
    st["n_selected"] = n
    return mask, index[:n], st


def highly_variable_genes(X_log: DeviceCSR, n_top_genes: int = 2000, n_bins: int = 20, flavor: str = "seurat",
                          ties: str = "cutoff"):
    """sc.pp.highly_variable_genes(flavor='seurat', n_top_genes, n_bins) on normalize_log1p output.
    Only the seurat flavour is implemented (cell_ranger / seurat_v3 need a loess fit or the raw
    counts' median dispersion; they are not on the north-star path).
    Returns (hvg_mask u8[G], hvg_index i32[H] sorted, stats dict)."""
    if flavor != "seurat":
        raise NotImplementedError(f"highly_variable_genes: flavor={flavor!r} (only 'seurat' is implemented)")
    sums = hvg_gene_sums(X_log)
    return hvg_select(sums, X_log.n_rows, n_top_genes, n_bins, ties)


# ----------------------------------------------------------------------------- regress (scale)
@dataclasses.dataclass
class Scaled:
    """Dense scaled HVG matrix Z[N][ld] (row-major): columns [0, H) are the HVGs, column
    ``ones_col`` = 1 (gives the column sums in the Gram), the rest zero.  Held as float32 ``Z``
    and/or as the BF16 operand planes ``Z_hi`` = bf16(Z), ``Z_lo`` = bf16(Z - hi) (the pipeline
    writes only the planes: Z = hi + lo to 2^-17 relative)."""
    Z: Optional[torch.Tensor]
    H: int
    ones_col: int
    mean: torch.Tensor
    inv_std: torch.Tensor
    Z_hi: Optional[torch.Tensor] = None
    Z_lo: Optional[torch.Tensor] = None

    @property
    def ld(self):
        return (self.Z if self.Z is not None else self.Z_hi).shape[1]

    @property
    def n_rows(self):
        return (self.Z if self.Z is not None else self.Z_hi).shape[0]

    @property
    def device(self):
        return (self.Z if self.Z is not None else self.Z_hi).device

    def dense(self) -> torch.Tensor:
        """float32 [N][ld]: Z, or hi + lo reconstructed from the planes."""
        if self.Z is not None:
            return self.Z
        return self.Z_hi.float() + self.Z_lo.float()

    def values(self):
        return self.dense()[:, : self.H]


def padded_width(H: int) -> int:
    return ((H + 1 + ONES_PAD - 1) // ONES_PAD) * ONES_PAD


def gene_slots(hvg_index: torch.Tensor, n_cols: int):
    slot = torch.full((n_cols,), -1, dtype=torch.int32, device=hvg_index.device)
    slot[hvg_index.long()] = torch.arange(hvg_index.numel(), dtype=torch.int32, device=hvg_index.device)
    return slot


def scale_gene_sums(X_log: DeviceCSR, slot, H, sums=None):
    if sums is None:
        sums = torch.zeros((2, 2, H), dtype=torch.int64, device=X_log.device)
    _lib.call("scb_scale_gene_sums", _ctx(X_log.data), _p(X_log.indptr), _p(X_log.indices), _p(X_log.data),
              X_log.n_rows, X_log.n_cols, _p(slot), H, _p(sums), _stream(X_log.device))
    return sums


def scale_finalize(sums, n_cells: int):
    H = sums.shape[-1]
    dev = sums.device
    mean = torch.empty(H, dtype=torch.float64, device=dev)
    inv = torch.empty(H, dtype=torch.float64, device=dev)
    _lib.call("scb_scale_finalize", _ctx(sums), _p(sums), H, int(n_cells), _p(mean), _p(inv), _stream(dev))
    return mean, inv


CLIPS = ("symmetric", "upper")


def clip_min(max_value: float, clip: str) -> float:
    """Lower clip bound: -max_value for Scanpy >= 1.10 / rapids-singlecell (zero_center=True),
    -inf for Scanpy <= 1.9 (upper clip only)."""
    if clip not in CLIPS:
        raise ValueError(f"clip must be one of {CLIPS}")
    return -float(max_value) if clip == "symmetric" else float("-inf")


def scale_dense(X_log: DeviceCSR, slot, H, mean, inv, max_value=10.0, out=None, clip: str = "symmetric",
                planes: bool = False) -> Scaled:
    """Dense clipped z-scores Z[N][ld] (float32) of the HVG columns, plus the ones column.  With
    ``planes`` the z-scores are written directly as the BF16 planes the Gram and the projection
    read (no float32 matrix, no split pass; bit-identical to splitting the float32 one)."""
    ld = padded_width(H)
    dev = X_log.device
    if planes:
        hi = torch.empty((X_log.n_rows, ld), dtype=_lib.plane_dtype(), device=dev)
        lo = torch.empty((X_log.n_rows, ld), dtype=_lib.plane_dtype(), device=dev)
        _lib.call("scb_scale_dense_planes", _ctx(X_log.data), _p(X_log.indptr), _p(X_log.indices), _p(X_log.data),
                  X_log.n_rows, X_log.n_cols, _p(slot), H, _p(mean), _p(inv), float(max_value),
                  clip_min(max_value, clip), _p(hi), _p(lo), ld, H, _stream(dev))
        return Scaled(None, H, H, mean, inv, hi, lo)
    Z = out if out is not None else torch.empty((X_log.n_rows, ld), dtype=torch.float32, device=dev)
    _lib.call("scb_scale_dense", _ctx(X_log.data), _p(X_log.indptr), _p(X_log.indices), _p(X_log.data),
              X_log.n_rows, X_log.n_cols, _p(slot), H, _p(mean), _p(inv), float(max_value),
              clip_min(max_value, clip), _p(Z), ld, H, _stream(dev))
    return Scaled(Z, H, H, mean, inv)


def _hvg_index(X_log: DeviceCSR, hvg: torch.Tensor) -> torch.Tensor:
    """Accept the HVG mask (bool/uint8 [n_cols]) or the sorted index list."""
    if hvg.dtype in (torch.bool, torch.uint8) and hvg.numel() == X_log.n_cols:
        return torch.nonzero(hvg.to(torch.bool)).view(-1).to(torch.int32)
    return hvg.to(torch.int32)


def scale(X_log: DeviceCSR, hvg_mask: torch.Tensor, max_value: float = 10.0, clip: str = "symmetric") -> Scaled:
    """sc.pp.scale(adata[:, hvg], max_value, zero_center=True) -> dense float32 (zero-centred, unit
    variance, clipped to [-max_value, max_value]; ``clip="upper"``: Scanpy <= 1.9's upper clip).
    ``hvg_mask``: uint8/bool mask over the columns (or the sorted HVG index list)."""
    hvg_index = _hvg_index(X_log, hvg_mask)
    H = int(hvg_index.numel())
    slot = gene_slots(hvg_index, X_log.n_cols)
    sums = scale_gene_sums(X_log, slot, H)
    mean, inv = scale_finalize(sums, X_log.n_rows)
    return scale_dense(X_log, slot, H, mean, inv, max_value, clip=clip)


# ----------------------------------------------------------------------------- regress_out
def regress_cov_sums(qc: dict, cell_mask: torch.Tensor) -> torch.Tensor:
    """float64[6] = (n, Σtc, Σtc², Σpct, Σpct², Σtc·pct) over the kept cells (all-reduce across ranks)."""
    tc, pc = qc["total_counts"], qc["pct_counts_mt"]
    out = torch.empty(6, dtype=torch.float64, device=tc.device)
    _lib.call("scb_regress_cov_sums", _ctx(tc), _p(tc), _p(pc), _p(cell_mask), tc.numel(), _p(out), _stream(tc.device))
    return out


def regress_design(qc: dict, cell_mask: torch.Tensor, sums6: torch.Tensor, n_kept: int) -> torch.Tensor:
    """Standardised covariates float64 [2][n_kept] (kept-row order)."""
    tc, pc = qc["total_counts"], qc["pct_counts_mt"]
    a = torch.empty((2, n_kept), dtype=torch.float64, device=tc.device)
    _lib.call("scb_regress_design", _ctx(tc), _p(tc), _p(pc), _p(cell_mask), tc.numel(), _p(sums6), int(n_kept),
              _p(a), _stream(tc.device))
    return a


def regress_dense_log(X_log: DeviceCSR, slot, H: int) -> Scaled:
    """Dense log values of the HVG columns (scale_dense with mean 0, inv_std 1, no clip)."""
    dev = X_log.device
    zeros = torch.zeros(H, dtype=torch.float64, device=dev)
    ones = torch.ones(H, dtype=torch.float64, device=dev)
    return scale_dense(X_log, slot, H, zeros, ones, float("inf"), clip="upper")


def regress_xty(L: Scaled, design: torch.Tensor, xty=None) -> torch.Tensor:
    """xty float64 [4][H] += (Σl, Σa1·l, Σa2·l, Σl²) per gene (all-reduce across ranks)."""
    if xty is None:
        xty = torch.zeros((4, L.H), dtype=torch.float64, device=L.Z.device)
    _lib.call("scb_regress_xty", _ctx(L.Z), _p(L.Z), L.Z.shape[0], L.ld, L.H, _p(design), _p(xty), _stream(L.Z.device))
    return xty


def regress_finalize(xty: torch.Tensor, sums6: torch.Tensor):
    H = xty.shape[1]
    beta = torch.empty((3, H), dtype=torch.float64, device=xty.device)
    inv = torch.empty(H, dtype=torch.float64, device=xty.device)
    _lib.call("scb_regress_finalize", _ctx(xty), _p(xty), _p(sums6), H, _p(beta), _p(inv), _stream(xty.device))
    return beta, inv


def regress_apply(L: Scaled, design, beta, inv, max_value: float = 10.0, clip: str = "symmetric") -> Scaled:
    """In place: Z[:, :H] = clip((l - fit) * inv_std, -max_value | -inf, max_value); returns the Scaled
    view (mean 0 -- the residual mean is zero by construction)."""
    _lib.call("scb_regress_apply", _ctx(L.Z), _p(L.Z), L.Z.shape[0], L.ld, L.H, _p(design), _p(beta), _p(inv),
              float(max_value), clip_min(max_value, clip), _stream(L.Z.device))
    L.mean = torch.zeros(L.H, dtype=torch.float64, device=L.Z.device)
    L.inv_std = inv
    return L


def regress_out_scale(X_log: DeviceCSR, hvg_index: torch.Tensor, qc: dict, cell_mask: torch.Tensor,
                      max_value: float = 10.0, clip: str = "symmetric") -> Scaled:
    """sc.pp.regress_out(adata[:, hvg], ["total_counts", "pct_counts_mt"]) + sc.pp.scale(max_value)
    (paper Table 1 step 4).  ``qc``/``cell_mask`` are the QC metrics and cell mask of the ORIGINAL
    rows; X_log holds the kept rows in order."""
    hvg_index = _hvg_index(X_log, hvg_index)
    H = int(hvg_index.numel())
    slot = gene_slots(hvg_index, X_log.n_cols)
    s6 = regress_cov_sums(qc, cell_mask)
    design = regress_design(qc, cell_mask, s6, X_log.n_rows)
    L = regress_dense_log(X_log, slot, H)
    beta, inv = regress_finalize(regress_xty(L, design), s6)
    return regress_apply(L, design, beta, inv, max_value, clip)


# ----------------------------------------------------------------------------- pca
@dataclasses.dataclass
class PCAResult:
    X_pca: torch.Tensor           # float32 [N][ld] (first n_comps columns valid, rest 0)
    components: torch.Tensor      # float32 [n_comps][H] (row j = component j, sign-canonical)
    variance: torch.Tensor        # float64 [n_comps]
    variance_ratio: torch.Tensor  # float64 [n_comps]
    col_mean: torch.Tensor        # float32 [ld_z] column means of Z (centring)
    n_comps: int


def split_planes(sc: Scaled) -> Scaled:
    """BF16 operand planes of Z for the Gram: hi = bf16(Z), lo = bf16(Z - hi) (one streaming pass)."""
    if sc.Z is None:  # already planes only
        return sc
    n, ld = sc.Z.shape
    if sc.Z_hi is None:
        sc.Z_hi = torch.empty((n, ld), dtype=_lib.plane_dtype(), device=sc.Z.device)
        sc.Z_lo = torch.empty((n, ld), dtype=_lib.plane_dtype(), device=sc.Z.device)
    _lib.call("scb_split_bf16", _ctx(sc.Z), _p(sc.Z), n, ld, _p(sc.Z_hi), _p(sc.Z_lo), _stream(sc.Z.device))
    return sc


def gram(sc: Scaled, out=None, planes: bool = True, keep_planes: bool = False):
    """Partial (local) Gram matrix Z^T Z, float64 [ld][ld] (tcgen05, 3xBF16).  ``planes`` (default)
    splits Z into BF16 hi/lo planes first and feeds them to the tensor cores by TMA; ``planes=False``
    converts fp32 tiles inside the Gram kernel instead (no extra 4 B/element of HBM, slower).  The
    planes (4 B per element) are released after the call unless ``keep_planes``."""
    ld = sc.ld
    dev = sc.device
    C = out if out is not None else torch.empty((ld, ld), dtype=torch.float64, device=dev)
    if planes or sc.Z is None:
        split_planes(sc)
        _lib.call("scb_gram_split", _ctx(sc.Z_hi), _p(sc.Z_hi), _p(sc.Z_lo), sc.n_rows, ld, _p(C), _stream(dev))
        if not keep_planes and sc.Z is not None:  # stream-ordered release (planes-only matrices keep them)
            sc.Z_hi = sc.Z_lo = None
    else:
        _lib.call("scb_gram", _ctx(sc.Z), _p(sc.Z), sc.Z.shape[0], ld, _p(C), _stream(sc.Z.device))
    return C


def pca_from_gram(sc: Scaled, C, n_cells: int, n_comps: int = 50):
    dev = sc.device
    ld = sc.ld
    npad = 64 if n_comps <= 64 else 128
    lam = torch.empty(n_comps, dtype=torch.float64, device=dev)
    comp_t = torch.empty((npad, ld), dtype=torch.float32, device=dev)
    mean = torch.empty(ld, dtype=torch.float32, device=dev)
    tr = torch.empty(1, dtype=torch.float64, device=dev)
    _lib.call("scb_pca_eig", _ctx(C), _p(C), sc.H, ld, sc.ones_col, int(n_cells), n_comps, npad, _p(lam), _p(comp_t),
              _p(mean), _p(tr), _stream(dev))
    return lam, comp_t, mean, tr


def project(sc: Scaled, comp_t, mean, n_comps: int, ld_out: int = 64):
    """X_pca = (Z - m) V: from the float32 matrix (3xTF32) or, for a planes-only matrix, from the
    BF16 planes (3xBF16, scb_project_planes)."""
    dev = sc.device
    npad = comp_t.shape[0]
    X = torch.empty((sc.n_rows, max(ld_out, npad)), dtype=torch.float32, device=dev)
    if sc.Z is None:
        _lib.call("scb_project_planes", _ctx(sc.Z_hi), _p(sc.Z_hi), _p(sc.Z_lo), sc.n_rows, sc.ld, _p(comp_t), _p(mean),
                  n_comps, npad, _p(X), X.shape[1], _stream(dev))
        return X
    _lib.call("scb_project", _ctx(sc.Z), _p(sc.Z), sc.Z.shape[0], sc.ld, _p(comp_t), _p(mean), n_comps, npad, _p(X),
              X.shape[1], _stream(dev))
    return X


def pca(sc: Scaled, n_comps: int = 50) -> PCAResult:
    """sc.tl.pca(n_comps, zero_center=True) on the scaled matrix: tcgen05 Gram, float64
    subspace-iteration eigensolve, tcgen05 projection."""
    C = gram(sc)
    N = sc.n_rows
    lam, comp_t, mean, tr = pca_from_gram(sc, C, N, n_comps)
    X = project(sc, comp_t, mean, n_comps)
    return PCAResult(X, comp_t[:n_comps, : sc.H], lam, lam / tr, mean, n_comps)


# ----------------------------------------------------------------------------- knn
def neighbors(X_pca: torch.Tensor, n_neighbors: int = 15, n_comps: Optional[int] = None,
              keys: Optional[torch.Tensor] = None, timer=None):
    """sc.pp.neighbors(n_neighbors, metric='euclidean') by brute force over every key: FP16
    tensor-core candidate scores (32 candidates per query for k <= 16) and an exact FP32 re-rank.
    Recall-checked (>= 0.999 against exact float64 neighbours in the tests), not certified exact:
    a true neighbour whose FP16 score misses the candidate lists is not reported.  Output:
    (indices int32 [Nq][k], distances float32 [Nq][k]) ordered by (distance, index), self
    included.  ``keys`` (default: X_pca itself) is the full embedding when the queries are a
    shard (multi-GPU); returned indices index ``keys``.  ``timer`` = (start, end) CUDA events
    recorded around the tensor-core candidate kernel (bench roofline)."""
    keys = X_pca if keys is None else keys
    d = X_pca.shape[1] if n_comps is None else n_comps
    dev = X_pca.device
    nq, nk = X_pca.shape[0], keys.shape[0]
    k = int(n_neighbors)
    kc = 32 if k <= 16 else 64
    idx = torch.empty((nq, k), dtype=torch.int32, device=dev)
    dist = torch.empty((nq, k), dtype=torch.float32, device=dev)
    e0 = e1 = 0
    if timer is not None:
        for ev in timer:
            ev.record()  # materialise the cudaEvent_t (torch creates events lazily)
        e0, e1 = timer[0].cuda_event, timer[1].cuda_event
    _lib.call("scb_knn_timed", _ctx(X_pca), _p(X_pca), nq, _p(keys), nk, d, X_pca.stride(0), k, kc, _p(idx), _p(dist),
              _stream(dev), e0, e1)
    return idx, dist


# ----------------------------------------------------------------------------- neighbors graph
@dataclasses.dataclass
class NeighborsGraph:
    """sc.pp.neighbors' sparse outputs for this rank's rows: `distances` (kNN distances without
    the self edge) and `connectivities` (umap fuzzy_simplicial_set), both CSR over all cells,
    plus the per-cell sigma/rho of the membership strengths."""
    distances: DeviceCSR
    connectivities: DeviceCSR
    sigma: torch.Tensor
    rho: torch.Tensor


def neighbors_graph(knn_idx: torch.Tensor, knn_dist: torch.Tensor, comm=None) -> NeighborsGraph:
    """Graph outputs of sc.pp.neighbors(method="umap") from the exact kNN (self included).
    With ``comm`` the rows are this rank's shard (in rank order); the membership strengths of
    all cells are all-gathered (N x k x 8 B) and each rank builds its own rows."""
    dev = knn_idx.device
    n, k = knn_idx.shape
    ctx, s = _ctx(knn_idx), _stream(dev)
    tot = torch.zeros(1, dtype=torch.float64, device=dev)
    _lib.call("scb_knn_dist_sum", ctx, _p(knn_dist), n * k, _p(tot), s)
    n_all, r0 = n, 0
    if comm is not None:
        comm.allreduce_(tot)
        counts = comm.allgather_rows(torch.tensor([[n]], dtype=torch.int64, device=dev)).view(-1).tolist()
        r0 = int(sum(counts[:comm.rank]))
        n_all = int(sum(counts))
    mean = tot / float(n_all * k)
    sigma = torch.empty(n, dtype=torch.float32, device=dev)
    rho = torch.empty(n, dtype=torch.float32, device=dev)
    w = torch.empty((n, k), dtype=torch.float32, device=dev)
    _lib.call("scb_umap_weights", ctx, _p(knn_idx), _p(knn_dist), n, k, r0, _p(mean), _p(sigma), _p(rho), _p(w), s)
    idx_all, w_all = knn_idx, w
    if comm is not None:
        idx_all, w_all = comm.allgather_rows(knn_idx), comm.allgather_rows(w)
    indptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    _lib.call("scb_fuzzy_union_rows", ctx, _p(idx_all), _p(w_all), n_all, k, r0, r0 + n, _p(indptr), s)
    nnz = int(indptr[n].item())
    cols = torch.empty(nnz, dtype=torch.int32, device=dev)
    vals = torch.empty(nnz, dtype=torch.float32, device=dev)
    _lib.call("scb_fuzzy_union_fill", ctx, _p(idx_all), _p(w_all), n_all, k, r0, r0 + n, _p(indptr), _p(cols),
              _p(vals), s)
    dptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    dcols = torch.empty(n * k, dtype=torch.int32, device=dev)
    dvals = torch.empty(n * k, dtype=torch.float32, device=dev)
    _lib.call("scb_knn_distances_csr", ctx, _p(knn_idx), _p(knn_dist), n, k, _p(dptr), _p(dcols), _p(dvals), s)
    dn = int(dptr[n].item())
    return NeighborsGraph(DeviceCSR(dptr, dcols[:dn], dvals[:dn], n_all), DeviceCSR(indptr, cols, vals, n_all),
                          sigma, rho)


# ----------------------------------------------------------------------------- umap layout
def umap_ab(min_dist: float = 0.5, spread: float = 1.0):
    """umap's find_ab_params: fit 1 / (1 + a x^(2b)) to the (min_dist, spread) target curve
    (scipy curve_fit on the host; two scalars)."""
    from scipy.optimize import curve_fit

    def curve(x, a, b):
        return 1.0 / (1.0 + a * x ** (2 * b))
    xv = np.linspace(0, spread * 3, 300)
    yv = np.where(xv < min_dist, 1.0, np.exp(-(xv - min_dist) / spread))
    (a, b), _ = curve_fit(curve, xv, yv)
    return float(a), float(b)


def umap_layout(connectivities: DeviceCSR, init: torch.Tensor, n_epochs: Optional[int] = None,
                min_dist: float = 0.5, spread: float = 1.0, negative_sample_rate: int = 5, seed: int = 0):
    """sc.tl.umap(min_dist, spread, init_pos=<obsm key>) on the device: umap-learn's
    optimize_layout_euclidean as edge-parallel SGD (see csrc/umap.cu).  ``init`` = [N][>=2]
    float32 starting coordinates (e.g. X_pca's first two columns); n_epochs defaults as umap
    (500 for <= 10k cells, else 200).  Returns float32 [N][2]."""
    n = connectivities.n_rows
    if n_epochs is None:
        n_epochs = 500 if n <= 10000 else 200
    a, b = umap_ab(min_dist, spread)
    w = connectivities.data
    w_max = float(w.max().item()) if w.numel() else 1.0
    emb = torch.empty((n, 2), dtype=torch.float32, device=w.device)
    init = init.contiguous()
    _lib.call("scb_umap_layout", _ctx(w), _p(connectivities.indptr), _p(connectivities.indices), _p(w), n,
              int(w.numel()), w_max, _p(init), init.stride(0), int(n_epochs), a, b, int(negative_sample_rate),
              int(seed), _p(emb), _stream(w.device))
    return emb


# ----------------------------------------------------------------------------- clustering
def _cluster(fn: str, G: DeviceCSR, resolution: float, max_levels: int, max_iters: int, seed: int):
    import ctypes
    lab = torch.empty(G.n_rows, dtype=torch.int32, device=G.data.device)
    nc = ctypes.c_int32(0)
    q = ctypes.c_double(0.0)
    _lib.call(fn, _ctx(G.data), _p(G.indptr), _p(G.indices), _p(G.data), G.n_rows, int(G.data.numel()),
              float(resolution), int(max_levels), int(max_iters), int(seed) & 0xFFFFFFFF, _p(lab),
              ctypes.addressof(nc), ctypes.addressof(q), _stream(G.data.device))
    return lab, int(nc.value), float(q.value)


def louvain(connectivities: DeviceCSR, resolution: float = 1.0, max_levels: int = 10, max_iters: int = 10,
            seed: int = 0):
    """sc.tl.louvain(resolution) on the neighbors graph, deterministic (csrc/cluster.cu).  Returns
    (labels int32 [N] ordered by decreasing community size, n_communities, modularity)."""
    return _cluster("scb_louvain", connectivities, resolution, max_levels, max_iters, seed)


def leiden(connectivities: DeviceCSR, resolution: float = 1.0, max_levels: int = 10, max_iters: int = 10,
           seed: int = 0):
    """sc.tl.leiden(resolution): local moving, refinement (well-connected sub-communities) and
    aggregation by the refined partition, deterministic (csrc/cluster.cu).  Returns (labels,
    n_communities, modularity)."""
    return _cluster("scb_leiden", connectivities, resolution, max_levels, max_iters, seed)


# ----------------------------------------------------------------------------- differential expression
def rank_genes_groups(X_log: DeviceCSR, labels: torch.Tensor, n_groups: Optional[int] = None) -> dict:
    """sc.tl.rank_genes_groups(groupby=labels, method="t-test", reference="rest") on the
    log-normalized kept matrix (csrc/de.cu).  Returns float64 [n_groups][G] scores,
    logfoldchanges, pvals, pvals_adj and int32 order (gene indices by decreasing score)."""
    dev = X_log.device
    K = int(labels.max().item()) + 1 if n_groups is None else int(n_groups)
    G = X_log.n_cols
    out = {k: torch.empty((K, G), dtype=torch.float64, device=dev)
           for k in ("scores", "logfoldchanges", "pvals", "pvals_adj")}
    out["order"] = torch.empty((K, G), dtype=torch.int32, device=dev)
    lab = labels.to(device=dev, dtype=torch.int32).contiguous()
    _lib.call("scb_rank_genes_groups", _ctx(X_log.data), _p(X_log.indptr), _p(X_log.indices), _p(X_log.data),
              X_log.n_rows, G, _p(lab), K, _p(out["scores"]), _p(out["logfoldchanges"]), _p(out["pvals"]),
              _p(out["pvals_adj"]), _p(out["order"]), _stream(dev))
    return out
