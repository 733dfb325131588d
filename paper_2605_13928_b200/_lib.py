"""ctypes binding of libscb_b200.so (the C ABI declared in include/scb.h).

There is no fallback: if the shared library is missing or no B200 is visible, every
step function raises.  The library is built in-tree by ``__graft_entry__.build()``
(``make -C paper_2605_13928_b200/csrc``).
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SCB_LIB_PATH") or os.path.join(_HERE, "libscb_b200.so")  # override: A/B experiments

c_i32, c_i64, c_u64, c_dbl, c_ptr = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p

# name -> argtypes (all functions return int status unless listed in _RESTYPE)
SIGNATURES = {
    "scb_abi_version": [],
    "scb_last_error": [],
    "scb_launch_count": [],
    "scb_ctx_create": [ctypes.c_int, ctypes.POINTER(c_ptr)],
    "scb_ctx_destroy": [c_ptr],
    "scb_nccl_unique_id": [c_ptr],
    "scb_ctx_create_comm": [ctypes.c_int, c_ptr, c_i32, c_i32, ctypes.POINTER(c_ptr)],
    "scb_comm_info": [c_ptr, c_ptr, c_ptr],
    "scb_comm_allreduce": [c_ptr, c_ptr, c_i64, c_i32, c_i32, c_ptr],
    "scb_comm_broadcast": [c_ptr, c_ptr, c_i64, c_i32, c_ptr],
    "scb_comm_allgather": [c_ptr, c_ptr, c_ptr, c_i64, c_ptr],
    "scb_qc_metrics": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                       c_ptr],
    "scb_hvg_tiles": [c_i32],
    "scb_filter_masks": [c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_i32, c_i32, c_i32, c_dbl, c_i32, c_ptr, c_ptr, c_ptr, c_ptr,
                         c_ptr],
    "scb_subset_rows_all_genes": [c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_dbl, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "scb_ctx_set_deferred_checks": [c_ptr, c_i32],
    "scb_ctx_copy_data_flag": [c_ptr, c_ptr, c_ptr],
    "scb_subset_count": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_dbl, c_ptr, c_ptr, c_ptr],
    "scb_subset_fill": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "scb_normalize_log1p": [c_ptr, c_ptr, c_ptr, c_i64, c_dbl, c_ptr, c_ptr, c_ptr],
    "scb_hvg_gene_sums": [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_i32, c_ptr, c_ptr, c_ptr],
    "scb_hvg_select": [c_ptr, c_ptr, c_i32, c_i64, c_i32, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "scb_scale_gene_sums": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_i32, c_ptr, c_ptr],
    "scb_scale_finalize": [c_ptr, c_ptr, c_i32, c_i64, c_ptr, c_ptr, c_ptr],
    "scb_scale_dense": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_i32, c_ptr, c_ptr, c_dbl, c_dbl, c_ptr, c_i64,
                        c_i32, c_ptr],
    "scb_gram": [c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr],
    "scb_gram_split": [c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr],
    "scb_split_bf16": [c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr],
    "scb_plane_format": [],
    "scb_subset_fill_scale_sums": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i32,
                                   c_ptr, c_ptr, c_ptr, c_ptr],
    "scb_umap_layout": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i64, ctypes.c_float, c_ptr, c_i64, c_i32, ctypes.c_float,
                        ctypes.c_float, c_i32, c_u64, c_ptr, c_ptr],
    "scb_louvain": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_dbl, c_i32, c_i32, ctypes.c_uint32, c_ptr, c_ptr, c_ptr,
                    c_ptr],
    "scb_leiden": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_dbl, c_i32, c_i32, ctypes.c_uint32, c_ptr, c_ptr, c_ptr,
                   c_ptr],
    "scb_rank_genes_groups": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                              c_ptr],
    "scb_knn_dist_sum": [c_ptr, c_ptr, c_i64, c_ptr, c_ptr],
    "scb_umap_weights": [c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "scb_fuzzy_union_rows": [c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_i64, c_i64, c_ptr, c_ptr],
    "scb_fuzzy_union_fill": [c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr],
    "scb_knn_distances_csr": [c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_ptr],
    "scb_mtx_parse": [c_ptr, c_ptr, c_i64, c_i64, c_i32, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr],
    "scb_coo_to_csr": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_ptr],
    "scb_regress_cov_sums": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_ptr],
    "scb_regress_design": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_ptr],
    "scb_regress_xty": [c_ptr, c_ptr, c_i64, c_i64, c_i32, c_ptr, c_ptr, c_ptr],
    "scb_regress_finalize": [c_ptr, c_ptr, c_ptr, c_i32, c_ptr, c_ptr, c_ptr],
    "scb_regress_apply": [c_ptr, c_ptr, c_i64, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_dbl, c_dbl, c_ptr],
    "scb_pca_eig": [c_ptr, c_ptr, c_i32, c_i32, c_i32, c_i64, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "scb_project": [c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_i32, c_i32, c_ptr, c_i32, c_ptr],
    "scb_knn": [c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_i32, c_i32, c_i32, c_i32, c_ptr, c_ptr, c_ptr],
    "scb_knn_ordered": [c_ptr, c_ptr, c_i64, c_i32, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "scb_knn_timed": [c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_i32, c_i32, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "scb_qc_metrics_u16": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                           c_ptr, c_ptr, c_ptr, c_i64, c_ptr],
    "scb_subset_count_u16": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_dbl, c_ptr, c_ptr,
                             c_ptr, c_ptr, c_i64, c_ptr],
    "scb_subset_fill_u16": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                            c_ptr, c_i64, c_ptr],
    "scb_subset_fill_scale_sums_u16": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                                       c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr],
    "scb_hvg_gene_sums_u16": [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_ptr,
                              c_i64, c_ptr],
    "scb_csr_u16_decode": [c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_ptr],
    "scb_csr_delta8_decode": [c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_i64,
                              c_ptr, c_ptr, c_ptr],
    "scb_scale_dense_planes": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_i32, c_ptr, c_ptr, c_dbl, c_dbl,
                               c_ptr, c_ptr, c_i64, c_i32, c_ptr],
    "scb_project_planes": [c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_i32, c_i32, c_ptr, c_i32, c_ptr],
    "scb_synth_logmean": [c_ptr, c_i64, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    "scb_synth_rows": [c_ptr, c_u64, c_i64, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
}
_RESTYPE = {"scb_last_error": ctypes.c_char_p, "scb_launch_count": ctypes.c_ulonglong, "scb_hvg_tiles": ctypes.c_int32,
            "scb_plane_format": ctypes.c_int32}

_lib = None
_lock = threading.Lock()


class ScbError(RuntimeError):
    """Raised when a C-ABI call returns a non-zero status (message from scb_last_error)."""

    def __init__(self, fn, code, msg):
        super().__init__(f"{fn} failed ({code}): {msg}")
        self.code = code


def load(path: str = LIB_PATH):
    """Load the shared library and bind every symbol in SIGNATURES (raises if any is missing)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                              " (or `make -C paper_2605_13928_b200/csrc`); there is no CPU fallback")
        lib = ctypes.CDLL(path)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)  # AttributeError if not exported
            fn.argtypes = argtypes
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
        _lib = lib
        return lib


def call(name, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    if name in _RESTYPE:
        return rc
    if rc != 0:
        msg = lib.scb_last_error()
        raise ScbError(name, rc, msg.decode() if msg else "")
    return rc


def launch_count() -> int:
    """Kernels launched by libscb_b200.so so far in this process."""
    return int(load().scb_launch_count())


_ctx = {}


def context(device: int):
    """Per-device scb_ctx (created lazily, destroyed at interpreter exit)."""
    with _lock:
        c = _ctx.get(device)
    if c is None:
        lib = load()
        p = c_ptr()
        rc = lib.scb_ctx_create(device, ctypes.byref(p))
        if rc != 0:
            raise ScbError("scb_ctx_create", rc, lib.scb_last_error().decode())
        with _lock:
            _ctx[device] = p.value
        c = p.value
    return c


def install_context(device: int, ptr: int):
    """Make ``ptr`` (e.g. a ctx that owns an NCCL communicator) the device's ctx for every step
    call; a previously created ctx of that device is destroyed at exit."""
    with _lock:
        old = _ctx.get(device)
        _ctx[device] = ptr
        if old is not None and old != ptr:
            _retired.append(old)


_retired = []


def _destroy_all():
    if _lib is None:
        return
    for c in list(_ctx.values()) + _retired:
        try:
            _lib.scb_ctx_destroy(c)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass
    _ctx.clear()
    _retired.clear()


import atexit  # noqa: E402

atexit.register(_destroy_all)


def plane_dtype():
    """torch dtype of the Gram / projection operand planes of this build (scb_plane_format)."""
    import torch
    return torch.bfloat16 if int(load().scb_plane_format()) == 0 else torch.float16
