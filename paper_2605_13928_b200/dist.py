"""Cell-sharded multi-GPU plumbing over torch.distributed (NCCL on B200s, gloo in CPU tests).

Rows (cells) are split into contiguous blocks balanced by nonzeros (``shard_rows_by_nnz``);
every collective of the path is one of
(SURVEY.md §8(e)): SUM all-reduce of per-gene integer sums / counts and of the partial
Gram matrix, a broadcast of the rank-0 eigenvectors, and a row all-gather of the PCA
embedding for the kNN keys.  Integer fixed-point gene sums make the HVG set and the scale
statistics bit-identical for any world size.
"""
from __future__ import annotations

import torch
import torch.distributed as td


def shard_rows(n: int, rank: int, world: int):
    """Contiguous [begin, end) row range of ``rank`` with balanced row counts."""
    base, rem = divmod(n, world)
    b = rank * base + min(rank, rem)
    return b, b + base + (1 if rank < rem else 0)


def shard_rows_by_nnz(indptr, rank: int, world: int):
    """Contiguous [begin, end) row range of ``rank`` balanced by nonzeros: the
    cut before shard r is the first row boundary with indptr >= Z * r / world.  ``indptr`` is the
    host (numpy or CPU tensor) int64 row-pointer array of the whole matrix."""
    import numpy as np
    ip = np.asarray(indptr, dtype=np.int64)
    n, Z = len(ip) - 1, int(ip[-1])
    if Z == 0:
        return shard_rows(n, rank, world)

    def cut(r):
        if r <= 0:
            return 0
        if r >= world:
            return n
        return int(min(n, np.searchsorted(ip, (Z * r + world - 1) // world, side="left")))
    return cut(rank), cut(rank + 1)


def row_shards_from_counts(row_nnz, world: int):
    """All ranks' nnz-balanced [begin, end) ranges from per-row nonzero counts."""
    import numpy as np
    ip = np.zeros(len(row_nnz) + 1, dtype=np.int64)
    np.cumsum(np.asarray(row_nnz, dtype=np.int64), out=ip[1:])
    return [shard_rows_by_nnz(ip, r, world) for r in range(world)]


class Comm:
    def __init__(self, group=None):
        self.group = group
        self.rank = td.get_rank(group)
        self.world = td.get_world_size(group)
        self.cpu_only = td.get_backend(group) == "gloo"

    def _dev(self, t):
        return t.cpu() if (self.cpu_only and t.is_cuda) else t

    def allreduce_(self, t: torch.Tensor, op=td.ReduceOp.SUM):
        x = self._dev(t)
        td.all_reduce(x, op=op, group=self.group)
        if x is not t:
            t.copy_(x)
        return t

    def allreduce_int(self, v: int) -> int:
        dev = "cpu" if self.cpu_only else torch.device("cuda", torch.cuda.current_device())
        t = torch.tensor([int(v)], dtype=torch.int64, device=dev)
        td.all_reduce(t, group=self.group)
        return int(t.item())

    def allreduce_max(self, v: float) -> float:
        dev = "cpu" if self.cpu_only else torch.device("cuda", torch.cuda.current_device())
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        td.all_reduce(t, op=td.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def broadcast_(self, t: torch.Tensor, src: int = 0):
        x = self._dev(t)
        td.broadcast(x, src, group=self.group)
        if x is not t:
            t.copy_(x)
        return t

    def allgather_rows(self, X: torch.Tensor) -> torch.Tensor:
        """Concatenate every rank's rows (possibly unequal counts) in rank order."""
        x = self._dev(X.contiguous())
        n = torch.tensor([x.shape[0]], dtype=torch.int64, device=x.device)
        ns = [torch.zeros_like(n) for _ in range(self.world)]
        td.all_gather(ns, n, group=self.group)
        ns = [int(v.item()) for v in ns]
        m = max(ns)
        pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        pad[: x.shape[0]] = x
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        td.all_gather(outs, pad, group=self.group)
        full = torch.cat([o[:k] for o, k in zip(outs, ns)], 0)
        return full.to(X.device) if full.device != X.device else full


_NCCL_DTYPES = {torch.int64: 0, torch.float64: 1, torch.float32: 2, torch.int32: 3}


class NcclComm:
    """The Comm interface over the C ABI's own NCCL communicator (scb_ctx_create_comm): the
    device's scb_ctx holds the ncclComm_t and every collective of the
    pipeline is a stream-ordered scb_comm_* call on the current torch stream.  The 128-byte
    NCCL id travels through an existing torch.distributed group (``from_torch_distributed``)
    or any side channel (``unique_id`` on rank 0, then the constructor on every rank)."""

    cpu_only = False

    @staticmethod
    def unique_id() -> bytes:
        import ctypes
        from . import _lib
        buf = (ctypes.c_uint8 * 128)()
        _lib.call("scb_nccl_unique_id", ctypes.addressof(buf))
        return bytes(buf)

    def __init__(self, device: int, rank: int, world: int, nccl_id: bytes):
        import ctypes
        from . import _lib
        if len(nccl_id) != 128:
            raise ValueError("nccl_id must be the 128 bytes of scb_nccl_unique_id")
        lib = _lib.load()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
        p = ctypes.c_void_p()
        rc = lib.scb_ctx_create_comm(int(device), ctypes.addressof(buf), int(rank), int(world), ctypes.byref(p))
        if rc != 0:
            raise _lib.ScbError("scb_ctx_create_comm", rc, lib.scb_last_error().decode())
        self.ctx = p.value
        _lib.install_context(int(device), self.ctx)
        self.device = int(device)
        self.rank = int(rank)
        self.world = int(world)

    @classmethod
    def from_torch_distributed(cls, device: int, group=None) -> "NcclComm":
        """Rank 0 creates the id and broadcasts it over an initialised torch.distributed group."""
        rank, world = td.get_rank(group), td.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        td.broadcast_object_list(obj, src=0, group=group)
        return cls(device, rank, world, obj[0])

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def allreduce_(self, t: torch.Tensor, op=None):
        from . import _lib
        if t.dtype not in _NCCL_DTYPES:
            raise TypeError(f"NcclComm.allreduce_: unsupported dtype {t.dtype}")
        x = t if t.is_contiguous() else t.contiguous()
        is_max = op is not None and op == td.ReduceOp.MAX
        _lib.call("scb_comm_allreduce", self.ctx, x.data_ptr(), x.numel(), _NCCL_DTYPES[x.dtype], 1 if is_max else 0,
                  self._stream())
        if x is not t:
            t.copy_(x)
        return t

    def allreduce_int(self, v: int) -> int:
        t = torch.tensor([int(v)], dtype=torch.int64, device=torch.device("cuda", self.device))
        return int(self.allreduce_(t).item())

    def allreduce_max(self, v: float) -> float:
        t = torch.tensor([float(v)], dtype=torch.float64, device=torch.device("cuda", self.device))
        return float(self.allreduce_(t, td.ReduceOp.MAX).item())

    def broadcast_(self, t: torch.Tensor, src: int = 0):
        from . import _lib
        x = t if t.is_contiguous() else t.contiguous()
        _lib.call("scb_comm_broadcast", self.ctx, x.data_ptr(), x.numel() * x.element_size(), int(src), self._stream())
        if x is not t:
            t.copy_(x)
        return t

    def allgather_rows(self, X: torch.Tensor) -> torch.Tensor:
        """Concatenate every rank's rows (possibly unequal counts) in rank order."""
        from . import _lib
        x = X.contiguous()
        dev = torch.device("cuda", self.device)
        n = torch.tensor([x.shape[0]], dtype=torch.int64, device=dev)
        ns = torch.empty(self.world, dtype=torch.int64, device=dev)
        _lib.call("scb_comm_allgather", self.ctx, n.data_ptr(), ns.data_ptr(), 8, self._stream())
        ns = [int(v) for v in ns.tolist()]
        m = max(ns)
        pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=dev)
        pad[: x.shape[0]] = x
        out = torch.empty((self.world * m,) + tuple(x.shape[1:]), dtype=x.dtype, device=dev)
        _lib.call("scb_comm_allgather", self.ctx, pad.data_ptr(), out.data_ptr(), pad.numel() * pad.element_size(),
                  self._stream())
        return torch.cat([out[r * m: r * m + k] for r, k in enumerate(ns)], 0)
