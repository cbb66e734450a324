"""Multi-GPU decomposition of the RSVD path.

Two shardings, both one process (or host thread) per rank:

* batch split (C2, C4): independent matrices are split contiguously across
  ranks, each rank uses its items' own seeds; no collective on the data path.
* row shard (C3, C5): one large A is split by rows; Omega is replicated from
  the seed, Y_p = A_p Omega and Q_p are local, and the only exchanges are sum
  all-reduces of the m-side l x l Grams and of the n x l panels A^T Q
  (engine.cu `orth` / `range_finder` / `svd_stage`), over NCCL
  (`attach_nccl`) or an in-process group (`Group`, used to emulate P ranks on
  one GPU: host barriers only, never a device-side wait).
"""
from __future__ import annotations

import ctypes
from typing import Optional, Tuple

from . import _lib
from .factorize import RsvdParams, TruncatedFactorization, _colmajor_torch, _MASK


def batch_partition(batch: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous split of `batch` items: (first item, count) of `rank`."""
    base, extra = divmod(batch, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def row_partition(m: int, world: int, rank: int, align: int = 16) -> Tuple[int, int]:
    """Contiguous split of m rows in multiples of `align` (the TMA A-pass wants
    16-row aligned local blocks); the last rank takes the remainder."""
    chunk = -(-m // world)
    chunk = -(-chunk // align) * align
    first = min(rank * chunk, m)
    return first, max(0, min(chunk, m - first))


class Group:
    """In-process group of `n` ranks for row-sharded calls (rsvd_group)."""

    def __init__(self, n: int):
        lib = _lib.load()
        g = ctypes.c_void_p()
        rc = lib.rsvd_group_create(ctypes.byref(g), int(n))
        if rc != _lib.RSVD_OK:
            raise _lib.InvalidArgument(f"rsvd_group_create({n}) failed")
        self._g = g
        self.n = n

    def attach(self, handle: _lib.Handle, rank: int) -> None:
        _lib.raise_for(_lib.load().rsvd_attach_group(handle.raw, self._g, int(rank)), handle.raw)

    def close(self):
        if getattr(self, "_g", None):
            _lib.load().rsvd_group_destroy(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = _lib.load().rsvd_nccl_unique_id(buf)
    if rc != _lib.RSVD_OK:
        raise _lib.DeviceError("rsvd_nccl_unique_id failed (NCCL unavailable?)")
    return buf.raw


def attach_nccl(handle: _lib.Handle, world: int, rank: int, uid: Optional[bytes] = None) -> None:
    """Create the handle's NCCL communicator.  Without `uid`, rank 0 makes one
    and torch.distributed broadcasts it (the process group must exist)."""
    if uid is None:
        import torch.distributed as dist

        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    _lib.raise_for(_lib.load().rsvd_attach_nccl(handle.raw, int(world), int(rank), uid), handle.raw)


def detach(handle: _lib.Handle) -> None:
    _lib.raise_for(_lib.load().rsvd_detach(handle.raw), handle.raw)


def rsvd_rowsharded(a_local, m_global: int, row_offset: int, params: RsvdParams,
                    handle: _lib.Handle) -> TruncatedFactorization:
    """This rank's part of rsvd(A) for the row block A[row_offset:row_offset+m_local]
    (a float64 CUDA tensor).  Returns left = the matching rows of U; sigma and
    right_adj are replicated."""
    import torch

    lib = _lib.load()
    a_local, lda = _colmajor_torch(a_local)
    m, n = a_local.shape
    kk = max(int(params.rank), 1)
    U = torch.empty((kk, m), dtype=torch.float64, device=a_local.device).t()
    S = torch.empty(kk, dtype=torch.float64, device=a_local.device)
    Vt = torch.empty((n, kk), dtype=torch.float64, device=a_local.device).t()
    r = ctypes.c_int64(0)
    dw = ctypes.c_double(0.0)
    with _lib.on_torch_stream(handle):
        rc = lib.rsvd_f64_rowsharded(handle.raw, a_local.data_ptr(), m, n, lda, int(m_global),
                                     int(row_offset), params.rank, params.oversample,
                                     params.power, params.seed & _MASK, U.data_ptr(), max(m, 1),
                                     S.data_ptr(), Vt.data_ptr(), kk, ctypes.byref(r),
                                     ctypes.byref(dw), _lib.PTR_DEVICE)
    _lib.raise_for(rc, handle.raw)
    rr = r.value
    return TruncatedFactorization(U[:, :rr], S[:rr], Vt[:rr, :], dw.value, False)
