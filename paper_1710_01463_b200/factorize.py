"""Reference-shaped factorization API over the B200 engine.

Mirrors rlftn's factorize.hpp (proj/include/rlftn/factorize.hpp):
``RsvdParams`` (hpp:40-45, ``oversample`` is the TOTAL sample width l),
``TruncatedFactorization`` (hpp:15-31), ``rsvd`` (hpp:62-63,
factorize.cpp:76-95), ``randomized_range`` (hpp:56-57, cpp:52-74) and
``reconstruction_error`` (hpp:68-70, cpp:97-104), with the same argument
errors (raised as ``InvalidArgument``, a ``ValueError``, for the reference's
``std::invalid_argument``) and messages.

Arrays: numpy float64 arrays go through the C ABI with host pointers (the
engine copies in and out); float64 CUDA tensors go with device pointers and
stay on the GPU.  Matrices are column-major on the device; numpy inputs are
converted with ``np.asfortranarray`` and torch inputs must be column-major
(``t.t().contiguous().t()``) or are converted.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import Any, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import InvalidArgument


@dataclass
class RsvdParams:
    """rlftn::RsvdParams (factorize.hpp:40-45)."""

    rank: int = 0
    oversample: int = 0  # total sample width l; 0 -> min(2*rank, min(m, n))
    power: int = 4
    seed: int = 0


@dataclass
class TruncatedFactorization:
    """rlftn::TruncatedFactorization (factorize.hpp:15-31)."""

    left: Any  # m x r
    sigma: Any  # r
    right_adj: Any  # r x n
    discarded_weight: float = 0.0
    discarded_exact: bool = True

    def rank(self) -> int:
        return int(self.sigma.shape[0])

    def reconstruct(self):
        return (self.left * self.sigma[None, :]) @ self.right_adj


class ErrorNorm(enum.Enum):
    frobenius = 0
    spectral = 1


def _is_torch_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and hasattr(a, "data_ptr") and bool(a.is_cuda)


def _is_complex(a) -> bool:
    """Complex instantiation (factorize.cpp:106-118): complex128 numpy arrays or
    torch tensors go to the *_z128 entry points."""
    if hasattr(a, "is_complex") and hasattr(a, "data_ptr"):
        return bool(a.is_complex())
    return bool(np.iscomplexobj(a))


def _np_dtype(cplx: bool):
    return np.complex128 if cplx else np.float64


def _torch_dtype(cplx: bool):
    import torch

    return torch.complex128 if cplx else torch.float64


def _colmajor_torch(a):
    import torch

    if a.dtype not in (torch.float64, torch.complex128):
        raise InvalidArgument("rsvd: expected a float64 or complex128 tensor")
    if a.dim() != 2:
        raise InvalidArgument("rsvd: expected a 2-D tensor")
    m, n = a.shape
    if a.stride(0) == 1 and (a.stride(1) >= max(m, 1)):
        return a, a.stride(1)
    a = a.t().contiguous().t()
    return a, max(m, 1)


def _torch_stream_guard(h):
    import torch

    lib = _lib.load()
    lib.rsvd_set_stream(h.raw, ctypes.c_void_p(_lib.torch_stream_ptr()))


def _resolve_ell(m: int, n: int, p: RsvdParams) -> int:
    ell = p.oversample
    if ell == 0:
        ell = min(2 * p.rank, min(m, n))
    return ell


def rsvd(a, params: RsvdParams, handle: Optional[_lib.Handle] = None) -> TruncatedFactorization:
    """rlftn::rsvd (factorize.cpp:76-95) on the GPU; complex128 input runs the
    complex instantiation (rsvd<std::complex<double>>)."""
    lib = _lib.load()
    h = handle or _lib.default_handle()
    out_rank = ctypes.c_int64(0)
    dw = ctypes.c_double(0.0)
    cplx = _is_complex(a)
    fn = lib.rsvd_z128 if cplx else lib.rsvd_f64
    if _is_torch_cuda(a):
        import torch

        a, lda = _colmajor_torch(a)
        m, n = a.shape
        k = max(int(params.rank), 0)
        kk = max(k, 1)
        U = torch.empty((kk, m), dtype=a.dtype, device=a.device).t()  # m x k col-major
        S = torch.empty(kk, dtype=torch.float64, device=a.device)
        Vt = torch.empty((n, kk), dtype=a.dtype, device=a.device).t()  # k x n col-major
        _torch_stream_guard(h)
        try:
            rc = fn(h.raw, a.data_ptr() if a.numel() else 0, m, n, lda, params.rank,
                              params.oversample, params.power, params.seed & _MASK, U.data_ptr(),
                              max(m, 1), S.data_ptr(), Vt.data_ptr(), kk, ctypes.byref(out_rank),
                              ctypes.byref(dw), _lib.PTR_DEVICE)
        finally:
            lib.rsvd_set_stream(h.raw, None)
        _lib.raise_for(rc, h.raw)
        r = out_rank.value
        return TruncatedFactorization(U[:, :r], S[:r], Vt[:r, :], dw.value, False)
    dt = _np_dtype(cplx)
    a = np.asfortranarray(np.asarray(a, dtype=dt))
    if a.ndim != 2:
        raise InvalidArgument("rsvd: expected a 2-D array")
    m, n = a.shape
    kk = max(int(params.rank), 1)
    U = np.zeros((m, kk), dtype=dt, order="F")
    S = np.zeros(kk)
    Vt = np.zeros((kk, n), dtype=dt, order="F")
    rc = fn(h.raw, a.ctypes.data if a.size else 0, m, n, max(m, 1), params.rank,
                      params.oversample, params.power, params.seed & _MASK, U.ctypes.data,
                      max(m, 1), S.ctypes.data, Vt.ctypes.data, kk, ctypes.byref(out_rank),
                      ctypes.byref(dw), _lib.PTR_HOST)
    _lib.raise_for(rc, h.raw)
    r = out_rank.value
    return TruncatedFactorization(U[:, :r].copy(order="F"), S[:r].copy(),
                                  Vt[:r, :].copy(order="F"), dw.value, False)


_MASK = (1 << 64) - 1


def tsvd(a, chi: int, handle: Optional[_lib.Handle] = None) -> TruncatedFactorization:
    """rlftn::tsvd (factorize.cpp:42-50): exact thin SVD truncated to
    r = min(chi, numerical rank), exact discarded weight.  Any size (the
    row-streamed Jacobi handles min(m, n) into the thousands)."""
    lib = _lib.load()
    h = handle or _lib.default_handle()
    r = ctypes.c_int64(0)
    dw = ctypes.c_double(0.0)
    cplx = _is_complex(a)
    fn = lib.rsvd_tsvd_z128 if cplx else lib.rsvd_tsvd_f64
    if _is_torch_cuda(a):
        import torch

        a, lda = _colmajor_torch(a)
        m, n = a.shape
        k = max(min(int(chi), m, n), 1)
        U = torch.empty((k, m), dtype=a.dtype, device=a.device).t()
        S = torch.empty(k, dtype=torch.float64, device=a.device)
        Vt = torch.empty((n, k), dtype=a.dtype, device=a.device).t()
        with _lib.on_torch_stream(h):
            rc = fn(h.raw, a.data_ptr() if a.numel() else 0, m, n, lda, int(chi),
                                   U.data_ptr(), max(m, 1), S.data_ptr(), Vt.data_ptr(), k,
                                   ctypes.byref(r), ctypes.byref(dw), _lib.PTR_DEVICE)
        _lib.raise_for(rc, h.raw)
        rr = r.value
        return TruncatedFactorization(U[:, :rr], S[:rr], Vt[:rr, :], dw.value, True)
    dt = _np_dtype(cplx)
    a = np.asfortranarray(np.asarray(a, dtype=dt))
    if a.ndim != 2:
        raise InvalidArgument("tsvd: expected a 2-D array")
    m, n = a.shape
    k = max(min(int(chi), m, n), 1)
    U = np.zeros((m, k), dtype=dt, order="F")
    S = np.zeros(k)
    Vt = np.zeros((k, n), dtype=dt, order="F")
    rc = fn(h.raw, a.ctypes.data if a.size else 0, m, n, max(m, 1), int(chi),
                           U.ctypes.data, max(m, 1), S.ctypes.data, Vt.ctypes.data, k,
                           ctypes.byref(r), ctypes.byref(dw), _lib.PTR_HOST)
    _lib.raise_for(rc, h.raw)
    rr = r.value
    return TruncatedFactorization(U[:, :rr].copy(order="F"), S[:rr].copy(),
                                  Vt[:rr, :].copy(order="F"), dw.value, True)


@dataclass
class BatchedFactorization:
    """Result of rsvd_batched: stacked buffers plus per-item ranks."""

    left: Any  # batch x m x k (column-major items)
    sigma: Any  # batch x k
    right_adj: Any  # batch x k x n
    ranks: List[int] = field(default_factory=list)
    discarded_weight: List[float] = field(default_factory=list)
    discarded_exact: bool = False

    def item(self, b: int) -> TruncatedFactorization:
        r = self.ranks[b]
        return TruncatedFactorization(self.left[b][:, :r], self.sigma[b][:r],
                                      self.right_adj[b][:r, :], self.discarded_weight[b],
                                      self.discarded_exact)


def _batched_buffers(a, k: int, who: str):
    """Stage a (batch, m, n) input and allocate (batch, m, k) / (batch, k) /
    (batch, k, n) outputs with column-major items.  Returns
    (bsz, m, n, flags, ptrs, U, S, Vt, Ub, Vb, keepalive)."""
    import torch

    if a.dim() != 3 or a.dtype not in (torch.float64, torch.complex128):
        raise InvalidArgument(f"{who}: expected a (batch, m, n) float64 or complex128 tensor")
    bsz, m, n = a.shape
    if not (a.stride(1) == 1 and a.stride(2) == m and a.stride(0) == m * n):
        a = a.transpose(1, 2).contiguous().transpose(1, 2)
    dev = a.device if a.is_cuda else None
    pin = (not a.is_cuda) and bool(a.is_pinned())
    kw = dict(device=dev) if dev is not None else dict(pin_memory=pin)
    U = torch.empty((bsz, k, m), dtype=a.dtype, **kw).transpose(1, 2)
    S = torch.empty((bsz, k), dtype=torch.float64, **kw)
    Vt = torch.empty((bsz, n, k), dtype=a.dtype, **kw).transpose(1, 2)
    flags = _lib.PTR_DEVICE if a.is_cuda else _lib.PTR_HOST
    return bsz, m, n, flags, (a.data_ptr(), U.data_ptr(), S.data_ptr(), Vt.data_ptr()), U, S, Vt, a


def tsvd_batched(a, chi: int, handle: Optional[_lib.Handle] = None) -> BatchedFactorization:
    """Batched tsvd over (batch, m, n) items of one shape (the exact route of
    block_factorize for equal-shape sectors, blocks.cpp:82)."""
    lib = _lib.load()
    h = handle or _lib.default_handle()
    cplx = _is_complex(a)
    fn = lib.rsvd_tsvd_z128_batched if cplx else lib.rsvd_tsvd_f64_batched
    if hasattr(a, "data_ptr") and hasattr(a, "is_pinned"):
        m_, n_ = int(a.shape[1]), int(a.shape[2])
        k = max(min(int(chi), m_, n_), 1)
        bsz, m, n, flags, ptrs, U, S, Vt, a = _batched_buffers(a, k, "tsvd_batched")
        Ub = None
    else:
        dt = _np_dtype(cplx)
        a = np.asarray(a, dtype=dt)
        if a.ndim != 3:
            raise InvalidArgument("tsvd_batched: expected a (batch, m, n) array")
        bsz, m, n = a.shape
        k = max(min(int(chi), m, n), 1)
        a = np.ascontiguousarray(np.transpose(a, (0, 2, 1)))
        Ub = np.zeros((bsz, k, m), dtype=dt)
        S = np.zeros((bsz, k))
        Vb = np.zeros((bsz, n, k), dtype=dt)
        flags = _lib.PTR_HOST
        ptrs = (a.ctypes.data, Ub.ctypes.data, S.ctypes.data, Vb.ctypes.data)
    ranks = (ctypes.c_int64 * max(bsz, 1))()
    dws = (ctypes.c_double * max(bsz, 1))()
    if flags == _lib.PTR_DEVICE:
        with _lib.on_torch_stream(h):
            rc = fn(h.raw, bsz, ptrs[0], m, n, m, m * n, int(chi), ptrs[1],
                    m, m * k, ptrs[2], k, ptrs[3], k, k * n, ranks, dws, flags)
    else:
        rc = fn(h.raw, bsz, ptrs[0], m, n, m, m * n, int(chi), ptrs[1], m,
                                       m * k, ptrs[2], k, ptrs[3], k, k * n, ranks, dws, flags)
    _lib.raise_for(rc, h.raw)
    if Ub is not None:
        U = np.transpose(Ub, (0, 2, 1))
        Vt = np.transpose(Vb, (0, 2, 1))
    return BatchedFactorization(U, S, Vt, [int(ranks[i]) for i in range(bsz)],
                                [float(dws[i]) for i in range(bsz)], True)


def rsvd_batched(a, params: RsvdParams, seeds: Sequence[int],
                 handle: Optional[_lib.Handle] = None, out: Optional[BatchedFactorization] = None
                 ) -> BatchedFactorization:
    """Batched rsvd: ``a`` is (batch, m, n) with column-major items (a CUDA
    tensor whose items have strides (1, m), or a numpy array of shape
    (batch, m, n)); item b uses ``seeds[b]``.  ``out`` (torch inputs only):
    a previous result of the same shapes and device whose buffers are reused,
    e.g. pinned host factors in a loop (no per-call pinned allocation)."""
    lib = _lib.load()
    h = handle or _lib.default_handle()
    if out is not None and hasattr(a, "data_ptr"):
        return _rsvd_batched_into(lib, h, a, params, seeds, out)
    cplx = _is_complex(a)
    fn = lib.rsvd_z128_batched if cplx else lib.rsvd_f64_batched
    if _is_torch_cuda(a):
        import torch

        if a.dim() != 3 or a.dtype not in (torch.float64, torch.complex128):
            raise InvalidArgument("rsvd_batched: expected a (batch, m, n) float64 tensor")
        bsz, m, n = a.shape
        if not (a.stride(1) == 1 and a.stride(2) == m and a.stride(0) == m * n):
            a = a.transpose(1, 2).contiguous().transpose(1, 2)
        k = max(int(params.rank), 1)
        U = torch.empty((bsz, k, m), dtype=a.dtype, device=a.device).transpose(1, 2)
        S = torch.empty((bsz, k), dtype=torch.float64, device=a.device)
        Vt = torch.empty((bsz, n, k), dtype=a.dtype, device=a.device).transpose(1, 2)
        flags = _lib.PTR_DEVICE
        ptrs = (a.data_ptr(), U.data_ptr(), S.data_ptr(), Vt.data_ptr())
        _torch_stream_guard(h)
    elif hasattr(a, "data_ptr") and hasattr(a, "is_pinned"):
        # Host torch tensor (ideally pinned): passed with host pointers, the
        # engine copies in and out inside the call (the end-to-end path).
        import torch

        if a.dim() != 3 or a.dtype not in (torch.float64, torch.complex128):
            raise InvalidArgument("rsvd_batched: expected a (batch, m, n) float64 tensor")
        bsz, m, n = a.shape
        if not (a.stride(1) == 1 and a.stride(2) == m and a.stride(0) == m * n):
            a = a.transpose(1, 2).contiguous().transpose(1, 2)
        k = max(int(params.rank), 1)
        pin = bool(a.is_pinned())
        U = torch.empty((bsz, k, m), dtype=a.dtype, pin_memory=pin).transpose(1, 2)
        S = torch.empty((bsz, k), dtype=torch.float64, pin_memory=pin)
        Vt = torch.empty((bsz, n, k), dtype=a.dtype, pin_memory=pin).transpose(1, 2)
        flags = _lib.PTR_HOST
        ptrs = (a.data_ptr(), U.data_ptr(), S.data_ptr(), Vt.data_ptr())
        Ub = Vb = None
    else:
        dt = _np_dtype(cplx)
        a = np.asarray(a, dtype=dt)
        if a.ndim != 3:
            raise InvalidArgument("rsvd_batched: expected a (batch, m, n) array")
        bsz, m, n = a.shape
        a = np.ascontiguousarray(np.transpose(a, (0, 2, 1)))  # items column-major
        k = max(int(params.rank), 1)
        Ub = np.zeros((bsz, k, m), dtype=dt)
        S = np.zeros((bsz, k))
        Vb = np.zeros((bsz, n, k), dtype=dt)
        flags = _lib.PTR_HOST
        ptrs = (a.ctypes.data, Ub.ctypes.data, S.ctypes.data, Vb.ctypes.data)
    if len(seeds) != bsz:
        raise InvalidArgument("rsvd_batched: need one seed per item")
    seeds_arr = (ctypes.c_uint64 * max(bsz, 1))(*[int(s) & _MASK for s in seeds])
    ranks = (ctypes.c_int64 * max(bsz, 1))()
    dws = (ctypes.c_double * max(bsz, 1))()
    try:
        rc = fn(h.raw, bsz, ptrs[0], m, n, m, m * n, params.rank,
                params.oversample, params.power, seeds_arr, ptrs[1], m, m * k,
                ptrs[2], k, ptrs[3], k, k * n, ranks, dws, flags)
    finally:
        if flags == _lib.PTR_DEVICE:
            lib.rsvd_set_stream(h.raw, None)
    _lib.raise_for(rc, h.raw)
    if flags == _lib.PTR_HOST and Ub is not None:
        U = np.transpose(Ub, (0, 2, 1))
        Vt = np.transpose(Vb, (0, 2, 1))
    return BatchedFactorization(U, S, Vt, [int(ranks[i]) for i in range(bsz)],
                                [float(dws[i]) for i in range(bsz)])


def _rsvd_batched_into(lib, h, a, params, seeds, out):
    import torch

    if a.dim() != 3 or a.dtype not in (torch.float64, torch.complex128):
        raise InvalidArgument("rsvd_batched: expected a (batch, m, n) float64 tensor")
    bsz, m, n = a.shape
    if not (a.stride(1) == 1 and a.stride(2) == m and a.stride(0) == m * n):
        a = a.transpose(1, 2).contiguous().transpose(1, 2)
    k = max(int(params.rank), 1)
    U, S, Vt = out.left, out.sigma, out.right_adj
    fn = lib.rsvd_z128_batched if a.is_complex() else lib.rsvd_f64_batched
    ok = (tuple(U.shape) == (bsz, m, k) and U.stride() == (m * k, 1, m) and
          tuple(S.shape) == (bsz, k) and S.is_contiguous() and
          tuple(Vt.shape) == (bsz, k, n) and Vt.stride() == (k * n, 1, k) and
          all(x.device == a.device for x in (U, S, Vt)) and U.dtype == a.dtype and
          Vt.dtype == a.dtype and S.dtype == torch.float64)
    if not ok:
        raise InvalidArgument("rsvd_batched: out= buffers do not match the input shapes")
    if len(seeds) != bsz:
        raise InvalidArgument("rsvd_batched: need one seed per item")
    seeds_arr = (ctypes.c_uint64 * max(bsz, 1))(*[int(s) & _MASK for s in seeds])
    ranks = (ctypes.c_int64 * max(bsz, 1))()
    dws = (ctypes.c_double * max(bsz, 1))()
    flags = _lib.PTR_DEVICE if a.is_cuda else _lib.PTR_HOST
    if flags == _lib.PTR_DEVICE:
        _torch_stream_guard(h)
    try:
        rc = fn(h.raw, bsz, a.data_ptr(), m, n, m, m * n, params.rank,
                                  params.oversample, params.power, seeds_arr, U.data_ptr(), m,
                                  m * k, S.data_ptr(), k, Vt.data_ptr(), k, k * n, ranks, dws, flags)
    finally:
        if flags == _lib.PTR_DEVICE:
            lib.rsvd_set_stream(h.raw, None)
    _lib.raise_for(rc, h.raw)
    return BatchedFactorization(U, S, Vt, [int(ranks[i]) for i in range(bsz)],
                                [float(dws[i]) for i in range(bsz)])


def randomized_range(a, ell: int, power: int, seed: int,
                     handle: Optional[_lib.Handle] = None):
    """rlftn::randomized_range (factorize.cpp:52-74): Q (m x ell)."""
    lib = _lib.load()
    h = handle or _lib.default_handle()
    cplx = _is_complex(a)
    fn = lib.rsvd_randomized_range_z128 if cplx else lib.rsvd_randomized_range_f64
    if _is_torch_cuda(a):
        import torch

        a, lda = _colmajor_torch(a)
        m, n = a.shape
        Q = torch.empty((max(ell, 1), m), dtype=a.dtype, device=a.device).t()
        _torch_stream_guard(h)
        try:
            rc = fn(h.raw, a.data_ptr() if a.numel() else 0, m, n,
                                               lda, ell, power, seed & _MASK, Q.data_ptr(),
                                               max(m, 1), _lib.PTR_DEVICE)
        finally:
            lib.rsvd_set_stream(h.raw, None)
        _lib.raise_for(rc, h.raw)
        return Q[:, :ell]
    dt = _np_dtype(cplx)
    a = np.asfortranarray(np.asarray(a, dtype=dt))
    m, n = a.shape
    Q = np.zeros((m, max(ell, 1)), dtype=dt, order="F")
    rc = fn(h.raw, a.ctypes.data if a.size else 0, m, n, max(m, 1),
                                       ell, power, seed & _MASK, Q.ctypes.data, max(m, 1),
                                       _lib.PTR_HOST)
    _lib.raise_for(rc, h.raw)
    return Q[:, :ell]


def reconstruction_error(a, f: TruncatedFactorization, norm: ErrorNorm = ErrorNorm.frobenius,
                         handle: Optional[_lib.Handle] = None) -> float:
    """rlftn::reconstruction_error (factorize.cpp:97-104).  Frobenius: the
    engine's fused residual kernel.  Spectral (the reference's gesdd('N') of
    the residual, lapack.cpp:130-144): the residual is formed on the device and
    its largest singular value taken with the engine's tsvd (exact, as
    gesdd('N'))."""
    if norm != ErrorNorm.frobenius:
        return _spectral_error(a, f, handle)
    lib = _lib.load()
    h = handle or _lib.default_handle()
    out = ctypes.c_double(0.0)
    r = f.rank()
    cplx = _is_complex(a)
    fn = lib.rsvd_reconstruction_error_z128 if cplx else lib.rsvd_reconstruction_error_f64
    if _is_torch_cuda(a):
        import torch

        a, lda = _colmajor_torch(a)
        m, n = a.shape
        U = f.left.to(a.dtype).t().contiguous().t() if r else torch.zeros(
            (m, 1), dtype=a.dtype, device=a.device)
        Vt = f.right_adj.to(a.dtype).t().contiguous().t() if r else torch.zeros(
            (1, n), dtype=a.dtype, device=a.device)
        S = f.sigma.contiguous() if r else torch.zeros(1, dtype=torch.float64, device=a.device)
        _torch_stream_guard(h)
        try:
            rc = fn(h.raw, a.data_ptr(), m, n, lda, U.data_ptr(),
                                                   m, S.data_ptr(), Vt.data_ptr(), max(r, 1), r,
                                                   ctypes.byref(out), _lib.PTR_DEVICE)
        finally:
            lib.rsvd_set_stream(h.raw, None)
    else:
        dt = _np_dtype(cplx)
        a = np.asfortranarray(np.asarray(a, dtype=dt))
        m, n = a.shape
        U = np.asfortranarray(np.asarray(f.left, dtype=dt) if r else np.zeros((m, 1), dtype=dt))
        Vt = np.asfortranarray(np.asarray(f.right_adj, dtype=dt) if r else np.zeros((1, n), dtype=dt))
        S = np.ascontiguousarray(f.sigma if r else np.zeros(1))
        rc = fn(h.raw, a.ctypes.data, m, n, m, U.ctypes.data, m,
                                               S.ctypes.data, Vt.ctypes.data, max(r, 1), r,
                                               ctypes.byref(out), _lib.PTR_HOST)
    _lib.raise_for(rc, h.raw)
    return out.value


def _spectral_error(a, f: TruncatedFactorization, handle) -> float:
    import torch

    dev = a.device if _is_torch_cuda(a) else torch.device("cuda", (handle.device if handle else 0))
    A = a if _is_torch_cuda(a) else torch.from_numpy(
        np.asarray(a, dtype=_np_dtype(_is_complex(a)))).to(dev)
    m, n = A.shape
    R = A.clone()
    if f.rank():
        U = torch.as_tensor(np.asarray(f.left) if not hasattr(f.left, "to") else f.left,
                            dtype=A.dtype).to(dev)
        S = torch.as_tensor(np.asarray(f.sigma) if not hasattr(f.sigma, "to") else f.sigma,
                            dtype=torch.float64).to(dev)
        Vt = torch.as_tensor(np.asarray(f.right_adj) if not hasattr(f.right_adj, "to")
                             else f.right_adj, dtype=A.dtype).to(dev)
        R = R - (U * S[None, :]) @ Vt
    if float(torch.linalg.norm(R)) == 0.0:
        return 0.0
    g = tsvd(R, 1, handle)
    return float(g.sigma[0]) if g.rank() else 0.0
