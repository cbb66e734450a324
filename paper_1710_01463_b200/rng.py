"""Seed derivation and the counter-based Gaussian stream (rlftn rng.hpp).

``mix64`` / ``derive_seed`` / ``seed_tag`` are exact integer restatements
(rng.hpp:11-29); they are pure host-side bookkeeping.  ``CounterRng.fill_gaussian``
produces the reference's Box-Muller normals on the GPU through the C ABI
(rng.hpp:62-64 -> rsvd_fill_gaussian_f64).
"""
from __future__ import annotations

import ctypes

from . import _lib

MASK64 = (1 << 64) - 1


def mix64(z: int) -> int:
    """SplitMix64 finalizer (rng.hpp:11-15)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def derive_seed(seed: int, tag: int) -> int:
    """seed XOR mix64(tag) (rng.hpp:20-22; docs/seeds.md)."""
    return (seed & MASK64) ^ mix64(tag)


class seed_tag:  # noqa: N801 - mirrors rlftn::seed_tag (rng.hpp:25-29)
    initial_state = 1
    rsvd_stream = 2
    bench_matrix = 3


class CounterRng:
    """rlftn::CounterRng (rng.hpp:34-78).  Integer words on the host; Gaussian
    fills on the device."""

    GOLDEN = 0x9E3779B97F4A7C15

    def __init__(self, seed: int):
        self.key = seed & MASK64
        self.counter = 0

    def next(self) -> int:
        self.counter += 1
        return mix64((self.key + self.counter * self.GOLDEN) & MASK64)

    def uniform(self) -> float:
        """((w >> 11) + 1) * 2^-53 in (0, 1] (rng.hpp:46)."""
        return float((self.next() >> 11) + 1) * (1.0 / 9007199254740992.0)

    def fill_gaussian(self, out, count: int | None = None, handle: _lib.Handle | None = None):
        """Fill ``out`` (a float64 torch CUDA tensor or numpy array) with the
        first ``count`` normals of this stream, computed on the GPU.  A
        complex128 ``out`` takes the complex fill (rng.hpp:66-71): entry t =
        (normal 2t+1, normal 2t) / sqrt 2 as the reference's g++ build orders
        the two unsequenced calls."""
        h = handle or _lib.default_handle()
        lib = _lib.load()
        try:
            import torch  # noqa: F401
            is_torch = hasattr(out, "data_ptr") and getattr(out, "is_cuda", False)
        except ImportError:  # pragma: no cover
            is_torch = False
        if is_torch:
            n = out.numel() if count is None else count
            cplx = bool(out.is_complex())
            if out.dtype.itemsize != (16 if cplx else 8) or not out.is_contiguous():
                raise _lib.InvalidArgument("fill_gaussian: need a contiguous float64 tensor")
            fn = lib.rsvd_fill_gaussian_z128 if cplx else lib.rsvd_fill_gaussian_f64
            lib.rsvd_set_stream(h.raw, ctypes.c_void_p(_lib.torch_stream_ptr()))
            rc = fn(h.raw, self.key, out.data_ptr(), n, _lib.PTR_DEVICE)
            lib.rsvd_set_stream(h.raw, None)
        else:
            import numpy as np
            cplx = out.dtype == np.complex128
            if (out.dtype != np.float64 and not cplx) or (
                    not out.flags.c_contiguous and not out.flags.f_contiguous):
                raise _lib.InvalidArgument("fill_gaussian: need a contiguous float64 array")
            n = out.size if count is None else count
            fn = lib.rsvd_fill_gaussian_z128 if cplx else lib.rsvd_fill_gaussian_f64
            rc = fn(h.raw, self.key, out.ctypes.data, n, _lib.PTR_HOST)
        _lib.raise_for(rc, h.raw)
        return out
