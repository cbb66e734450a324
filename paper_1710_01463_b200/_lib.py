"""ctypes binding of librsvd_b200.so (the C ABI declared in include/rsvd_c.h).

The product path has no CPU fallback: if the CUDA library is missing or fails
to load, every entry point raises.  Build it with ``python -c "import
__graft_entry__ as g; g.build()"`` (or ``make -C paper_1710_01463_b200/csrc``).
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librsvd_b200.so")

RSVD_OK = 0
RSVD_ERR_INVALID = 1
RSVD_ERR_NUMERICAL = 2
RSVD_ERR_CUDA = 3
PTR_HOST = 0
PTR_DEVICE = 1

# Every symbol include/rsvd_c.h declares, with its ctypes signature.
_c_i64 = ctypes.c_int64
_c_u64 = ctypes.c_uint64
_c_int = ctypes.c_int
_c_vp = ctypes.c_void_p
_c_dp = ctypes.c_void_p  # double* passed as raw addresses (host or device)

SIGNATURES = {
    "rsvd_create": (_c_int, [ctypes.POINTER(_c_vp), _c_int]),
    "rsvd_destroy": (_c_int, [_c_vp]),
    "rsvd_last_error": (ctypes.c_char_p, [_c_vp]),
    "rsvd_set_stream": (_c_int, [_c_vp, _c_vp]),
    "rsvd_trim": (_c_int, [_c_vp]),
    "rsvd_version": (ctypes.c_char_p, []),
    "rsvd_mix64": (_c_u64, [_c_u64]),
    "rsvd_derive_seed": (_c_u64, [_c_u64, _c_u64]),
    "rsvd_fill_gaussian_f64": (_c_int, [_c_vp, _c_u64, _c_dp, _c_i64, _c_int]),
    "rsvd_f64": (
        _c_int,
        [_c_vp, _c_dp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_int, _c_u64, _c_dp, _c_i64,
         _c_dp, _c_dp, _c_i64, ctypes.POINTER(_c_i64), ctypes.POINTER(ctypes.c_double), _c_int],
    ),
    "rsvd_f64_batched": (
        _c_int,
        [_c_vp, _c_i64, _c_dp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_int,
         ctypes.POINTER(_c_u64), _c_dp, _c_i64, _c_i64, _c_dp, _c_i64, _c_dp, _c_i64, _c_i64,
         ctypes.POINTER(_c_i64), ctypes.POINTER(ctypes.c_double), _c_int],
    ),
    "rsvd_randomized_range_f64": (
        _c_int, [_c_vp, _c_dp, _c_i64, _c_i64, _c_i64, _c_i64, _c_int, _c_u64, _c_dp, _c_i64, _c_int]
    ),
    "rsvd_validate_params": (
        _c_int, [_c_i64, _c_i64, _c_i64, _c_i64, _c_int, ctypes.POINTER(_c_i64), ctypes.c_char_p,
                 _c_i64]
    ),
    "rsvd_tsvd_f64": (
        _c_int,
        [_c_vp, _c_dp, _c_i64, _c_i64, _c_i64, _c_i64, _c_dp, _c_i64, _c_dp, _c_dp, _c_i64,
         ctypes.POINTER(_c_i64), ctypes.POINTER(ctypes.c_double), _c_int],
    ),
    "rsvd_tsvd_f64_batched": (
        _c_int,
        [_c_vp, _c_i64, _c_dp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_dp, _c_i64, _c_i64,
         _c_dp, _c_i64, _c_dp, _c_i64, _c_i64, ctypes.POINTER(_c_i64),
         ctypes.POINTER(ctypes.c_double), _c_int],
    ),
    "rsvd_group_create": (_c_int, [ctypes.POINTER(_c_vp), _c_int]),
    "rsvd_group_destroy": (_c_int, [_c_vp]),
    "rsvd_attach_group": (_c_int, [_c_vp, _c_vp, _c_int]),
    "rsvd_nccl_unique_id": (_c_int, [ctypes.c_char_p]),
    "rsvd_attach_nccl": (_c_int, [_c_vp, _c_int, _c_int, ctypes.c_char_p]),
    "rsvd_detach": (_c_int, [_c_vp]),
    "rsvd_f64_rowsharded": (
        _c_int,
        [_c_vp, _c_dp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_int, _c_u64,
         _c_dp, _c_i64, _c_dp, _c_dp, _c_i64, ctypes.POINTER(_c_i64),
         ctypes.POINTER(ctypes.c_double), _c_int],
    ),
    "rsvd_kernel_launches": (_c_u64, []),
    "rsvd_profile_enable": (_c_int, [_c_vp, _c_int]),
    "rsvd_profile_read": (_c_int, [_c_vp, ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(_c_i64), _c_int]),
    "rsvd_profile_stage_name": (ctypes.c_char_p, [_c_int]),
    "rsvd_last_jacobi_sweeps": (_c_int, [_c_vp]),
    "rsvd_last_gemm_path": (_c_int, [_c_vp]),
    "rsvd_testing_dgemm": (
        _c_int,
        [_c_vp, _c_int, _c_i64, _c_i64, _c_i64, _c_dp, _c_i64, _c_i64, _c_dp, _c_i64, _c_i64, _c_dp,
         _c_i64, _c_i64, _c_i64],
    ),
    "rsvd_testing_ozaki_gemm": (
        _c_int,
        [_c_vp, _c_int, _c_i64, _c_i64, _c_i64, _c_dp, _c_i64, _c_i64, _c_dp, _c_i64, _c_i64, _c_dp,
         _c_i64, _c_i64, _c_i64],
    ),
    "rsvd_block_factorize_f64": (
        _c_int,
        [_c_vp, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_i64, _c_int, _c_i64, _c_int, _c_i64,
         _c_int, _c_u64, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_dp, _c_vp,
         _c_int],
    ),
    "rsvd_combine_blocks": (_c_int, [_c_vp, _c_int, _c_i64, _c_vp, _c_i64, _c_vp]),
    "rsvd_grouped_gemm": (_c_int, [_c_vp, _c_int, _c_i64, _c_vp]),
    "rsvd_block_sqnorms": (_c_int, [_c_vp, _c_int, _c_i64, _c_vp, _c_vp, _c_dp]),
    "rsvd_qr_f64": (
        _c_int,
        [_c_vp, _c_i64, _c_dp, _c_i64, _c_i64, _c_i64, _c_i64, _c_dp, _c_i64, _c_i64, _c_dp,
         _c_i64, _c_i64, _c_int],
    ),
    "rsvd_reconstruction_error_f64": (
        _c_int,
        [_c_vp, _c_dp, _c_i64, _c_i64, _c_i64, _c_dp, _c_i64, _c_dp, _c_dp, _c_i64, _c_i64,
         ctypes.POINTER(ctypes.c_double), _c_int],
    ),
}
# Complex instantiation: same signatures as the double entry points.
for _z, _d in (("rsvd_z128", "rsvd_f64"), ("rsvd_z128_batched", "rsvd_f64_batched"),
               ("rsvd_tsvd_z128", "rsvd_tsvd_f64"),
               ("rsvd_tsvd_z128_batched", "rsvd_tsvd_f64_batched"),
               ("rsvd_randomized_range_z128", "rsvd_randomized_range_f64"),
               ("rsvd_reconstruction_error_z128", "rsvd_reconstruction_error_f64"),
               ("rsvd_fill_gaussian_z128", "rsvd_fill_gaussian_f64")):
    SIGNATURES[_z] = SIGNATURES[_d]

# Table rows of rsvd_combine_blocks / rsvd_grouped_gemm / rsvd_block_sqnorms
# (include/rsvd_c.h): all fields 8 bytes wide, so the packed numpy layout is
# the C struct layout.
BLOCK_TERM = np.dtype([("src", "u8"), ("rs", "i8"), ("cs", "i8"), ("row_scale", "u8"),
                       ("col_scale", "u8"), ("coef_re", "f8"), ("coef_im", "f8")])
BLOCK_JOB = np.dtype([("dst", "u8"), ("rs", "i8"), ("cs", "i8"), ("rows", "i8"), ("cols", "i8"),
                      ("term_begin", "i8"), ("term_count", "i8")])
GEMM_JOB = np.dtype([("A", "u8"), ("a_rs", "i8"), ("a_cs", "i8"), ("B", "u8"), ("b_rs", "i8"),
                     ("b_cs", "i8"), ("C", "u8"), ("c_rs", "i8"), ("c_cs", "i8"), ("M", "i8"),
                     ("N", "i8"), ("K", "i8")])

_lib = None
_lock = threading.Lock()


class LibraryMissing(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    """Load librsvd_b200.so (once).  Raises LibraryMissing when absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not built: run `make -C paper_1710_01463_b200/csrc` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class InvalidArgument(ValueError):
    """Mirrors the reference's std::invalid_argument."""


class NumericalError(RuntimeError):
    """Mirrors the reference's std::runtime_error from LAPACK failures."""


class DeviceError(RuntimeError):
    """CUDA / driver failure inside the engine."""


def raise_for(rc: int, handle) -> None:
    if rc == RSVD_OK:
        return
    msg = load().rsvd_last_error(handle)
    msg = msg.decode() if msg else ""
    if rc == RSVD_ERR_INVALID:
        raise InvalidArgument(msg)
    if rc == RSVD_ERR_NUMERICAL:
        raise NumericalError(msg)
    raise DeviceError(msg or f"rsvd error code {rc}")


class Handle:
    """Owns one rsvd_handle (device workspace + stream).  One per thread."""

    def __init__(self, device: int = 0):
        lib = load()
        h = ctypes.c_void_p()
        rc = lib.rsvd_create(ctypes.byref(h), int(device))
        if rc != RSVD_OK:
            msg = lib.rsvd_last_error(h) if h else b"rsvd_create failed"
            if h:
                lib.rsvd_destroy(h)
            raise DeviceError((msg or b"").decode())
        self._h = h
        self.device = device

    @property
    def raw(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            load().rsvd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_handles = threading.local()


def default_handle(device: int = 0) -> Handle:
    d = getattr(_handles, "by_device", None)
    if d is None:
        d = _handles.by_device = {}
    h = d.get(device)
    if h is None:
        h = d[device] = Handle(device)
    return h


def validate_params(m: int, n: int, rank: int, oversample: int, power: int) -> int:
    """Host-only argument check (rsvd_validate_params); returns l or raises
    InvalidArgument with the reference's message."""
    lib = load()
    ell = ctypes.c_int64(0)
    buf = ctypes.create_string_buffer(256)
    rc = lib.rsvd_validate_params(m, n, rank, oversample, power, ctypes.byref(ell), buf, 256)
    if rc != RSVD_OK:
        raise InvalidArgument(buf.value.decode())
    return ell.value


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the legacy default stream


def torch_stream_ptr() -> int:
    """torch's current stream as a cudaStream_t for rsvd_set_stream.  torch
    reports its default stream as 0; NULL means "the handle's own stream" to
    the engine, so the legacy default stream is passed explicitly."""
    import torch

    s = torch.cuda.current_stream().cuda_stream
    return s if s else CUDA_STREAM_LEGACY


class on_torch_stream:
    """Context manager: run engine calls of `handle` on torch's current stream."""

    def __init__(self, handle: "Handle"):
        self.h = handle

    def __enter__(self):
        load().rsvd_set_stream(self.h.raw, ctypes.c_void_p(torch_stream_ptr()))
        return self.h

    def __exit__(self, *exc):
        load().rsvd_set_stream(self.h.raw, None)
        return False


def kernel_launches() -> int:
    return int(load().rsvd_kernel_launches())


def profile_enable(handle: Handle, on: bool = True) -> None:
    raise_for(load().rsvd_profile_enable(handle.raw, int(on)), handle.raw)


def profile_read(handle: Handle) -> dict:
    lib = load()
    n = 16
    ms = (ctypes.c_double * n)()
    calls = (ctypes.c_int64 * n)()
    k = lib.rsvd_profile_read(handle.raw, ms, calls, n)
    return {lib.rsvd_profile_stage_name(i).decode(): (ms[i], int(calls[i])) for i in range(k)}


def last_jacobi_sweeps(handle: Handle) -> int:
    return int(load().rsvd_last_jacobi_sweeps(handle.raw))


def last_gemm_path(handle: Handle) -> str:
    """'ozaki' (emulated FP64 on the INT8 tensor cores) or 'dmma'."""
    return "ozaki" if load().rsvd_last_gemm_path(handle.raw) == 1 else "dmma"
