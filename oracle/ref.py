"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front-end of oracle/_ref/librlftn_ref.so: the REFERENCE's own
proj/src/factorize.cpp, lapack.cpp and blocks.cpp compiled unmodified (against
the Eigen/LAPACKE shims in oracle/refshim/, recipe oracle/Makefile `ref`).
This is the parity anchor: the restatement (oracle/oracle.py) and the CUDA
engine are both checked against it.  Same call shapes as oracle.py.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module; the product package never does.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "librlftn_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB} not built (needs /root/reference; make -C oracle ref)")
        L = ctypes.CDLL(LIB)
        i64, u64, vp, dbl, ci = (ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p,
                                 ctypes.c_double, ctypes.c_int)
        pi64, pdbl = ctypes.POINTER(i64), ctypes.POINTER(dbl)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_set_threads.argtypes = [ci]
        L.ref_get_threads.restype = ci
        L.ref_mix64.restype = u64
        L.ref_mix64.argtypes = [u64]
        L.ref_derive_seed.restype = u64
        L.ref_derive_seed.argtypes = [u64, u64]
        L.ref_fill_gaussian.argtypes = [u64, vp, i64]
        L.ref_zfill_gaussian.argtypes = [u64, vp, i64]
        for s in "dz":
            getattr(L, f"ref_rsvd_{s}").argtypes = [vp, i64, i64, i64, i64, i64, ci, u64, vp, vp,
                                                    vp, i64, pi64, pdbl]
            getattr(L, f"ref_tsvd_{s}").argtypes = [vp, i64, i64, i64, i64, vp, vp, vp, i64, pi64,
                                                    pdbl]
            getattr(L, f"ref_randomized_range_{s}").argtypes = [vp, i64, i64, i64, i64, ci, u64,
                                                                vp]
            getattr(L, f"ref_reconstruction_error_{s}").argtypes = [vp, i64, i64, vp, vp, vp, i64,
                                                                    i64, ci, pdbl]
            getattr(L, f"ref_block_factorize_{s}").argtypes = [i64, i64, vp, vp, vp, vp, i64, ci, i64,
                                                               ci, i64, ci, u64, i64, pdbl,
                                                               ctypes.POINTER(ci)]
            getattr(L, f"ref_block_sector_{s}").argtypes = [i64, vp, vp, vp, pi64, pdbl]
            getattr(L, f"ref_matrix_with_spectrum_{s}").argtypes = [i64, i64, vp, i64, u64, vp]
        L.ref_orthonormal_columns_d.argtypes = [vp, i64, i64, vp]
        L.ref_singular_values_d.argtypes = [vp, i64, i64, vp]
        L.ref_sector_request.argtypes = [ci, i64, i64, vp, i64, vp]
        _lib = L
    return _lib


class RefInvalid(ValueError):
    """std::invalid_argument thrown by the reference."""


class RefNumerical(RuntimeError):
    """std::runtime_error thrown by the reference (LAPACK failure)."""


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().ref_last_error().decode()
    raise (RefInvalid if rc == 1 else RefNumerical)(msg)


def _arr(a, z: bool) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.complex128 if z else np.float64))


def _dt(z: bool):
    return np.complex128 if z else np.float64


def _is_z(a) -> bool:
    return np.iscomplexobj(a)


M64 = (1 << 64) - 1


def set_threads(n: int) -> None:
    lib().ref_set_threads(int(n))


def get_threads() -> int:
    return lib().ref_get_threads()


def mix64(z: int) -> int:
    return lib().ref_mix64(z & M64)


def derive_seed(s: int, t: int) -> int:
    return lib().ref_derive_seed(s & M64, t & M64)


def fill_gaussian(seed: int, n: int, complex_: bool = False) -> np.ndarray:
    out = np.zeros(n, dtype=_dt(complex_))
    fn = lib().ref_zfill_gaussian if complex_ else lib().ref_fill_gaussian
    fn(seed & M64, out.ctypes.data, n)
    return out


def rsvd(a, rank: int, oversample: int, power: int, seed: int):
    """rlftn::rsvd (factorize.cpp:76-95) -> (U m x r, S r, Vt r x n, discarded_weight)."""
    z = _is_z(a)
    a = _arr(a, z)
    m, n = a.shape
    k = max(rank, 1)
    U = np.zeros((m, k), dtype=_dt(z), order="F")
    S = np.zeros(k)
    Vt = np.zeros((k, n), dtype=_dt(z), order="F")
    r, dw = ctypes.c_int64(0), ctypes.c_double(0.0)
    fn = lib().ref_rsvd_z if z else lib().ref_rsvd_d
    _check(fn(a.ctypes.data if a.size else None, m, n, max(m, 1), rank, oversample, power,
              seed & M64, U.ctypes.data, S.ctypes.data, Vt.ctypes.data, k, ctypes.byref(r),
              ctypes.byref(dw)))
    rr = r.value
    return U[:, :rr].copy(order="F"), S[:rr].copy(), Vt[:rr, :].copy(order="F"), dw.value


def tsvd(a, chi: int):
    """rlftn::tsvd (factorize.cpp:42-50)."""
    z = _is_z(a)
    a = _arr(a, z)
    m, n = a.shape
    kk = max(min(max(chi, 1), min(m, n)) if m and n else 1, 1)
    U = np.zeros((m, kk), dtype=_dt(z), order="F")
    S = np.zeros(kk)
    Vt = np.zeros((kk, n), dtype=_dt(z), order="F")
    r, dw = ctypes.c_int64(0), ctypes.c_double(0.0)
    fn = lib().ref_tsvd_z if z else lib().ref_tsvd_d
    _check(fn(a.ctypes.data if a.size else None, m, n, max(m, 1), chi, U.ctypes.data,
              S.ctypes.data, Vt.ctypes.data, kk, ctypes.byref(r), ctypes.byref(dw)))
    rr = r.value
    return U[:, :rr].copy(order="F"), S[:rr].copy(), Vt[:rr, :].copy(order="F"), dw.value


def randomized_range(a, ell: int, power: int, seed: int) -> np.ndarray:
    """rlftn::randomized_range (factorize.cpp:52-74)."""
    z = _is_z(a)
    a = _arr(a, z)
    m, n = a.shape
    Q = np.zeros((m, max(ell, 1)), dtype=_dt(z), order="F")
    fn = lib().ref_randomized_range_z if z else lib().ref_randomized_range_d
    _check(fn(a.ctypes.data if a.size else None, m, n, max(m, 1), ell, power, seed & M64,
              Q.ctypes.data))
    return Q[:, :ell]


def reconstruction_error(a, U, S, Vt, spectral: bool = False) -> float:
    """rlftn::reconstruction_error (factorize.cpp:97-104)."""
    z = _is_z(a) or _is_z(U)
    a = _arr(a, z)
    m, n = a.shape
    r = len(S)
    U = _arr(U, z) if r else np.zeros((m, 1), dtype=_dt(z), order="F")
    Vt = _arr(Vt, z) if r else np.zeros((1, n), dtype=_dt(z), order="F")
    S = np.ascontiguousarray(S, dtype=np.float64) if r else np.zeros(1)
    out = ctypes.c_double(0.0)
    fn = lib().ref_reconstruction_error_z if z else lib().ref_reconstruction_error_d
    _check(fn(a.ctypes.data, m, n, U.ctypes.data, S.ctypes.data, Vt.ctypes.data, max(r, 1), r,
              int(spectral), ctypes.byref(out)))
    return out.value


def orthonormal_columns(a) -> np.ndarray:
    """rlftn::lapack::orthonormal_columns (lapack.cpp:211-215)."""
    a = _arr(a, False)
    m, n = a.shape
    Q = np.zeros((m, min(m, n)), order="F")
    _check(lib().ref_orthonormal_columns_d(a.ctypes.data, m, n, Q.ctypes.data))
    return Q


def singular_values(a) -> np.ndarray:
    a = _arr(a, False)
    m, n = a.shape
    s = np.zeros(min(m, n))
    _check(lib().ref_singular_values_d(a.ctypes.data, m, n, s.ctypes.data))
    return s


def sector_request(maximal: bool, chi: int, slack: int, dims) -> np.ndarray:
    d = np.asarray(dims, dtype=np.int64)
    out = np.zeros(len(d), dtype=np.int64)
    _check(lib().ref_sector_request(int(maximal), chi, slack, d.ctypes.data, len(d),
                                    out.ctypes.data))
    return out


def block_factorize(blocks, charges, chi: int, maximal: bool = False, slack: int = -1,
                    kind: str = "tsvd", oversample: int = 0, power: int = 4, seed: int = 0,
                    min_dim: int = 32):
    """rlftn::block_factorize (blocks.cpp:38-118).  Same return shape as
    oracle.block_factorize: ([(U, S, Vt, dw) per sector], total_dw, exact)."""
    z = any(_is_z(b) for b in blocks)
    bl = [_arr(b, z) for b in blocks]
    ns = len(bl)
    ch = np.asarray(charges, dtype=np.int64)
    rows = np.asarray([b.shape[0] for b in bl], dtype=np.int64)
    cols = np.asarray([b.shape[1] for b in bl], dtype=np.int64)
    P = ctypes.c_void_p * max(ns, 1)
    bp = P(*[b.ctypes.data if b.size else None for b in bl])
    tot, ex = ctypes.c_double(0.0), ctypes.c_int(0)
    L = lib()
    fn = L.ref_block_factorize_z if z else L.ref_block_factorize_d
    sec = L.ref_block_sector_z if z else L.ref_block_sector_d
    _check(fn(ns, len(ch), ch.ctypes.data, bp, rows.ctypes.data, cols.ctypes.data, chi, int(maximal),
              slack, 1 if kind == "rsvd" else 0, oversample, power, seed & M64, min_dim,
              ctypes.byref(tot), ctypes.byref(ex)))
    out = []
    for s in range(ns):
        r, dw = ctypes.c_int64(0), ctypes.c_double(0.0)
        _check(sec(s, None, None, None, ctypes.byref(r), ctypes.byref(dw)))
        k, m, n = r.value, int(rows[s]), int(cols[s])
        U = np.zeros((m, max(k, 1)), dtype=_dt(z), order="F")
        S = np.zeros(max(k, 1))
        Vt = np.zeros((max(k, 1), n), dtype=_dt(z), order="F")
        _check(sec(s, U.ctypes.data, S.ctypes.data, Vt.ctypes.data, ctypes.byref(r),
                   ctypes.byref(dw)))
        out.append((U[:, :k].copy(order="F"), S[:k].copy(), Vt[:k, :].copy(order="F"),
                    dw.value))
    return out, tot.value, bool(ex.value)


def matrix_with_spectrum(rows: int, cols: int, sigma, gen_seed: int, complex_: bool = False):
    """The reference tests' input generator (tests/helpers.hpp:47-88):
    std::mt19937_64(gen_seed) Gaussians -> Householder isometries U, V ->
    U diag(sigma) V^H."""
    s = np.ascontiguousarray(sigma, dtype=np.float64)
    out = np.zeros((rows, cols), dtype=_dt(complex_), order="F")
    fn = lib().ref_matrix_with_spectrum_z if complex_ else lib().ref_matrix_with_spectrum_d
    _check(fn(rows, cols, s.ctypes.data, len(s), gen_seed & M64, out.ctypes.data))
    return out


def spectrum_family(family: int, n: int) -> np.ndarray:
    """tests/helpers.hpp:91-103: 0 -> 2^-k, 1 -> (k+1)^-3, 2 -> 0.8^k."""
    k = np.arange(n, dtype=np.float64)
    if family == 0:
        return np.power(2.0, -k)
    if family == 1:
        return 1.0 / ((k + 1) * (k + 1) * (k + 1))
    return np.power(0.8, k)
