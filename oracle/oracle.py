"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front-end of oracle/liboracle.so, the CPU restatement of the reference
rsvd path (see rsvd_oracle.cpp for the file:line map).  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / reference arm may import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_KAT = os.path.join(HERE, "_ref", "rng_kat")

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        i64, u64, vp, dbl = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_double
        L.oracle_last_error.restype = ctypes.c_char_p
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_get_threads.restype = ctypes.c_int
        L.oracle_mix64.restype = u64
        L.oracle_mix64.argtypes = [u64]
        L.oracle_derive_seed.restype = u64
        L.oracle_derive_seed.argtypes = [u64, u64]
        L.oracle_rng_words.argtypes = [u64, vp, i64]
        L.oracle_fill_gaussian.argtypes = [u64, vp, i64]
        L.oracle_rsvd.argtypes = [vp, i64, i64, i64, i64, i64, ctypes.c_int, u64, vp, vp, vp, vp,
                                  i64, ctypes.POINTER(i64), ctypes.POINTER(dbl)]
        L.oracle_tsvd.argtypes = [vp, i64, i64, i64, i64, vp, vp, vp, i64, ctypes.POINTER(i64),
                                  ctypes.POINTER(dbl)]
        L.oracle_randomized_range.argtypes = [vp, i64, i64, i64, i64, ctypes.c_int, u64, vp, vp]
        L.oracle_reconstruction_error.argtypes = [vp, i64, i64, i64, vp, vp, vp, i64, i64,
                                                  ctypes.c_int, ctypes.POINTER(dbl)]
        L.oracle_orthonormal_columns.argtypes = [vp, i64, i64, vp]
        L.oracle_singular_values.argtypes = [vp, i64, i64, vp]
        L.oracle_sector_request.argtypes = [ctypes.c_int, i64, i64, vp, i64, vp]
        L.oracle_block_factorize.argtypes = [i64, vp, vp, vp, vp, i64, ctypes.c_int, i64,
                                             ctypes.c_int, i64, ctypes.c_int, u64, i64, vp, vp, vp,
                                             vp, vp, ctypes.POINTER(dbl),
                                             ctypes.POINTER(ctypes.c_int)]
        L.oracle_zfill_gaussian.argtypes = [u64, vp, i64]
        L.oracle_zrsvd.argtypes = [vp, i64, i64, i64, i64, i64, ctypes.c_int, u64, vp, vp, vp, vp,
                                   i64, ctypes.POINTER(i64), ctypes.POINTER(dbl)]
        L.oracle_ztsvd.argtypes = [vp, i64, i64, i64, i64, vp, vp, vp, i64, ctypes.POINTER(i64),
                                   ctypes.POINTER(dbl)]
        L.oracle_zrandomized_range.argtypes = [vp, i64, i64, i64, i64, ctypes.c_int, u64, vp, vp]
        L.oracle_zreconstruction_error.argtypes = [vp, i64, i64, i64, vp, vp, vp, i64, i64,
                                                   ctypes.c_int, ctypes.POINTER(dbl)]
        L.oracle_zorthonormal_columns.argtypes = [vp, i64, i64, vp]
        L.oracle_zsingular_values.argtypes = [vp, i64, i64, vp]
        _lib = L
    return _lib


class OracleInvalid(ValueError):
    pass


class OracleNumerical(RuntimeError):
    pass


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().oracle_last_error().decode()
    if rc == 1:
        raise OracleInvalid(msg)
    raise OracleNumerical(msg)


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return lib().oracle_get_threads()


def mix64(z: int) -> int:
    return lib().oracle_mix64(z)


def derive_seed(s: int, t: int) -> int:
    return lib().oracle_derive_seed(s, t)


def rng_words(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    lib().oracle_rng_words(seed, out.ctypes.data, n)
    return out


def fill_gaussian(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n)
    lib().oracle_fill_gaussian(seed, out.ctypes.data, n)
    return out


def gaussian_matrix(seed: int, rows: int, cols: int) -> np.ndarray:
    """rows x cols column-major fill, exactly as randomized_range fills Omega."""
    return fill_gaussian(seed, rows * cols).reshape(cols, rows).T.copy(order="F")


def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def rsvd(a, rank: int, oversample: int, power: int, seed: int, omega=None):
    """rlftn::rsvd -> (U m x r, S r, Vt r x n, discarded_weight)."""
    a = _f(a)
    m, n = a.shape
    k = max(rank, 1)
    U = np.zeros((m, k), order="F")
    S = np.zeros(k)
    Vt = np.zeros((k, n), order="F")
    r = ctypes.c_int64(0)
    dw = ctypes.c_double(0.0)
    om = None if omega is None else _f(omega)
    _check(lib().oracle_rsvd(a.ctypes.data if a.size else None, m, n, max(m, 1), rank, oversample,
                             power, seed & ((1 << 64) - 1),
                             None if om is None else om.ctypes.data, U.ctypes.data, S.ctypes.data,
                             Vt.ctypes.data, k, ctypes.byref(r), ctypes.byref(dw)))
    rr = r.value
    return U[:, :rr].copy(order="F"), S[:rr].copy(), Vt[:rr, :].copy(order="F"), dw.value


def tsvd(a, chi: int):
    a = _f(a)
    m, n = a.shape
    k = max(chi, 1)
    kk = min(k, min(m, n)) if m and n else 1
    U = np.zeros((m, max(kk, 1)), order="F")
    S = np.zeros(max(kk, 1))
    Vt = np.zeros((max(kk, 1), n), order="F")
    r = ctypes.c_int64(0)
    dw = ctypes.c_double(0.0)
    _check(lib().oracle_tsvd(a.ctypes.data if a.size else None, m, n, max(m, 1), chi,
                             U.ctypes.data, S.ctypes.data, Vt.ctypes.data, max(kk, 1),
                             ctypes.byref(r), ctypes.byref(dw)))
    rr = r.value
    return U[:, :rr].copy(order="F"), S[:rr].copy(), Vt[:rr, :].copy(order="F"), dw.value


def randomized_range(a, ell: int, power: int, seed: int, omega=None) -> np.ndarray:
    a = _f(a)
    m, n = a.shape
    Q = np.zeros((m, max(ell, 1)), order="F")
    om = None if omega is None else _f(omega)
    _check(lib().oracle_randomized_range(a.ctypes.data if a.size else None, m, n, max(m, 1), ell,
                                         power, seed & ((1 << 64) - 1),
                                         None if om is None else om.ctypes.data, Q.ctypes.data))
    return Q[:, :ell]


def reconstruction_error(a, U, S, Vt, spectral: bool = False) -> float:
    a = _f(a)
    m, n = a.shape
    r = len(S)
    U = _f(U) if r else np.zeros((m, 1), order="F")
    Vt = _f(Vt) if r else np.zeros((1, n), order="F")
    S = np.ascontiguousarray(S, dtype=np.float64) if r else np.zeros(1)
    out = ctypes.c_double(0.0)
    _check(lib().oracle_reconstruction_error(a.ctypes.data, m, n, m, U.ctypes.data, S.ctypes.data,
                                             Vt.ctypes.data, max(r, 1), r, int(spectral),
                                             ctypes.byref(out)))
    return out.value


def orthonormal_columns(a) -> np.ndarray:
    a = _f(a)
    m, n = a.shape
    Q = np.zeros((m, min(m, n)), order="F")
    _check(lib().oracle_orthonormal_columns(a.ctypes.data, m, n, Q.ctypes.data))
    return Q


def singular_values(a) -> np.ndarray:
    a = _f(a)
    m, n = a.shape
    s = np.zeros(min(m, n))
    _check(lib().oracle_singular_values(a.ctypes.data, m, n, s.ctypes.data))
    return s


def sector_request(maximal: bool, chi: int, slack: int, dims) -> np.ndarray:
    d = np.asarray(dims, dtype=np.int64)
    out = np.zeros(len(d), dtype=np.int64)
    _check(lib().oracle_sector_request(int(maximal), chi, slack, d.ctypes.data, len(d),
                                       out.ctypes.data))
    return out


def block_factorize(blocks, charges, chi: int, maximal: bool = False, slack: int = -1,
                    kind: str = "tsvd", oversample: int = 0, power: int = 4, seed: int = 0,
                    min_dim: int = 32):
    """rlftn::block_factorize (blocks.cpp:38-118).  Returns
    (factors [(U, S, Vt, dw) per sector], total_dw, exact)."""
    bl = [_f(b) for b in blocks]
    ns = len(bl)
    ch = np.asarray(charges, dtype=np.int64)
    rows = np.asarray([b.shape[0] for b in bl], dtype=np.int64)
    cols = np.asarray([b.shape[1] for b in bl], dtype=np.int64)
    us = [np.zeros(max(int(r) * int(min(r, c)), 1)) for r, c in zip(rows, cols)]
    vts = [np.zeros(max(int(c) * int(min(r, c)), 1)) for r, c in zip(rows, cols)]
    P = ctypes.c_void_p * max(ns, 1)
    bp = P(*[b.ctypes.data if b.size else None for b in bl])
    up = P(*[u.ctypes.data for u in us])
    vp_ = P(*[v.ctypes.data for v in vts])
    ranks = np.zeros(max(ns, 1), dtype=np.int64)
    dws = np.zeros(max(ns, 1))
    sig = np.zeros(max(int(np.minimum(rows, cols).sum()), 1))
    tot = ctypes.c_double(0.0)
    ex = ctypes.c_int(0)
    _check(lib().oracle_block_factorize(ns, ch.ctypes.data, bp, rows.ctypes.data, cols.ctypes.data,
                                        chi, int(maximal), slack, 1 if kind == "rsvd" else 0,
                                        oversample, power, seed & ((1 << 64) - 1), min_dim,
                                        ranks.ctypes.data, dws.ctypes.data, sig.ctypes.data, up,
                                        vp_, ctypes.byref(tot), ctypes.byref(ex)))
    out, off = [], 0
    for s in range(ns):
        k, m, n = int(ranks[s]), int(rows[s]), int(cols[s])
        U = us[s][:m * k].reshape(k, m).T.copy(order="F")
        Vt = vts[s][:k * n].reshape(n, k).T.copy(order="F")
        out.append((U, sig[off:off + k].copy(), Vt, float(dws[s])))
        off += k
    return out, tot.value, bool(ex.value)


def haar(seed: int, rows: int, cols: int) -> np.ndarray:
    """Haar-distributed orthonormal columns: Householder Q of a CounterRng
    Gaussian, columns sign-fixed by diag(R) = diag(Q^T G)."""
    g = gaussian_matrix(seed, rows, cols)
    q = orthonormal_columns(g)
    d = np.sign(np.einsum("ij,ij->j", q, g))
    d[d == 0] = 1.0
    return np.asfortranarray(q * d[None, :])


def reference_rng_kat(nwords: int = 64, nnormal: int = 257):
    """Run the reference's own CounterRng (oracle/_ref/rng_kat, compiled from
    /root/reference/proj/include/rlftn/rng.hpp) if it was built here."""
    if not os.path.exists(REF_KAT):
        return None
    out = subprocess.run([REF_KAT, str(nwords), str(nnormal)], check=True, capture_output=True,
                         text=True).stdout
    return json.loads(out)


# ------------------------------------------------------------------ complex
# The reference's std::complex<double> instantiation of the same path
# (factorize.cpp:106-118; lapack.cpp:73-110, 154-177): zgemm, zgeqrf+zungqr,
# zgesdd -> zgesvd, complex CounterRng fill (rng.hpp:66-71).


def _z(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.complex128))


def zfill_gaussian(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.complex128)
    lib().oracle_zfill_gaussian(seed & ((1 << 64) - 1), out.ctypes.data, n)
    return out


def zgaussian_matrix(seed: int, rows: int, cols: int) -> np.ndarray:
    """Complex Omega exactly as randomized_range<complex> fills it (column-major)."""
    return zfill_gaussian(seed, rows * cols).reshape(cols, rows).T.copy(order="F")


def zrsvd(a, rank: int, oversample: int, power: int, seed: int, omega=None):
    """rlftn::rsvd<complex<double>> -> (U m x r, S r, Vt r x n, discarded_weight)."""
    a = _z(a)
    m, n = a.shape
    k = max(rank, 1)
    U = np.zeros((m, k), dtype=np.complex128, order="F")
    S = np.zeros(k)
    Vt = np.zeros((k, n), dtype=np.complex128, order="F")
    r = ctypes.c_int64(0)
    dw = ctypes.c_double(0.0)
    om = None if omega is None else _z(omega)
    _check(lib().oracle_zrsvd(a.ctypes.data if a.size else None, m, n, max(m, 1), rank, oversample,
                              power, seed & ((1 << 64) - 1),
                              None if om is None else om.ctypes.data, U.ctypes.data, S.ctypes.data,
                              Vt.ctypes.data, k, ctypes.byref(r), ctypes.byref(dw)))
    rr = r.value
    return U[:, :rr].copy(order="F"), S[:rr].copy(), Vt[:rr, :].copy(order="F"), dw.value


def ztsvd(a, chi: int):
    a = _z(a)
    m, n = a.shape
    kk = max(min(max(chi, 1), min(m, n)) if m and n else 1, 1)
    U = np.zeros((m, kk), dtype=np.complex128, order="F")
    S = np.zeros(kk)
    Vt = np.zeros((kk, n), dtype=np.complex128, order="F")
    r = ctypes.c_int64(0)
    dw = ctypes.c_double(0.0)
    _check(lib().oracle_ztsvd(a.ctypes.data if a.size else None, m, n, max(m, 1), chi,
                              U.ctypes.data, S.ctypes.data, Vt.ctypes.data, kk, ctypes.byref(r),
                              ctypes.byref(dw)))
    rr = r.value
    return U[:, :rr].copy(order="F"), S[:rr].copy(), Vt[:rr, :].copy(order="F"), dw.value


def zrandomized_range(a, ell: int, power: int, seed: int, omega=None) -> np.ndarray:
    a = _z(a)
    m, n = a.shape
    Q = np.zeros((m, max(ell, 1)), dtype=np.complex128, order="F")
    om = None if omega is None else _z(omega)
    _check(lib().oracle_zrandomized_range(a.ctypes.data if a.size else None, m, n, max(m, 1), ell,
                                          power, seed & ((1 << 64) - 1),
                                          None if om is None else om.ctypes.data, Q.ctypes.data))
    return Q[:, :ell]


def zreconstruction_error(a, U, S, Vt, spectral: bool = False) -> float:
    a = _z(a)
    m, n = a.shape
    r = len(S)
    U = _z(U) if r else np.zeros((m, 1), dtype=np.complex128, order="F")
    Vt = _z(Vt) if r else np.zeros((1, n), dtype=np.complex128, order="F")
    S = np.ascontiguousarray(S, dtype=np.float64) if r else np.zeros(1)
    out = ctypes.c_double(0.0)
    _check(lib().oracle_zreconstruction_error(a.ctypes.data, m, n, m, U.ctypes.data, S.ctypes.data,
                                              Vt.ctypes.data, max(r, 1), r, int(spectral),
                                              ctypes.byref(out)))
    return out.value


def zorthonormal_columns(a) -> np.ndarray:
    a = _z(a)
    m, n = a.shape
    Q = np.zeros((m, min(m, n)), dtype=np.complex128, order="F")
    _check(lib().oracle_zorthonormal_columns(a.ctypes.data, m, n, Q.ctypes.data))
    return Q


def zsingular_values(a) -> np.ndarray:
    a = _z(a)
    m, n = a.shape
    s = np.zeros(min(m, n))
    _check(lib().oracle_zsingular_values(a.ctypes.data, m, n, s.ctypes.data))
    return s


def zhaar(seed: int, rows: int, cols: int) -> np.ndarray:
    """Haar-distributed complex isometry: Householder Q of a complex CounterRng
    Gaussian, columns phase-fixed so that diag(R) = diag(Q^H G) is real > 0."""
    g = zgaussian_matrix(seed, rows, cols)
    q = zorthonormal_columns(g)
    d = np.einsum("ij,ij->j", q.conj(), g)
    ph = np.where(np.abs(d) > 0, d / np.where(np.abs(d) > 0, np.abs(d), 1.0), 1.0)
    return np.asfortranarray(q * ph[None, :])
