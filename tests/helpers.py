"""Shared test utilities (test infrastructure; may use the oracle)."""
from __future__ import annotations

import numpy as np


def spectrum_family(family: int, n: int) -> np.ndarray:
    """helpers.hpp spectrum_family: 0 -> 2^-k, 1 -> (k+1)^-3, 2 -> 0.8^k."""
    k = np.arange(n, dtype=np.float64)
    if family == 0:
        return 2.0 ** -k
    if family == 1:
        return 1.0 / (k + 1) ** 3
    return 0.8 ** k


def matrix_with_spectrum(oracle, seed: int, rows: int, cols: int, sigma) -> np.ndarray:
    """A = U diag(sigma) V^T with Haar isometries (helpers.hpp matrix_with_spectrum,
    regenerated from CounterRng + the oracle's Householder QR)."""
    sigma = np.asarray(sigma, dtype=np.float64)
    r = len(sigma)
    u = oracle.haar(oracle.derive_seed(seed, 1), rows, r)
    v = oracle.haar(oracle.derive_seed(seed, 2), cols, r)
    return np.asfortranarray((u * sigma[None, :]) @ v.T)


def rel_sigma_err(s, s_ref) -> float:
    s = np.asarray(s)
    s_ref = np.asarray(s_ref)
    k = min(len(s), len(s_ref))
    if k == 0:
        return 0.0
    return float(np.max(np.abs(s[:k] - s_ref[:k]) / np.abs(s_ref[:k])))


def subspace_distance(U, U_ref) -> float:
    """||U U^T - U_ref U_ref^T||_2 for orthonormal U, U_ref (same column count),
    computed as ||U - U_ref (U_ref^T U)||_2 (stable below 1e-8)."""
    U = np.asarray(U)
    U_ref = np.asarray(U_ref)
    if U.shape[1] == 0:
        return 0.0
    d = U - U_ref @ (U_ref.conj().T @ U)
    return float(np.linalg.norm(d, 2))


def isometry_err(U) -> float:
    U = np.asarray(U)
    r = U.shape[1]
    return float(np.max(np.abs(U.conj().T @ U - np.eye(r)))) if r else 0.0


def zmatrix_with_spectrum(oracle, seed: int, rows: int, cols: int, sigma) -> np.ndarray:
    """Complex A = U diag(sigma) V^H with Haar complex isometries
    (helpers.hpp:78-88 matrix_with_spectrum<Complex>, regenerated from the
    complex CounterRng fill + the oracle's zgeqrf/zungqr)."""
    sigma = np.asarray(sigma, dtype=np.float64)
    r = len(sigma)
    u = oracle.zhaar(oracle.derive_seed(seed, 1), rows, r)
    v = oracle.zhaar(oracle.derive_seed(seed, 2), cols, r)
    return np.asfortranarray((u * sigma[None, :]) @ v.conj().T)


def ulp_distance(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    ai = np.asarray(a, dtype=np.float64).view(np.int64)
    bi = np.asarray(b, dtype=np.float64).view(np.int64)
    # map to a monotonic integer line
    ai = np.where(ai < 0, np.int64(-(2**63)) - ai, ai)
    bi = np.where(bi < 0, np.int64(-(2**63)) - bi, bi)
    return np.abs(ai - bi)
