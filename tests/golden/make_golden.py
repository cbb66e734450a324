"""Regenerate the committed golden fixtures (run in the build container, where
/root/reference exists).  TEST INFRASTRUCTURE ONLY.

  rng_kat.json    : first 64 SplitMix64 words and 257 Box-Muller normals of
                    six seeds, produced by the REFERENCE's own rng.hpp
                    (oracle/_ref/rng_kat, compiled from
                    /root/reference/proj/include/rlftn/rng.hpp).
  rsvd_small.npz  : small rsvd/tsvd known-answer cases computed by the
                    REFERENCE's own factorize.cpp/lapack.cpp compiled unmodified
                    (oracle/_ref/librlftn_ref.so, 1 BLAS thread as lapack.cpp:225)
                    on CounterRng inputs; the restatement must agree bitwise.
  zrsvd_small.npz : the same cases for the complex instantiation
                    (rsvd/tsvd<std::complex<double>>, complex CounterRng inputs).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from oracle import ref  # noqa: E402


def spectrum_family(family, n):
    k = np.arange(n, dtype=np.float64)
    if family == 0:
        return 2.0 ** -k
    if family == 1:
        return 1.0 / (k + 1) ** 3
    return 0.8 ** k


def matrix_with_spectrum(seed, rows, cols, sigma):
    r = len(sigma)
    u = oracle.haar(oracle.derive_seed(seed, 1), rows, r)
    v = oracle.haar(oracle.derive_seed(seed, 2), cols, r)
    return np.asfortranarray((u * np.asarray(sigma)[None, :]) @ v.T)


# (name, rows, cols, spectrum-or-None(gaussian), rank, oversample, power, seed)
CASES = [
    ("geom_50x30", 50, 30, ("fam", 0, 30), 10, 20, 4, 123),
    ("gauss_40x25", 40, 25, None, 8, 16, 4, 11),
    ("exact3_60x40", 60, 40, ("list", [5.0 / (1 + i) for i in range(3)]), 10, 20, 4, 5),
    ("exact7_60x40", 60, 40, ("list", [5.0 / (1 + i) for i in range(7)]), 10, 20, 4, 5),
    ("gauss_48x32", 48, 32, None, 6, 12, 4, 77),
    ("wide_30x70", 30, 70, ("fam", 2, 30), 8, 16, 2, 99),
    ("odd_37x53", 37, 53, ("fam", 1, 37), 5, 13, 1, 2024),
    ("q0_64x64", 64, 64, ("fam", 2, 64), 12, 20, 0, 7),
    ("exp_200x160", 200, 160, ("exp", 32.0, 160), 32, 42, 2, 31337),
]


def build_case(i, rows, cols, spec):
    seed = oracle.derive_seed(0x601DE5, i)
    if spec is None:
        return oracle.gaussian_matrix(seed, rows, cols)
    if spec[0] == "fam":
        s = spectrum_family(spec[1], spec[2])
    elif spec[0] == "exp":
        s = np.exp(-np.arange(spec[2]) / spec[1])
    else:
        s = np.asarray(spec[1])
    return matrix_with_spectrum(seed, rows, cols, s)


def zbuild_case(i, rows, cols, spec):
    """Complex counterpart of build_case: Haar complex isometries (complex
    CounterRng fill + zgeqrf/zungqr, phase-fixed) or a complex Gaussian."""
    seed = oracle.derive_seed(0x2601DE5, i)
    if spec is None:
        return oracle.zgaussian_matrix(seed, rows, cols)
    if spec[0] == "fam":
        s = spectrum_family(spec[1], spec[2])
    elif spec[0] == "exp":
        s = np.exp(-np.arange(spec[2]) / spec[1])
    else:
        s = np.asarray(spec[1])
    r = len(s)
    u = oracle.zhaar(oracle.derive_seed(seed, 1), rows, r)
    v = oracle.zhaar(oracle.derive_seed(seed, 2), cols, r)
    return np.asfortranarray((u * s[None, :]) @ v.conj().T)


def _same(x, y, name):
    assert all(np.array_equal(p, q) for p, q in zip(x[:3], y[:3])) and x[3] == y[3], name


def main():
    oracle.build()
    kat = oracle.reference_rng_kat(64, 257)
    if kat is None:
        raise SystemExit("oracle/_ref/rng_kat missing: needs /root/reference to build")
    with open(os.path.join(HERE, "rng_kat.json"), "w") as f:
        json.dump(kat, f, indent=1)
    oracle.set_threads(1)
    ref.set_threads(1)
    out = {}
    for i, (name, rows, cols, spec, k, ell, q, seed) in enumerate(CASES):
        a = build_case(i, rows, cols, spec)
        U, S, Vt, dw = ref.rsvd(a, k, ell, q, seed)
        Ut, St, Vtt, dwt = ref.tsvd(a, k)
        _same(oracle.rsvd(a, k, ell, q, seed), (U, S, Vt, dw), name)
        out[f"{name}/a"] = a
        out[f"{name}/params"] = np.array([k, ell, q, seed], dtype=np.uint64)
        out[f"{name}/U"] = U
        out[f"{name}/S"] = S
        out[f"{name}/Vt"] = Vt
        out[f"{name}/dw"] = np.array([dw])
        out[f"{name}/S_tsvd"] = St
        out[f"{name}/dw_tsvd"] = np.array([dwt])
        out[f"{name}/omega"] = oracle.gaussian_matrix(seed, cols, ell)
    np.savez_compressed(os.path.join(HERE, "rsvd_small.npz"), **out)
    print("wrote", len(CASES), "cases")
    zout = {}
    for i, (name, rows, cols, spec, k, ell, q, seed) in enumerate(CASES):
        a = zbuild_case(i, rows, cols, spec)
        U, S, Vt, dw = ref.rsvd(a, k, ell, q, seed)
        Ut, St, Vtt, dwt = ref.tsvd(a, k)
        _same(oracle.zrsvd(a, k, ell, q, seed), (U, S, Vt, dw), name)
        zout[f"{name}/a"] = a
        zout[f"{name}/params"] = np.array([k, ell, q, seed], dtype=np.uint64)
        zout[f"{name}/U"] = U
        zout[f"{name}/S"] = S
        zout[f"{name}/Vt"] = Vt
        zout[f"{name}/dw"] = np.array([dw])
        zout[f"{name}/S_tsvd"] = St
        zout[f"{name}/dw_tsvd"] = np.array([dwt])
        zout[f"{name}/omega"] = oracle.zgaussian_matrix(seed, cols, ell)
    np.savez_compressed(os.path.join(HERE, "zrsvd_small.npz"), **zout)
    print("wrote", len(CASES), "complex cases")


if __name__ == "__main__":
    main()
