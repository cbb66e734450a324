"""Pins the complex instantiation of the CPU oracle (rsvd<complex<double>>,
factorize.cpp:106-118) before it checks the GPU: the complex CounterRng fill
bit-exact against the reference-built KAT (rng.hpp:66-71 as compiled by g++),
and the reference's own complex factorization tests
(proj/tests/test_factorize.cpp:105-131) restated on CounterRng inputs."""
import json
import os

import numpy as np
import pytest

from tests.helpers import isometry_err, spectrum_family, subspace_distance, zmatrix_with_spectrum

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KAT = json.load(open(os.path.join(ROOT, "tests", "golden", "rng_kat.json")))


def test_complex_fill_matches_reference_kat(oracle_mod):
    for s in KAT["streams"]:
        seed = int(s["seed"], 16)
        want = s["complex"]
        got = oracle_mod.zfill_gaussian(seed, len(want) // 2).view(np.uint64)
        assert [f"{int(x):016x}" for x in got] == want


def test_complex_fill_is_the_real_stream_swapped_and_scaled(oracle_mod):
    # g++ evaluates the imaginary argument first: entry t = (n[2t+1], n[2t]) / sqrt 2.
    n = oracle_mod.fill_gaussian(42, 40)
    z = oracle_mod.zfill_gaussian(42, 20)
    inv = 0.70710678118654752440
    assert np.array_equal(z.real, n[1::2] * inv)
    assert np.array_equal(z.imag, n[0::2] * inv)


@pytest.mark.parametrize("r", [3, 7])
def test_complex_exact_rank_reconstructs(oracle_mod, r):
    # test_factorize.cpp:105-120 (complex half)
    sigma = [5.0 / (1.0 + k) for k in range(r)]
    a = zmatrix_with_spectrum(oracle_mod, 17 + r, 60, 40, sigma)
    U, S, Vt, dw = oracle_mod.zrsvd(a, 10, 20, 4, 5)
    assert oracle_mod.zreconstruction_error(a, U, S, Vt) <= 1e-10 * np.linalg.norm(a)
    assert len(S) <= 10
    assert isometry_err(U) < 1e-12


def test_complex_tsvd_and_rsvd_agree(oracle_mod):
    # test_factorize.cpp:122-131
    sigma = spectrum_family(2, 24)
    a = zmatrix_with_spectrum(oracle_mod, 29, 36, 24, sigma)
    Ut, St, Vtt, dwt = oracle_mod.ztsvd(a, 8)
    U, S, Vt, dw = oracle_mod.zrsvd(a, 8, 16, 4, 99)
    assert np.all(np.abs(St - sigma[:8]) <= 1e-11 * sigma[:8])
    assert np.all(np.abs(S - St) / St < 1e-9)
    assert subspace_distance(U[:, :4], Ut[:, :4]) < 1e-8
    assert 0 < dw <= dwt * (1 + 1e-8)


def test_complex_rsvd_is_deterministic_and_seed_dependent(oracle_mod):
    a = zmatrix_with_spectrum(oracle_mod, 5, 30, 20, spectrum_family(0, 20))
    f1 = oracle_mod.zrsvd(a, 5, 10, 2, 7)
    f2 = oracle_mod.zrsvd(a, 5, 10, 2, 7)
    assert np.array_equal(f1[0], f2[0]) and np.array_equal(f1[1], f2[1])
    om = oracle_mod.zgaussian_matrix(7, 20, 10)
    f3 = oracle_mod.zrsvd(a, 5, 10, 2, 0, omega=om)
    assert np.array_equal(f1[0], f3[0])


def test_complex_invalid_arguments(oracle_mod):
    a = np.ones((4, 3), dtype=np.complex128)
    with pytest.raises(oracle_mod.OracleInvalid, match="rank must be >= 1"):
        oracle_mod.zrsvd(a, 0, 0, 1, 0)
    with pytest.raises(oracle_mod.OracleInvalid, match="oversample must be >= rank"):
        oracle_mod.zrsvd(a, 2, 1, 1, 0)
    with pytest.raises(oracle_mod.OracleInvalid, match="need 1 <= ell"):
        oracle_mod.zrsvd(a, 2, 4, 1, 0)


def test_complex_oracle_reproduces_committed_golden(oracle_mod):
    """tests/golden/zrsvd_small.npz (made by tests/golden/make_golden.py) is
    reproduced by the oracle here: the fixture and the restatement agree."""
    g = np.load(os.path.join(ROOT, "tests", "golden", "zrsvd_small.npz"))
    names = sorted({k.split("/")[0] for k in g.files})
    assert len(names) == 9
    for name in names:
        a = g[f"{name}/a"]
        k, ell, q, seed = (int(x) for x in g[f"{name}/params"])
        assert np.array_equal(oracle_mod.zgaussian_matrix(seed, a.shape[1], ell), g[f"{name}/omega"])
        U, S, Vt, dw = oracle_mod.zrsvd(a, k, ell, q, seed)
        np.testing.assert_allclose(S, g[f"{name}/S"], rtol=1e-12)
        assert dw == pytest.approx(float(g[f"{name}/dw"][0]), rel=1e-9, abs=1e-30)
        St = oracle_mod.ztsvd(a, k)[1]
        np.testing.assert_allclose(St, g[f"{name}/S_tsvd"], rtol=1e-12, atol=1e-15)
