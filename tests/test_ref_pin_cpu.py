"""Pins the restatement oracle (oracle/liboracle.so) to the REFERENCE ITSELF.

oracle/_ref/librlftn_ref.so is the reference's own proj/src/factorize.cpp,
lapack.cpp and blocks.cpp compiled unmodified (oracle/Makefile `ref`, Eigen and
LAPACKE shims in oracle/refshim/).  Both libraries drive the same OpenBLAS, so
the restatement must reproduce the reference BIT FOR BIT: factors, singular
values, discarded weight, error messages -- on the committed golden cases, on
the block/sector dispatch, and on BASELINE's C1 and a C2 item at full size.
The committed golden fixtures are checked against the reference build too.
"""
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KAT = json.load(open(os.path.join(ROOT, "tests", "golden", "rng_kat.json")))


@pytest.fixture
def one_thread(ref_mod, oracle_mod):
    """The reference protocol pins BLAS to one thread (lapack.cpp:225,
    main.cpp:7); the golden fixtures were produced that way, and a 1-thread
    OpenBLAS result does not depend on the host's core count."""
    rt, ot = ref_mod.get_threads(), oracle_mod.get_threads()
    ref_mod.set_threads(1)
    oracle_mod.set_threads(1)
    yield
    ref_mod.set_threads(rt)
    oracle_mod.set_threads(ot)


def _bitwise(x, y, label):
    for name, a, b in zip(("U", "S", "Vt"), x[:3], y[:3]):
        assert a.shape == b.shape, (label, name, a.shape, b.shape)
        assert np.array_equal(a, b), (label, name, float(np.max(np.abs(a - b))))
    assert x[3] == y[3], (label, "dw", x[3], y[3])


def _cases(golden):
    names = sorted({k.split("/")[0] for k in golden.keys()})
    for nm in names:
        p = golden[f"{nm}/params"]
        yield nm, np.asfortranarray(golden[f"{nm}/a"]), [int(v) for v in p]


def test_reference_rng_is_the_kat(ref_mod):
    for s in KAT["streams"]:
        seed = int(s["seed"], 16)
        normals = ref_mod.fill_gaussian(seed, len(s["normals"]))
        assert [f"{int(x):016x}" for x in normals.view(np.uint64)] == s["normals"]
    for t, h in enumerate(KAT["mix64"]):
        assert f"{ref_mod.mix64(t):016x}" == h


def test_golden_fixtures_are_reference_outputs(ref_mod, golden_small, one_thread):
    """tests/golden/rsvd_small.npz holds exactly what the reference computes."""
    for nm, a, (k, ell, q, seed) in _cases(golden_small):
        U, S, Vt, dw = ref_mod.rsvd(a, k, ell, q, seed)
        assert np.array_equal(S, golden_small[f"{nm}/S"]), nm
        assert np.array_equal(U, golden_small[f"{nm}/U"]), nm
        assert np.array_equal(Vt, golden_small[f"{nm}/Vt"]), nm
        assert dw == float(golden_small[f"{nm}/dw"][0]), nm
        _, St, _, dwt = ref_mod.tsvd(a, k)
        assert np.array_equal(St, golden_small[f"{nm}/S_tsvd"]), nm
        assert dwt == float(golden_small[f"{nm}/dw_tsvd"][0]), nm


def test_restatement_bitwise_on_golden_cases(ref_mod, oracle_mod, golden_small):
    for nm, a, (k, ell, q, seed) in _cases(golden_small):
        _bitwise(oracle_mod.rsvd(a, k, ell, q, seed), ref_mod.rsvd(a, k, ell, q, seed), nm)
        _bitwise(oracle_mod.tsvd(a, k), ref_mod.tsvd(a, k), nm + "/tsvd")
        assert np.array_equal(oracle_mod.randomized_range(a, ell, q, seed),
                              ref_mod.randomized_range(a, ell, q, seed)), nm
        U, S, Vt, _ = ref_mod.rsvd(a, k, ell, q, seed)
        for spectral in (False, True):
            assert (oracle_mod.reconstruction_error(a, U, S, Vt, spectral)
                    == ref_mod.reconstruction_error(a, U, S, Vt, spectral)), nm


def test_restatement_bitwise_complex(ref_mod, oracle_mod, one_thread):
    z = np.load(os.path.join(ROOT, "tests", "golden", "zrsvd_small.npz"))
    names = sorted({k.split("/")[0] for k in z.keys()})
    assert names
    for nm in names:
        a = np.asfortranarray(z[f"{nm}/a"])
        k, ell, q, seed = [int(v) for v in z[f"{nm}/params"]]
        R = ref_mod.rsvd(a, k, ell, q, seed)
        _bitwise(oracle_mod.zrsvd(a, k, ell, q, seed), R, nm)
        _bitwise(oracle_mod.ztsvd(a, k), ref_mod.tsvd(a, k), nm + "/tsvd")
        assert np.array_equal(R[1], z[f"{nm}/S"]), nm
        assert np.array_equal(R[0], z[f"{nm}/U"]), nm
        assert R[3] == float(z[f"{nm}/dw"][0]), nm


@pytest.mark.parametrize("args", [
    # (m, n, rank, oversample, power) -- test_factorize.cpp:175-184 error cases
    (10, 8, 0, 0, 4), (10, 8, 4, 3, 4), (10, 8, 4, 9, 4), (10, 8, 4, 6, -1), (0, 8, 4, 6, 1),
])
def test_error_messages_match_reference(ref_mod, oracle_mod, args):
    m, n, k, ell, q = args
    a = np.ones((m, n))
    with pytest.raises(ref_mod.RefInvalid) as er:
        ref_mod.rsvd(a, k, ell, q, 1)
    with pytest.raises(oracle_mod.OracleInvalid) as eo:
        oracle_mod.rsvd(a, k, ell, q, 1)
    assert str(er.value) == str(eo.value)


def test_tsvd_error_messages_match_reference(ref_mod, oracle_mod):
    for a, chi in ((np.zeros((0, 3)), 1), (np.ones((3, 3)), 0)):
        with pytest.raises(ref_mod.RefInvalid) as er:
            ref_mod.tsvd(a, chi)
        with pytest.raises(oracle_mod.OracleInvalid) as eo:
            oracle_mod.tsvd(a, chi)
        assert str(er.value) == str(eo.value)


@pytest.mark.parametrize("chi,slack,maximal,dims", [
    (10, -1, False, [5, 7, 9]), (64, 3, False, [40, 10]), (7, -1, True, [3, 12, 7]),
    (100, -1, False, [64, 64, 64, 64]),
])
def test_sector_request_matches_reference(ref_mod, oracle_mod, chi, slack, maximal, dims):
    assert np.array_equal(ref_mod.sector_request(maximal, chi, slack, dims),
                          oracle_mod.sector_request(maximal, chi, slack, dims))


def _sectors(seed, shapes, decay=6.0):
    rng = np.random.default_rng(seed)
    out = []
    for (m, n) in shapes:
        g = rng.standard_normal((m, n)) * np.exp(-np.arange(n) / decay)[None, :]
        out.append(np.asfortranarray(g))
    return out


@pytest.mark.parametrize("kind,shapes,charges,chi,over", [
    ("rsvd", [(40, 36), (48, 40)], [0, 1], 16, 0),
    ("rsvd", [(64, 40), (20, 30), (33, 50)], [3, 0, 1], 24, 20),   # mixed rsvd / tsvd (< 32)
    ("tsvd", [(12, 9), (7, 15)], [1, 0], 10, 0),
    ("rsvd", [(36, 36), (36, 36)], [5, 2], 40, 500),                # oversample clipped
    ("rsvd", [(40, 40), (0, 5)], [0, 1], 8, 4),                     # empty sector, lifted ell
])
def test_block_factorize_bitwise(ref_mod, oracle_mod, kind, shapes, charges, chi, over):
    bl = _sectors(sum(charges) + chi, shapes)
    R = ref_mod.block_factorize(bl, charges, chi, kind=kind, oversample=over, power=2, seed=99)
    O = oracle_mod.block_factorize(bl, charges, chi, kind=kind, oversample=over, power=2, seed=99)
    assert R[1] == O[1] and R[2] == O[2]
    for s, (fr, fo) in enumerate(zip(R[0], O[0])):
        _bitwise(fo, fr, f"sector {s}")


def test_block_factorize_errors_match_reference(ref_mod):
    """The product's host-side checks (blocks.py) raise the reference's
    messages (blocks.cpp:42-46), checked against the reference build."""
    from paper_1710_01463_b200 import blocks as B
    from paper_1710_01463_b200 import InvalidArgument

    a = np.ones((4, 4))
    for bl, ch in (([a, a], [0, 0]), ([a], [0, 1]), ([], [])):
        with pytest.raises(ref_mod.RefInvalid) as er:
            ref_mod.block_factorize(bl, ch, 2)
        with pytest.raises(InvalidArgument) as ep:
            B.block_factorize(B.BlockDiagMatrix(ch, bl), 2, B.SectorRankRequest(),
                              B.BlockMethod.deterministic())
        assert str(er.value) == str(ep.value)


def test_reference_input_generator_has_the_prescribed_spectrum(ref_mod):
    """matrix_with_spectrum (helpers.hpp:78-88, mt19937_64 draws) really has
    the requested singular values -- the A1/A2 inputs."""
    s = ref_mod.spectrum_family(2, 40)
    a = ref_mod.matrix_with_spectrum(60, 40, s, 9000)
    assert np.max(np.abs(np.linalg.svd(a, compute_uv=False) - s)) < 1e-13
    z = ref_mod.matrix_with_spectrum(30, 20, s[:5], 77000, complex_=True)
    assert np.iscomplexobj(z)
    sv = np.linalg.svd(z, compute_uv=False)
    assert np.max(np.abs(sv[:5] - s[:5])) < 1e-13 and np.max(sv[5:]) < 1e-13


def test_restatement_bitwise_c1_full_size(ref_mod, oracle_mod):
    """BASELINE C1 (1024^2, k=64, l=74, q=2) on a host-built input."""
    rng = np.random.default_rng(1)
    n = 1024
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = np.asfortranarray((u * np.exp(-np.arange(n) / 32.0)) @ v.T)
    seed = ref_mod.derive_seed(ref_mod.derive_seed(1, 2), 0)
    _bitwise(oracle_mod.rsvd(a, 64, 74, 2, seed), ref_mod.rsvd(a, 64, 74, 2, seed), "C1")


def test_restatement_bitwise_c2_item(ref_mod, oracle_mod):
    rng = np.random.default_rng(2)
    n = 256
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = (np.arange(n) + 1.0) ** -1.5
    a = np.asfortranarray((u * (s / np.linalg.norm(s))) @ v.T)
    _bitwise(oracle_mod.rsvd(a, 128, 138, 2, 7), ref_mod.rsvd(a, 128, 138, 2, 7), "C2")
