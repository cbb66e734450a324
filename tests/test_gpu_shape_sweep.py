"""Seeded sweep over shapes, ranks, sample widths, power counts, batch sizes
and scalar types against the oracle (restated reference): catches layout /
tiling corner cases (odd leading dimensions, 96-multiple sample widths,
l = min(m, n), k = l, wide and tall inputs) that the named configs miss.
Same tolerances as tests/test_gpu_rsvd.py (north_star)."""
import numpy as np
import pytest

from tests.helpers import (isometry_err, matrix_with_spectrum, rel_sigma_err, spectrum_family,
                           zmatrix_with_spectrum)

pytestmark = pytest.mark.gpu


def _cases(n=28, seed=20261020):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        m = int(rng.integers(3, 420))
        nn = int(rng.integers(3, 420))
        p = min(m, nn)
        ell = int(rng.integers(1, p + 1))
        k = int(rng.integers(1, ell + 1))
        q = int(rng.integers(0, 4))
        batch = int(rng.choice([1, 1, 2, 5]))
        cplx = bool(rng.integers(0, 2))
        out.append((i, m, nn, k, ell, q, batch, cplx))
    # hand-picked corners
    out += [(100, 97, 193, 96, 96, 2, 3, False), (101, 193, 97, 96, 96, 1, 1, True),
            (102, 288, 301, 200, 288, 1, 2, False), (103, 65, 64, 64, 64, 0, 1, True),
            (104, 1, 50, 1, 1, 2, 2, False), (105, 50, 1, 1, 1, 2, 1, True)]
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"c{c[0]}-{c[1]}x{c[2]}-k{c[3]}-l{c[4]}-q{c[5]}-b{c[6]}-{'z' if c[7] else 'd'}")
def test_sweep_rsvd_against_oracle(cuda, oracle_mod, case):
    from paper_1710_01463_b200 import RsvdParams, rsvd_batched

    i, m, n, k, ell, q, batch, cplx = case
    p = min(m, n)
    sig = np.exp(-np.arange(p) / max(2.0, p / 8.0))
    mk = zmatrix_with_spectrum if cplx else matrix_with_spectrum
    mats = [mk(oracle_mod, 1000 * i + b, m, n, sig) for b in range(batch)]
    seeds = [17 * i + b for b in range(batch)]
    f = rsvd_batched(np.stack(mats), RsvdParams(k, ell, q, 0), seeds)
    ref_fn = oracle_mod.zrsvd if cplx else oracle_mod.rsvd
    for b in range(batch):
        U, S, Vt, dw = ref_fn(mats[b], k, ell, q, seeds[b])
        fb = f.item(b)
        assert fb.rank() == len(S), (case, b)
        assert rel_sigma_err(fb.sigma, S) < 1e-10, (case, b, rel_sigma_err(fb.sigma, S))
        left = np.asarray(fb.left)
        assert isometry_err(left) < 1e-12, (case, b)
        rec = (left * np.asarray(fb.sigma)[None, :]) @ np.asarray(fb.right_adj)
        e_gpu = np.linalg.norm(mats[b] - rec)
        e_ref = np.linalg.norm(mats[b] - (U * S[None, :]) @ Vt)
        scale = np.linalg.norm(mats[b])
        if e_ref > 1e-12 * scale:  # a real truncation error: 1e-10 relative (north_star)
            assert abs(e_gpu - e_ref) <= 1e-10 * e_ref, (case, b, e_gpu, e_ref)
        else:  # exact reconstruction: roundoff on both sides (test_factorize.cpp:105-120 bound)
            assert e_gpu <= 1e-10 * scale, (case, b, e_gpu, e_ref)
        assert fb.discarded_weight == pytest.approx(dw, rel=1e-8, abs=1e-24 * scale ** 2), (case, b)


@pytest.mark.parametrize("case", [(i, m, n, c) for i, (m, n, c) in enumerate(
    [(31, 77, False), (77, 31, True), (129, 128, False), (200, 3, True), (5, 5, False),
     (256, 255, True), (97, 193, False)])], ids=lambda c: f"t{c[0]}-{c[1]}x{c[2]}-{'z' if c[3] else 'd'}")
def test_sweep_tsvd_against_oracle(cuda, oracle_mod, case):
    from paper_1710_01463_b200 import tsvd

    i, m, n, cplx = case
    p = min(m, n)
    sig = spectrum_family(2, p)
    a = (zmatrix_with_spectrum if cplx else matrix_with_spectrum)(oracle_mod, 77 + i, m, n, sig)
    for chi in sorted({1, max(1, p // 2), p}):
        f = tsvd(a, chi)
        _, S, _, dw = (oracle_mod.ztsvd if cplx else oracle_mod.tsvd)(a, chi)
        assert f.rank() == len(S)
        # 0.8^k runs down to ~1e-25: like gesdd the small values are accurate to
        # O(u ||A||) absolute; 1e-10 relative where that is meaningful.
        sv = np.asarray(f.sigma)
        assert np.all(np.abs(sv - S) <= 1e-10 * S + 1e-12 * S[0]), (case, chi)
        assert f.discarded_weight == pytest.approx(dw, rel=1e-9, abs=1e-22 * S[0] ** 2)
