"""GPU tsvd and block_factorize against the oracle.

tsvd restates test_factorize.cpp:33-83,199-207 on the GPU path; block_factorize
restates test_blocks.cpp:82-279 and checks every sector against the oracle's
block_factorize (same sector requests, sample widths and per-charge seeds).
Tolerances as test_gpu_rsvd.py (BASELINE.json north_star)."""
import numpy as np
import pytest

from tests.helpers import (isometry_err, matrix_with_spectrum, rel_sigma_err, spectrum_family,
                           subspace_distance)

pytestmark = pytest.mark.gpu

SIG_TOL = 1e-10
ISO_TOL = 1e-12


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


# ------------------------------------------------------------------ tsvd ---

def test_tsvd_diagonal(cuda):  # test_factorize.cpp:33-55
    from paper_1710_01463_b200 import reconstruction_error, tsvd

    a = np.diag([3.0, 2.0, 1.0])
    f = tsvd(a, 2)
    assert f.discarded_exact
    np.testing.assert_allclose(f.sigma, [3.0, 2.0], rtol=1e-14)
    assert f.discarded_weight == pytest.approx(1.0, rel=1e-14)
    assert reconstruction_error(a, f) == pytest.approx(1.0, rel=1e-12)
    f = tsvd(a, 1)
    assert f.discarded_weight == pytest.approx(5.0, rel=1e-14)


def test_tsvd_geometric_spectrum(cuda, oracle_mod):  # test_factorize.cpp:57-71
    from paper_1710_01463_b200 import reconstruction_error, tsvd

    sigma = spectrum_family(0, 30)
    a = matrix_with_spectrum(oracle_mod, 42, 50, 30, sigma)
    f = tsvd(a, 10)
    assert f.rank() == 10
    assert rel_sigma_err(f.sigma, sigma[:10]) < 1e-12
    tail = float(np.sum(sigma[10:] ** 2))
    assert f.discarded_weight == pytest.approx(tail, rel=1e-10)
    err = reconstruction_error(a, f)
    assert err * err == pytest.approx(tail, rel=1e-9)


@pytest.mark.parametrize("m,n,chi", [(40, 25, 8), (25, 40, 8), (64, 64, 64), (200, 96, 30),
                                     (96, 300, 50), (17, 5, 9), (1, 7, 3), (7, 1, 3),
                                     (576, 600, 100)])
def test_tsvd_vs_oracle(cuda, oracle_mod, m, n, chi, ref_mod):
    from paper_1710_01463_b200 import tsvd

    a = oracle_mod.gaussian_matrix(1000 + m + 7 * n, m, n)
    f = tsvd(a, chi)
    U, S, Vt, dw = ref_mod.tsvd(a, chi)
    assert f.rank() == len(S)
    assert rel_sigma_err(f.sigma, S) < SIG_TOL
    assert isometry_err(f.left) < ISO_TOL and isometry_err(f.right_adj.T) < ISO_TOL
    assert f.discarded_weight == pytest.approx(dw, rel=1e-9, abs=1e-28)
    # Gaussian spectra are gapped: the leading subspaces must agree.
    j = f.rank() - 1 if f.rank() < min(m, n) else f.rank()
    if j > 0:
        assert subspace_distance(f.left[:, :j], U[:, :j]) < 1e-8
        assert subspace_distance(f.right_adj[:j].T, Vt[:j].T) < 1e-8


def test_tsvd_zero_and_rank_deficient(cuda, oracle_mod):  # test_factorize.cpp:199-207
    from paper_1710_01463_b200 import tsvd

    f = tsvd(np.zeros((12, 9)), 4)
    assert f.rank() == 0 and f.discarded_weight == 0.0
    sig = np.array([5.0, 3.0, 1.0])
    a = matrix_with_spectrum(oracle_mod, 5, 30, 20, sig)
    f = tsvd(a, 10)
    assert f.rank() == 3
    np.testing.assert_allclose(f.sigma, sig, rtol=1e-12)


def test_tsvd_invalid(cuda):  # factorize.cpp:44-45
    from paper_1710_01463_b200 import InvalidArgument, tsvd

    with pytest.raises(InvalidArgument, match="tsvd: empty matrix"):
        tsvd(np.zeros((0, 4)), 2)
    with pytest.raises(InvalidArgument, match="tsvd: rank must be >= 1"):
        tsvd(np.eye(4), 0)


def test_tsvd_batched_and_device(cuda, oracle_mod, ref_mod):
    import torch

    from paper_1710_01463_b200 import tsvd, tsvd_batched

    items = [oracle_mod.gaussian_matrix(77 + b, 48, 36) for b in range(5)]
    bf = tsvd_batched(np.stack(items), 12)
    at = torch.from_numpy(np.stack(items)).to(cuda)
    bd = tsvd_batched(at, 12)
    for b, a in enumerate(items):
        U, S, Vt, dw = ref_mod.tsvd(a, 12)
        fb = bf.item(b)
        assert fb.discarded_exact
        assert rel_sigma_err(fb.sigma, S) < SIG_TOL
        assert fb.discarded_weight == pytest.approx(dw, rel=1e-9)
        fd = bd.item(b)
        assert np.array_equal(_np(fd.sigma), fb.sigma)  # same kernels, same bits
        fs = tsvd(torch.from_numpy(a).to(cuda), 12)
        assert rel_sigma_err(_np(fs.sigma), S) < SIG_TOL


# ------------------------------------------------------- block_factorize ---

def _req(chi=0, maximal=False, slack=-1):
    from paper_1710_01463_b200 import RankPolicy, SectorRankRequest

    return SectorRankRequest(RankPolicy.maximal if maximal else RankPolicy.per_sector_estimate,
                             chi, slack)


def _merged(f):
    return sorted(np.concatenate([_np(x.sigma) for x in f.factors]).tolist(), reverse=True)


def test_block_global_selection(cuda):  # test_blocks.cpp:82-95
    from paper_1710_01463_b200 import BlockDiagMatrix, BlockMethod, block_factorize

    a = BlockDiagMatrix([0, 1], [np.diag([3.0, 1.0]), np.diag([2.0, 0.5])])
    f = block_factorize(a, 2, _req(maximal=True), BlockMethod.deterministic())
    assert [x.rank() for x in f.factors] == [1, 1]
    assert f.factors[0].sigma[0] == pytest.approx(3.0, rel=1e-14)
    assert f.factors[1].sigma[0] == pytest.approx(2.0, rel=1e-14)
    assert f.total_rank() == 2
    assert f.discarded_weight == pytest.approx(1.25, rel=1e-14)
    assert f.discarded_exact


def test_block_order_and_ties(cuda):  # test_blocks.cpp:97-140
    from paper_1710_01463_b200 import BlockDiagMatrix, BlockMethod, block_factorize

    det = BlockMethod.deterministic()
    even, odd = np.diag([3.0, 1.0]), np.diag([2.0, 0.5])
    fa = block_factorize(BlockDiagMatrix([0, 1], [even, odd]), 3, _req(maximal=True), det)
    fb = block_factorize(BlockDiagMatrix([1, 0], [odd, even]), 3, _req(maximal=True), det)
    assert _merged(fa) == _merged(fb)
    assert fa.factors[0].rank() == fb.factors[1].rank()
    t = np.diag([2.0, 1.0])
    f = block_factorize(BlockDiagMatrix([0, 1], [t, t.copy()]), 3, _req(maximal=True), det)
    assert [x.rank() for x in f.factors] == [2, 1]
    g = block_factorize(BlockDiagMatrix([1, 0], [t, t.copy()]), 3, _req(maximal=True), det)
    assert [x.rank() for x in g.factors] == [1, 2]


def test_block_single_sector_is_dense(cuda):  # test_blocks.cpp:142-156
    from paper_1710_01463_b200 import BlockDiagMatrix, BlockMethod, block_factorize, tsvd

    blk = np.random.default_rng(21).standard_normal((30, 22))
    f = block_factorize(BlockDiagMatrix([0], [blk]), 6, _req(maximal=True),
                        BlockMethod.deterministic())
    d = tsvd(blk, 6)
    assert f.factors[0].rank() == d.rank()
    assert np.array_equal(f.factors[0].sigma, d.sigma)
    assert f.discarded_weight == pytest.approx(d.discarded_weight, rel=1e-14)


def test_block_dense_embedding(cuda):  # test_blocks.cpp:158-183
    from paper_1710_01463_b200 import BlockDiagMatrix, BlockMethod, block_factorize, tsvd

    rng = np.random.default_rng(33)
    b0, b1 = rng.standard_normal((18, 14)), rng.standard_normal((16, 20))
    dense = np.zeros((34, 34))
    dense[:18, :14] = b0
    dense[18:, 14:] = b1
    f = block_factorize(BlockDiagMatrix([0, 1], [b0, b1]), 9, _req(maximal=True),
                        BlockMethod.deterministic())
    ft = tsvd(dense, 9)
    np.testing.assert_allclose(_merged(f), ft.sigma, rtol=1e-12)
    assert f.discarded_weight == pytest.approx(ft.discarded_weight, rel=1e-10)


def test_block_randomized_matches_deterministic(cuda, oracle_mod):  # test_blocks.cpp:185-203
    from paper_1710_01463_b200 import BlockDiagMatrix, BlockMethod, block_factorize

    a = BlockDiagMatrix([0, 1], [
        matrix_with_spectrum(oracle_mod, 8, 64, 48, spectrum_family(0, 40)),
        matrix_with_spectrum(oracle_mod, 9, 56, 60, spectrum_family(2, 40))])
    fd = block_factorize(a, 24, _req(), BlockMethod.deterministic())
    fr = block_factorize(a, 24, _req(), BlockMethod.randomized(4, 2024))
    assert not fr.discarded_exact
    assert fr.total_rank() == fd.total_rank()
    sd, sr = np.array(_merged(fd)), np.array(_merged(fr))
    assert np.max(np.abs(sr - sd) / sd) < 1e-8


def test_block_size_floor_takes_exact_path(cuda):  # test_blocks.cpp:205-220
    from paper_1710_01463_b200 import BlockDiagMatrix, BlockMethod, block_factorize

    rng = np.random.default_rng(13)
    a = BlockDiagMatrix([0, 1], [rng.standard_normal((8, 8)), rng.standard_normal((10, 9))])
    m = BlockMethod.randomized(4, 5)
    f = block_factorize(a, 6, _req(maximal=True), m)
    assert f.discarded_exact
    fd = block_factorize(a, 6, _req(maximal=True), BlockMethod.deterministic())
    assert _merged(f) == _merged(fd)


def test_block_seed_derivation(cuda, oracle_mod):  # test_blocks.cpp:222-243
    from paper_1710_01463_b200 import (BlockDiagMatrix, BlockMethod, RsvdParams, block_factorize,
                                       derive_seed, rsvd)

    blk = matrix_with_spectrum(oracle_mod, 44, 64, 64, spectrum_family(2, 50))
    m = BlockMethod.randomized(4, 99)
    m.rsvd_min_dim = 1
    f = block_factorize(BlockDiagMatrix([1], [blk]), 10, _req(maximal=True), m)
    d = rsvd(blk, RsvdParams(10, 20, 4, derive_seed(99, 1)))
    assert np.array_equal(f.factors[0].sigma, d.sigma)
    assert np.array_equal(f.factors[0].left, d.left)


def test_block_oversample_clamped(cuda):  # test_blocks.cpp:245-262
    from paper_1710_01463_b200 import BlockDiagMatrix, BlockMethod, block_factorize

    blk = np.random.default_rng(50).standard_normal((40, 36))
    m = BlockMethod.randomized(2, 7)
    m.rsvd_min_dim = 1
    for ov in (4, 500):
        m.rsvd.oversample = ov
        assert block_factorize(BlockDiagMatrix([0], [blk]), 12, _req(maximal=True),
                               m).total_rank() == 12


def test_block_rank_zero_sector(cuda):  # test_blocks.cpp:260-279
    from paper_1710_01463_b200 import BlockDiagMatrix, BlockMethod, block_factorize

    a = BlockDiagMatrix([0, 1], [np.diag([9.0, 8.0, 7.0]), np.diag([0.2, 0.1])])
    f = block_factorize(a, 3, _req(maximal=True), BlockMethod.deterministic())
    assert [x.rank() for x in f.factors] == [3, 0]
    assert f.factors[1].left.shape == (2, 0)
    assert f.discarded_weight == pytest.approx(0.05, rel=1e-12)


@pytest.mark.parametrize("kind", ["tsvd", "rsvd"])
@pytest.mark.parametrize("device", [False, True])
def test_block_many_sectors_vs_oracle(cuda, oracle_mod, kind, device, ref_mod):
    """A TEBD-like bond: 7 sectors, three sharing one shape (one batched engine
    call), ragged others, a sector below rsvd_min_dim, one zero-width sector;
    per-sector results against the oracle's block_factorize."""
    import torch

    from paper_1710_01463_b200 import BlockDiagMatrix, BlockMethod, block_factorize

    shapes = [(96, 80), (96, 80), (96, 80), (120, 64), (40, 150), (20, 30), (0, 12)]
    charges = [3, -1, 0, 5, 2, 7, 4]
    blocks = []
    for i, (r, c) in enumerate(shapes):
        if r == 0:
            blocks.append(np.zeros((0, c)))
            continue
        blocks.append(matrix_with_spectrum(oracle_mod, 300 + i, r, c,
                                           spectrum_family(i % 3, min(r, c)) * (1.0 + 0.1 * i)))
    chi = 90
    meth = BlockMethod.randomized(3, 4242) if kind == "rsvd" else BlockMethod.deterministic()
    ins = [torch.from_numpy(b).to(cuda) for b in blocks] if device else blocks
    if device:
        ins[-1] = np.zeros((0, 12))  # empty sector stays on the host path
    f = block_factorize(BlockDiagMatrix(charges, ins), chi, _req(), meth)
    ref, dw, exact = ref_mod.block_factorize(blocks, charges, chi, kind=kind, power=3,
                                                seed=4242)
    assert f.discarded_exact == exact
    assert f.total_rank() == sum(len(x[1]) for x in ref)
    for s, (U, S, Vt, dws) in enumerate(ref):
        g = f.factors[s]
        assert g.rank() == len(S), s
        if len(S) == 0:
            continue
        assert rel_sigma_err(_np(g.sigma), S) < SIG_TOL, s
        assert isometry_err(_np(g.left)) < ISO_TOL
        assert g.discarded_weight == pytest.approx(dws, rel=1e-8, abs=1e-26), s
    assert f.discarded_weight == pytest.approx(dw, rel=1e-8)


def test_tsvd_rank_deficient_graded_block(cuda, oracle_mod, ref_mod):
    """A TEBD sector block (24 x 21, numerical rank 15, values 0.79 .. 5e-15)
    captured from the bond-update tests: every value to O(u ||A||)
    absolutely, like the oracle's gesdd."""
    import os

    from paper_1710_01463_b200 import tsvd

    a = np.load(os.path.join(os.path.dirname(__file__), "golden", "theta_rankdef_24x21.npy"))
    _, S, _, dw = ref_mod.tsvd(a, 100)
    for x in (a, a.T.copy()):
        f = tsvd(x, 100)
        assert f.rank() == len(S)
        assert np.max(np.abs(np.asarray(f.sigma) - S)) < 1e-14  # ~50 u ||A||
        assert f.discarded_weight == pytest.approx(dw, abs=1e-28)


@pytest.mark.parametrize("kind", ["tsvd", "rsvd"])
def test_block_factorize_complex_vs_oracle(cuda, oracle_mod, kind):
    """block_factorize<Complex> (blocks.cpp:122): complex sectors through the
    complex engine, global selection over the merged spectra as for real."""
    from paper_1710_01463_b200 import BlockDiagMatrix, BlockMethod, block_factorize
    from tests.helpers import zmatrix_with_spectrum

    blocks = [zmatrix_with_spectrum(oracle_mod, 70 + i, 48 + 8 * i, 40, np.exp(-np.arange(40) / (5.0 + i)))
              for i in range(3)]
    a = BlockDiagMatrix([0, 1, 2], blocks)
    meth = BlockMethod.randomized(4, 77) if kind == "rsvd" else BlockMethod.deterministic()
    f = block_factorize(a, 24, _req(), meth)
    assert f.total_rank() == 24
    merged = np.sort(np.concatenate([np.asarray(x.sigma) for x in f.factors]))[::-1]
    want = np.sort(np.concatenate([np.exp(-np.arange(40) / (5.0 + i)) for i in range(3)]))[::-1][:24]
    np.testing.assert_allclose(merged, want, rtol=1e-9)
    for x, b in zip(f.factors, blocks):
        assert np.asarray(x.left).dtype == np.complex128
        r = x.rank()
        if r:
            rec = (np.asarray(x.left) * np.asarray(x.sigma)[None, :]) @ np.asarray(x.right_adj)
            tail = np.linalg.norm(b - rec) ** 2
            assert tail == pytest.approx(np.linalg.norm(b) ** 2 - np.sum(np.asarray(x.sigma) ** 2),
                                         rel=1e-8, abs=1e-20)
