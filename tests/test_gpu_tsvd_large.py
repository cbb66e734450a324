"""GPU full-SVD truncation (tsvd, factorize.cpp:42-50) at BASELINE's large
shapes -- the comparator the configs name ("compare against full SVD
truncated") -- against the reference's own tsvd (oracle/_ref, gesdd).  The
row-streamed Jacobi (jacobi_rs_kernel) has no l-dependent shared memory, so
min(m, n) is not capped at the old 1600."""
import numpy as np
import pytest

from tests.helpers import isometry_err, rel_sigma_err, subspace_distance

pytestmark = pytest.mark.gpu


def _check(a, f, ref, label):
    from paper_1710_01463_b200 import reconstruction_error

    U, S, Vt, dw = ref
    assert f.rank() == len(S), (label, f.rank(), len(S))
    assert rel_sigma_err(f.sigma, S) < 1e-10, (label, rel_sigma_err(f.sigma, S))
    left, right = np.asarray(f.left), np.asarray(f.right_adj)
    assert isometry_err(left) < 1e-12 and isometry_err(right.T) < 1e-12, label
    e, er = reconstruction_error(a, f), float(np.linalg.norm(a - (U * S[None, :]) @ Vt))
    assert abs(e - er) / er < 1e-10, (label, e, er)
    assert f.discarded_weight == pytest.approx(dw, rel=1e-8), label
    # gapped leading subspace
    j = next((j for j in range(len(S) - 1, 0, -1) if S[j - 1] - S[j] > 1e-3 * S[0]), 0)
    if j:
        assert subspace_distance(left[:, :j], U[:, :j]) < 1e-8, label


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_tsvd_4096_square(cuda, ref_mod, name):
    import torch

    from paper_1710_01463_b200 import synth, tsvd

    cfg = synth.CONFIGS[name]
    A = synth.make_matrix(cfg, 0, cuda)
    a = np.asfortranarray(A.cpu().numpy())
    f = tsvd(A, cfg.rank)
    torch.cuda.synchronize()
    ff = type(f)(f.left.cpu().numpy(), f.sigma.cpu().numpy(), f.right_adj.cpu().numpy(),
                 f.discarded_weight, f.discarded_exact) if hasattr(f.left, "cpu") else f
    _check(a, ff, ref_mod.tsvd(a, cfg.rank), f"{name} tsvd")


@pytest.mark.slow
def test_tsvd_c5_tall(cuda, ref_mod):
    import torch

    from paper_1710_01463_b200 import synth, tsvd

    cfg = synth.CONFIGS["C5"]
    A = synth.make_matrix(cfg, 0, cuda)
    a = np.asfortranarray(A.cpu().numpy())
    f = tsvd(A, cfg.rank)
    torch.cuda.synchronize()
    ff = type(f)(f.left.cpu().numpy(), f.sigma.cpu().numpy(), f.right_adj.cpu().numpy(),
                 f.discarded_weight, f.discarded_exact)
    _check(a, ff, ref_mod.tsvd(a, cfg.rank), "C5 tsvd")


@pytest.mark.parametrize("m,n", [(2000, 1800), (1700, 2100)])
def test_tsvd_beyond_old_cap(cuda, oracle_mod, ref_mod, m, n):
    from paper_1710_01463_b200 import tsvd
    from tests.helpers import matrix_with_spectrum

    p = min(m, n)
    a = matrix_with_spectrum(oracle_mod, 17, m, n, np.exp(-np.arange(p) / 64.0))
    _check(a, tsvd(a, 100), ref_mod.tsvd(a, 100), f"tsvd {m}x{n}")


def test_complex_tsvd_beyond_old_cap(cuda, oracle_mod, ref_mod):
    from paper_1710_01463_b200 import tsvd
    from tests.helpers import zmatrix_with_spectrum

    a = zmatrix_with_spectrum(oracle_mod, 5, 1800, 1700, np.exp(-np.arange(1700) / 64.0))
    _check(a, tsvd(a, 80), ref_mod.tsvd(a, 80), "complex tsvd 1800x1700")
