"""The rest of test_factorize.cpp on the GPU path, plus boundary shapes and
pointer layouts (k = 1, full sample width, tall / wide, odd sizes, strided
device buffers through the C ABI, many tiny matrices, extreme scales)."""
import ctypes

import numpy as np
import pytest

from tests.helpers import isometry_err, matrix_with_spectrum, rel_sigma_err, spectrum_family

pytestmark = pytest.mark.gpu


def test_tsvd_scale_equivariant(cuda):  # test_factorize.cpp:148-155
    from paper_1710_01463_b200 import tsvd

    a = np.random.default_rng(55).standard_normal((20, 20))
    f1, f2 = tsvd(a, 5), tsvd(3.0 * a, 5)
    np.testing.assert_allclose(f2.sigma, 3.0 * f1.sigma, rtol=1e-13)


def test_rank_clamps_to_matrix_size(cuda):  # test_factorize.cpp:157-161
    from paper_1710_01463_b200 import tsvd

    f = tsvd(np.diag([3.0, 2.0, 1.0]), 10)
    assert f.rank() == 3 and f.discarded_weight == 0.0


def test_rank_one_recovered_exactly(cuda):  # test_factorize.cpp:186-197
    from paper_1710_01463_b200 import reconstruction_error, tsvd

    rng = np.random.default_rng(9)
    u, v = rng.standard_normal(12), rng.standard_normal(9)
    a = 2.0 * np.outer(u / np.linalg.norm(u), v / np.linalg.norm(v))
    f = tsvd(a, 1)
    assert f.rank() == 1 and f.sigma[0] == pytest.approx(2.0, rel=1e-12)
    assert reconstruction_error(a, f) <= 1e-12


def test_truncation_error_is_spectral_tail(cuda):  # test_factorize.cpp:228-238
    from paper_1710_01463_b200 import reconstruction_error, tsvd

    a = np.random.default_rng(77).standard_normal((40, 40))
    f = tsvd(a, 8)
    tail = float(np.sum(np.linalg.svd(a, compute_uv=False)[8:] ** 2))
    assert reconstruction_error(a, f) ** 2 == pytest.approx(tail, rel=1e-10)
    assert f.discarded_weight == pytest.approx(tail, rel=1e-10)


def test_spectral_reconstruction_error(cuda, oracle_mod):  # test_factorize.cpp:240-252
    from paper_1710_01463_b200 import ErrorNorm, reconstruction_error, rsvd, RsvdParams, tsvd

    a = matrix_with_spectrum(oracle_mod, 63, 28, 20, spectrum_family(1, 20))
    f = tsvd(a, 6)
    r = a - (f.left * f.sigma) @ f.right_adj
    rs = np.linalg.svd(r, compute_uv=False)
    assert reconstruction_error(a, f, ErrorNorm.spectral) == pytest.approx(rs[0], rel=1e-10)
    assert reconstruction_error(a, f) == pytest.approx(np.linalg.norm(r), rel=1e-12)
    big = matrix_with_spectrum(oracle_mod, 64, 700, 650, 0.97 ** np.arange(650))
    g = rsvd(big, RsvdParams(40, 80, 3, 5))
    rb = big - (g.left * g.sigma) @ g.right_adj
    assert reconstruction_error(big, g, ErrorNorm.spectral) == pytest.approx(
        np.linalg.svd(rb, compute_uv=False)[0], rel=1e-8)


@pytest.mark.parametrize("m,n,k,ell,q", [(64, 48, 1, 1, 0), (64, 48, 1, 2, 3), (50, 30, 30, 30, 0),
                                         (50, 30, 12, 30, 2), (5000, 30, 8, 20, 2),
                                         (30, 5000, 8, 20, 2), (257, 129, 17, 37, 1),
                                         (1, 300, 1, 1, 2), (300, 1, 1, 1, 2)])
def test_boundary_shapes_vs_oracle(cuda, oracle_mod, m, n, k, ell, q, ref_mod):
    from paper_1710_01463_b200 import RsvdParams, rsvd

    a = matrix_with_spectrum(oracle_mod, 7 + m + n, m, n, 0.8 ** np.arange(min(m, n)))
    f = rsvd(a, RsvdParams(k, ell, q, 99))
    U, S, Vt, dw = ref_mod.rsvd(a, k, ell, q, 99)
    assert f.rank() == len(S)
    big = S > 1e-6 * S[0]
    assert rel_sigma_err(f.sigma[big], S[big]) < 1e-10
    assert isometry_err(f.left) < 1e-12 and isometry_err(f.right_adj.T) < 1e-12
    assert f.discarded_weight == pytest.approx(dw, rel=1e-8, abs=1e-28)


def test_strided_device_buffers_through_the_c_abi(cuda, oracle_mod, ref_mod):
    """lda > m, ldu > m, ldvt > k and item strides with padding, device pointers."""
    import torch

    from paper_1710_01463_b200 import _lib

    lib = _lib.load()
    h = _lib.Handle(0)
    m, n, k, ell, bsz = 70, 50, 6, 14, 3
    lda, ldu, ldvt = 80, 75, 9
    sa, su, ss, sv = lda * n + 13, ldu * k + 7, k + 3, ldvt * n + 5
    mats = [matrix_with_spectrum(oracle_mod, 40 + b, m, n, 0.7 ** np.arange(n)) for b in range(bsz)]
    A = torch.zeros(bsz * sa, dtype=torch.float64, device=cuda)
    for b, a in enumerate(mats):
        view = A[b * sa:b * sa + lda * n].view(n, lda)
        view[:, :m] = torch.from_numpy(a.T.copy()).to(cuda)
    U = torch.zeros(bsz * su, dtype=torch.float64, device=cuda)
    S = torch.zeros(bsz * ss, dtype=torch.float64, device=cuda)
    V = torch.zeros(bsz * sv, dtype=torch.float64, device=cuda)
    seeds = (ctypes.c_uint64 * bsz)(*[500 + b for b in range(bsz)])
    ranks = (ctypes.c_int64 * bsz)()
    dws = (ctypes.c_double * bsz)()
    with _lib.on_torch_stream(h):
        rc = lib.rsvd_f64_batched(h.raw, bsz, A.data_ptr(), m, n, lda, sa, k, ell, 2, seeds,
                                  U.data_ptr(), ldu, su, S.data_ptr(), ss, V.data_ptr(), ldvt, sv,
                                  ranks, dws, _lib.PTR_DEVICE)
    _lib.raise_for(rc, h.raw)
    for b, a in enumerate(mats):
        Uo, So, Vto, dwo = ref_mod.rsvd(a, k, ell, 2, 500 + b)
        s = S[b * ss:b * ss + k].cpu().numpy()
        assert ranks[b] == len(So) and rel_sigma_err(s, So) < 1e-10
        u = U[b * su:b * su + ldu * k].view(k, ldu)[:, :m].t().cpu().numpy()
        assert isometry_err(u) < 1e-12
        assert float(torch.abs(U[b * su + ldu * k:(b + 1) * su]).max()) == 0.0  # gaps untouched
    h.close()


def test_many_tiny_matrices(cuda, oracle_mod, ref_mod):
    import torch

    from paper_1710_01463_b200 import RsvdParams, rsvd_batched

    bsz, m, n = 1500, 8, 6
    rng = np.random.default_rng(3)
    mats = rng.standard_normal((bsz, m, n))
    A = torch.from_numpy(np.ascontiguousarray(np.transpose(mats, (0, 2, 1)))).to(cuda).transpose(1, 2)
    seeds = list(range(bsz))
    bf = rsvd_batched(A, RsvdParams(2, 4, 1, 0), seeds)
    for b in range(0, bsz, 149):
        _, S, _, _ = ref_mod.rsvd(mats[b], 2, 4, 1, b)
        assert rel_sigma_err(bf.sigma[b][:len(S)].cpu().numpy(), S) < 1e-10


@pytest.mark.parametrize("scale", [2.0 ** -500, 2.0 ** 500, 1e-150, 1e150])
def test_extreme_scales(cuda, oracle_mod, scale):
    """sigma scales with A; factors unchanged (the reference's Householder
    bases are scale-free; Gram-based bases must not under/overflow)."""
    from paper_1710_01463_b200 import RsvdParams, rsvd, tsvd

    a = matrix_with_spectrum(oracle_mod, 12, 90, 70, 0.9 ** np.arange(70))
    f0 = rsvd(a, RsvdParams(10, 20, 2, 3))
    f1 = rsvd(a * scale, RsvdParams(10, 20, 2, 3))
    assert f1.rank() == f0.rank()
    np.testing.assert_allclose(f1.sigma / scale, f0.sigma, rtol=1e-12)
    t0, t1 = tsvd(a, 10), tsvd(a * scale, 10)
    np.testing.assert_allclose(t1.sigma / scale, t0.sigma, rtol=1e-12)
