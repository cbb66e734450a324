"""The engine's table-driven TEBD bond-update kernels through the C ABI
(rsvd_combine_blocks, rsvd_grouped_gemm, rsvd_block_sqnorms, rsvd_qr_f64),
each against a plain fp64 reference of the same operation (mps.cpp:130-137,
157-268, 307-316; lapack.cpp:180-201 for the QR)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_1710_01463_b200 import _lib as L

    return L, L.default_handle()


def _view(t):
    return t.data_ptr(), t.stride(0), t.stride(1)


@pytest.mark.parametrize("cplx", [False, True])
def test_combine_blocks_matches_reference(cuda, cplx):
    import torch

    L, h = _lib()
    dt = torch.complex128 if cplx else torch.float64
    g = torch.Generator(device="cpu").manual_seed(3)

    def rnd(r, c):
        x = torch.randn(r, c, generator=g, dtype=torch.float64)
        if cplx:
            x = x + 1j * torch.randn(r, c, generator=g, dtype=torch.float64)
        return x.to(dt).to(cuda)

    srcs = [rnd(7, 5), rnd(5, 7).t(), rnd(7, 5)]          # strided views too
    rs = torch.rand(7, dtype=torch.float64, device=cuda)
    cs = torch.rand(5, dtype=torch.float64, device=cuda)
    dst = torch.empty((5, 9), dtype=dt, device=cuda).t()[1:8]  # 7 x 5 column-major slice
    dst2 = torch.empty(3, 4, dtype=dt, device=cuda)            # zero-term job
    coefs = [1.5, -0.25 + (0.5j if cplx else 0.0), 2.0]
    terms = [(_view(srcs[0])[0], *_view(srcs[0])[1:], rs.data_ptr(), 0, coefs[0].real, 0.0),
             (_view(srcs[1])[0], *_view(srcs[1])[1:], 0, cs.data_ptr(), complex(coefs[1]).real,
              complex(coefs[1]).imag),
             (_view(srcs[2])[0], *_view(srcs[2])[1:], rs.data_ptr(), cs.data_ptr(), coefs[2], 0.0)]
    jobs = [(*_view(dst), 7, 5, 0, 3), (*_view(dst2), 3, 4, 3, 0)]
    J = np.array(jobs, dtype=L.BLOCK_JOB)
    T = np.array(terms, dtype=L.BLOCK_TERM)
    with L.on_torch_stream(h):
        L.raise_for(L.load().rsvd_combine_blocks(h.raw, int(cplx), 2, J.ctypes.data, 3,
                                                 T.ctypes.data), h.raw)
    torch.cuda.synchronize()
    ref = (coefs[0] * rs[:, None] * srcs[0] + coefs[1] * srcs[1] * cs[None, :]
           + coefs[2] * rs[:, None] * srcs[2] * cs[None, :])
    assert torch.allclose(dst, ref, rtol=1e-14, atol=1e-14)
    assert torch.count_nonzero(dst2).item() == 0


@pytest.mark.parametrize("cplx", [False, True])
def test_grouped_gemm_matches_reference(cuda, cplx):
    import torch

    L, h = _lib()
    dt = torch.complex128 if cplx else torch.float64
    shapes = [(1, 1, 1), (70, 33, 129), (130, 65, 8), (64, 64, 64), (5, 200, 0)]
    jobs, refs, outs, keep = [], [], [], []
    for (M, N, K) in shapes:
        A = torch.randn(M, K, dtype=dt, device=cuda)
        B = torch.randn(N, K, dtype=dt, device=cuda).t()  # strided operand
        C = torch.empty((N, M), dtype=dt, device=cuda).t()
        jobs.append((*_view(A), *_view(B), *_view(C), M, N, K))
        refs.append(A @ B if K else torch.zeros(M, N, dtype=dt, device=cuda))
        outs.append(C)
        keep += [A, B]  # the job table holds raw pointers
    J = np.array(jobs[:-1], dtype=L.GEMM_JOB)
    with L.on_torch_stream(h):
        L.raise_for(L.load().rsvd_grouped_gemm(h.raw, int(cplx), len(J), J.ctypes.data), h.raw)
    torch.cuda.synchronize()
    for C, R, (M, N, K) in zip(outs[:-1], refs[:-1], shapes[:-1]):
        assert torch.allclose(C, R, rtol=1e-13, atol=1e-12 * max(K, 1)), (M, N, K)


def test_block_sqnorms_is_deterministic(cuda):
    import torch

    L, h = _lib()
    blocks = [torch.randn(37, 11, dtype=torch.float64, device=cuda),
              torch.randn(5, 300, dtype=torch.float64, device=cuda).t(),
              torch.randn(1, 1, dtype=torch.float64, device=cuda)]
    tab = np.array([(*_view(b), b.shape[0], b.shape[1], 0, 0) for b in blocks], dtype=L.BLOCK_JOB)
    begin = np.array([0, 2, 2, 3], dtype=np.int64)  # slot 1 is empty
    outs = []
    for _ in range(2):
        out = torch.empty(3, dtype=torch.float64, device=cuda)
        with L.on_torch_stream(h):
            L.raise_for(L.load().rsvd_block_sqnorms(h.raw, 0, 3, begin.ctypes.data,
                                                    tab.ctypes.data, out.data_ptr()), h.raw)
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    ref = [float((blocks[0] ** 2).sum() + (blocks[1] ** 2).sum()), 0.0, float(blocks[2][0, 0] ** 2)]
    np.testing.assert_allclose(outs[0], ref, rtol=1e-13)


@pytest.mark.parametrize("m,n,rank", [(200, 48, 48), (96, 96, 96), (150, 40, 7), (64, 1, 1)])
def test_qr_f64_against_reference_qr(cuda, ref_mod, m, n, rank):
    """x = Q R with Q orthonormal; at full rank R is upper triangular and equals
    the reference's Householder R up to row signs (lapack.cpp:180-201).  On
    rank-deficient x the pivoted fallback leaves a column-permuted triangle;
    x = Q R still holds, which is all the product form needs (mps.cpp:265)."""
    import torch

    L, h = _lib()
    rng = np.random.default_rng(m + n)
    x = rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n))
    batch = np.stack([x, 2.0 * x[:, ::-1]])
    X = torch.from_numpy(np.ascontiguousarray(batch.transpose(0, 2, 1))).to(cuda).transpose(1, 2)
    Q = torch.empty((2, n, m), dtype=torch.float64, device=cuda).transpose(1, 2)
    R = torch.empty((2, n, n), dtype=torch.float64, device=cuda).transpose(1, 2)
    L.raise_for(L.load().rsvd_qr_f64(h.raw, 2, X.data_ptr(), m, n, m, m * n, Q.data_ptr(), m,
                                     m * n, R.data_ptr(), n, n * n, L.PTR_DEVICE), h.raw)
    torch.cuda.synchronize()
    for b in range(2):
        q, r, a = Q[b].cpu().numpy(), R[b].cpu().numpy(), batch[b]
        assert np.max(np.abs(q.T @ q - np.eye(n))) < 1e-12
        assert np.linalg.norm(a - q @ r) <= 1e-13 * np.linalg.norm(a)
        if rank == n:  # full rank: R is upper triangular, unique up to row signs
            assert np.allclose(np.tril(r, -1), 0.0)
            rr = np.linalg.qr(a, mode="r")
            np.testing.assert_allclose(np.abs(np.diag(r)), np.abs(np.diag(rr)), rtol=1e-10)


def test_qr_f64_rejects_wide(cuda):
    import torch

    from paper_1710_01463_b200 import InvalidArgument

    L, h = _lib()
    X = torch.zeros(4, 8, dtype=torch.float64, device=cuda)
    rc = L.load().rsvd_qr_f64(h.raw, 1, X.data_ptr(), 4, 8, 4, 32, X.data_ptr(), 4, 32,
                              X.data_ptr(), 8, 64, L.PTR_DEVICE)
    with pytest.raises(InvalidArgument, match="m >= n"):
        L.raise_for(rc, h.raw)


@pytest.mark.parametrize("log_kappa", [2, 6, 9, 12, 15])
def test_qr_fallback_range(cuda, log_kappa):
    """The engine's orthonormalisation (the reference's Householder QR,
    lapack.cpp:180-201 -> shifted CholeskyQR with pivoted completion here,
    DESIGN.md §4) over a kappa(Y) sweep: Q stays orthonormal to 1e-12
    throughout; Y = Q R holds to working precision up to kappa = 1e12 and to
    ~4e-12 relative at kappa = 1e15 (numerically rank deficient: Householder
    would keep ~1e-16 there -- the documented limit of the fallback), while
    plain CholeskyQR2 (restated in numpy below) has already broken down from
    kappa ~ 1e8 (the Gram loses definiteness)."""
    import torch

    L, h = _lib()
    m, n = 300, 40
    rng = np.random.default_rng(log_kappa)
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    y = (u * np.logspace(0, -log_kappa, n)) @ v.T
    X = torch.from_numpy(np.asfortranarray(y).T.copy()).to(cuda).t()
    Q = torch.empty((n, m), dtype=torch.float64, device=cuda).t()
    R = torch.empty((n, n), dtype=torch.float64, device=cuda).t()
    L.raise_for(L.load().rsvd_qr_f64(h.raw, 1, X.data_ptr(), m, n, m, m * n, Q.data_ptr(), m,
                                     m * n, R.data_ptr(), n, n * n, L.PTR_DEVICE), h.raw)
    torch.cuda.synchronize()
    q, r = Q.cpu().numpy(), R.cpu().numpy()
    assert np.max(np.abs(q.T @ q - np.eye(n))) < 1e-12
    tol = 1e-13 if log_kappa <= 12 else 1e-11
    assert np.linalg.norm(y - q @ r) <= tol * np.linalg.norm(y)

    def cholqr2(a):
        for _ in range(2):
            rr = np.linalg.cholesky(a.T @ a).T
            a = np.linalg.solve(rr.T, a.T).T
        return a

    try:
        qq = cholqr2(y)
        plain_ok = np.max(np.abs(qq.T @ qq - np.eye(n))) < 1e-12
    except np.linalg.LinAlgError:
        plain_ok = False
    if log_kappa >= 9:
        assert not plain_ok  # the range the fallback exists for
