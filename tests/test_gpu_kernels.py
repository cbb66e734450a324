"""Kernel-level GPU checks: the device CounterRng against the reference's own
KAT, and the DMMA GEMM against a torch float64 reference."""
import ctypes
import json
import os

import numpy as np
import pytest

from tests.helpers import ulp_distance

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KAT = json.load(open(os.path.join(ROOT, "tests", "golden", "rng_kat.json")))


def test_device_gaussian_matches_reference_kat(cuda):
    import torch
    from paper_1710_01463_b200 import CounterRng

    exact = total = 0
    for s in KAT["streams"]:
        seed = int(s["seed"], 16)
        ref = np.array([int(h, 16) for h in s["normals"]], dtype=np.uint64).view(np.float64)
        out = torch.empty(len(ref), dtype=torch.float64, device=cuda)
        CounterRng(seed).fill_gaussian(out)
        got = out.cpu().numpy()
        d = ulp_distance(got, ref)
        assert d.max() <= 4, (seed, d.max())
        exact += int((d == 0).sum())
        total += len(d)
    assert exact / total > 0.5


def test_device_gaussian_large_stream_vs_oracle(cuda, oracle_mod):
    import torch
    from paper_1710_01463_b200 import CounterRng

    n = 1_000_001  # odd: last element uses the cos half of its pair
    ref = oracle_mod.fill_gaussian(0xABCDEF, n)
    out = torch.empty(n, dtype=torch.float64, device=cuda)
    CounterRng(0xABCDEF).fill_gaussian(out)
    d = ulp_distance(out.cpu().numpy(), ref)
    # |x| < tiny values can have larger relative ulp counts; bound absolute error too
    assert np.max(np.abs(out.cpu().numpy() - ref)) < 1e-14
    assert np.mean(d == 0) > 0.5


def _dgemm(trans_a, A, B, M, N, K, batch, lda, ldb, sA, sB, fn="rsvd_testing_dgemm"):
    import torch
    from paper_1710_01463_b200 import _lib

    h = _lib.default_handle()
    C = torch.zeros(batch * M * N + 7, dtype=torch.float64, device=A.device)
    lib = _lib.load()
    lib.rsvd_set_stream(h.raw, ctypes.c_void_p(_lib.torch_stream_ptr()))
    try:
        rc = getattr(lib, fn)(h.raw, int(trans_a), M, N, K, A.data_ptr(), lda, sA,
                              B.data_ptr(), ldb, sB, C.data_ptr(), M, M * N, batch)
    finally:
        lib.rsvd_set_stream(h.raw, None)
    _lib.raise_for(rc, h.raw)
    return C[: batch * M * N].reshape(batch, N, M).transpose(1, 2)


@pytest.mark.parametrize("trans_a", [False, True])
@pytest.mark.parametrize(
    "M,N,K,batch",
    [(128, 96, 64, 1), (1000, 74, 1024, 1), (257, 33, 129, 3), (80, 80, 4096, 2),
     (4096, 280, 4096, 1), (5, 3, 7, 2), (1024, 144, 2048, 4)],
)
def test_dgemm_vs_torch(cuda, trans_a, M, N, K, batch):
    import torch

    g = torch.Generator(device=cuda).manual_seed(M * 7 + N * 13 + K)
    if trans_a:
        A = torch.randn(batch, M, K, dtype=torch.float64, device=cuda, generator=g)  # K x M col-major
        lda, sA = K, M * K
        Aflat = A.contiguous()
        ref_A = Aflat  # item b: row i of (M,K) = column i of stored K x M
    else:
        A = torch.randn(batch, K, M, dtype=torch.float64, device=cuda, generator=g)  # M x K col-major
        lda, sA = M, M * K
        Aflat = A.contiguous()
        ref_A = Aflat.transpose(1, 2)  # (batch, M, K)
    B = torch.randn(batch, N, K, dtype=torch.float64, device=cuda, generator=g).contiguous()  # K x N col-major
    C = _dgemm(trans_a, Aflat, B, M, N, K, batch, lda, K, sA, N * K)
    ref = torch.matmul(ref_A, B.transpose(1, 2))
    err = (C - ref).abs().max().item()
    scale = (ref_A.abs().max() * B.abs().max() * K).item()
    assert err <= 1e-14 * scale, err


def test_dgemm_odd_leading_dimension(cuda):
    """8-byte cp.async path (odd ld) gives the same result."""
    import torch

    M, N, K = 131, 17, 99
    A2 = torch.randn(K, M, dtype=torch.float64, device=cuda)  # lda = M = 131 odd
    B = torch.randn(N, K, dtype=torch.float64, device=cuda)
    C = _dgemm(False, A2, B, M, N, K, 1, M, K, 0, 0)[0]
    ref = A2.t() @ B.t()
    assert (C - ref).abs().max().item() < 1e-12


@pytest.mark.parametrize("trans_a", [False, True])
@pytest.mark.parametrize(
    "M,N,K,batch,grade",
    [(128, 64, 32, 1, 0), (128, 48, 64, 2, 0), (256, 288, 512, 3, 0), (1024, 80, 1024, 1, 0),
     (1024, 96, 2048, 2, 12), (4096, 288, 4096, 2, 0), (2048, 544, 32768, 1, 0),
     (512, 64, 256, 1, 300), (4096, 288, 2048, 8, 6), (4096, 256, 1024, 8, 0),
     (272, 96, 1040, 2, 0)],
)
def test_ozaki_gemm_vs_torch(cuda, trans_a, M, N, K, batch, grade):
    """Emulated FP64 (7 signed 8-bit slices per operand on the INT8 tensor
    cores, ozaki.cu) against torch float64: elementwise within 8e-15 of
    |op(A)| |B| (an FP64 GEMM's K u |A||B| bound is ~1e-12 here), normwise
    within 1e-14; `grade` spreads the K columns of op(A) over 10^-grade
    (per-row exponents keep the small entries), 300 = extreme magnitudes.
    The shapes cover the three launch forms: 128 x 32 tiles (small grids),
    128 x 64 tiles (8 x 4096 x 256), and the mixed grid of 64-wide tiles plus
    one 32-wide remainder tile (544 columns; 288 columns on 8 items)."""
    import torch

    g = torch.Generator(device=cuda).manual_seed(M * 5 + N * 11 + K)
    opA = torch.randn(batch, M, K, dtype=torch.float64, device=cuda, generator=g)
    if grade == 300:
        opA = opA * 1e-300
    elif grade:
        opA = opA * torch.logspace(0, -grade, K, dtype=torch.float64, device=cuda)
    if trans_a:
        Aflat, lda = opA.contiguous(), K  # stored K x M column-major
    else:
        Aflat, lda = opA.transpose(1, 2).contiguous(), M  # stored M x K
    B = torch.randn(batch, N, K, dtype=torch.float64, device=cuda, generator=g)
    if grade == 300:
        B = B * 1e250
    C = _dgemm(trans_a, Aflat, B, M, N, K, batch, lda, K, M * K, N * K, fn="rsvd_testing_ozaki_gemm")
    ref = torch.matmul(opA, B.transpose(1, 2))
    bound = torch.matmul(opA.abs(), B.abs().transpose(1, 2))
    assert ((C - ref).abs() <= 8e-15 * bound).all(), ((C - ref).abs() / bound).max().item()
    assert ((C - ref).norm() / ref.norm()).item() < 1e-14


def test_ozaki_gemm_zero_lines_and_rejects(cuda):
    """All-zero rows / columns (no exponent) give exact zeros; shapes off the
    16-multiple grid are refused with InvalidArgument."""
    import torch

    from paper_1710_01463_b200 import InvalidArgument

    M, N, K = 256, 64, 128
    opA = torch.randn(1, M, K, dtype=torch.float64, device=cuda)
    opA[:, 5, :] = 0
    opA[:, :, 7] = 0
    B = torch.randn(1, N, K, dtype=torch.float64, device=cuda)
    B[:, 3, :] = 0
    C = _dgemm(False, opA.transpose(1, 2).contiguous(), B, M, N, K, 1, M, K, M * K, N * K,
               fn="rsvd_testing_ozaki_gemm")
    ref = torch.matmul(opA, B.transpose(1, 2))
    assert (C[0, 5, :] == 0).all() and (C[0, :, 3] == 0).all()
    assert ((C - ref).abs().max() <= 1e-13 * ref.abs().max()).item()
    with pytest.raises(InvalidArgument):
        _dgemm(False, opA.transpose(1, 2).contiguous(), B, M, N, K - 8, 1, M, K, M * K, N * K,
               fn="rsvd_testing_ozaki_gemm")
