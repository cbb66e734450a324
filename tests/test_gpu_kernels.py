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


def _dgemm(trans_a, A, B, M, N, K, batch, lda, ldb, sA, sB):
    import torch
    from paper_1710_01463_b200 import _lib

    h = _lib.default_handle()
    C = torch.zeros(batch * M * N + 7, dtype=torch.float64, device=A.device)
    lib = _lib.load()
    lib.rsvd_set_stream(h.raw, ctypes.c_void_p(_lib.torch_stream_ptr()))
    try:
        rc = lib.rsvd_testing_dgemm(h.raw, int(trans_a), M, N, K, A.data_ptr(), lda, sA,
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
