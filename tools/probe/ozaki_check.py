"""Probe: emulated-FP64 (Ozaki / INT8 tcgen05) GEMM against torch fp64 and the
engine's DMMA GEMM; accuracy (normwise, elementwise vs |A||B|) and call time."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1710_01463_b200 import _lib  # noqa: E402


def run(fn, trans_a, M, N, K, A, lda, sA, B, ldb, sB, batch):
    h = _lib.default_handle()
    C = torch.zeros(batch * M * N, dtype=torch.float64, device="cuda")
    lib = _lib.load()
    lib.rsvd_set_stream(h.raw, ctypes.c_void_p(_lib.torch_stream_ptr()))
    try:
        rc = getattr(lib, fn)(h.raw, int(trans_a), M, N, K, A.data_ptr(), lda, sA, B.data_ptr(),
                              ldb, sB, C.data_ptr(), M, M * N, batch)
    finally:
        lib.rsvd_set_stream(h.raw, None)
    _lib.raise_for(rc, h.raw)
    return C.reshape(batch, N, M).transpose(1, 2)


def case(trans_a, M, N, K, batch, reps=5, steep=False):
    g = torch.Generator(device="cuda").manual_seed(M + 3 * N + 7 * K)
    if trans_a:
        A = torch.randn(batch, M, K, dtype=torch.float64, device="cuda", generator=g)
        lda, sA = K, M * K
        opA = A  # (b, M, K): row i of op(A) = column i of stored K x M
    else:
        A = torch.randn(batch, K, M, dtype=torch.float64, device="cuda", generator=g)
        lda, sA = M, M * K
        opA = A.transpose(1, 2)
    if steep:
        opA = opA * torch.logspace(0, -12, opA.shape[-1], dtype=torch.float64, device="cuda")
        A = opA.contiguous() if trans_a else opA.transpose(1, 2).contiguous()
    B = torch.randn(batch, N, K, dtype=torch.float64, device="cuda", generator=g)
    ldb, sB = K, N * K
    ref = opA @ B.transpose(1, 2)
    bound = opA.abs() @ B.abs().transpose(1, 2)
    out = {}
    for fn in ("rsvd_testing_ozaki_gemm", "rsvd_testing_dgemm"):
        C = run(fn, trans_a, M, N, K, A, lda, sA, B, ldb, sB, batch)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            run(fn, trans_a, M, N, K, A, lda, sA, B, ldb, sB, batch)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        err = (C - ref)
        out[fn] = dict(
            norm_rel=float(err.norm() / ref.norm()),
            elem_vs_bound=float((err.abs() / bound.clamp_min(1e-300)).max()),
            ms=dt * 1e3,
            tflops=2.0 * M * N * K * batch / dt / 1e12,
        )
    print(f"trans_a={int(trans_a)} M={M} N={N} K={K} batch={batch} steep={steep}")
    for k, v in out.items():
        print(f"   {k:26s} " + " ".join(f"{a}={b:.3e}" for a, b in v.items()))
    sys.stdout.flush()


def big_only():
    torch.cuda.init()
    case(False, 4096, 288, 4096, 32, reps=1)
    case(True, 4096, 288, 4096, 32, reps=1)


if __name__ == "__main__" and len(sys.argv) > 1:
    big_only()
elif __name__ == "__main__":
    torch.cuda.init()
    case(False, 128, 64, 32, 1)
    case(False, 128, 64, 64, 1)
    case(True, 128, 64, 64, 1)
    case(False, 256, 128, 512, 2)
    case(True, 512, 96, 256, 2)
    case(False, 1024, 80, 1024, 1)
    case(False, 1024, 80, 1024, 1, steep=True)
    case(True, 1024, 80, 1024, 1, steep=True)
    case(False, 4096, 288, 4096, 8)
    case(True, 4096, 288, 4096, 8)
    case(False, 4096, 288, 4096, 32, reps=3)
    case(True, 4096, 288, 4096, 32, reps=3)
