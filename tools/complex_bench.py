"""Throughput of the complex instantiation (rsvd<std::complex<double>>) on the
BASELINE shapes, HBM-resident inputs, device pointers.  Not the headline bench
(BASELINE.json's metric is real FP64); reported in DESIGN.md.

    python tools/complex_bench.py [--config C2|C4|C1|C3] [--steps K] [--warmup W]

Inputs: A = U diag(sigma) V^H with U, V from the QR of seeded complex
Gaussians (torch on the device; synthetic, the config's spectrum), Omega from
the reference's complex CounterRng fill.  Prints one JSON line: truncations/s,
ms/step, per-stage device ms (CUDA events around each stage, separate pass),
and the complex-GEMM flop rate of the A-passes.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CFG = {  # m, n, batch, k, ell, q, spectrum
    "C1": (1024, 1024, 1, 64, 74, 2, "exp32"),
    "C2": (256, 256, 256, 128, 138, 2, "pow1.5"),
    "C3": (4096, 4096, 1, 256, 272, 1, "c3"),
    "C4": (4096, 4096, 32, 256, 276, 2, "exp0.02"),
}


def spectrum(kind, n, torch):
    i = torch.arange(n, dtype=torch.float64)
    if kind == "exp32":
        return torch.exp(-i / 32)
    if kind == "pow1.5":
        s = (i + 1) ** -1.5
        return s / s.norm()
    if kind == "c3":
        s = 1.0 / (i + 1)
        s[512:] *= 1e-8
        return s
    return torch.exp(-0.02 * i)


def main():
    import torch
    from paper_1710_01463_b200 import RsvdParams, _lib, rsvd_batched

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--batch", type=int, default=0)
    o = ap.parse_args()
    m, n, batch, k, ell, q, kind = CFG[o.config]
    if o.batch:
        batch = o.batch
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(1234)
    sig = spectrum(kind, min(m, n), torch).to(dev)
    A = torch.empty((batch, n, m), dtype=torch.complex128, device=dev).transpose(1, 2)
    for b in range(batch):
        u, _ = torch.linalg.qr(torch.randn(m, min(m, n), dtype=torch.complex128, device=dev,
                                           generator=g))
        v, _ = torch.linalg.qr(torch.randn(n, min(m, n), dtype=torch.complex128, device=dev,
                                           generator=g))
        A[b] = (u * sig[None, :]) @ v.conj().T
    seeds = [0xC0FFEE + b for b in range(batch)]
    p = RsvdParams(k, ell, q, 0)
    h = _lib.default_handle()
    f = None
    for _ in range(o.warmup):  # factor buffers reused (out=): the call replays its CUDA graph
        f = rsvd_batched(A, p, seeds, out=f)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(o.steps):
        f = rsvd_batched(A, p, seeds, out=f)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / o.steps
    _lib.profile_enable(h, True)
    rsvd_batched(A, p, seeds)
    torch.cuda.synchronize()
    prof = _lib.profile_read(h)
    _lib.profile_enable(h, False)
    # complex A-pass flops: 8 m n l per pass, 2q + 2 passes
    apass_ms = prof["apass_nn"][0] + prof["apass_tn"][0]
    fl = 8.0 * m * n * ell * (2 * q + 2) * batch
    print(json.dumps({
        "metric": "complex128 RSVD truncations/sec", "config": o.config, "m": m, "n": n,
        "batch": batch, "k": k, "ell": ell, "q": q, "value": batch / (ms / 1e3),
        "ms_per_step": ms, "stage_ms": {kk: v[0] for kk, v in prof.items()},
        "apass_tflops": fl / (apass_ms / 1e3) / 1e12 if apass_ms else None,
        "rank_ok": all(r == k for r in f.ranks), "sigma0": float(f.sigma[0][0]),
        "jacobi_sweeps": _lib.last_jacobi_sweeps(h),
    }))


if __name__ == "__main__":
    main()
