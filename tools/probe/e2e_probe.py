"""Host-buffer (e2e) path of C4: raw pinned H2D / D2H bandwidth and the
pipelined rsvd_batched call time for several chunk counts.
    python tools/probe/e2e_probe.py [chunks ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1710_01463_b200 import RsvdParams, rsvd_batched, synth  # noqa: E402
from paper_1710_01463_b200 import _lib  # noqa: E402

cfg = synth.CONFIGS["C4"]
A = synth.make_batch(cfg, device="cuda:0")
seeds = synth.omega_seeds(cfg)
p = RsvdParams(cfg.rank, cfg.ell, cfg.power, 0)
Ah = torch.empty_strided(A.shape, A.stride(), dtype=A.dtype, pin_memory=True)
Ah.copy_(A)
torch.cuda.synchronize()
# raw bandwidth
for _ in range(2):
    t0 = time.perf_counter()
    A.copy_(Ah, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
print(f"H2D {Ah.numel() * 8 / 1e9:.2f} GB: {(t1 - t0) * 1e3:.1f} ms = {Ah.numel() * 8 / (t1 - t0) / 1e9:.1f} GB/s")
t0 = time.perf_counter()
Ah.copy_(A, non_blocking=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"D2H: {(t1 - t0) * 1e3:.1f} ms = {Ah.numel() * 8 / (t1 - t0) / 1e9:.1f} GB/s")
# device-resident
f = rsvd_batched(A, p, seeds)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    f = rsvd_batched(A, p, seeds, out=f)
torch.cuda.synchronize()
print(f"device-resident call: {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms")
del A, f
torch.cuda.empty_cache()
specs = sys.argv[1:] or ["7"]
for c in specs:
    # "7" = chunk count; "2,3,5,5/4" = chunk sizes / compute streams
    os.environ.pop("RSVD_HOST_SIZES", None)
    os.environ.pop("RSVD_HOST_STREAMS", None)
    if "," in c or "/" in c:
        sz, _, ns = c.partition("/")
        if sz:
            os.environ["RSVD_HOST_SIZES"] = sz
        if ns:
            os.environ["RSVD_HOST_STREAMS"] = ns
    else:
        os.environ["RSVD_HOST_CHUNKS"] = c
    h = _lib.Handle()
    fe = rsvd_batched(Ah, p, seeds, handle=h)
    fe = rsvd_batched(Ah, p, seeds, handle=h, out=fe)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        fe = rsvd_batched(Ah, p, seeds, handle=h, out=fe)
        _ = fe.sigma[0, 0].item()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"chunks {c}: host-buffer call {min(ts):.1f} ms (median {sorted(ts)[len(ts) // 2]:.1f})")
    del fe, h
    torch.cuda.empty_cache()
