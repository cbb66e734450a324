"""Host-pointer call time vs chunk count (C4, pinned in/out reused)."""
import os, sys, time
import torch
sys.path.insert(0, os.getcwd())
from paper_1710_01463_b200 import Handle, RsvdParams, rsvd_batched, synth

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
A = synth.make_batch(cfg, device="cuda:0")
seeds = synth.omega_seeds(cfg)
p = RsvdParams(cfg.rank, cfg.ell, cfg.power, 0)
h = Handle(0)
Ah = torch.empty_strided(A.shape, A.stride(), dtype=A.dtype, pin_memory=True)
Ah.copy_(A)
del A
torch.cuda.empty_cache()
out = rsvd_batched(Ah, p, seeds, handle=h)
for c in sys.argv[2:] or ["1", "2", "3", "4", "8"]:
    os.environ["RSVD_HOST_CHUNKS"] = c
    out = rsvd_batched(Ah, p, seeds, handle=h, out=out)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        out = rsvd_batched(Ah, p, seeds, handle=h, out=out)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"chunks {c}: ms per call {[round(x, 1) for x in ts]}  -> {cfg.batch / (min(ts) / 1e3):.1f} trunc/s best")
