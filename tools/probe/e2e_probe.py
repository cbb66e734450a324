import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_1710_01463_b200 import RsvdParams, rsvd_batched, synth, Handle
cfg = synth.CONFIGS["C4"]
A = synth.make_batch(cfg, device="cuda:0")
seeds = synth.omega_seeds(cfg)
p = RsvdParams(cfg.rank, cfg.ell, cfg.power, 0)
h = Handle(0)
Ah = torch.empty_strided(A.shape, A.stride(), dtype=A.dtype, pin_memory=True); Ah.copy_(A)
print("pinned", Ah.is_pinned(), Ah.stride())
def t(f, n=3):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1000
print("device call ms", t(lambda: rsvd_batched(A, p, seeds, handle=h)))
print("torch H2D of A ms", t(lambda: A.copy_(Ah, non_blocking=True)))
for c in ("1", "2", "4"):
    os.environ["RSVD_HOST_CHUNKS"] = c
    print("host call chunks", c, "ms", t(lambda: rsvd_batched(Ah, p, seeds, handle=h)))
