"""Per-stage device ms and call counts of one call (rsvd_profile) for a config."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1710_01463_b200 import RsvdParams, rsvd_batched, synth, _lib

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
A = synth.make_batch(cfg, device="cuda:0")
seeds = synth.omega_seeds(cfg)
p = RsvdParams(cfg.rank, cfg.ell, cfg.power, 0)
h = _lib.default_handle()
f = rsvd_batched(A, p, seeds)
_lib.profile_enable(h, True)
rsvd_batched(A, p, seeds)
torch.cuda.synchronize()
for k, (ms, n) in _lib.profile_read(h).items():
    print(f"{k:10s} {ms:8.3f} ms {n:4d} calls {ms / max(n, 1) * 1e3:8.1f} us/call")
