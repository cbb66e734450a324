"""One pipeline call of a BASELINE config bracketed by cudaProfilerStart/Stop,
for `ncu --profile-from-start off` launch lists / captures:
    ncu --profile-from-start off ... python tools/probe/one_call.py C1 [tsvd]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1710_01463_b200 import RsvdParams, rsvd_batched, synth, tsvd_batched  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
mode = sys.argv[2] if len(sys.argv) > 2 else "rsvd"
A = synth.make_batch(cfg, device="cuda:0")
seeds = synth.omega_seeds(cfg)
p = RsvdParams(cfg.rank, cfg.ell, cfg.power, 0)
run = (lambda: rsvd_batched(A, p, seeds)) if mode == "rsvd" else (lambda: tsvd_batched(A, cfg.rank))
f = None
for _ in range(3):
    f = run()
torch.cuda.synchronize()
torch.cuda.profiler.start()
f = run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ranks", f.ranks[:4])
