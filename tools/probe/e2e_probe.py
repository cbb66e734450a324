"""e2e (host-pointer) timing of C4 under different chunkings: one line per
RSVD_HOST_SPLIT / RSVD_HOST_CHUNKS setting given on the command line (each in
a fresh process so the engine reads its env)."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    from paper_1710_01463_b200 import RsvdParams, rsvd_batched, synth, _lib
    cfg = synth.CONFIGS["C4"]
    A = synth.make_batch(cfg, device="cuda:0")
    seeds = synth.omega_seeds(cfg)
    p = RsvdParams(cfg.rank, cfg.ell, cfg.power, 0)
    A_host = torch.empty_strided(A.shape, A.stride(), dtype=A.dtype, pin_memory=True)
    A_host.copy_(A)
    del A
    torch.cuda.empty_cache()
    fe = rsvd_batched(A_host, p, seeds)
    fe = rsvd_batched(A_host, p, seeds, out=fe)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        fe = rsvd_batched(A_host, p, seeds, out=fe)
        _ = fe.sigma[0, 0].item()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(json.dumps({"split": os.environ.get("RSVD_HOST_SPLIT"),
                      "chunks": os.environ.get("RSVD_HOST_CHUNKS"),
                      "ms": [round(t, 1) for t in ts],
                      "trunc_s": 32 / (min(ts) / 1e3)}))
    sys.exit(0)

for spec in sys.argv[1:]:
    env = dict(os.environ)
    if spec.startswith("c"):
        env["RSVD_HOST_CHUNKS"] = spec[1:]
    elif spec != "default":
        env["RSVD_HOST_SPLIT"] = spec
    out = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True,
                         text=True)
    print(out.stdout.strip() or out.stderr[-500:], flush=True)
    if env.get("RSVD_PIPE_TRACE"):
        print("\n".join(out.stderr.strip().splitlines()[-3:]), flush=True)
