"""One row-sharded rsvd call (C5 or C3) bracketed by cudaProfilerStart/Stop,
under torch.distributed.run (NCCL), for an ncu launch list:
    ncu --profile-from-start off ... python -m torch.distributed.run --nproc-per-node 1 \
        tools/probe/rowshard_call.py C5"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1710_01463_b200 import Handle, RsvdParams, sharding, synth  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
A = synth.make_matrix(cfg, 0, dev)
first, count = sharding.row_partition(cfg.m, world, rank)
a_loc = A[first:first + count].t().contiguous().t()
del A
p = RsvdParams(cfg.rank, cfg.ell, cfg.power, synth.omega_seed(cfg, 0))
h = Handle(local)
sharding.attach_nccl(h, world, rank)
for _ in range(3):
    f = sharding.rsvd_rowsharded(a_loc, cfg.m, first, p, h)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    f = sharding.rsvd_rowsharded(a_loc, cfg.m, first, p, h)
torch.cuda.synchronize()
print("rowsharded call ms (wall):", (time.perf_counter() - t0) / 3 * 1e3)
flush = torch.empty(count * cfg.n, dtype=torch.float64, device=dev)
pairs = []
for _ in range(3):
    flush.zero_()
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es.record()
    f = sharding.rsvd_rowsharded(a_loc, cfg.m, first, p, h)
    ee.record()
    pairs.append((es, ee))
torch.cuda.synchronize()
print("with flush, event ms:", [round(a.elapsed_time(b), 2) for a, b in pairs])
torch.cuda.profiler.start()
f = sharding.rsvd_rowsharded(a_loc, cfg.m, first, p, h)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
dist.destroy_process_group()
