import torch, time
n = 1 << 27  # 1 GiB of doubles
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device='cuda')
for name, f in [("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    print(name, "GB/s", 5 * n * 8 / e0.elapsed_time(e1) / 1e6)
# 2D copy via cudaMemcpy2DAsync equivalent: strided column copy
import ctypes
