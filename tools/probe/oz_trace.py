"""Phase timing of oz_gemm_kernel tiles (library built with
`make -C paper_1710_01463_b200/csrc EXTRA=-DRSVD_OZ_TRACE`): per-CTA
%globaltimer stamps of the last launch -> mean / median phase durations.
    python tools/probe/oz_trace.py [M N K batch trans]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1710_01463_b200 import _lib  # noqa: E402

M, N, K, batch, trans = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (4096, 288, 4096, 32, 0)))
torch.cuda.init()
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn(batch, K, M, dtype=torch.float64, device="cuda", generator=g)
B = torch.randn(batch, N, K, dtype=torch.float64, device="cuda", generator=g)
C = torch.zeros(batch * M * N, dtype=torch.float64, device="cuda")
h = _lib.default_handle()
lib = _lib.load()
lda = K if trans else M
for _ in range(3):
    rc = lib.rsvd_testing_ozaki_gemm(h.raw, trans, M, N, K, A.data_ptr(), lda, M * K, B.data_ptr(), K, N * K,
                                     C.data_ptr(), M, M * N, batch)
    _lib.raise_for(rc, h.raw)
torch.cuda.synchronize()
nt = min(8192, -(-N // 64) * -(-M // 128) * batch)
buf = (ctypes.c_ulonglong * (nt * 8))()
lib.rsvd_testing_oz_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int64]
lib.rsvd_testing_oz_trace_read(buf, nt * 8)
t = np.frombuffer(buf, dtype=np.uint64).reshape(nt, 8).astype(np.int64)
d = np.diff(t, axis=1) / 1e3
names = ["setup (barriers, TMEM alloc)", "first stage lands", "main loop (MMAs)", "drain columns 0-31 (7 x tcgen05.ld x32 + Horner)",
         "stores 0-31", "drain columns 32-63", "stores 32-63, sync, dealloc"]
print(f"M={M} N={N} K={K} batch={batch} trans={trans}: {nt} CTAs traced, K steps {K // 32}")
for i, nm in enumerate(names):
    print(f"  {nm:50s} mean {d[:, i].mean():8.2f} us  median {np.median(d[:, i]):8.2f}  p95 {np.percentile(d[:, i], 95):8.2f}")
tot = (t[:, 7] - t[:, 0]) / 1e3
print(f"  {'CTA lifetime':32s} mean {tot.mean():8.2f} us  median {np.median(tot):8.2f}")
span = (t[:, 7].max() - t[:, 0].min()) / 1e3
print(f"  launch span {span:.1f} us; sum of lifetimes / 148 SMs = {tot.sum() / 148:.1f} us "
      f"(gap share {1 - tot.sum() / 148 / span:.3f})")
