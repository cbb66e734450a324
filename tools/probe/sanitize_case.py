"""Small shapes that exercise every kernel family once (for compute-sanitizer
memcheck / racecheck / synccheck): TMA + cp.async GEMMs, gchol (grid,
cluster and per-item modes), the dataflow and cluster Jacobi kernels, the
fallback Cholesky kernels, RNG, the TEBD table kernels and the thin QR."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1710_01463_b200 import RsvdParams, rsvd, rsvd_batched, tsvd  # noqa: E402
from paper_1710_01463_b200 import _lib as L  # noqa: E402

dev = "cuda:0"
rng = np.random.default_rng(0)
# batch -> dataflow Jacobi (tasks > SMs / 4), gchol grid mode
a = torch.from_numpy(rng.standard_normal((48, 80, 96))).to(dev).transpose(1, 2)
f = rsvd_batched(a, RsvdParams(20, 40, 1, 0), list(range(48)))
# single matrix -> cluster Jacobi, per-item gchol (l_p = 96)
b = rng.standard_normal((512, 400)) * np.exp(-np.arange(400) / 30.0)
g = rsvd(b, RsvdParams(64, 74, 2, 5))
# l_p = 224 single -> cluster gchol; steep spectrum -> shifted / pivoted fallback
c = rng.standard_normal((320, 300)) * (2.0 ** -np.arange(300))
h = rsvd(c, RsvdParams(100, 200, 1, 7))
t = tsvd(rng.standard_normal((130, 120)), 30)
# TEBD table kernels + thin QR
H = L.default_handle()
x = torch.from_numpy(rng.standard_normal((60, 50))).to(dev)
y = torch.empty((60, 50), dtype=torch.float64, device=dev)
J = np.array([(y.data_ptr(), 50, 1, 60, 50, 0, 1)], dtype=L.BLOCK_JOB)
T = np.array([(x.data_ptr(), 50, 1, 0, 0, 2.0, 0.0)], dtype=L.BLOCK_TERM)
L.raise_for(L.load().rsvd_combine_blocks(H.raw, 0, 1, J.ctypes.data, 1, T.ctypes.data), H.raw)
C = torch.empty((60, 60), dtype=torch.float64, device=dev)
G = np.array([(x.data_ptr(), 50, 1, x.data_ptr(), 1, 50, C.data_ptr(), 60, 1, 60, 60, 50)],
             dtype=L.GEMM_JOB)
L.raise_for(L.load().rsvd_grouped_gemm(H.raw, 0, 1, G.ctypes.data), H.raw)
q = torch.empty((50, 60), dtype=torch.float64, device=dev).t()
r = torch.empty((50, 50), dtype=torch.float64, device=dev).t()
xc = x.t().contiguous().t()
L.raise_for(L.load().rsvd_qr_f64(H.raw, 1, xc.data_ptr(), 60, 50, 60, 3000, q.data_ptr(), 60, 3000,
                                 r.data_ptr(), 50, 2500, L.PTR_DEVICE), H.raw)
torch.cuda.synchronize()
print("sanitize case ok", f.ranks[:2], g.rank(), h.rank(), t.rank())
