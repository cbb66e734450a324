import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1710_01463_b200 import _lib as L
h = L.default_handle()
def v(t): return t.data_ptr(), t.stride(0), t.stride(1)
for (M,N,K) in [(2,2,1),(2,2,16),(2,2,17),(3,2,20),(70,33,16),(70,33,129),(64,64,64)]:
    for mode in range(4):
        A = torch.randn(M, K, dtype=torch.float64, device='cuda')
        B = torch.randn(K, N, dtype=torch.float64, device='cuda')
        if mode & 1: A = A.t().contiguous().t()
        if mode & 2: B = B.t().contiguous().t()
        C = torch.empty(M, N, dtype=torch.float64, device='cuda')
        J = np.array([(*v(A), *v(B), *v(C), M, N, K)], dtype=L.GEMM_JOB)
        with L.on_torch_stream(h):
            L.raise_for(L.load().rsvd_grouped_gemm(h.raw, 0, 1, J.ctypes.data), h.raw)
        torch.cuda.synchronize()
        err = (C - A @ B).abs().max().item()
        print(M,N,K,mode, 'err', err, 'strides', A.stride(), B.stride())
