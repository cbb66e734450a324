"""Time the engine's DMMA GEMM on the RSVD A-pass shapes (C4: 32 x 4096^2, l=288)."""
import ctypes, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1710_01463_b200 import _lib
dev = torch.device('cuda:0')
h = _lib.default_handle()
lib = _lib.load()
def run(tr, M, N, K, b, reps=5):
    A = torch.randn(b * M * K, dtype=torch.float64, device=dev)
    B = torch.randn(b * N * K, dtype=torch.float64, device=dev)
    C = torch.empty(b * M * N, dtype=torch.float64, device=dev)
    lda = K if tr else M
    lib.rsvd_set_stream(h.raw, ctypes.c_void_p(_lib.torch_stream_ptr()))
    f = lambda: lib.rsvd_testing_dgemm(h.raw, int(tr), M, N, K, A.data_ptr(), lda, M * K, B.data_ptr(), K, N * K, C.data_ptr(), M, M * N, b)
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, 2.0 * M * N * K * b / ms / 1e9
v = os.environ.get('RSVD_GEMM_VARIANT', '0')
for (tr, M, N, K, b) in [(False, 4096, 288, 4096, 32), (True, 4096, 288, 4096, 32), (False, 4096, 276, 4096, 32)]:
    ms, tf = run(tr, M, N, K, b)
    print(f"variant {v} {'TN' if tr else 'NN'} {M}x{N}x{K} b{b}: {ms:.3f} ms  {tf:.2f} TF")
