import sys, torch
sys.path.insert(0, '.')
from tests.test_gpu_kernels import _dgemm
dev = torch.device('cuda:0')
for (M,N,K,b) in [(4096,96,4096,1),(4096,280,4096,1)]:
    for tr in (True, False):
        g = torch.Generator(device=dev).manual_seed(1)
        if tr:
            A = torch.randn(b, M, K, dtype=torch.float64, device=dev, generator=g).contiguous(); lda=K; refA=A
        else:
            A = torch.randn(b, K, M, dtype=torch.float64, device=dev, generator=g).contiguous(); lda=M; refA=A.transpose(1,2)
        B = torch.randn(b, N, K, dtype=torch.float64, device=dev, generator=g).contiguous()
        C = _dgemm(tr, A, B, M, N, K, b, lda, K, M*K, N*K)
        ref = refA @ B.transpose(1,2)
        ref2 = (refA.cpu() @ B.transpose(1,2).cpu()).to(dev)
        d = (C-ref).abs(); d2 = (C-ref2).abs(); d3=(ref-ref2).abs()
        print(M,N,K,b,'TN' if tr else 'NN', 'err_vs_torchgpu %.3e' % d.max().item(), 'err_vs_cpu %.3e' % d2.max().item(), 'torchgpu_vs_cpu %.3e' % d3.max().item(), C[0,0,:3].tolist(), ref2[0,0,:3].tolist())
