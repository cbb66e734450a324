"""cuBLAS DGEMM peak probe (the FP64 roofline denominator; MEASURED_PEAKS.json has none)."""
import json, torch
dev = torch.device("cuda:0")
res = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"dgemm_{n}"] = {"ms": best, "tflops": 2 * n**3 / best / 1e9}
# skinny shapes representative of the A-passes
for (m, k, nn) in ((4096, 4096, 276), (4096, 4096, 288), (32768, 2048, 544), (1024, 1024, 74)):
    a = torch.randn(m, k, dtype=torch.float64, device=dev)
    b = torch.randn(k, nn, dtype=torch.float64, device=dev)
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"dgemm_{m}x{k}x{nn}"] = {"ms": best, "tflops": 2 * m * k * nn / best / 1e9}
print(json.dumps(res, indent=1))
