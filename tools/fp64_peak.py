"""cuBLAS DGEMM 8192^3 (torch.matmul float64), best of 10 with CUDA events: the
FP64 denominator for the factor roofline (MEASURED_PEAKS.json has none)."""
import json
import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"probe": "cublas_dgemm_8192", "tflops": 2 * n**3 / best / 1e9, "ms": best}))
