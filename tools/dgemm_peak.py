"""cuBLAS FP64 GEMM (torch.matmul float64, 8192^3) as the attainable FP64 ceiling."""
import json
import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.matmul(a, b)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e-3)
print(json.dumps({"kernel": "torch.matmul float64 8192^3 (cuBLAS DGEMM)", "tflops_best": 2 * n ** 3 / min(ts) / 1e12,
                  "tflops_median": 2 * n ** 3 / sorted(ts)[2] / 1e12}))
