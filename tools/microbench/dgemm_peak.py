"""Measures the FP64 roofline denominator: cuBLAS DGEMM (torch.matmul fp64) on this B200."""
import json, torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
for _ in range(3): a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
e0.record()
for _ in range(20): c = a @ b
e1.record(); torch.cuda.synchronize(); sus = e0.elapsed_time(e1) / 20
print(json.dumps({"dgemm_tflops_burst": 2 * n**3 / best / 1e9, "dgemm_tflops_sustained": 2 * n**3 / sus / 1e9}))
