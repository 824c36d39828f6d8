"""Measured FP64 dense peak on this GPU (cuBLAS DGEMM via torch.matmul, 8192^3, best of 10 with
CUDA events) -- the denominator for the setup kernels' FP64 tensor-pipe utilisation."""
import json
import sys

import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a @ b
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
tf = 2.0 * n ** 3 / (best * 1e-3) / 1e12
json.dump({"fp64_dgemm_tflops": tf, "n": n, "ms": best, "how": "torch.matmul fp64 8192^3, best of 10"}, sys.stdout)
print()
