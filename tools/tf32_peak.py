"""Measured dense TF32 tensor-core peak of this B200 (cuBLAS, the denominator
for the tcgen05 kind::tf32 kernels' tensor-pipe fraction): fp32 8192^3 matmul
with TF32 allowed, best of 10 (burst) and back to back for 4 s (sustained),
CUDA events. Our kernels issue 3 TF32 MMAs per fp32 product (3xTF32), so
their fp32-equivalent ceiling is a third of this."""
import json
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
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
flop = 2.0 * n ** 3
t0 = time.perf_counter()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
k = 0
while time.perf_counter() - t0 < 4.0:
    for _ in range(8):
        a @ b
    k += 8
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
print(json.dumps({"tf32_tflops_burst": flop / (best / 1e3) / 1e12,
                  "tf32_tflops_sustained": k * flop / (e0.elapsed_time(e1) / 1e3) / 1e12,
                  "how": "torch.matmul fp32 8192^3 with allow_tf32 (cuBLAS), best of 10 / 4 s back to back",
                  "gpu": torch.cuda.get_device_name()}))
