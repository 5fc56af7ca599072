"""Measured FP64 dense throughput of this B200 (cuBLAS DGEMM through torch),
the roofline denominator of the DMMA dense kernels: best of 10 and the
median of 10, 8192^3 (2*N^3 flop), CUDA events."""
import json

import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
ts = []
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    a @ b
    e.record()
    e.synchronize()
    ts.append(s.elapsed_time(e) / 1e3)
ts.sort()
fl = 2 * n**3
print(json.dumps({"fp64_dgemm_tflops_best": round(fl / ts[0] / 1e12, 2),
                  "fp64_dgemm_tflops_median": round(fl / ts[len(ts) // 2] / 1e12, 2), "n": n}))
