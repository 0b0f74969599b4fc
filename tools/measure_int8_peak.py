"""Measures the dense int8 tensor-core peak on this B200 with cuBLASLt
(torch._int_mm, s8 x s8 -> s32), burst (best of 10) and sustained (4 s loop),
the same way the driver measures bf16 for MEASURED_PEAKS.json.  Writes
profiles/int8_peak.json; bench.py uses it as the GEMM roofline denominator."""
import json
import os
import time

import torch

N = 8192
a = torch.randint(-128, 127, (N, N), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (N, N), dtype=torch.int8, device="cuda")
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
ops = 2.0 * N ** 3
burst = ops / (best / 1e3) / 1e12
t0 = time.time()
n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    for _ in range(20):
        torch._int_mm(a, b)
    n += 20
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
sustained = ops * n / (e0.elapsed_time(e1) / 1e3) / 1e12
out = {"int8_tops_burst": burst, "int8_tops_sustained": sustained,
       "how": f"torch._int_mm (cuBLASLt s8xs8->s32) {N}^3, 2*N^3 ops: best of 10 (burst), 4 s back-to-back (sustained)",
       "gpu": torch.cuda.get_device_name()}
os.makedirs(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles"), exist_ok=True)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "int8_peak.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out))
