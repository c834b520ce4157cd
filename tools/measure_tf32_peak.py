"""Measure the dense TF32 tensor peak the way MEASURED_PEAKS.json measures bf16:
torch.matmul of fp32 8192^3 with TF32 allowed (cuBLAS, tcgen05 kind::tf32),
best of 10 (burst) and back to back for 4 s (sustained).  Writes
profiles/measured_tf32.json, which bench.py uses as the 3xTF32/TF32 roof."""
import json
import time
from pathlib import Path

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
burst = 2 * n ** 3 / (best / 1e3) / 1e12
t0 = time.time()
cnt = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    for _ in range(10):
        a @ b
    cnt += 10
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
sustained = 2 * n ** 3 * cnt / (e0.elapsed_time(e1) / 1e3) / 1e12
out = {"tf32_tflops": burst, "tf32_tflops_sustained": sustained,
       "how": "torch.matmul fp32 8192^3 with allow_tf32 (cuBLAS): best of 10 (burst) and back to back for 4 s (sustained)",
       "gpu": torch.cuda.get_device_name(0)}
# under gpurun only gpurun_out/ comes back: write there too and copy it into profiles/
for d in ("profiles", "gpurun_out"):
    Path(d).mkdir(exist_ok=True)
    Path(d, "measured_tf32.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out))
