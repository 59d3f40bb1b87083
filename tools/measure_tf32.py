"""TF32 dense tensor-core peak on this box, measured the way MEASURED_PEAKS.json
measures bf16: torch.matmul 8192^3 (2 N^3 FLOP), best of 10 (burst) and back to
back for 4 s (sustained), CUDA events.  Written to profiles/measured_tf32.json;
bench.py's training roofline divides by the sustained figure."""
import json
import os
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = True
torch.backends.cudnn.allow_tf32 = True
N = 8192
a = torch.randn(N, N, device="cuda")
b = torch.randn(N, N, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
best = 0.0
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a @ b
    e1.record()
    e1.synchronize()
    best = max(best, 2 * N ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
n, t0 = 0, time.perf_counter()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.perf_counter() - t0 < 4.0:
    a @ b
    n += 1
e1.record()
e1.synchronize()
sustained = n * 2 * N ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12
out = {"tf32_tflops": round(best, 1), "tf32_tflops_sustained": round(sustained, 1),
       "gpu_name": torch.cuda.get_device_name(0), "torch": torch.__version__,
       "how": "torch.matmul fp32 inputs with allow_tf32, 8192^3 (2*N^3): best of 10 (burst) and back to back for 4 s (sustained), CUDA events"}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "measured_tf32.json")
os.makedirs(os.path.dirname(path), exist_ok=True)
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out))
