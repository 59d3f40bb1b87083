"""Kernel timeline of one decode step (workload argv[1], default cfg2) (torch.profiler / CUPTI): per-kernel
durations and the idle gaps between consecutive kernels on the device."""
import collections
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2404_10162_b200 import _cabi  # noqa: E402
from paper_2404_10162_b200.synth import descriptors  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
bench.W = bench.WORKLOADS[wl]
bench.KERNEL, bench.BEAM = bench.W["kernel"], bench.W["beam"]
path = bench.model_path()
eng = _cabi.Engine(path, 0, "f16x3")
B = bench.W.get("configs", 65536)
K = bench.BEAM
tok = eng.encode(descriptors(B, bench.KERNEL))
with open(path, "rb") as f:
    head = f.read(8192).split(b"\n\n")[0].decode().split("\n")
names = [l.split(": ", 1)[1].split(" = ")[0] for l in head if l.startswith("param.")]
values = [[int(x) for x in l.split(" = ")[1].split(",")] for l in head if l.startswith("param.")]
preds = [] if bench.W["greedy"] else bench.predicates(names, values)
T = eng.T
d_tok = torch.from_numpy(tok).cuda()
d_out = {"tokens": torch.empty((B, K, T), dtype=torch.int32, device="cuda"),
         "log_prob": torch.empty((B, K), dtype=torch.float64, device="cuda"),
         "count": torch.empty(B, dtype=torch.int32, device="cuda"),
         "status": torch.empty(B, dtype=torch.int32, device="cuda"),
         "fail_pred": torch.empty(B, dtype=torch.int32, device="cuda"),
         "fail_step": torch.empty(B, dtype=torch.int32, device="cuda")}
ptrs = {k: v.data_ptr() for k, v in d_out.items()}
stream = torch.cuda.current_stream()
for _ in range(3):
    eng.beam_device(d_tok.data_ptr(), 0, B, K, preds, ptrs, stream.cuda_stream)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    eng.beam_device(d_tok.data_ptr(), 0, B, K, preds, ptrs, stream.cuda_stream)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev])
per = collections.defaultdict(float)
gaps = []
for i, (s, e, n) in enumerate(ev):
    per[n[:60]] += (e - s) / 1000.0
    if i:
        gaps.append((s - ev[i - 1][1]) / 1000.0)
span = (ev[-1][1] - ev[0][0]) / 1000.0
busy = sum(per.values())
print(f"kernels {len(ev)}  span {span:.3f} ms  busy {busy:.3f} ms  idle {span - busy:.3f} ms")
for n, t in sorted(per.items(), key=lambda x: -x[1]):
    print(f"  {t:8.3f} ms  {n}")
g = np.array(gaps)
print("largest gaps (ms):", np.round(np.sort(g)[-10:], 3).tolist())
for i in np.argsort(g)[-5:]:
    print(f"  gap {g[i]:.3f} ms after {ev[i][2][:50]} before {ev[i + 1][2][:50]}")
