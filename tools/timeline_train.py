"""Kernel timeline of one cfg4 training step (torch.profiler / CUPTI): busy vs
span on the device and the largest inter-kernel gaps."""
import collections
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2404_10162_b200.dptrain import DataParallelTrainer  # noqa: E402

bench.W = bench.WORKLOADS["cfg4"]
bench.KERNEL = bench.W["kernel"]
path = bench.model_path()
GB = bench.W["configs"]
tok, tgt, ck = bench.train_data(path, GB)
dp = DataParallelTrainer(path, 0, 1)
stream = torch.cuda.current_stream()
d_tok = torch.from_numpy(tok).cuda()
d_tgt = torch.from_numpy(tgt).cuda()
d_idx = torch.arange(0, GB, dtype=torch.int64, device="cuda")
for e in range(3):
    dp.step(d_tok, d_tgt, d_idx, GB, e + 1, 1, bench.TRAIN_LR, 5.0, stream)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    dp.step(d_tok, d_tgt, d_idx, GB, 9, 1, bench.TRAIN_LR, 5.0, stream)
    torch.cuda.synchronize()
ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
            if e.device_type == torch.autograd.DeviceType.CUDA)
per = collections.defaultdict(float)
gaps = []
for i, (s, e, n) in enumerate(ev):
    per[n[:60]] += (e - s) / 1000.0
    if i:
        gaps.append((s - ev[i - 1][1]) / 1000.0)
span = (ev[-1][1] - ev[0][0]) / 1000.0
print(f"kernels {len(ev)}  span {span:.3f} ms  busy {sum(per.values()):.3f} ms  gaps {sum(g for g in gaps if g > 0):.3f} ms")
for n, t in sorted(per.items(), key=lambda x: -x[1])[:12]:
    print(f"  {t:8.3f} ms  {n}")
