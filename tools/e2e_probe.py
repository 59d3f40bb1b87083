import time, numpy as np, sys, os
sys.path.insert(0, "/root/repo")
import bench
from paper_2404_10162_b200 import _cabi
from paper_2404_10162_b200.synth import descriptors
path = bench.model_path()
eng = _cabi.Engine(path, 0, "f16x3")
B = 65536
tok = eng.encode(descriptors(B, bench.KERNEL))
with open(path, "rb") as f:
    head = f.read(8192).split(b"\n\n")[0].decode().split("\n")
names = [l.split(": ", 1)[1].split(" = ")[0] for l in head if l.startswith("param.")]
values = [[int(x) for x in l.split(" = ")[1].split(",")] for l in head if l.startswith("param.")]
preds = bench.predicates(names, values)
out = None
for i in range(8):
    t0 = time.perf_counter()
    r = eng.beam(tok, 5, None, preds, out=out)
    out = r
    dt = time.perf_counter() - t0
    print(f"call {i}: {dt*1e3:.2f} ms")
import torch
d_tok = torch.from_numpy(tok).cuda()
T = eng.T
d_out = {"tokens": torch.empty((B, 5, T), dtype=torch.int32, device="cuda"), "log_prob": torch.empty((B, 5), dtype=torch.float64, device="cuda"),
         "count": torch.empty(B, dtype=torch.int32, device="cuda"), "status": torch.empty(B, dtype=torch.int32, device="cuda"),
         "fail_pred": torch.empty(B, dtype=torch.int32, device="cuda"), "fail_step": torch.empty(B, dtype=torch.int32, device="cuda")}
ptrs = {k: v.data_ptr() for k, v in d_out.items()}
for i in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    eng.beam_device(d_tok.data_ptr(), 0, B, 5, preds, ptrs, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize(); print(f"device {i}: {(time.perf_counter()-t0)*1e3:.2f} ms")
