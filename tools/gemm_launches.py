"""Per gate-GEMM launch of one decode (GPU box): CUDA-event ms, useful TFLOP/s
(reference formula) and issued TFLOP/s, for a workload's benched batch.

  python tools/gemm_launches.py [cfg2|cfg5|cfg1] [precision]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2404_10162_b200 import _cabi
    from paper_2404_10162_b200 import workloads as W

    wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    prec = sys.argv[2] if len(sys.argv) > 2 else "f16x3"
    w = W.WORKLOADS[wl]
    path = W.DEFAULT_CKPT if w["model"] == "default" else W.cfg5_checkpoint_ours()
    e = _cabi.Engine(path, 0, prec)
    B = w["configs"]
    tok = e.encode(e.synthetic(B, W.SEED, 0))
    preds = [] if w["greedy"] else W.predicate_dicts(path)
    k = max(1, w["beam"])
    d_tok = torch.from_numpy(tok).cuda()
    out = {"tokens": torch.empty((B, k, e.T), dtype=torch.int32, device="cuda"),
           "log_prob": torch.empty((B, k), dtype=torch.float64, device="cuda"),
           "count": torch.empty(B, dtype=torch.int32, device="cuda"),
           "status": torch.empty(B, dtype=torch.int32, device="cuda"),
           "fail_pred": torch.empty(B, dtype=torch.int32, device="cuda"),
           "fail_step": torch.empty(B, dtype=torch.int32, device="cuda")}
    ptrs = {kk: v.data_ptr() for kk, v in out.items()}
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        e.beam_device(d_tok.data_ptr(), 0, B, k, preds, ptrs, s)
    torch.cuda.synchronize()
    reps = int(os.environ.get("REPS", "5"))
    runs = []
    for _ in range(reps):  # median over repeated decodes (the clock under the power cap wanders)
        e.profile_reset(True)
        e.beam_device(d_tok.data_ptr(), 0, B, k, preds, ptrs, s)
        torch.cuda.synchronize()
        ms, fl, ex = e.profile_launches()
        e.profile_reset(False)
        runs.append(ms)
    ms = np.median(np.stack(runs), axis=0)
    for i in range(len(ms)):
        print(f"launch {i:2d}: {ms[i]:7.3f} ms  useful {fl[i] / ms[i] / 1e9:7.1f} TF/s  issued "
              f"{ex[i] / ms[i] / 1e9:7.1f} TF/s  useful {fl[i] / 1e12:6.3f} TFLOP")
    print(f"total {ms.sum():.3f} ms, useful {fl.sum() / ms.sum() / 1e9:.1f} TF/s, issued {ex.sum() / ms.sum() / 1e9:.1f}")


if __name__ == "__main__":
    main()
