"""Data-parallel teacher-forced training (BASELINE config 4) over the C-ABI
trainer (ks_trainer_*, paper_2404_10162_b200/csrc/ks_train.cu).

Reference: train_model (proj/src/models.cpp:862-969) sums per-sample gradients
over CPU worker threads (models.cpp:907-942), divides by the batch, clips to
global norm 5.0 and takes one Adam step.  Here one process per GPU owns a
contiguous shard of the global batch; each rank's summed gradients are
all-reduced (NCCL over NVLink via torch.distributed; gloo in the CPU tests)
and every rank applies the identical optimiser step to its replica -- the
all-reduce sits exactly where the reference's in-process gradient sum is.

Only plumbing lives here (buffers, streams, the collective); the math is the
CUDA trainer.  There is no CPU fallback.
"""
from __future__ import annotations

import numpy as np

from .parallel import shard_bounds


def shard_batch(global_batch: int, rank: int, world: int):
    """Rows [lo, hi) of the global batch owned by `rank` (balanced, contiguous)."""
    return shard_bounds(global_batch, rank, world)


def allreduce_sum(tensors, world: int):
    """Sum-all-reduce of per-rank gradient / statistics tensors in place
    (the reference's add_into over workers, models.cpp:936-942)."""
    if world == 1:
        return
    import torch.distributed as dist

    for t in tensors:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)


class DataParallelTrainer:
    """One replica per GPU.  `step` takes this rank's shard already on the
    device and returns nothing (statistics stay on the device until `stats`)."""

    def __init__(self, checkpoint: str, device: int = 0, world: int = 1):
        import torch

        from ._cabi import Trainer

        self.tr = Trainer(checkpoint, device)
        self.world = world
        self.grads = torch.empty(self.tr.num_params, dtype=torch.float32, device=f"cuda:{device}")
        self.loss = torch.zeros(1, dtype=torch.float64, device=f"cuda:{device}")
        self.match = torch.zeros(1, dtype=torch.int64, device=f"cuda:{device}")
        self.stats_buf = torch.zeros(2, dtype=torch.float64, device=f"cuda:{device}")

    @property
    def num_params(self) -> int:
        return self.tr.num_params

    def step(self, d_tok, d_tgt, d_idx, global_batch: int, epoch: int, seed: int, lr: float,
             clip: float = 5.0, stream=None):
        """d_tok / d_tgt / d_idx: torch CUDA tensors (this rank's shard)."""
        import torch

        s = stream if stream is not None else torch.cuda.current_stream()
        B = int(d_tok.shape[0])
        self.tr.loss_grads_device(d_tok.data_ptr(), d_tgt.data_ptr(),
                                  d_idx.data_ptr() if d_idx is not None else None, B, epoch, seed,
                                  self.grads.data_ptr(), 0, self.loss.data_ptr(), self.match.data_ptr(),
                                  s.cuda_stream)
        with torch.cuda.stream(s):
            self.stats_buf[0] = self.loss[0]
            self.stats_buf[1] = self.match[0].double()
            allreduce_sum([self.grads, self.stats_buf], self.world)
        self.tr.apply_device(self.grads.data_ptr(), global_batch, lr, clip, s.cuda_stream)

    def stats(self):
        """(global loss sum, global per-position argmax matches) of the last step."""
        v = self.stats_buf.cpu().numpy()
        return float(v[0]), int(v[1])

    def export(self) -> np.ndarray:
        return self.tr.export()
