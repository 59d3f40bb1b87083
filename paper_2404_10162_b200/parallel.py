"""Multi-GPU plumbing for the decode path: problem configs are independent
(the reference stripes them over CPU threads, proj/src/eval.cpp:105-137), so
N GPUs take contiguous shards with no collective on the data path.  The only
collectives are outside the timed work: gathering decoded beams to rank 0 and
the max-over-ranks timing reduction.  One process per GPU (torchrun); NCCL on
GPU, gloo in the CPU tests.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(n: int, rank: int, world: int):
    """Balanced contiguous shard [lo, hi) of n items for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def weak_shard(per_rank: int, rank: int):
    """Weak scaling: every rank owns `per_rank` configs of a rank-major global batch."""
    return rank * per_rank, (rank + 1) * per_rank


def gather_rows(local: np.ndarray, n_total: int, world: int):
    """All-gathers row-sharded numpy arrays (balanced shards) into the global
    array on every rank, preserving config order."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    rows = [shard_bounds(n_total, r, world) for r in range(world)]
    width = max(hi - lo for lo, hi in rows)
    pad = np.zeros((width,) + local.shape[1:], local.dtype)
    pad[: len(local)] = local
    backend = dist.get_backend()
    dev = "cuda" if backend == "nccl" else "cpu"
    t = torch.from_numpy(pad).to(dev)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)
    parts = [o.cpu().numpy()[: hi - lo] for o, (lo, hi) in zip(outs, rows)]
    return np.concatenate(parts, 0)


def max_over_ranks(x: float, world: int) -> float:
    import torch
    import torch.distributed as dist

    if world == 1:
        return x
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
