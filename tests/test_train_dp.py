"""Data-parallel training plumbing on CPU (world_size 2, gloo): each rank
computes the summed gradients of its batch shard (the fp64 training oracle
stands in for the CUDA trainer here), `allreduce_sum` combines them, and the
result equals the full-batch sum -- then the optimiser step (÷ global batch,
clip, Adam) is identical on every rank.  Mirrors train_model's per-worker sum
(proj/src/models.cpp:907-947)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2404_10162_b200.dptrain import shard_batch
from tests.util import golden_path


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch(ck, B, seed):
    rng = np.random.default_rng(seed)
    tok = np.stack([rng.integers(0, len(ck.inputs[f]), B) for f in range(7)], 1)
    tgt = np.stack([rng.integers(0, v, B) for v in ck.vsizes], 1)
    return tok, tgt


def _worker(rank, world, port, B, out_dir):
    import torch
    import torch.distributed as dist

    from oracle import train_oracle as TO
    from paper_2404_10162_b200.dptrain import allreduce_sum, shard_batch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ck = TO.Checkpoint(golden_path("tiny_attn_s3423.ckpt"))
    tok, tgt = _batch(ck, B, 1)
    lo, hi = shard_batch(B, rank, world)
    loss, G, match = TO.loss_and_grads(ck, ck.tensors, tok[lo:hi], tgt[lo:hi])
    g = torch.from_numpy(ck.flat(G))
    stats = torch.tensor([loss, float(match)], dtype=torch.float64)
    allreduce_sum([g, stats], world)
    # identical optimiser step on every replica
    adam = TO.Adam(lr=3e-3)
    new = adam.apply(ck.flat(), TO.clip_global_norm(g.numpy() / B, 5.0))
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.concatenate([g.numpy(), stats.numpy(), new]))
    dist.barrier()
    dist.destroy_process_group()


def test_shards_partition_the_batch():
    for B in (1, 7, 4096):
        for world in (1, 2, 8):
            rows = [shard_batch(B, r, world) for r in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))


def test_two_rank_allreduce_equals_full_batch(tmp_path):
    from oracle import train_oracle as TO

    B = 13
    port = _free_port()
    mp.spawn(_worker, args=(2, port, B, str(tmp_path)), nprocs=2, join=True)
    ck = TO.Checkpoint(golden_path("tiny_attn_s3423.ckpt"))
    tok, tgt = _batch(ck, B, 1)
    loss, G, match = TO.loss_and_grads(ck, ck.tensors, tok, tgt)
    full = ck.flat(G)
    n = len(full)
    r0, r1 = (np.load(tmp_path / f"r{r}.npy") for r in range(2))
    np.testing.assert_array_equal(r0, r1)  # replicas stay identical
    np.testing.assert_allclose(r0[:n], full, rtol=1e-12, atol=1e-15)
    assert abs(r0[n] - loss) <= 1e-12 * loss and r0[n + 1] == match
    adam = TO.Adam(lr=3e-3)
    np.testing.assert_allclose(r0[n + 2:], adam.apply(ck.flat(), TO.clip_global_norm(full / B, 5.0)),
                               rtol=0, atol=1e-12)
