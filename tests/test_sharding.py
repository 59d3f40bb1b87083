"""Multi-process (world_size 2, gloo, CPU) coverage of the sharding plumbing
used by bench.py and the batched API: shards partition the configs, gathers
preserve config order, timing reduces with MAX."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2404_10162_b200.parallel import shard_bounds, weak_shard


def test_shard_bounds_partition():
    for n in (0, 1, 7, 65536, 1048577):
        for world in (1, 2, 3, 8):
            got = [shard_bounds(n, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [hi - lo for lo, hi in got]
            assert max(sizes) - min(sizes) <= 1
    assert weak_shard(65536, 3) == (196608, 262144)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out_dir):
    import torch.distributed as dist

    from paper_2404_10162_b200.parallel import gather_rows, max_over_ranks, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_bounds(n, rank, world)
    # stand-in for a per-rank decode: rows carry their global config index
    local = np.stack([np.arange(lo, hi), np.arange(lo, hi) * 3], 1).astype(np.int64)
    full = gather_rows(local, n, world)
    t = max_over_ranks(float(rank + 1) * 1.5, world)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.concatenate([full.ravel(), [int(t * 10)]]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [5, 1001])
def test_two_rank_gather_and_max(tmp_path, n):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, n, str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        a = np.load(tmp_path / f"r{r}.npy")
        full, t = a[:-1].reshape(n, 2), a[-1]
        assert (full[:, 0] == np.arange(n)).all() and (full[:, 1] == 3 * np.arange(n)).all()
        assert t == 30  # max(1.5, 3.0) * 10
