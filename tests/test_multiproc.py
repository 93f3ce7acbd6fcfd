"""World-size-2 gloo tests of the N>1 host path (CPU): the Proc. 3 shard
ranges used by bench.py and st_eval_sharded, and the label gather."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1111_1373_b200.shard import gather_labels, shard_range, shard_ranges


def test_shard_ranges_cover_exactly():
    for m in (0, 1, 7, 100, 15_625_000, 10**9):
        for n in (1, 2, 3, 4, 8):
            r = shard_ranges(m, n)
            assert r[0][0] == 0 and r[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(m, rank, world)
        # stand-in for this rank's kernel output: label = record index * 7 mod 13
        local = torch.arange(lo, hi, dtype=torch.int64).mul_(7).remainder_(13).to(torch.int32)
        full = gather_labels(local, m)
        # max-over-ranks timing reduction used by bench.py
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, full.numpy().tobytes(), float(t.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m", [(2, 1001), (2, 2), (3, 100)])
def test_gloo_label_gather(world, m):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, q)) for r in range(world)]
    [p.start() for p in procs]
    res = [q.get(timeout=120) for _ in procs]
    [p.join(timeout=60) for p in procs]
    want = (np.arange(m, dtype=np.int64) * 7 % 13).astype(np.int32)
    for rank, buf, tmax in res:
        assert np.array_equal(np.frombuffer(buf, dtype=np.int32), want)
        assert tmax == float(world)
