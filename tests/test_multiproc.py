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


def test_bench_self_spawn_two_ranks():
    """`bench.py --gpus 2` without torchrun re-launches itself as two ranks
    under torch.distributed.run (127.0.0.1 rendezvous): exercised here on CPU
    through the reference arm, which rank 0 alone runs and prints -- exactly
    one JSON line with n_gpus 2, every rank exits 0."""
    import json
    import subprocess
    import sys

    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--workload", "C1",
                        "--steps", "1", "--warmup", "3", "--ref-sample", "20000"],
                       cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def test_bench_rank_parity_hashes_cover_eight_ranks():
    """bench.py checks every rank's labels against the reference hash of its
    own batch: the committed golden file holds C2 / C4 hashes for ranks 0-7
    and all 64 C5 shards at every depth (rank 0 / shard 0 = Appendix A)."""
    import bench

    g = bench.golden()
    assert len(g["c2_ranks"]["labels_fnv"]) == 8 and len(g["c4_ranks"]["vote_fnv"]) == 8
    assert bench.golden_labels(bench.WORKLOADS["C2"], 0) == 0x9e7e87e9cc15c4e0
    assert int(g["c4_ranks"]["vote_fnv"][0], 16) == 0x1b2543c41e436ce0
    assert sorted(int(d) for d in g["c5"]["depths"]) == [8, 10, 12, 14, 16, 18, 20]
    for d, want in ((8, 0xa41b18f5886a3516), (12, 0x8a36c71851f61114), (16, 0x4bbe70e47d70a501),
                    (20, 0x894ffd1cd01ac0a5)):
        row = g["c5"]["depths"][str(d)]
        assert len(row["labels_fnv"]) == 64 and int(row["labels_fnv"][0], 16) == want
        assert bench.golden_labels(bench.WORKLOADS[f"C5d{d}"], 0) == want
    # Appendix A d_mu of shard 0
    assert abs(g["c5"]["depths"]["16"]["depth_sum"][0] / 15_625_000 - 7.7637) < 5e-5
    assert abs(g["c5"]["depths"]["20"]["depth_sum"][0] / 15_625_000 - 7.3201) < 5e-5
