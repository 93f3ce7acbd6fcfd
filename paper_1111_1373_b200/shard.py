"""Sample sharding across ranks / GPUs.

The partition is the reference's Proc. 3 contiguous-range rule
(eval_data_parallel.cpp:47-51) applied to devices: shard k of n
owns records [floor(k*m/n), floor((k+1)*m/n)).  The tree is replicated; the
only exchange is the label gather (a copy, not a reduction), so there is no
collective in the hot loop.
"""
from __future__ import annotations

from typing import List, Tuple


def shard_range(m: int, k: int, n: int) -> Tuple[int, int]:
    if n <= 0 or not (0 <= k < n):
        raise ValueError("shard index out of range")
    return (m * k) // n, (m * (k + 1)) // n


def shard_ranges(m: int, n: int) -> List[Tuple[int, int]]:
    return [shard_range(m, k, n) for k in range(n)]


def gather_labels(local, m: int, group=None):
    """Gather every rank's label shard into the full label vector on every
    rank (torch.distributed all_gather of equal-padded shards; NCCL over
    NVLink on GPUs, gloo on CPU).  ``local`` is this rank's 1-D int32 tensor."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(m, rank, world)
    assert local.numel() == hi - lo
    width = max(b - a for a, b in shard_ranges(m, world))
    buf = torch.zeros(width, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[: b - a] for p, (a, b) in zip(parts, shard_ranges(m, world))])
