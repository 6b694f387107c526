"""Input (batch) sharding across GPUs — the only multi-GPU structure the path needs.

Every input's hidden state H_b is private and every output row b*x + k depends
only on (H_b, Y_{b,k}, weights), so a batch of B inputs is
split into contiguous blocks, one per rank, and each rank runs its decode steps
with no collective.  After the step, one all_gather brings the output rows to
every rank (NCCL over NVLink on GPUs; gloo on CPU for the tests).  Weights are
replicated.
"""
from __future__ import annotations

from typing import Tuple


def shard_range(B: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [b0, b1) of inputs owned by `rank` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(B, world)
    b0 = rank * base + min(rank, extra)
    return b0, b0 + base + (1 if rank < extra else 0)


def gather_outputs(local_out, B: int, x: int, group=None):
    """All-gather per-rank output rows [B_local*x, d_m] into the full [B*x, d_m] in
    input order.  Uneven shards are padded to the largest shard for the collective."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    d_m = local_out.shape[1]
    sizes = [shard_range(B, r, world) for r in range(world)]
    max_rows = max(b1 - b0 for b0, b1 in sizes) * x
    b0, b1 = sizes[rank]
    if local_out.shape[0] != (b1 - b0) * x:
        raise ValueError("local output rows do not match this rank's shard")
    padded = local_out.new_zeros((max_rows, d_m))
    padded[: local_out.shape[0]] = local_out
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[: (e - s) * x] for p, (s, e) in zip(parts, sizes)], dim=0)
