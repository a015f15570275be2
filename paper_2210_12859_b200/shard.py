"""Multi-GPU plumbing for the query-sharded path.

One process per GPU; torch.distributed carries the only exchange the path
has: the level-order tree is built once on rank 0 and broadcast (NCCL over
NVLink on the GPU box; gloo in the CPU tests).  Queries are independent, so
each rank walks its own contiguous block with no per-query communication,
and results land in disjoint slots.  Timing is reduced as the max over ranks.
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np


def shard_range(m: int, world: int, rank: int, align: int = 32) -> Tuple[int, int]:
    """Contiguous block of a batch of m walk positions for `rank`, block
    boundaries rounded to `align` (a warp) so no warp straddles two GPUs."""
    if world <= 1:
        return 0, m
    per = -(-m // world)
    per = -(-per // align) * align
    lo = min(m, rank * per)
    return lo, min(m, lo + per)


def query_stream(rank: int) -> int:
    """RNG stream of a rank's own queries in the weak-scaling bench: rank 0
    uses the reference's query stream (rng.hpp:24), others private streams."""
    return 2 if rank == 0 else 1000 + rank


def replicate_tree(nodes: Optional[np.ndarray], n: int, dim: int, device, group=None):
    """Broadcast the level-order array from rank 0; returns a tensor on
    `device` (CUDA for NCCL, CPU for gloo) holding the identical bytes."""
    import torch
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_rank(group) != 0:
        t = torch.empty((n, dim), dtype=torch.float32, device=device)
    else:
        t = torch.from_numpy(np.ascontiguousarray(nodes, np.float32)).to(device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(t, src=0, group=group)
    return t


def max_over_ranks(value: float, device, group=None) -> float:
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
