"""Multi-GPU plumbing for the query-sharded path.

One process per GPU; torch.distributed carries the exchanges (NCCL over
NVLink / NVSwitch on the GPU box; gloo in the CPU tests):

* the level-order tree is built once on rank 0 and broadcast
  (:func:`replicate_tree`);
* block sharding (default, no data-path collective): queries are
  independent, each rank walks its own contiguous block and results land in
  disjoint slots;
* Morton-range partition (optional, SURVEY §8(e) "then" step): the ranks
  split the key space of the whole batch into equal-count ranges
  (:func:`morton_range_owner` — one all-reduce of a key histogram), send
  every query to the rank that owns its key range and the answers back
  (:func:`MortonExchange` — two all-to-all rounds), so each GPU walks one
  1/G region of space and touches ~1/G of the tree's leaf levels.

Timing is reduced as the max over ranks.
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


# ---------------------------------------------------------------- Morton-range partition

def morton_range_owner(keys, key_bits: int, world: int, group=None, hist_bits: int = 16):
    """Owner rank of every bin of the top ``hist_bits`` key bits: the global
    histogram (all-reduce SUM over the ranks' local histograms) is cut into
    ``world`` equal-count ranges in key order; a bin belongs to the range its
    first element falls in.  Returns an int64 tensor of 2^hist_bits owners
    (identical on every rank)."""
    import torch
    import torch.distributed as dist

    hb = max(0, min(hist_bits, key_bits))
    top = (keys.to(torch.int64) >> (key_bits - hb)) if hb else torch.zeros_like(keys, dtype=torch.int64)
    hist = torch.bincount(top, minlength=1 << hb).to(torch.int64)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hist, group=group)
    total = int(hist.sum().item())
    first = torch.cumsum(hist, 0) - hist  # elements before each bin
    if total == 0:
        return torch.zeros(1 << hb, dtype=torch.int64, device=keys.device)
    return torch.clamp((first * world) // total, max=world - 1)


class MortonExchange:
    """Sends each local query to the rank owning its key range and brings
    the answers back to the original slots.

        ex = MortonExchange(queries, keys, key_bits, world, group)
        counts, hits = walk(ex.local_queries)        # this rank's key range
        counts, hits = ex.return_results(counts, hits, stride)

    ``queries`` (m, dim) and ``keys`` (m) live on the collective's device
    (CUDA for NCCL, CPU for gloo); the returned arrays are in the caller's
    original query order."""

    def __init__(self, queries, keys, key_bits: int, world: int, group=None, hist_bits: int = 16):
        import torch

        self.group = group
        self.world = world
        owner = morton_range_owner(keys, key_bits, world, group, hist_bits)
        hb = max(0, min(hist_bits, key_bits))
        top = (keys.to(torch.int64) >> (key_bits - hb)) if hb else torch.zeros_like(keys, dtype=torch.int64)
        dest = owner[top]
        self.order = torch.argsort(dest, stable=True)  # send order: grouped by destination
        self.send_counts = torch.bincount(dest, minlength=world).to(torch.int64)
        self.recv_counts = self._a2a_counts(self.send_counts)
        self.local_queries = self._a2a(queries[self.order].contiguous(), self.send_counts, self.recv_counts)

    def _a2a_counts(self, send):
        import torch
        import torch.distributed as dist

        if not (dist.is_initialized() and dist.get_world_size(self.group) > 1):
            return send.clone()
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=self.group)
        return recv

    def _a2a(self, x, send_counts, recv_counts):
        import torch
        import torch.distributed as dist

        if not (dist.is_initialized() and dist.get_world_size(self.group) > 1):
            return x
        out = torch.empty((int(recv_counts.sum().item()),) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        dist.all_to_all_single(out, x, output_split_sizes=recv_counts.tolist(),
                               input_split_sizes=send_counts.tolist(), group=self.group)
        return out

    def return_results(self, counts, hits, stride: int):
        """counts (m_local,) int32 and hits (m_local * stride,) 8-byte slots of
        the local walk -> the same arrays for the caller's original queries."""
        import torch

        c_back = self._a2a(counts.contiguous(), self.recv_counts, self.send_counts)
        h_back = self._a2a(hits.reshape(-1, stride).contiguous(), self.recv_counts, self.send_counts)
        out_c = torch.empty_like(c_back)
        out_h = torch.empty_like(h_back)
        out_c[self.order] = c_back
        out_h[self.order] = h_back
        return out_c, out_h.reshape(-1)
