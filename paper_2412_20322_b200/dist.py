"""Multi-GPU sharding of timing chains.

Timing chains are independent; CI/lifetime scenarios only enter the Alg. 1
epilogue.  Each rank simulates a contiguous block of chains, then ONE
all_gather of the 80-byte gl_chain_stats records (NCCL over NVLink on the GPU
box, gloo in the CPU tests) gives every rank all statistics, and every rank
runs gl_argmin_feasible on the full grid -> identical Optimal on all ranks.
Integers on the wire make the result bit-identical for any world size.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

STATS_BYTES = 80


def shard_bounds(n_chains: int, world: int):
    """Balanced contiguous blocks: the first n % world ranks get one extra chain."""
    base, extra = divmod(n_chains, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def all_gather_stats(local: torch.Tensor, gathered: torch.Tensor, bounds, n_chains: int,
                     group=None) -> torch.Tensor:
    """local: uint8 [max_shard, 80] (this rank's chains first); gathered: uint8
    [world * max_shard, 80] scratch.  Returns the [n_chains, 80] stats in chain
    order (a view when the shards are even, else a compacted copy)."""
    dist.all_gather_into_tensor(gathered, local, group=group)
    max_shard = local.shape[0]
    if all(hi - lo == max_shard for lo, hi in bounds):
        return gathered[:n_chains]
    parts = [gathered[r * max_shard: r * max_shard + (hi - lo)] for r, (lo, hi) in enumerate(bounds)]
    return torch.cat(parts, dim=0)


def evaluate_sharded(n_chains: int, compute_shard, argmin, device, group=None):
    """Host-side flow of one distributed evaluation.

    compute_shard(lo, hi, out_uint8[hi-lo, 80]) fills this rank's stats;
    argmin(full_stats_uint8[n_chains, 80]) runs Alg. 1.  Returns argmin's result.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bounds = shard_bounds(n_chains, world)
    lo, hi = bounds[rank]
    max_shard = max(h - l for l, h in bounds)
    local = torch.zeros((max_shard, STATS_BYTES), dtype=torch.uint8, device=device)
    gathered = torch.empty((world * max_shard, STATS_BYTES), dtype=torch.uint8, device=device)
    if hi > lo:
        compute_shard(lo, hi, local[: hi - lo])
    full = all_gather_stats(local, gathered, bounds, n_chains, group)
    return argmin(full)
