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
    """Equal-count contiguous blocks: the first n % world ranks get one extra chain."""
    base, extra = divmod(n_chains, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


W_DSD = 1  # a speculative chain also draws its K_j (k_dsd_demand)


def chain_costs(grid) -> list:
    """SURVEY §8(e)'s cost estimate per timing chain: N (1 + w_DSD), N = requests of
    its trace, w_DSD = 1 for the speculative modes (DSD, co-located SpecDecode)."""
    return [grid.traces[c.trace_idx].n * (1 + (W_DSD if c.mode in (1, 3) else 0))
            for c in grid.chains]


def shard_bounds_cost(costs, world: int):
    """Contiguous blocks of chains, one per rank, minimising the largest block cost
    (the linear-partition problem: binary search on the bound, greedy packing).
    Deterministic; ranks past the last chain get empty blocks at the end."""
    costs = [int(c) for c in costs]
    n = len(costs)
    if n == 0:
        return [(0, 0)] * world

    def blocks(limit):  # greedy: fill each block up to `limit`
        out, lo, acc = [], 0, 0
        for i, c in enumerate(costs):
            if acc + c > limit and i > lo:
                out.append((lo, i))
                lo, acc = i, 0
            acc += c
        out.append((lo, n))
        return out

    lo_b, hi_b = max(costs), sum(costs)
    while lo_b < hi_b:
        mid = (lo_b + hi_b) // 2
        if len(blocks(mid)) <= world:
            hi_b = mid
        else:
            lo_b = mid + 1
    out = blocks(lo_b)
    # split the largest multi-chain blocks until every rank has one (keeps the bound)
    while len(out) < world and any(h - l > 1 for l, h in out):
        k = max(range(len(out)), key=lambda i: (out[i][1] - out[i][0] > 1,
                                                 sum(costs[out[i][0]:out[i][1]])))
        l, h = out[k]
        half, acc, m = sum(costs[l:h]) / 2, 0, l
        while m < h - 1 and acc + costs[m] <= half:
            acc += costs[m]
            m += 1
        m = max(m, l + 1)
        out[k:k + 1] = [(l, m), (m, h)]
    while len(out) < world:
        out.append((n, n))
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


def evaluate_sharded(n_chains: int, compute_shard, argmin, device, group=None, costs=None):
    """Host-side flow of one distributed evaluation.

    compute_shard(lo, hi, out_uint8[hi-lo, 80]) fills this rank's stats;
    argmin(full_stats_uint8[n_chains, 80]) runs Alg. 1.  Returns argmin's result.
    ``costs`` (one per chain, e.g. chain_costs(grid)) selects cost-balanced
    contiguous shards; without it the shards have equal counts.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bounds = shard_bounds(n_chains, world) if costs is None else shard_bounds_cost(costs, world)
    lo, hi = bounds[rank]
    max_shard = max(h - l for l, h in bounds)
    local = torch.zeros((max_shard, STATS_BYTES), dtype=torch.uint8, device=device)
    gathered = torch.empty((world * max_shard, STATS_BYTES), dtype=torch.uint8, device=device)
    if hi > lo:
        compute_shard(lo, hi, local[: hi - lo])
    full = all_gather_stats(local, gathered, bounds, n_chains, group)
    return argmin(full)
