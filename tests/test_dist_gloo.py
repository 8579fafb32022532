"""Multi-rank host logic of the sharded evaluation on CPU (gloo, world 2, 3 and 4).

The shard computation is substituted by oracle statistics (no GPU here); what
is tested is the product's sharding, the single all_gather of 80-byte records
and the reassembly that every rank feeds to Alg. 1 (T5 in SURVEY.md §4).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_20322_b200.dist import (chain_costs, evaluate_sharded, shard_bounds,
                                        shard_bounds_cost)

STATS_DTYPE = np.dtype([("n", "<i8"), ("slo_ok", "<i8"), ("tokens", "<i8"),
                        ("busy_new_us", "<i8"), ("busy_old_us", "<i8"), ("e_new_uj", "<i8"),
                        ("e_old_uj", "<i8"), ("makespan_us", "<i8"), ("req_hash", "<u8"),
                        ("status", "<u4"), ("capacity_ok", "<u4")])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_records(grid):
    from oracle import oracle as O
    rec = np.zeros(len(grid.chains), STATS_DTYPE)
    for i, ch in enumerate(grid.chains):
        st, _, _ = O.simulate_chain(grid.traces[ch.trace_idx], ch, False)
        for f in STATS_DTYPE.names:
            rec[i][f] = st[f]
    return rec


def _alg1(grid, rec):
    from oracle import oracle as O
    rows, cols = grid.rows, grid.cols
    total = np.zeros((rows, cols))
    ok = np.zeros((rows, cols), np.int64)
    n = np.ones((rows, cols), np.int64)
    pres = np.zeros((rows, cols), np.uint8)
    cap = np.zeros((rows, cols), np.uint8)
    cells = grid.cell_chain.reshape(rows, cols)
    for r in range(rows):
        sc = grid.scenarios[grid.row_scenario[r]]
        for c in range(cols):
            k = cells[r, c]
            if k < 0:
                continue
            d = {f: int(rec[k][f]) for f in STATS_DTYPE.names}
            ch = grid.chains[k]
            total[r, c] = O.carbon(d, ch.ce_new_g, ch.ce_old_g, *sc)[2]
            ok[r, c], n[r, c], pres[r, c], cap[r, c] = d["slo_ok"], d["n"], 1, ch.capacity_ok
    return O.alg1(total, ok, n, pres, cap, grid.slo_num, grid.slo_den, grid.priority,
                  grid.default_col)


def _worker(rank, world, port, n_chains_take, result_dir, cost_balanced=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2412_20322_b200.inputs import build_config, subset_chains
    grid = build_config(2, n=300)
    grid = subset_chains(grid, range(n_chains_take))
    rec = _oracle_records(grid)
    computed = []

    def compute(lo, hi, out):
        computed.append((lo, hi))
        out.copy_(torch.from_numpy(rec[lo:hi].view(np.uint8).reshape(hi - lo, 80).copy()))

    full_holder = {}

    def argmin(full):
        full_holder["full"] = full.numpy().copy()
        return _alg1(grid, full.numpy().view(STATS_DTYPE).reshape(-1))

    choice, fb = evaluate_sharded(len(grid.chains), compute, argmin, torch.device("cpu"),
                                  costs=chain_costs(grid) if cost_balanced else None)
    np.savez(os.path.join(result_dir, f"r{rank}.npz"), full=full_holder["full"], choice=choice,
             fb=fb, computed=np.array(computed))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_chains,cost", [(2, 40, False), (2, 5, False), (3, 40, False),
                                                (3, 7, False), (4, 40, False), (4, 3, False),
                                                (2, 40, True), (3, 7, True), (4, 3, True)])
def test_sharded_gather_matches_single_process(tmp_path, world, n_chains, cost):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, n_chains, str(tmp_path), cost), nprocs=world, join=True)
    from paper_2412_20322_b200.inputs import build_config, subset_chains
    grid = subset_chains(build_config(2, n=300), range(n_chains))
    rec = _oracle_records(grid)
    want_c, want_f = _alg1(grid, rec)
    bounds = shard_bounds_cost(chain_costs(grid), world) if cost else shard_bounds(n_chains, world)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        assert z["full"].tobytes() == rec.view(np.uint8).tobytes()
        assert np.array_equal(z["choice"], want_c) and np.array_equal(z["fb"], want_f)
        lo, hi = bounds[r]
        if hi > lo:
            assert z["computed"].tolist() == [[lo, hi]]


def test_shard_bounds():
    for n in (1, 5, 64, 320):
        for w in (1, 2, 3, 4, 8):
            b = shard_bounds(n, w)
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            sizes = [h - l for l, h in b]
            assert max(sizes) - min(sizes) <= 1


def test_shard_bounds_cost_optimal_and_contiguous():
    """The cost-balanced partition is contiguous, covers every chain,
    gives every rank a block, and its largest block cost equals the brute-force
    optimum over all contiguous partitions."""
    import itertools
    rng = np.random.default_rng(3)
    for _ in range(200):
        n = int(rng.integers(1, 9))
        w = int(rng.integers(1, 5))
        costs = rng.integers(1, 20, n).tolist()
        b = shard_bounds_cost(costs, w)
        assert len(b) == w and b[0][0] == 0 and b[-1][1] == n
        assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
        assert all(h >= l for l, h in b)
        if n >= w:
            assert all(h > l for l, h in b)
        got = max(sum(costs[l:h]) for l, h in b)
        best = sum(costs)
        for cuts in itertools.combinations(range(1, n), min(w, n) - 1):
            edges = [0, *cuts, n]
            best = min(best, max(sum(costs[edges[i]:edges[i + 1]]) for i in range(len(edges) - 1)))
        assert got == best, (costs, w, b)


def test_chain_costs_weights_speculative_chains():
    from paper_2412_20322_b200.inputs import build_config
    g = build_config(4, n=1000)
    c = chain_costs(g)
    for ch, x in zip(g.chains, c):
        assert x == (2000 if ch.mode in (1, 3) else 1000)
    b = shard_bounds_cost(c, 8)
    assert [h - l for l, h in b] == [8] * 8  # alternating DPD / DSD: equal blocks
