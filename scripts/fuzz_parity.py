"""Randomised parity campaign on a B200 (test infrastructure: imports oracle/ through
tests/oracle_pool.py): random grids mixing every mode, caps on both sides of the
32-lane boundary, stage groups (chains with identical tables on one trace, so
secondaries are cloned), DSD families (several (alpha, gamma) on one set of draws),
bursts, o = 1 requests, far gaps, with or without co-located chains (which switches
the deferred DSD demand off), and a random launch-order hint; some grids also go
through gl_link_demand (random payloads and windows) against oracle_link_demand.
Each grid also carries a random Alg. 1 matrix (scenarios, absent cells, capacity
flags, SLO targets from easy to impossible, both fallback priorities) for
gl_argmin_feasible, and some go end to end through gl_evaluate_host.  Every request's
(TTFT, finish), every chain statistic, every link field, every carbon cell (bit for
bit), choice and fallback flag must equal the oracle's.

usage: python scripts/fuzz_parity.py [seconds] [seed]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from oracle import oracle as O  # noqa: E402
from paper_2412_20322_b200 import api  # noqa: E402
from paper_2412_20322_b200.inputs import GridSpec, custom_trace  # noqa: E402
from tests import oracle_pool  # noqa: E402
from tests.helpers import make_chain, make_tables  # noqa: E402

INT_FIELDS = ("n", "slo_ok", "tokens", "busy_new_us", "busy_old_us", "e_new_uj", "e_old_uj",
              "makespan_us", "req_hash", "status", "capacity_ok")


def random_grid(rng):
    traces, chains = [], []
    colo = rng.random() < 0.3
    for t in range(int(rng.integers(1, 6))):
        n = int(rng.choice([1, 2, 31, 128, 129, 700, 2500, 6000]))
        gaps = rng.exponential(float(rng.choice([20, 200, 2000, 20000])), n)
        if rng.random() < 0.2:
            gaps[rng.integers(0, n)] += 3e9  # a gap beyond 2^31 us
        a = np.cumsum(gaps).astype(np.int64)
        if rng.random() < 0.3:
            a[: n // 3] = a[0]  # a burst
            a = np.sort(a)
        P = 8
        p = rng.integers(1, P + 1, n)
        o = rng.integers(1, int(rng.choice([4, 40, 300])), n)
        o[rng.random(n) < 0.1] = 1
        traces.append(custom_trace(a, p, o))
        for _ in range(int(rng.integers(1, 4))):  # stage groups: shared tables
            cap = int(rng.choice([1, 2, 5, 16, 31, 32, 40, 64, 100, 256]))
            tab = make_tables(P, cap, rng.integers(1, 400, P + 1), rng.integers(0, 300, P + 1),
                              np.sort(rng.integers(5, 900, cap + 1)),
                              b2=rng.integers(0, 50, P + 1), e1=rng.integers(0, 999, P + 1),
                              e2=rng.integers(0, 999, P + 1), sbn=rng.integers(0, 50, cap + 1),
                              sbo=rng.integers(0, 50, cap + 1), sen=rng.integers(0, 9999, cap + 1),
                              seo=rng.integers(0, 9999, cap + 1))
            slo = dict(ttft_slo=int(rng.integers(100, 50000)), tpot_slo=int(rng.integers(10, 2000)))
            modes = [0, 1] + ([2, 3] if colo else [])
            for _ in range(int(rng.integers(1, 5))):
                mode = int(rng.choice(modes))
                spec = mode in (1, 3)
                gamma = int(rng.integers(1, 9)) if spec else 0
                alpha = float(rng.choice([0.0, 0.5, 0.6, 0.8, 0.9, 1.0])) if spec else 0.0
                chains.append(make_chain(tab, mode, cap, gamma, alpha, seed=0xF00D + t,
                                         trace_idx=t, **slo))
    # an Alg. 1 grid over the chains: random scenarios (CI, lifetimes), rows x cols cells
    # (absent ones included), random capacity flags, both fallback priorities, and SLO
    # targets from easy to impossible (the fallback path)
    k = len(chains)
    for c in chains:
        c.capacity_ok = int(rng.random() < 0.9)
    S = int(rng.integers(1, 5))
    yr = 365 * 24 * 3600.0
    scen = np.stack([rng.choice([0.0, 17.0, 261.0, 501.0, 1000.0], S),
                     rng.uniform(1, 10, S) * yr, rng.uniform(1, 10, S) * yr], axis=1)
    cols = int(rng.integers(1, 7))
    rows = int(rng.integers(1, 9))
    cells = rng.integers(0, k, rows * cols).astype(np.int32)
    cells[rng.random(rows * cols) < 0.15] = -1
    target = [(9, 10), (1, 2), (1, 1), (0, 1)][int(rng.integers(0, 4))]
    prio = int(rng.integers(0, 2))
    return GridSpec("fuzz", traces, chains, scen, rng.integers(0, S, rows).astype(np.int32),
                    cells, rows, cols, slo_num=target[0], slo_den=target[1], priority=prio,
                    default_col=int(rng.integers(-1, cols)))


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 600.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    t0 = time.time()
    grids = chains = reqs = links = e2e = 0
    while time.time() - t0 < budget:
        g = random_grid(rng)
        dg = api.DeviceGrid(g)
        nc = len(g.chains)
        hint = None
        if nc >= 2 and rng.random() < 0.5:
            lo = int(rng.integers(0, nc - 1))
            hint = (lo, int(rng.integers(lo + 1, nc + 1)))
        stats, pr = api.eval_grid(dg, per_request=True, schedule=hint or False)
        torch.cuda.synchronize()
        st = api.stats_numpy(stats)
        ref = oracle_pool.evaluate_grid(g, gpu_per_request=pr.cpu().numpy())
        for ci in range(nc):
            for f in INT_FIELDS:
                if int(st[ci][f]) != int(ref["stats"][ci][f]):
                    raise SystemExit(f"MISMATCH grid {grids} seed {seed} chain {ci} {f}: "
                                     f"{int(st[ci][f])} != {int(ref['stats'][ci][f])} (hint {hint})")
        if ref["mismatch"]:
            raise SystemExit(f"MISMATCH grid {grids} seed {seed} rows: "
                             f"{dict(list(ref['mismatch'].items())[:2])} (hint {hint})")
        # Alg. 1 on the grid (gl_argmin_feasible): carbon bit for bit, choice, fallback
        carbon, choice, fb = api.argmin_feasible(dg, stats)
        m = ref["present"].astype(bool)
        if not (np.array_equal(carbon.cpu().numpy()[m], ref["carbon"][m]) and
                np.array_equal(choice.cpu().numpy(), ref["choice"]) and
                np.array_equal(fb.cpu().numpy(), ref["via_fallback"])):
            raise SystemExit(f"ALG1 MISMATCH grid {grids} seed {seed}")
        if rng.random() < 0.1:  # end to end from host buffers, same answers
            res = api.evaluate_host(dg, dg.pinned_traces(), want_carbon=True,
                                    schedule=hint or False)
            if not (np.array_equal(res.stats.view(np.uint8).reshape(nc, -1), stats.cpu().numpy())
                    and np.array_equal(res.choice, ref["choice"])):
                raise SystemExit(f"E2E MISMATCH grid {grids} seed {seed}")
            e2e += 1
        if rng.random() < 0.15 and not any(c.mode in (2, 3) for c in g.chains):
            # gl_link_demand (NEXT #2) with random payloads and window, chain by chain
            window = int(rng.choice([1, 1000, 250_000, 1_000_000]))
            params = [(int(rng.integers(0, 5000)), int(rng.integers(0, 9000))) for _ in range(nc)]
            _, link = api.link_demand(dg, window, params=params)
            torch.cuda.synchronize()
            lk = api.link_numpy(link)
            for ci, ch in enumerate(g.chains):
                want = O.link_demand(g.traces[ch.trace_idx], ch, window, *params[ci])
                for f in ("total_bytes", "peak_bytes", "peak_t_us", "n_impulses"):
                    if int(lk[ci][f]) != want[f]:
                        raise SystemExit(f"LINK MISMATCH grid {grids} seed {seed} chain {ci} {f}: "
                                         f"{int(lk[ci][f])} != {want[f]}")
            links += 1
        grids += 1
        chains += nc
        reqs += sum(g.traces[c.trace_idx].n for c in g.chains)
        if grids % 20 == 0:
            print(f"{time.time() - t0:7.1f} s: {grids} grids, {chains} chains, {reqs} chain-requests, "
                  "all equal", flush=True)
    print(f"fuzz_parity seed {seed}: {grids} random grids ({links} also through gl_link_demand, "
          f"{e2e} through gl_evaluate_host), {chains} chains, {reqs} chain-requests: every "
          "request, statistic, link field, carbon cell (bit for bit), choice and fallback flag "
          "equal to the oracle")


if __name__ == "__main__":
    main()
