"""CUDA path (through the C ABI) vs the CPU oracle, element by element.

Integer results (per-request TTFT / finish, every chain statistic, Alg. 1
choice) must be bit-exact; fp64 carbon must be within 1e-9 relative (it is
bit-identical by construction: same expression order, no contraction).
"""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_20322_b200 import api
from paper_2412_20322_b200 import native as N
from paper_2412_20322_b200.inputs import (MODE_DPD, MODE_DSD, MODE_SPEC_COLO, MODE_STANDALONE,
                                          GridSpec, build_config, custom_trace, subset_chains)

ALL_MODES = (MODE_DPD, MODE_DSD, MODE_STANDALONE, MODE_SPEC_COLO)
from tests import oracle_pool
from tests.helpers import make_chain, make_tables, random_case

pytestmark = pytest.mark.gpu

INT_FIELDS = ("n", "slo_ok", "tokens", "busy_new_us", "busy_old_us", "e_new_uj", "e_old_uj",
              "makespan_us", "req_hash", "status", "capacity_ok")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    N.lib()


def grid_of(pairs, name="cases"):
    """GridSpec with one trace and one chain per (trace, chain) pair, one row per chain."""
    traces, chains = [], []
    for i, (tr, ch) in enumerate(pairs):
        traces.append(tr)
        chains.append(dataclasses.replace(ch, trace_idx=i))
    k = len(chains)
    lt = 7 * 365 * 24 * 3600.0
    return GridSpec(name, traces, chains, np.array([[261.0, lt, lt]]), np.zeros(k, np.int32),
                    np.arange(k, dtype=np.int32), k, 1)


_LAST_PER_TOKEN = {}


def run_gpu(g, per_request=True):
    dg = api.DeviceGrid(g)
    stats, pr = api.eval_grid(dg, per_request=per_request)
    ptok = torch.empty((g.rows, g.cols), dtype=torch.float64, device="cuda")
    carbon, choice, fb = api.argmin_feasible(dg, stats, per_token_out=ptok)
    torch.cuda.synchronize()
    _LAST_PER_TOKEN["v"] = ptok.cpu().numpy()
    return (api.stats_numpy(stats), None if pr is None else pr.cpu().numpy(),
            carbon.cpu().numpy(), choice.cpu().numpy(), fb.cpu().numpy())


def assert_parity(g, chain_ids=None, per_request=True, check_grid=True):
    """Every chain's statistics (and, with per_request, every request's (ttft,
    finish)) against the oracle -- fanned over all host cores (tests/oracle_pool.py)
    -- then, over the whole grid, carbon bit for bit, choice and via_fallback."""
    st, pr, carbon, choice, fb = run_gpu(g, per_request)
    ids = range(len(g.chains)) if chain_ids is None else chain_ids
    ref = oracle_pool.evaluate_grid(g, chain_ids=ids, gpu_per_request=pr if per_request else None)
    for ci in ids:
        want = ref["stats"][ci]
        for f in INT_FIELDS:
            assert int(st[ci][f]) == int(want[f]), (g.name, ci, f, int(st[ci][f]), int(want[f]))
    assert not ref["mismatch"], (g.name, dict(list(ref["mismatch"].items())[:3]))
    if check_grid and chain_ids is None:
        m = ref["present"].astype(bool)
        assert np.array_equal(carbon[m], ref["carbon"][m])  # bit-identical (R34)
        np.testing.assert_allclose(carbon[m], ref["carbon"][m], rtol=1e-9)
        # carbon per token: one division after the total, bit-identical too
        ptok = _LAST_PER_TOKEN["v"]
        assert np.array_equal(ptok[m], ref["carbon_per_token"][m], equal_nan=True)
        assert np.all(np.isnan(ptok[~m]))
        assert np.array_equal(choice, ref["choice"])
        assert np.array_equal(fb, ref["via_fallback"])
    return st


# ----------------------------------------------------------- random tiny cases
def test_random_tiny_cases_vs_oracle():
    rng = np.random.default_rng(20322)
    pairs = [random_case(rng) for _ in range(400)]
    assert_parity(grid_of(pairs), check_grid=True)


@pytest.mark.parametrize("cap", [1, 2, 3, 16, 31, 32, 33, 64, 100, 128, 200, 256])
def test_caps_and_slot_layouts(cap):
    """SPL = 1/2/4/8 slots per lane, caps at and across the 32-lane boundaries."""
    rng = np.random.default_rng(cap)
    pairs = []
    for mode in ALL_MODES:
        for n in (1, 7, 129, 1000):
            tr, ch = random_case(rng, n=n, mode=mode, cap=cap)
            a = np.sort(rng.integers(0, 40 * n, n))  # dense enough to fill big batches
            pairs.append((custom_trace(a, tr.prompt_len, tr.output_len), ch))
    assert_parity(grid_of(pairs))


def test_medium_random_traces():
    """Several chunks, ring wrap-around, ragged tails, mixed o = 1."""
    rng = np.random.default_rng(5)
    pairs = []
    for n in (127, 128, 129, 255, 256, 257, 1000, 4099, 20000):
        for mode in ALL_MODES:
            tr, ch = random_case(rng, n=n, mode=mode, cap=int(rng.integers(1, 40)))
            a = np.sort(rng.integers(0, int(rng.integers(1, 200)) * n, n))
            pairs.append((custom_trace(a, tr.prompt_len, tr.output_len), ch))
    assert_parity(grid_of(pairs))


# ------------------------------------------------------------------ edge cases
def _edge_chain(cap=4, mode=MODE_DPD, gamma=0, alpha=0.0, t2zero=False, max_prompt=8, **kw):
    tab = make_tables(max_prompt, cap, lambda p: 10 * p, (lambda p: 0) if t2zero else (lambda p: 3 * p),
                      [0] + [20 + b for b in range(1, cap + 1)], e1=lambda p: 7 * p,
                      b2=lambda p: p, e2=lambda p: 2 * p, sbn=[0] + [5] * cap,
                      sbo=[0] + [20 + b for b in range(1, cap + 1)], sen=[0] + [9] * cap,
                      seo=[0] + [11 * b for b in range(1, cap + 1)])
    return make_chain(tab, mode, cap, gamma, alpha, ttft_slo=300, tpot_slo=40, **kw)


def test_edge_cases():
    pairs = []
    # one request; o = 1 everywhere; equal arrivals; cap = 1; cap >= N
    pairs.append((custom_trace([5], [3], [4]), _edge_chain()))
    pairs.append((custom_trace([0, 0, 0, 0, 9], [1, 2, 3, 4, 5], [1, 1, 1, 1, 1]), _edge_chain()))
    pairs.append((custom_trace([0] * 300, [2] * 300, [5] * 300), _edge_chain(cap=1)))
    pairs.append((custom_trace(np.arange(50), [1] * 50, [3] * 50), _edge_chain(cap=256)))
    # all-zero stage-2 table; r == boundary ties
    pairs.append((custom_trace(np.arange(0, 2000, 21), [1] * 96, [4] * 96), _edge_chain(t2zero=True)))
    # DSD alpha 0 / 1, gamma 1 / 16
    for g, a in ((1, 0.0), (1, 1.0), (16, 1.0), (16, 0.5), (4, 0.8)):
        pairs.append((custom_trace(np.arange(0, 3000, 13), [2] * 231, [1 + (i % 40) for i in range(231)]),
                      _edge_chain(mode=MODE_DSD, gamma=g, alpha=a)))
    # int64-large timestamps
    big = 2**52 + np.arange(0, 500 * 37, 37)
    pairs.append((custom_trace(big, [3] * 500, [6] * 500), _edge_chain(cap=8)))
    # co-located modes: o = 1 only, bursts, cap 1, cap >= N, large timestamps
    for m, g, a in ((MODE_STANDALONE, 0, 0.0), (MODE_SPEC_COLO, 3, 0.7)):
        pairs.append((custom_trace([0, 0, 0, 0, 9], [1, 2, 3, 4, 5], [1, 1, 1, 1, 1]),
                      _edge_chain(mode=m, gamma=g, alpha=a)))
        pairs.append((custom_trace([0] * 300, [2] * 300, [5] * 300), _edge_chain(cap=1, mode=m, gamma=g, alpha=a)))
        pairs.append((custom_trace(np.arange(50), [1] * 50, [3] * 50), _edge_chain(cap=256, mode=m, gamma=g, alpha=a)))
        pairs.append((custom_trace(big, [3] * 500, [6] * 500), _edge_chain(cap=8, mode=m, gamma=g, alpha=a)))
        pairs.append((custom_trace([5], [3], [4]), _edge_chain(mode=m, gamma=g, alpha=a)))
    # large prompt tables (GL_MAX_PROMPT) and a 1-entry table
    pairs.append((custom_trace(np.arange(300) * 50, np.arange(1, 301) * 50, [3] * 300),
                  _edge_chain(max_prompt=16384)))
    pairs.append((custom_trace([0, 1, 2], [1, 1, 1], [2, 3, 4]), _edge_chain(max_prompt=1)))
    assert_parity(grid_of(pairs))


def _phased_case(rng, n, mode, cap, monotone=True):
    """Quiet and busy phases of random length: many idle points, long busy periods,
    candidates that are not idle (a loose step_min when the step table is not
    monotone), runs that extend past several candidates."""
    gaps = []
    while len(gaps) < n:
        busy = rng.random() < 0.5
        gaps.extend(rng.exponential(300.0 if busy else 40000.0, int(rng.integers(20, 3000))))
    a = np.cumsum(np.asarray(gaps[:n])).astype(np.int64)
    p = rng.integers(1, 9, n)
    o = rng.integers(1, 300, n)
    if monotone:
        step = [0] + [40 + 25 * b for b in range(1, cap + 1)]
    else:
        step = [0] + [int(x) for x in rng.integers(1, 400, cap)]
    tab = make_tables(8, cap, lambda q: 30 * q, lambda q: 7 * q, step, b2=lambda q: q,
                      e1=lambda q: 5 * q, e2=lambda q: 3 * q, sbn=[0] + [3] * cap,
                      sbo=[0] + [4] * cap, sen=[0] + [7] * cap, seo=[0] + [9] * cap)
    spec = mode in (MODE_DSD, MODE_SPEC_COLO)
    ch = make_chain(tab, mode, cap, 4 if spec else 0, 0.8 if spec else 0.0,
                    seed=int(rng.integers(0, 2**63)), ttft_slo=5000, tpot_slo=700)
    return custom_trace(a, p, o), ch


@pytest.mark.parametrize("n_chains,n", [(6, 30000), (100, 3000)])
def test_decode_speculation_stress(n_chains, n):
    """Leader / helper protocol of k_decode: few chains (many helpers each: long
    helper runs, aborts, waits) and many chains (few helpers: the leader walks
    unclaimed candidates).  Every request's finish must match the oracle."""
    rng = np.random.default_rng(n_chains * 7919 + n)
    pairs = []
    for i in range(n_chains):
        pairs.append(_phased_case(rng, n, ALL_MODES[i % 4], int(rng.choice([4, 16, 31, 48])),
                                  monotone=(i % 2 == 0)))
    assert_parity(grid_of(pairs))


@pytest.mark.parametrize("n_chains", [1, 37, 49, 74, 149])
def test_stage_split_block_boundaries(n_chains):
    # k_stages splits a chain over S blocks (S = 4, 4, 3, 2, 4 here; 149 chains
    # x 4 = 596 blocks is more than one wave, so later blocks start as earlier finish):
    # lengths around the 128-request chunk and 2048-request block-run boundaries, so
    # the decoupled look-back carries stage maps and decode counts across ragged runs
    rng = np.random.default_rng(9000 + n_chains)
    lens = [1, 127, 128, 129, 2047, 2048, 2049, 4097, 6143, 8191, 8193]
    pairs = []
    for i in range(n_chains):
        n = lens[i % len(lens)] if n_chains > 1 else 12289
        tr, ch = random_case(rng, n=n, mode=ALL_MODES[i % 4], cap=int(rng.choice([1, 3, 8, 40])))
        tr = dataclasses.replace(tr, arrival_us=np.sort(rng.integers(0, 40 * n + 1, n)))
        pairs.append((tr, ch))
    assert_parity(grid_of(pairs))


def test_iteration_rebase_and_far_gaps():
    """> 2^31 decode iterations (the 32-bit iteration counter rebases) and joins
    more than 2^31 us after the current boundary (the exact 64-bit path), in
    both the single-row (cap <= 31) and the multi-row (cap 40) loops."""
    pairs = []
    for cap in (2, 40):
        tab = make_tables(4, cap, lambda p: 3 * p, lambda p: p, [0] + [4] * cap,
                          sbo=[0] + [4] * cap, seo=[0] + [1] * cap)
        ch = make_chain(tab, MODE_DPD, cap, ttft_slo=100, tpot_slo=4)
        a = [0, 3_000_000_000, 3_000_000_010, 6_000_000_000, 6_000_000_001, 9_500_000_000,
             15_000_000_000, 16_000_000_000]
        o = [1_000_000_000, 5, 7, 1_070_000_000, 600_000_000, 3, 300_000_000, 1000]
        pairs.append((custom_trace(a, [1, 2, 3, 4, 1, 2, 3, 4], o), ch))
        if cap == 2:  # the co-located fast paths (prefill at every admission) rebase too
            pairs.append((custom_trace(a, [1, 2, 3, 4, 1, 2, 3, 4], o),
                          make_chain(tab, MODE_STANDALONE, cap, ttft_slo=100, tpot_slo=4)))
    assert_parity(grid_of(pairs))


def test_status_bits_match_oracle():
    pairs = [(custom_trace([5, 3, 7], [1, 1, 1], [2, 2, 2]), _edge_chain()),
             (custom_trace([0, 3], [0, 99], [2, 2]), _edge_chain()),
             (custom_trace([0, 3], [1, 1], [0, 2]), _edge_chain()),
             (custom_trace([-4, 3], [1, 1], [1, 2]), _edge_chain())]
    st, *_ = run_gpu(grid_of(pairs), per_request=False)
    for i, (tr, ch) in enumerate(pairs):
        want, _, _ = O.simulate_chain(tr, ch, per_request=False)
        assert st[i]["status"] == want["status"] != 0
        # R55: only n and the status survive; every other statistic is 0 on both sides
        for f in INT_FIELDS:
            assert int(st[i][f]) == int(want[f]), (i, f)
    # table errors are device-only (GL_ST_TABLE)
    bad = make_tables(4, 2, lambda p: 1, lambda p: 1, [0, 0, 3])
    st, *_ = run_gpu(grid_of([(custom_trace([0], [1], [3]), make_chain(bad))]), per_request=False)
    assert st[0]["status"] & N.ST_TABLE
    assert all(int(st[0][f]) == 0 for f in INT_FIELDS if f not in ("n", "status", "capacity_ok"))


def test_invalid_chains_never_feasible():
    """R55: a chain with status bits -- a device-only table error or an
    input violation -- is excluded from Alg. 1's feasible set like a capacity-
    infeasible one, and its statistics are deterministic (0) whatever the scratch
    memory held before."""
    tr = custom_trace(np.arange(0, 4000, 40), [2] * 100, [5] * 100)
    good = _edge_chain(cap=8)  # feasible: generous SLOs below
    good = dataclasses.replace(good, ttft_slo_us=10**9, tpot_slo_us=10**9, ce_new_g=99999.0)
    badtab = make_tables(8, 8, lambda p: 1, lambda p: 1, [0, 0] + [3] * 7)  # step[1] = 0
    cheap = make_chain(badtab, MODE_DPD, 8, ttft_slo=10**9, tpot_slo=10**9, ce_new=1.0, ce_old=1.0)
    unsorted = custom_trace(np.arange(100)[::-1].copy(), [2] * 100, [5] * 100)
    traces = [tr, unsorted]
    chains = [dataclasses.replace(good, trace_idx=0), dataclasses.replace(cheap, trace_idx=0),
              dataclasses.replace(cheap, trace_idx=1, tables=_edge_chain(cap=8).tables)]
    lt = 7 * 365 * 24 * 3600.0
    # row 0: all three; row 1: only the two invalid chains; row 2: only the table error
    cells = np.array([0, 1, 2, -1, 1, 2, -1, 1, -1], np.int32)
    for prio, dcol in ((0, -1), (1, 2)):
        g = GridSpec("invalid", traces, chains, np.array([[261.0, lt, lt]]), np.zeros(3, np.int32),
                     cells, 3, 3, 9, 10, prio, dcol)
        for rep in range(3):  # fill the pool with garbage between runs
            junk = torch.full((1 << 24,), -7, dtype=torch.int64, device="cuda")
            del junk
            st, _, carbon, choice, fb = run_gpu(g, per_request=False)
            assert st[1]["status"] & N.ST_TABLE and st[2]["status"] & 1
            ref = O.evaluate_grid(g, chain_ids=[0, 2])  # (the oracle has no table check)
            for ci in (0, 2):
                for f in INT_FIELDS:
                    assert int(st[ci][f]) == int(ref["stats"][ci][f]), (ci, f)
            assert choice[0] == 0 and fb[0] == 0
            assert fb[1] == 1 and fb[2] == 1
            if prio == 1:
                assert choice[1] == 2 and choice[2] == 2
            else:  # SLO fallback: both count as ok = 0 / +inf -> the lower column
                assert choice[1] == 1 and choice[2] == 1


# ------------------------------------------------------------ BASELINE configs
@pytest.mark.parametrize("mode,rate", [("dist", 1.0), ("fixed", 1.0), ("dist", 0.5), ("fixed", 0.5)])
def test_config1(mode, rate):
    assert_parity(build_config(1, mode=mode, rate=rate))


def test_config2_full():
    assert_parity(build_config(2))


def test_config3_reduced_all_chains():
    assert_parity(build_config(3, n=5000))


def test_config4_reduced_all_chains():
    assert_parity(build_config(4, n=5000))


def test_config3_full_size_all_chains():
    """BASELINE config 3 at its stated size: 128 chains (13B, both modes, 8 link
    bandwidths x 8 rates; the Fig. 13 bandwidth axis) x 100k requests.
    Every request's (ttft, finish), every statistic, all 64 x 2 Alg. 1 cells."""
    assert_parity(build_config(3))


def test_config4_full_size_all_chains():
    """The bench workload at full size (64 chains x 100k requests): every request,
    every statistic, carbon / choice / fallback of all 8,192 x 8 cells."""
    assert_parity(build_config(4))


def test_config5_full_size_all_chains():
    """BASELINE config 5 at its stated size: 320 chains (70B/7B DSD, gamma 1..8 x
    alpha 0.5..0.9 x 8 rates) x 1M LongBench requests (Table 2).  Every
    statistic of every chain -- including the 64-bit hash over every request's
    (ttft, finish) -- and all 40 x 8 Alg. 1 cells bit for bit (the oracle fanned
    over every host core)."""
    g = build_config(5)
    st = assert_parity(g, per_request=False)
    assert np.all(st["status"] == 0)


def test_config7_humaneval_full_size():
    """The paper's third workload (HumanEval code lengths, Table 2) over its
    QPS window 0.5-11 req/s: 80 chains (7B DPD / DSD on four GPU pairs,
    Standalone, SpecDecode) x 100k requests, every request and every Alg. 1 cell
    of 8,192 x 10, carbon and carbon per token bit for bit."""
    assert_parity(build_config(7))


def test_config6_colocated_columns_full_size():
    """NEXT #1 at the bench size: config 4 plus the Standalone / SpecDecode A100
    columns (80 chains x 100k requests), every request, every chain, every Alg. 1
    row of 8,192 x 10."""
    assert_parity(build_config(6))


# ------------------------------------------------------------ determinism
def test_determinism_and_chain_order_invariance():
    g = build_config(4, n=3000)
    a, *_ = run_gpu(g, per_request=False)
    b, *_ = run_gpu(g, per_request=False)
    assert a.tobytes() == b.tobytes()
    perm = np.random.default_rng(1).permutation(len(g.chains))
    gp = dataclasses.replace(g, chains=[g.chains[i] for i in perm],
                             cell_chain=np.array([np.nonzero(perm == c)[0][0] for c in g.cell_chain],
                                                 np.int32))
    c, *_ = run_gpu(gp, per_request=False)
    assert c[np.argsort(perm)].tobytes() == a.tobytes()
    # shard boundaries do not matter
    dg = api.DeviceGrid(g)
    full = torch.empty((len(g.chains), 80), dtype=torch.uint8, device="cuda")
    for lo, hi in ((0, 5), (5, 6), (6, 40), (40, 64)):
        api.eval_grid(dg, lo, hi, stats=full[lo:hi])
    torch.cuda.synchronize()
    assert api.stats_numpy(full).tobytes() == a.tobytes()


def test_concurrent_calls_on_two_streams():
    # two gl_eval_grid calls in flight at once on different streams, each splitting
    # its chains over several k_stages blocks (decoupled look-back, ticket order) and
    # running speculative decode helpers: no deadlock, results equal to one at a time
    gs = [build_config(4, n=6000), subset_chains(build_config(2, n=4000), list(range(8)))]
    dgs = [api.DeviceGrid(g) for g in gs]
    want = [api.stats_numpy(api.eval_grid(dg)[0]) for dg in dgs]
    outs = [torch.empty((dg.n_chains, 80), dtype=torch.uint8, device="cuda") for dg in dgs]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    for rep in range(3):
        for dg, out, st in zip(dgs, outs, streams):
            api.eval_grid(dg, stats=out, stream=st)
        torch.cuda.synchronize()
        for w, out in zip(want, outs):
            assert api.stats_numpy(out).tobytes() == w.tobytes()


# ------------------------------------------------------------------- Alg. 1
def test_argmin_random_stats_vs_oracle():
    """GPU Alg. 1 on synthetic stats (ties, absents, capacity, both priorities)."""
    rng = np.random.default_rng(11)
    base = build_config(2, n=200)
    for it in range(30):
        k = 24
        st = np.zeros(k, N.STATS_DTYPE)
        st["n"] = rng.integers(5, 20, k)
        st["slo_ok"] = np.minimum(st["n"], rng.integers(0, 21, k))
        st["busy_new_us"] = rng.choice([10**6, 2 * 10**6, 3 * 10**6], k)
        st["busy_old_us"] = rng.choice([0, 10**6], k)
        st["e_new_uj"] = rng.choice([0, 10**9, 2 * 10**9], k)
        st["e_old_uj"] = rng.choice([0, 10**9], k)
        chains = [dataclasses.replace(base.chains[0], capacity_ok=int(rng.random() > 0.2),
                                      ce_new_g=float(rng.choice([26340.0, 20000.0])))
                  for _ in range(k)]
        rows, cols = 37, 40
        cells = rng.integers(-1, k, rows * cols).astype(np.int32)
        scen = np.array([[rng.choice([0.0, 17.0, 261.0]), 7 * 3.15e7, rng.choice([5, 10]) * 3.15e7]
                         for _ in range(3)])
        rs = rng.integers(0, 3, rows).astype(np.int32)
        prio = int(it % 3 == 2)
        g = GridSpec("argmin", base.traces, chains, scen, rs, cells, rows, cols, 9, 10, prio,
                     int(rng.integers(-1, cols)))
        dg = api.DeviceGrid(g)
        stats = torch.from_numpy(st.view(np.uint8).reshape(k, 80).copy()).cuda()
        carbon, choice, fb = api.argmin_feasible(dg, stats)
        torch.cuda.synchronize()
        total = np.zeros((rows, cols))
        ok = np.zeros((rows, cols), np.int64)
        n = np.ones((rows, cols), np.int64)
        present = cells.reshape(rows, cols) >= 0
        cap = np.zeros((rows, cols), np.uint8)
        for r in range(rows):
            for c in range(cols):
                kk = cells[r * cols + c]
                if kk < 0:
                    continue
                d = {f: int(st[kk][f]) for f in INT_FIELDS}
                sc = scen[rs[r]]
                total[r, c] = O.carbon(d, chains[kk].ce_new_g, chains[kk].ce_old_g, *sc)[2]
                ok[r, c], n[r, c], cap[r, c] = d["slo_ok"], d["n"], chains[kk].capacity_ok
        want_c, want_f = O.alg1(total, ok, n, present, cap, 9, 10, prio, g.default_col)
        assert np.array_equal(choice.cpu().numpy(), want_c), it
        assert np.array_equal(fb.cpu().numpy(), want_f), it
        got = carbon.cpu().numpy()
        assert np.array_equal(got[present], total[present])
        assert np.all(np.isnan(got[~present]))


# --------------------------------------------------------- end-to-end host path
def test_evaluate_host_matches_device_path():
    g = build_config(4, n=4000)
    dg = api.DeviceGrid(g)
    stats, _ = api.eval_grid(dg)
    eval_launches = dg.last_launches
    carbon, choice, fb = api.argmin_feasible(dg, stats)
    torch.cuda.synchronize()
    ptok = torch.empty((g.rows, g.cols), dtype=torch.float64, device="cuda")
    api.argmin_feasible(dg, stats, per_token_out=ptok)
    torch.cuda.synchronize()
    res = api.evaluate_host(dg, dg.pinned_traces(), want_carbon=True, want_per_token=True)
    assert res.stats.tobytes() == api.stats_numpy(stats).tobytes()
    assert np.array_equal(res.choice, choice.cpu().numpy())
    assert np.array_equal(res.via_fallback, fb.cpu().numpy())
    assert np.array_equal(res.carbon, carbon.cpu().numpy())
    assert np.array_equal(res.carbon_per_token, ptok.cpu().numpy())
    # the same kernels as gl_eval_grid (DSD demand, stages, fill, segments, decode,
    # finalize) plus k_argmin
    assert res.launches == eval_launches + 1 == 7 and res.h2d_bytes > 0


def test_evaluate_host_pageable_inputs_other_stream_both_families():
    # pageable host arrays (synchronous staging), a non-default stream, and a grid
    # with disaggregated and co-located chains (both side streams in use)
    g = build_config(6, n=2500)
    dg = api.DeviceGrid(g)
    stats, _ = api.eval_grid(dg)
    _, choice, fb = api.argmin_feasible(dg, stats)
    torch.cuda.synchronize()
    cache = {}
    host = []
    for tr in g.traces:
        arrs = []
        for x in (tr.arrival_us, tr.prompt_len, tr.output_len):
            if id(x) not in cache:
                cache[id(x)] = torch.from_numpy(np.ascontiguousarray(x).copy())
            arrs.append(cache[id(x)])
        host.append(tuple(arrs))
    st = torch.cuda.Stream()
    for _ in range(2):
        res = api.evaluate_host(dg, host, stream=st)
        assert res.stats.tobytes() == api.stats_numpy(stats).tobytes()
        assert np.array_equal(res.choice, choice.cpu().numpy())
        assert np.array_equal(res.via_fallback, fb.cpu().numpy())


def test_abi_errors():
    g = build_config(1)
    dg = api.DeviceGrid(g)
    ch = dg.gl_chains[0]
    bad = N.GlChain.from_buffer_copy(ch)
    bad.batch_cap = 0
    stats = torch.empty((1, 80), dtype=torch.uint8, device="cuda")
    with pytest.raises(N.GreenLLMError) as e:
        N.eval_grid(dg.gl_traces, [bad], stats.data_ptr(), None, 0)
    assert e.value.status == N.GL_E_INVALID
    bad = N.GlChain.from_buffer_copy(ch)
    bad.trace_idx = 5
    with pytest.raises(N.GreenLLMError) as e:
        N.eval_grid(dg.gl_traces, [bad], stats.data_ptr(), None, 0)
    assert e.value.status == N.GL_E_LOOKUP
    bad = N.GlChain.from_buffer_copy(ch)
    bad.mode, bad.gamma, bad.alpha = 1, 4, 1.5
    with pytest.raises(N.GreenLLMError) as e:
        N.eval_grid(dg.gl_traces, [bad], stats.data_ptr(), None, 0)
    assert e.value.status == N.GL_E_DOMAIN
    with pytest.raises(N.GreenLLMError) as e:
        N.argmin_feasible(stats.data_ptr(), [ch], np.array([[-1.0, 1.0, 1.0]]), 1, 1,
                          np.zeros(1), np.zeros(1), 9, 10, 0, -1, None,
                          stats.data_ptr(), stats.data_ptr(), 0)
    assert e.value.status == N.GL_E_DOMAIN


def test_eval_grid_on_copied_traces():
    """api.eval_grid(traces=...) computes on the given device buffers (the
    distributed end-to-end path copies its shard's traces from the host and
    evaluates on the copies); results equal the resident path, and a copy with a
    changed arrival changes the result."""
    g = build_config(4, n=3000)
    dg = api.DeviceGrid(g)
    want = api.stats_numpy(api.eval_grid(dg, 8, 24)[0])
    host = dg.pinned_traces()
    copies = [tuple(x.to("cuda") for x in t) for t in host]
    got = api.stats_numpy(api.eval_grid(dg, 8, 24, traces=copies)[0])
    assert got.tobytes() == want.tobytes()
    copies[1][0][5:] += 1000  # shift trace 1 (chains 8..15) by 1 ms after request 5
    moved = api.stats_numpy(api.eval_grid(dg, 8, 24, traces=copies)[0])
    assert moved[:8].tobytes() != want[:8].tobytes() and moved[8:].tobytes() == want[8:].tobytes()


def test_dsd_demand_families():
    """k_dsd_family: chains on ONE trace with several (alpha, gamma) -- including alpha 0
    and 1, gamma 1..8, absent table cells, o = 1 requests and a gamma-16 chain that
    stays on the per-group kernel -- draw the same words once for all groups; every
    request's finish must equal the oracle's (which draws per member-step)."""
    rng = np.random.default_rng(77)
    n = 3000
    a = np.cumsum(rng.exponential(400.0, n)).astype(np.int64)
    p = rng.integers(1, 9, n)
    o = rng.integers(1, 400, n)
    o[rng.random(n) < 0.1] = 1
    tr = custom_trace(a, p, o)
    chains = []
    for alpha in (0.0, 0.3, 0.65, 0.9, 1.0):
        for gamma in (1, 3, 8):
            if (alpha, gamma) == (0.3, 3):
                continue  # an absent cell of the family table
            tab = make_tables(8, 16, lambda q: 30 * q, lambda q: 7 * q,
                              [0] + [40 + 10 * b for b in range(1, 17)], b2=lambda q: q,
                              sbn=[0] + [3] * 16, sbo=[0] + [4] * 16, sen=[0] + [5] * 16,
                              seo=[0] + [6] * 16)
            chains.append(make_chain(tab, MODE_DSD, 16, gamma, alpha, seed=0xABCDEF,
                                     ttft_slo=5000, tpot_slo=600))
    chains.append(dataclasses.replace(chains[0], gamma=16, alpha=0.8))  # per-group kernel
    chains.append(dataclasses.replace(chains[1], mode=MODE_SPEC_COLO))  # co-located, same draws
    k = len(chains)
    lt = 7 * 365 * 24 * 3600.0
    g = GridSpec("families", [tr], chains, np.array([[261.0, lt, lt]]), np.zeros(k, np.int32),
                 np.arange(k, dtype=np.int32), k, 1)
    assert_parity(g)


@pytest.mark.parametrize("per_request", [True, False])
def test_stage_groups_clone(per_request):
    """k_stage_clone: chains of one mode on one trace with the same prompt-indexed
    tables share one k_stages run (the primary) -- the secondaries differ in gamma,
    alpha, step table (one invalid: step[2] = 0), batch cap and capacity flag.  With
    per-request rows they get copies; without, k_finalize reads the primary's."""
    g = build_config(5, n=4000)
    chains = list(g.chains[:24])
    bad = make_tables(4096, 16, lambda q: 1, lambda q: 1, [0, 5, 0] + [9] * 14)
    chains[5] = dataclasses.replace(chains[5], tables=dataclasses.replace(
        chains[5].tables, step_us=bad.step_us))
    chains[7] = dataclasses.replace(chains[7], cap=8, capacity_ok=1)
    cells = np.arange(24, dtype=np.int32)
    gg = GridSpec("clone", g.traces, chains, g.scenarios, np.zeros(3, np.int32), cells, 3, 8)
    st, pr, _, _, _ = run_gpu(gg, per_request=per_request)
    assert st[5]["status"] & N.ST_TABLE
    ids = [i for i in range(24) if i != 5]
    ref = oracle_pool.evaluate_grid(gg, chain_ids=ids, gpu_per_request=pr if per_request else None)
    for ci in ids:
        for f in INT_FIELDS:
            assert int(st[ci][f]) == int(ref["stats"][ci][f]), (ci, f)
    assert not ref["mismatch"]


@pytest.mark.parametrize("cfg,n", [(4, 6000), (5, 2500), (3, 3000), (2, 2000)])
def test_schedule_hint_never_changes_results(cfg, n):
    """gl_eval_grid_sched / gl_evaluate_host_sched (greenllm.h gl_schedule): any hinted
    range -- the predicted one, single chains, ranges that split a stage group (their
    primary outside the range) or a trace, the first / last chains, a shard-relative
    range -- gives byte-identical statistics and per-request rows; a bad range is
    GL_E_INVALID and launches nothing."""
    g = build_config(cfg, n=n)
    dg = api.DeviceGrid(g)
    nc = dg.n_chains
    st0, pr0 = api.eval_grid(dg, per_request=True, schedule=False)
    st0, pr0 = st0.cpu().numpy(), pr0.cpu().numpy()
    ranges = [dg.first_range(), (0, 1), (nc - 1, nc), (min(3, nc - 1), min(17, nc)),
              (nc // 2, nc), (0, nc // 3), (0, nc), (2, 2)]
    for r in ranges:
        if r is None:
            continue
        st, pr = api.eval_grid(dg, per_request=True, schedule=r)
        assert np.array_equal(st.cpu().numpy(), st0), (cfg, r)
        assert np.array_equal(pr.cpu().numpy(), pr0), (cfg, r)
    if nc >= 6:  # a shard with a shard-relative hint
        lo, hi = 1, nc - 1
        st, _ = api.eval_grid(dg, lo, hi, schedule=(1, 3))
        assert np.array_equal(st.cpu().numpy(), st0[lo:hi])
    for bad in [(3, 2), (-1, 2), (0, nc + 1)]:
        with pytest.raises(N.GreenLLMError) as ei:
            api.eval_grid(dg, schedule=bad)
        assert ei.value.status == N.GL_E_INVALID
    # end to end with and without the hint
    host = dg.pinned_traces()
    a = api.evaluate_host(dg, host, want_carbon=True, schedule=False)
    sa, ca, cha = a.stats.copy(), a.carbon.copy(), a.choice.copy()
    b = api.evaluate_host(dg, host, want_carbon=True, schedule=dg.first_range() or (0, 1))
    assert np.array_equal(b.stats, sa) and np.array_equal(b.carbon, ca)
    assert np.array_equal(b.choice, cha)
    assert np.array_equal(sa.view(np.uint8).reshape(nc, -1), st0)


def test_deferred_demand_random_disaggregated():
    """Only disaggregated chains (no co-located SpecDecode), so the DSD demand is
    deferred: k_stages of the DSD primaries runs beside the demand kernels and the
    fill pass writes K_j.  Random traces (chunk and block boundaries, o = 1 requests)
    each carry stage groups -- DSD chains with identical tables and several
    (alpha, gamma) (one primary, secondaries cloned; a family when >= 2 groups share
    the draws) -- next to a DPD chain and a lone DSD chain (per-group kernel); every
    request against the oracle, with and without launch-order hints."""
    rng = np.random.default_rng(424242)
    traces, chains = [], []
    for t in range(10):
        n = int(rng.choice([1, 5, 129, 600, 2049, 4500]))
        a = np.sort(rng.integers(0, int(rng.integers(50, 400)) * n + 1, n))
        p = rng.integers(1, 9, n)
        o = rng.integers(1, 60, n)
        o[rng.random(n) < 0.1] = 1
        traces.append(custom_trace(a, p, o))
        cap = int(rng.choice([3, 8, 16, 40]))
        tab = make_tables(8, cap, lambda q: 30 * q, lambda q: 7 * q,
                          [0] + [40 + 10 * b for b in range(1, cap + 1)], b2=lambda q: q,
                          sbn=[0] + [3] * cap, sbo=[0] + [4] * cap, sen=[0] + [5] * cap,
                          seo=[0] + [6] * cap)
        for alpha, gamma in [(0.5, 1), (0.8, 4), (0.95, 8), (0.0, 2)][: int(rng.integers(1, 5))]:
            chains.append(make_chain(tab, MODE_DSD, cap, gamma, alpha, seed=0xC0FFEE + t,
                                     ttft_slo=4000, tpot_slo=500, trace_idx=t))
        chains.append(make_chain(tab, MODE_DPD, cap, ttft_slo=4000, tpot_slo=500, trace_idx=t))
        lone = make_tables(8, cap, lambda q: 20 * q, lambda q: 5 * q,
                           [0] + [35 + 9 * b for b in range(1, cap + 1)], b2=lambda q: q)
        chains.append(make_chain(lone, MODE_DSD, cap, 12, 0.7, seed=77 + t, ttft_slo=4000,
                                 tpot_slo=500, trace_idx=t))
    k = len(chains)
    lt = 7 * 365 * 24 * 3600.0
    g = GridSpec("deferred", traces, chains, np.array([[261.0, lt, lt]]), np.zeros(k, np.int32),
                 np.arange(k, dtype=np.int32), k, 1)
    st = assert_parity(g)
    dg = api.DeviceGrid(g)
    base, pr0 = api.eval_grid(dg, per_request=True)
    for h in [(0, 3), (k // 2, k), (5, k - 5)]:
        st2, pr2 = api.eval_grid(dg, per_request=True, schedule=h)
        assert torch.equal(st2, base) and torch.equal(pr2, pr0), h
