"""Pins of the oracle's link bandwidth-demand metric (
Fig. 4; readings R45-R47 in DESIGN.md §2).

Each test checks oracle_link_demand against something other than itself:
closed forms for isolated requests, SPEC's bandwidth accounting with
acceptance draws made independently, the max-plus prefill scan, and a 1-us tick
brute force that scans EVERY integer window start.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_20322_b200.inputs import (MODE_DPD, MODE_DSD, MODE_SPEC_COLO, MODE_STANDALONE,
                                          build_config, custom_trace)
from paper_2412_20322_b200.inputs.tables import VOCAB, dsd_member_step_bytes
from tests.bruteforce import _draw, _thresholds, tick_simulate, window_peak_bruteforce
from tests.helpers import make_chain, make_tables, random_case

pytestmark = pytest.mark.filterwarnings("ignore")


def test_member_step_bytes_formula():
    # R21 payloads: gamma IDs (4 B) + gamma fp16 distributions over the vocab + gamma+1 IDs back
    assert VOCAB == 32000
    assert dsd_member_step_bytes(4) == 16 + 4 * 32000 * 2 + 20 == 256036
    assert dsd_member_step_bytes(1) == 4 + 64000 + 8


def test_single_dpd_request_closed_form():
    # one request: one KV payload of bpt*(p+1) bytes at its prefill completion a + t1[p]
    tab = make_tables(8, 2, lambda p: 10 * p, lambda p: 7 * p, lambda b: 5 + b)
    ch = make_chain(tab, MODE_DPD, 2)
    tr = custom_trace([1000], [6], [4])
    d = O.link_demand(tr, ch, 1_000_000, bytes_per_token=524288, bytes_per_member_step=0)
    assert d["total_bytes"] == 524288 * 7
    assert d["peak_bytes"] == 524288 * 7
    assert d["peak_t_us"] == 1000 + 60
    assert d["n_impulses"] == 1
    # o = 1: no stage 2, no payload (R13)
    d1 = O.link_demand(custom_trace([1000], [6], [1]), ch, 1_000_000, 524288, 0)
    assert (d1["total_bytes"], d1["peak_bytes"], d1["peak_t_us"], d1["n_impulses"]) == (0, 0, -1, 0)


@pytest.mark.parametrize("gamma,o", [(1, 9), (4, 40), (3, 2)])
def test_isolated_dsd_request_closed_form(gamma, o):
    # alpha = 1: every step accepts gamma+1 tokens, so K = ceil((o-1)/(gamma+1)) steps at
    # r, r+S, ..., r+(K-1)S with r = c + t2[p]; the handoff (4(p+1) B) is issued at c.
    S = 50
    tab = make_tables(8, 2, lambda p: 10 * p, lambda p: 1000, lambda b: S)
    ch = make_chain(tab, MODE_DSD, 2, gamma=gamma, alpha=1.0)
    p, a = 5, 300
    tr = custom_trace([a], [p], [o])
    pm = dsd_member_step_bytes(gamma)
    K = -(-(o - 1) // (gamma + 1))
    c, r = a + 50, a + 50 + 1000
    hand = 4 * (p + 1)
    big = O.link_demand(tr, ch, 10**9, 4, pm)
    assert big["total_bytes"] == hand + K * pm
    assert big["peak_bytes"] == hand + K * pm and big["peak_t_us"] == c
    assert big["n_impulses"] == 1 + K
    one = O.link_demand(tr, ch, 1, 4, pm)  # 1-us window: the largest single impulse
    assert one["peak_bytes"] == pm and one["peak_t_us"] == r
    for m in (1, 2, 3):  # m steps fit in a window of m*S (the handoff is 1000 us earlier)
        d = O.link_demand(tr, ch, m * S, 4, pm)
        assert d["peak_bytes"] == min(m, K) * pm and d["peak_t_us"] == r


def test_colocated_modes_have_no_link():
    for mode in (MODE_STANDALONE, MODE_SPEC_COLO):
        tab = make_tables(8, 2, lambda p: 10 * p, lambda p: 0, lambda b: 20)
        ch = make_chain(tab, mode, 2, gamma=2 if mode == MODE_SPEC_COLO else 0, alpha=0.5)
        d = O.link_demand(custom_trace([0, 5, 9], [3, 4, 5], [6, 7, 1]), ch, 1000, 4, 1000)
        assert (d["total_bytes"], d["peak_bytes"], d["peak_t_us"], d["n_impulses"]) == (0, 0, -1, 0)


def _member_steps(seed, j, o, gamma, alpha):
    """K_j drawn independently (numpy Philox of the input module, R22)."""
    thr = _thresholds(alpha, gamma)
    rem, s = o - 1, 0
    while rem > 0:
        u = _draw(seed, j, s)
        rem -= 1 + sum(1 for t in thr if u < t)
        s += 1
    return s


@pytest.mark.parametrize("seed", range(4))
def test_bandwidth_accounting_S372(seed):
    # DPD bytes = sum of KV(p+1) over transferred requests; DSD bytes = sum
    # of per-step payload totals = handoffs + pm * (total member-steps), whatever the batching
    rng = np.random.default_rng(100 + seed)
    n = 200
    a = np.sort(rng.integers(0, 40_000, n))
    p = rng.integers(1, 9, n)
    o = rng.integers(1, 30, n)
    tr = custom_trace(a, p, o)
    gamma, alpha, cap = int(rng.integers(1, 6)), float(rng.choice([0.3, 0.7, 0.9])), 4
    tab = make_tables(8, cap, lambda q: 3 + q, lambda q: 2 * q, lambda b: 20 + 7 * b)
    ch = make_chain(tab, MODE_DSD, cap, gamma=gamma, alpha=alpha, seed=777 + seed)
    pm = dsd_member_step_bytes(gamma)
    d = O.link_demand(tr, ch, 500, 4, pm)
    steps = sum(_member_steps(ch.seed, j, int(o[j]), gamma, alpha) for j in range(n) if o[j] > 1)
    assert d["total_bytes"] == 4 * int(((p + 1) * (o > 1)).sum()) + pm * steps
    dpd = make_chain(tab, MODE_DPD, cap)
    d2 = O.link_demand(tr, dpd, 500, 524288, 0)
    assert d2["total_bytes"] == 524288 * int(((p + 1) * (o > 1)).sum())
    assert d2["n_impulses"] == int((o > 1).sum())


def test_dpd_peak_is_window_over_prefill_completions():
    # DPD: impulses at c_i = a_i + TTFT_i (o_i > 1); brute-force O(n^2) window over them,
    # with c_i from the max-plus closed form c_i = max_k (a_k + sum_{m=k..i} t1[p_m])
    rng = np.random.default_rng(5)
    n = 150
    a = np.sort(rng.integers(0, 200_000, n)).astype(np.int64)
    p = rng.integers(1, 9, n)
    o = rng.integers(1, 5, n)
    tab = make_tables(8, 3, lambda q: 500 * q, lambda q: 100 * q, lambda b: 900)
    ch = make_chain(tab, MODE_DPD, 3)
    s1 = np.array([int(tab.t1_us[x]) for x in p], np.int64)
    c = np.array([max(int(a[k]) + int(s1[k:i + 1].sum()) for k in range(i + 1)) for i in range(n)])
    for W in (1, 999, 10_000, 50_000):
        d = O.link_demand(custom_trace(a, p, o), ch, W, 1000, 0)
        imp = [(int(c[i]), 1000 * (int(p[i]) + 1)) for i in range(n) if o[i] > 1]
        sums = [sum(w for u, w in imp if t <= u < t + W) for t, _ in imp]
        best = max(sums)
        assert d["peak_bytes"] == best
        assert d["peak_t_us"] == min(t for (t, _), v in zip(imp, sums) if v == best)


@pytest.mark.parametrize("seed", range(40))
def test_link_vs_tick_bruteforce(seed):
    rng = np.random.default_rng(9000 + seed)
    mode = MODE_DPD if seed % 2 == 0 else MODE_DSD
    tr, ch = random_case(rng, mode=mode)
    bpt = int(rng.integers(1, 50))
    pm = int(rng.integers(1, 80)) if mode == MODE_DSD else 0
    W = int(rng.choice([1, 2, 7, 20, 60]))
    tk = tick_simulate(tr, ch, link=(bpt, pm))
    total, best, at = window_peak_bruteforce(tk["impulses"], W)
    d = O.link_demand(tr, ch, W, bpt, pm)
    assert d["total_bytes"] == total
    assert d["peak_bytes"] == best
    assert d["peak_t_us"] == at
    assert d["n_impulses"] == len(tk["impulses"])


def test_invariants_cfg2_subset():
    g = build_config(2, n=2000)
    for ch in g.chains[::7]:
        tr = g.traces[ch.trace_idx]
        d = O.link_demand(tr, ch)
        big = O.link_demand(tr, ch, window_us=10**13)
        assert 0 < d["peak_bytes"] <= d["total_bytes"] == big["total_bytes"]
        assert big["peak_bytes"] == big["total_bytes"]
        assert d["peak_bytes"] >= ch.tables.link_bytes_per_member_step  # one step of one member
        # a longer window never lowers the peak
        d2 = O.link_demand(tr, ch, window_us=2_000_000)
        assert d2["peak_bytes"] >= d["peak_bytes"]
        # the metric does not perturb the simulation
        st, _, _ = O.simulate_chain(tr, ch, per_request=False)
        for f in ("slo_ok", "busy_new_us", "busy_old_us", "makespan_us", "req_hash"):
            assert d["stats"][f] == st[f]


def test_trend_vs_fig4():
    """Trend check against Fig. 4: DSD needs far less link bandwidth than
    DPD, and DPD's demand grows with QPS.  Magnitudes are parity-unpinned: under the
    full-vocabulary fp16 probability payload (R21) the ratio is ~9-14x, below the
    paper's 65-434x (DESIGN.md §2 R47)."""
    from paper_2412_20322_b200.inputs import make_trace
    from paper_2412_20322_b200.inputs.grids import RATES8, _chain
    from paper_2412_20322_b200.inputs.tables import dpd_tables, dsd_tables
    prev = 0
    for rate in (0.5, 1.0, 2.0, 4.0):
        tr = make_trace("chat", 1500, rate, RATES8.index(rate), "fixed")
        dpd = _chain(MODE_DPD, 0, 16, dpd_tables("A100", "T4", "7B", 16), "chat", "A100", "T4",
                     "7B", None)
        dsd = _chain(MODE_DSD, 0, 16, dsd_tables("A100", "T4", "7B", "1B", 4, 16), "chat",
                     "A100", "T4", "7B", "1B", gamma=4, alpha=0.8)
        a, b = O.link_demand(tr, dpd), O.link_demand(tr, dsd)
        assert a["peak_bytes"] > 5 * b["peak_bytes"]
        assert a["peak_bytes"] >= prev
        prev = a["peak_bytes"]
