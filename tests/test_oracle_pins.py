"""Pins of the CPU oracle to things other than itself.

Each test names what fixes the expected value: the paper (cited), a closed
form, a textbook recursion, an independent brute force, or an invariant.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_20322_b200.inputs import (MODE_DPD, MODE_DSD, MODE_SPEC_COLO, MODE_STANDALONE,
                                          custom_trace)
from tests.bruteforce import tick_simulate
from tests.helpers import make_chain, make_tables, random_case

GOLD = os.path.join(os.path.dirname(__file__), "golden")
YEAR = 365 * 24 * 3600
WE = json.load(open(os.path.join(GOLD, "worked_examples.json")))


def _kat():
    rows = []
    for line in open(os.path.join(GOLD, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        rows.append((v[:4], v[4:6], v[6:10]))
    return rows


# --------------------------------------------------------------- Philox (R22)
@pytest.mark.parametrize("ctr,key,out", _kat())
def test_oracle_philox_kat(ctr, key, out):
    assert list(O.philox(ctr, *key)) == out


# ------------------------------------------------------- acceptance (R22, A.3)
def test_thresholds_worked_example_A3():
    ex = WE["A3_dsd_accept"]
    thr = O.thresholds(ex["alpha"], ex["gamma"])
    assert thr == ex["thr"]
    accs = [O.accept_count(int(u, 16), thr, ex["gamma"]) for u in ex["draws"]]
    assert accs == ex["acc"]
    # cumulative 3, 4, 6 >= 5 tokens: K = 3 steps for o = 6
    need, tot, k = 6 - 1, 0, 0
    while tot < need:
        tot += accs[k]
        k += 1
    assert k == ex["K_for_o6"]


@pytest.mark.parametrize("gamma", range(1, 9))
@pytest.mark.parametrize("alpha", [0.0, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0])
def test_expected_accept_closed_form(gamma, alpha):
    """E[acc] = (1 - alpha^(g+1)) / (1 - alpha) (Appendix B table),
    exactly sum_c thr_c / 2^32 under the quantised thresholds."""
    thr = O.thresholds(alpha, gamma)
    exact = 1.0 + sum(t / 2.0**32 for t in thr)
    closed = gamma + 1.0 if alpha == 1.0 else (1 - alpha ** (gamma + 1)) / (1 - alpha)
    assert abs(exact - closed) <= gamma * 2.0**-32
    if alpha == 0.0:
        assert thr == [0] * gamma
    if alpha == 1.0:
        assert thr == [2**32] * gamma


def test_appendix_b_eacc_table():
    """SURVEY Appendix B's printed E[acc] table (4 decimals)."""
    table = {4: [1.9375, 2.3056, 2.7731, 3.3616, 4.0951],
             8: [1.9961, 2.4748, 3.1988, 4.3289, 6.1258]}
    for g, vals in table.items():
        for a, v in zip([0.5, 0.6, 0.7, 0.8, 0.9], vals):
            thr = O.thresholds(a, g)
            assert abs(1 + sum(t / 2**32 for t in thr) - v) < 6e-5


def test_accept_distribution_chi2():
    """P(acc = c) = alpha^(c-1)(1-alpha) for c <= g, P(g+1) = alpha^g;
    10^5 Philox draws through the oracle's own generator + count rule."""
    from paper_2412_20322_b200.inputs.philox import philox4x32_10
    gamma, alpha = 4, 0.8
    thr = O.thresholds(alpha, gamma)
    # draws from the oracle's Philox must equal the inputs' numpy Philox
    for i in range(5):
        assert list(O.philox((i, 7, 0x41434350, 0), 5, 9)) == \
            [int(x) for x in philox4x32_10(i, 7, 0x41434350, 0, 5, 9)]
    w = np.stack(philox4x32_10(np.arange(25000), 3, 0x41434350, 0, 11, 13)).ravel()
    counts = np.zeros(gamma + 2)
    for u in w:
        counts[O.accept_count(int(u), thr, gamma)] += 1
    probs = [0.0] + [alpha ** (c - 1) * (1 - alpha) for c in range(1, gamma + 1)] + [alpha ** gamma]
    exp = np.array(probs) * len(w)
    chi2 = float(((counts[1:] - exp[1:]) ** 2 / exp[1:]).sum())
    assert chi2 < 15.09  # chi2_{0.99}(5 dof)
    mean = (np.arange(gamma + 2) * counts).sum() / len(w)
    assert abs(mean - (1 - alpha ** (gamma + 1)) / (1 - alpha)) < 0.01 * 3.3616


# ------------------------------------------------------------- hash rule
def test_mix64_splitmix_vector():
    """SplitMix64 finaliser: mix(0,0,0) of z=0 is 0; z = 1 -> known value."""
    assert O.mix64(0, 0, 0) == 0
    # SplitMix64 finaliser applied to 1 (Steele et al.; independently recomputed)
    z = 1
    z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & (2**64 - 1)
    z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & (2**64 - 1)
    z ^= z >> 31
    assert O.mix64(1, 0, 0) == z


def _kat_splitmix():
    rows = []
    with open(os.path.join(os.path.dirname(__file__), "golden", "splitmix64_kat.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                k, st, out = line.split()
                rows.append((int(k), int(st, 16), int(out, 16)))
    return rows


def _rotr(x, r):
    return ((x >> r) | (x << (64 - r))) & (2**64 - 1)


def test_mix64_splitmix_published_vectors():
    """The finaliser against SplitMix64's published seed-0 outputs
    (tests/golden/splitmix64_kat.txt), entering through each of the three inputs
    of the hash rule: j, rotl(ttft, 21) and rotl(finish, 42)."""
    rows = _kat_splitmix()
    assert len(rows) == 3
    for k, state, out in rows:
        assert (k * 0x9E3779B97F4A7C15) % 2**64 == state
        assert O.mix64(state, 0, 0) == out
        t = _rotr(state, 21)  # rotl(t, 21) == state
        assert O.mix64(0, t - 2**64 if t >= 2**63 else t, 0) == out
        f = _rotr(state, 42)
        assert O.mix64(0, 0, f - 2**64 if f >= 2**63 else f) == out


def test_carbon_per_token_closed_form_and_argmin_equivalence():
    """Carbon per token: S:73-74's Eq. 3 example (0.4 kWh + 3600 s on an
    A100 at CI 261, 7 y) = 104.82954990215... g spread over 1,000 tokens; and R33 --
    a row's cells share one trace, so Alg. 1 on per-token carbon (explicit matrices,
    fractional attainment) picks exactly what the integer Alg. 1 on totals picks."""
    lt7 = 7 * 365 * 24 * 3600.0
    st = _stats(e_new=1.44e12, busy_new=3600e6)
    st["tokens"] = 1000
    tot = O.carbon(st, 26340.0, 10300.0, 261.0, lt7, lt7)[2]
    assert O.carbon_per_token(st, tot) == pytest.approx(0.10482954990215264, rel=1e-13)
    assert O.carbon_per_token(st, tot) == tot / 1000.0
    st["tokens"] = 0  # void statistics (R55): IEEE total / 0
    assert O.carbon_per_token(st, tot) == math.inf
    from paper_2412_20322_b200.inputs import build_config
    g = build_config(4, n=600)
    ref = O.evaluate_grid(g)
    att = np.array([[ref["stats"][int(k)]["slo_ok"] / ref["stats"][int(k)]["n"] for k in row]
                    for row in g.cell_chain.reshape(g.rows, g.cols)])
    ch, fb = O.alg1_matrices(ref["carbon_per_token"], att, ref["present"], 0.9, g.priority,
                             g.default_col)
    assert np.array_equal(ch, ref["choice"]) and np.array_equal(fb, ref["via_fallback"])
    assert np.unique(ref["choice"]).size > 1  # the rows do not all pick one column


# ----------------------------------------------------- worked examples A.1/A.2
def _a1_chain(cap):
    ex = WE["A1_dpd_cap2"]
    tab = make_tables(4, cap, lambda p: ex["t1_per_token_us"] * p,
                      lambda p: ex["t2_per_token_us"] * p,
                      [0, 30, 40, 40][: cap + 1], e1=lambda p: 400 * 100 * p,
                      sbo=[0, 30, 40, 40][: cap + 1],
                      seo=[0, 30 * 70, 40 * 70, 40 * 70][: cap + 1])
    tr = custom_trace(ex["arrival_us"], ex["prompt_len"], ex["output_len"])
    return tr, make_chain(tab, MODE_DPD, cap, ttft_slo=ex["ttft_slo_us"], tpot_slo=ex["tpot_slo_us"])


def test_worked_example_A1_dpd_cap2():
    ex = WE["A1_dpd_cap2"]["expect"]
    tr, ch = _a1_chain(2)
    st, ttft, fin, r = O.simulate_chain(tr, ch, ready=True)
    assert list(ttft) == ex["ttft"]
    assert list(ttft + tr.arrival_us) == ex["c"]
    assert list(r) == ex["ready"]
    assert list(fin) == ex["finish"]
    assert st["busy_old_us"] == ex["busy_old_us"] and st["busy_new_us"] == ex["busy_new_us"]
    assert st["slo_ok"] == ex["slo_ok"]
    assert st["e_new_uj"] == 160000 and st["e_old_uj"] == 11200  # A.4 inputs


def test_worked_example_A2_cap1():
    ex = WE["A2_dpd_cap1"]["expect"]
    tr, ch = _a1_chain(1)
    st, ttft, fin = O.simulate_chain(tr, ch)
    assert list(fin) == ex["finish"]
    assert st["busy_old_us"] == ex["busy_old_us"]


# ------------------------------------------------------------ carbon Eqs. 1-3
def _stats(e_new=0, e_old=0, busy_new=0, busy_old=0, tokens=1):
    return dict(n=1, slo_ok=1, tokens=tokens, busy_new_us=int(busy_new), busy_old_us=int(busy_old),
                e_new_uj=int(e_new), e_old_uj=int(e_old), makespan_us=0, req_hash=0, status=0,
                capacity_ok=1)


def test_carbon_closed_forms():
    cf = WE["carbon_closed_forms"]
    lt7 = 7 * YEAR
    assert lt7 == 220_752_000
    op, emb, tot = O.carbon(_stats(busy_new=3600e6), 26340.0, 10300.0, 261.0, lt7, lt7)
    assert op == 0.0 and emb == pytest.approx(cf["embodied_3600s_A100_7y"], rel=1e-13)
    op, emb, tot = O.carbon(_stats(busy_new=lt7 * 1e6), 26340.0, 10300.0, 261.0, lt7, lt7)
    assert emb == pytest.approx(cf["embodied_LT_A100"], rel=1e-15)
    op, emb, tot = O.carbon(_stats(e_new=3.6e12), 26340.0, 10300.0, 261.0, lt7, lt7)
    assert op == cf["op_1kwh_261"] and emb == 0.0
    op, emb, tot = O.carbon(_stats(e_old=1.8e12), 26340.0, 10300.0, 501.0, lt7, lt7)
    assert op == cf["op_half_kwh_501"]
    op, emb, tot = O.carbon(_stats(e_new=1.44e12, busy_new=3600e6), 26340.0, 10300.0, 261.0, lt7, lt7)
    assert tot == pytest.approx(cf["total_0p4kwh_3600s_A100"], rel=1e-13)
    assert tot == op + emb
    # two identical GPUs -> exactly twice one GPU (linearity)
    one = O.carbon(_stats(e_new=1.44e12, busy_new=3600e6), 26340.0, 26340.0, 261.0, lt7, lt7)[2]
    two = O.carbon(_stats(e_new=1.44e12, e_old=1.44e12, busy_new=3600e6, busy_old=3600e6),
                   26340.0, 26340.0, 261.0, lt7, lt7)[2]
    assert two == 2 * one


def test_carbon_worked_example_A4():
    ex = WE["A4_carbon"]
    lt = ex["lt_years"] * YEAR
    op, emb, tot = O.carbon(_stats(ex["e_new_uj"], ex["e_old_uj"], ex["busy_new_us"],
                                   ex["busy_old_us"]), ex["ce_new_g"], ex["ce_old_g"], ex["ci"],
                            lt, lt)
    e = ex["expect"]
    for got, want in ((op, e["op"]), (emb, e["emb"]), (tot, e["total"]),
                      (tot / ex["tokens"], e["per_token"])):
        assert got == pytest.approx(want, rel=e["rel_tol"])


def test_break_even_ci_A5():
    """Argmin along CI switches at CI* = (emb_X - emb_Y)/(kwh_Y - kwh_X) (Eq. 5)."""
    ex = WE["A5_break_even"]
    lt = ex["lt_years"] * YEAR
    X = _stats(e_new=ex["X"]["e_uj"], busy_new=ex["X"]["busy_new_us"], busy_old=ex["X"]["busy_old_us"])
    Y = _stats(e_new=ex["Y"]["e_uj"], busy_new=ex["Y"]["busy_new_us"], busy_old=ex["Y"]["busy_old_us"])
    ce = (ex["ce_new_g"], ex["ce_old_g"])
    ex_e = ex["expect"]
    assert O.carbon(X, *ce, 0.0, lt, lt)[1] == pytest.approx(ex_e["emb_X"], rel=1e-11)
    assert O.carbon(Y, *ce, 0.0, lt, lt)[1] == pytest.approx(ex_e["emb_Y"], rel=1e-11)
    star = ex_e["ci_star"]
    for ci, want in ((star * 0.999, 1), (star * 1.001, 0), (0.0, 1), (501.0, 0)):
        tx = O.carbon(X, *ce, ci, lt, lt)[2]
        ty = O.carbon(Y, *ce, ci, lt, lt)[2]
        choice, fb = O.alg1(np.array([[tx, ty]]), np.array([[1, 1]]), np.array([[1, 1]]),
                            np.ones((1, 2)), np.ones((1, 2)))
        assert choice[0] == want and fb[0] == 0


def test_ci_limits_and_lower_envelope():
    """CI limits (Eq. 4): at CI = 0 Alg. 1 picks the
    least embodied chain, as CI grows it ends on the least-energy chain, and in
    between the choice is piecewise constant, walking down the lower envelope of
    the lines total(CI) = emb + CI kWh -- each switch goes to a chain with strictly
    less energy and more embodied carbon.  Embodied carbon is monotone in busy time
    (Eq. 1) and kWh in integer energy (Eq. 2), so the extremes are fixed by integers."""
    rng = np.random.default_rng(77)
    lt = 7 * YEAR
    for trial in range(20):
        k = int(rng.integers(2, 9))
        e = rng.choice(np.arange(1, 10_000), size=k, replace=False) * 10**9  # distinct uJ
        busy = rng.choice(np.arange(1, 10_000), size=k, replace=False) * 10**6  # distinct us
        st = [_stats(e_new=e[i], busy_new=busy[i]) for i in range(k)]

        def choose(ci):
            tot = np.array([[O.carbon(x, 26340.0, 10300.0, ci, lt, lt)[2] for x in st]])
            c, fb = O.alg1(tot, np.ones((1, k)), np.ones((1, k)), np.ones((1, k)), np.ones((1, k)))
            assert fb[0] == 0
            return int(c[0])
        assert choose(0.0) == int(np.argmin(busy))        # least embodied
        assert choose(1e12) == int(np.argmin(e))          # least energy
        path = [choose(ci) for ci in np.geomspace(1e-6, 1e12, 200)]
        switches = [(a, b) for a, b in zip(path, path[1:]) if a != b]
        assert len(switches) <= k - 1
        for a_, b_ in switches:                            # down the lower envelope
            assert e[b_] < e[a_] and busy[b_] > busy[a_]
        assert len(set(path)) == len(switches) + 1         # no chain chosen twice


def test_eq5_savings_ratio_from_totals():
    """Eq. 5: ratio of Case-2 to Case-1 totals equals
    ((N_A'+N_B) a + E_A'+E_B) / (N_A a + E_A); SPEC S:500 example 183.5/261.5."""
    lt = 7 * YEAR
    ce = 26340.0
    # embodied E_A = 0.5 g and E_A' + E_B = 0.8 g via busy times; N in kWh
    busy_a = 0.5 / ce * lt * 1e6
    busy_b = 0.8 / ce * lt * 1e6
    c1 = O.carbon(_stats(e_new=3.6e12, busy_new=round(busy_a)), ce, ce, 261.0, lt, lt)[2]
    c2 = O.carbon(_stats(e_new=0.7 * 3.6e12, busy_new=round(busy_b)), ce, ce, 261.0, lt, lt)[2]
    assert c2 / c1 == pytest.approx(183.5 / 261.5, rel=1e-9)
    # alpha = 0 limit: pure embodied ratio (E_A' + E_B) / E_A
    c1 = O.carbon(_stats(e_new=3.6e12, busy_new=round(busy_a)), ce, ce, 0.0, lt, lt)[2]
    c2 = O.carbon(_stats(e_new=0.7 * 3.6e12, busy_new=round(busy_b)), ce, ce, 0.0, lt, lt)[2]
    assert c2 / c1 == pytest.approx(0.8 / 0.5, rel=1e-9)


def test_lifetime_monotonicity():
    """Carbon strictly decreases in each LT when busy > 0 (Eq. 1)."""
    st = _stats(e_new=1e9, busy_new=5e9, busy_old=7e9)
    prev = None
    for lt_old in np.linspace(5, 10, 6) * YEAR:
        tot = O.carbon(st, 26340.0, 10300.0, 261.0, 7 * YEAR, lt_old)[2]
        assert prev is None or tot < prev
        prev = tot


# --------------------------------------------------------------- Alg. 1
def _alg1_from_att(att, carbon, target=0.9, priority=0, default_col=-1, cap=None):
    att = np.asarray(att, float)
    n = np.full(att.shape, 10000, np.int64)
    ok = np.round(att * 10000).astype(np.int64)
    num, den = int(round(target * 100)), 100
    cap = np.ones(att.shape) if cap is None else cap
    return O.alg1(np.asarray(carbon, float), ok, n, np.ones(att.shape), cap, num, den,
                  priority, default_col)


def test_alg1_spec_examples():
    ex = WE["alg1_examples"]
    ch, fb = _alg1_from_att(ex["feasible"]["slo_att"], ex["feasible"]["carbon"])
    assert ch[0] == ex["feasible"]["choice"] and fb[0] == 0
    ch, fb = _alg1_from_att(ex["fallback"]["slo_att"], ex["fallback"]["carbon"])
    assert ch[0] == ex["fallback"]["choice"] and fb[0] == 1
    ch, fb = _alg1_from_att(ex["fallback"]["slo_att"], ex["fallback"]["carbon"], priority=1,
                            default_col=2)
    assert ch[0] == 2 and fb[0] == 1


def _alg1_brute(total, ok, n, present, cap, num, den, priority, default_col):
    """Definition by enumeration + sort keys (an independent formulation)."""
    from fractions import Fraction
    rows, cols = total.shape
    choice, fb = [], []
    for r in range(rows):
        cand = [c for c in range(cols) if present[r, c]]
        feas = [c for c in cand if cap[r, c] and den * ok[r, c] >= num * n[r, c]]
        if feas:
            best = sorted(feas, key=lambda c: (total[r, c], -Fraction(int(ok[r, c]), int(n[r, c])), c))[0]
            choice.append(best)
            fb.append(0)
        elif priority == 1:
            choice.append(default_col)
            fb.append(1)
        elif not cand:
            choice.append(-1)
            fb.append(1)
        else:
            def key(c):
                okc = ok[r, c] if cap[r, c] else 0
                tc = total[r, c] if cap[r, c] else math.inf
                return (-Fraction(int(okc), int(n[r, c])), tc, c)
            choice.append(sorted(cand, key=key)[0])
            fb.append(1)
    return np.array(choice), np.array(fb)


def test_alg1_vs_brute_force_1000():
    """1,000 random 6x8 matrices, with ties, absents, capacity."""
    rng = np.random.default_rng(2412)
    for it in range(1000):
        rows, cols = 6, 8
        total = rng.choice([1.0, 2.0, 3.0, 2.5, 0.5], size=(rows, cols)) if it % 3 == 0 \
            else rng.random((rows, cols))
        n = rng.integers(5, 15, (rows, cols))
        ok = np.minimum(n, rng.integers(0, 16, (rows, cols)))
        present = rng.random((rows, cols)) > 0.1
        if it % 50 == 0:
            present[0] = False
        cap = rng.random((rows, cols)) > 0.15
        prio = int(it % 4 == 3)
        dcol = int(rng.integers(-1, cols))
        got = O.alg1(total, ok, n, present, cap, 9, 10, prio, dcol)
        want = _alg1_brute(total, ok, n, present, cap, 9, 10, prio, dcol)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), it


def test_alg1_invariants():
    """Optimality, scale equivariance and target monotonicity."""
    rng = np.random.default_rng(7)
    for _ in range(200):
        total = rng.random((4, 8)) + 0.1
        n = np.full((4, 8), 20)
        ok = rng.integers(10, 21, (4, 8))
        ones = np.ones((4, 8))
        ch, fb = O.alg1(total, ok, n, ones, ones, 9, 10)
        ch2, _ = O.alg1(total * 3.7, ok, n, ones, ones, 9, 10)
        assert np.array_equal(ch, ch2)
        for r in range(4):
            if not fb[r]:
                feas = [c for c in range(8) if 10 * ok[r, c] >= 9 * n[r, c]]
                assert all(total[r, c] >= total[r, ch[r]] for c in feas)
                ch95, fb95 = O.alg1(total, ok, n, ones, ones, 95, 100)
                if not fb95[r]:
                    assert total[r, ch95[r]] >= total[r, ch[r]]


# ---------------------------------------------- queueing: textbook / closed form
def _const_chain(n_prompt=8, t1=lambda p: 10 * p, t2=lambda p: 3 * p, step=None, cap=4, **kw):
    step = step if step is not None else [0] + [7 + b for b in range(1, cap + 1)]
    tab = make_tables(n_prompt, cap, t1, t2, step, sbo=step, seo=[0] + [5] * cap)
    return make_chain(tab, cap=cap, **kw)


def test_stage_scans_are_maxplus_longest_paths():
    """c_i = max_k (a_k + sum_{m=k..i} s1_m); r likewise over c (textbook max-plus)."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        n = int(rng.integers(1, 40))
        a = np.sort(rng.integers(0, 500, n))
        p = rng.integers(1, 9, n)
        o = rng.integers(1, 6, n)
        ch = _const_chain()
        st, ttft, fin, r = O.simulate_chain(custom_trace(a, p, o), ch, ready=True)
        c = ttft + a
        s1 = ch.tables.t1_us[p].astype(np.int64)
        s2 = np.where(o > 1, ch.tables.t2_us[p], 0).astype(np.int64)
        for i in range(n):
            assert c[i] == max(a[k] + s1[k:i + 1].sum() for k in range(i + 1))
            assert r[i] == max(c[k] + s2[k:i + 1].sum() for k in range(i + 1))


def test_cap1_is_lindley():
    """cap = 1: finish_j = max(finish_prev, r_j) + (o_j - 1) * S[1] (Lindley)."""
    rng = np.random.default_rng(4)
    for _ in range(50):
        n = int(rng.integers(1, 60))
        a = np.sort(rng.integers(0, 3000, n))
        p = rng.integers(1, 9, n)
        o = rng.integers(1, 12, n)
        ch = _const_chain(cap=1, step=[0, 13])
        st, ttft, fin, r = O.simulate_chain(custom_trace(a, p, o), ch, ready=True)
        prev = -10**18
        for j in range(n):
            if o[j] == 1:
                assert fin[j] == ttft[j] + a[j]
                continue
            want = max(prev, r[j]) + (o[j] - 1) * 13
            assert fin[j] == want
            prev = want


def test_isolated_request_closed_form():
    """TTFT = t1[p]; finish = c + t2[p] + (o-1) S[1]."""
    for p_, o_ in ((1, 1), (5, 2), (8, 30)):
        ch = _const_chain()
        st, ttft, fin = O.simulate_chain(custom_trace([1000], [p_], [o_]), ch)
        t1, t2 = 10 * p_, 3 * p_
        assert ttft[0] == t1
        assert fin[0] == (1000 + t1 if o_ == 1 else 1000 + t1 + t2 + (o_ - 1) * 8)


def test_dd1_overload_closed_form():
    """Gaps D < service s: c_i = a_0 + (i+1)s, TTFT_i = (i+1)s - i D."""
    s, D, n = 50, 20, 30
    a = 100 + D * np.arange(n)
    ch = _const_chain(t1=lambda p: s)
    st, ttft, fin = O.simulate_chain(custom_trace(a, np.ones(n), np.ones(n)), ch)
    for i in range(n):
        assert ttft[i] + a[i] == 100 + (i + 1) * s
        assert ttft[i] == (i + 1) * s - i * D


def test_dsd_isolated_steps_match_eacc():
    """Isolated DSD requests: (finish - r)/S[1] = K_j steps, and the average
    accepted tokens per step approaches E[acc]."""
    n, o_ = 400, 60
    a = np.arange(n) * 10**6
    gamma, alpha = 4, 0.8
    ch = _const_chain(mode=MODE_DSD, gamma=gamma, alpha=alpha, cap=2, step=[0, 9, 9])
    st, ttft, fin, r = O.simulate_chain(custom_trace(a, np.ones(n), np.full(n, o_)), ch, ready=True)
    K = (fin - r) / 9
    assert np.all(K == np.round(K))
    eacc = (1 - alpha ** (gamma + 1)) / (1 - alpha)
    # each request needs o-1 tokens; the last step overshoots by < gamma+1
    assert abs((o_ - 1) / K.mean() - eacc) < 0.25


# ------------------------------------------------------------ brute force
@pytest.mark.parametrize("seed", range(300))
def test_oracle_vs_tick_bruteforce(seed):
    rng = np.random.default_rng(seed)
    tr, ch = random_case(rng)
    st, ttft, fin, r = O.simulate_chain(tr, ch, ready=True)
    bf = tick_simulate(tr, ch)
    assert list(ttft) == bf["ttft"]
    assert list(fin) == bf["finish"]
    for i, rr in enumerate(bf["ready"]):
        if rr is not None:
            assert r[i] == rr
    for k in ("slo_ok", "busy_new_us", "busy_old_us", "e_new_uj", "e_old_uj", "tokens",
              "makespan_us", "req_hash"):
        assert st[k] == bf[k], k


def test_exhaustive_tiny_enumeration():
    """All N<=2 traces with arrivals on 0..6, p, o in {1,2,3}, cap in {1,2}, two
    step tables (SURVEY §8(c.4) exhaustive row, reduced to run in seconds)."""
    import itertools
    count = 0
    for cap in (1, 2):
        for steps in ([0, 3, 5], [0, 4, 4]):
            tab = make_tables(3, cap, lambda p: 2 * p, lambda p: p, steps[: cap + 1],
                              sbo=steps[: cap + 1])
            ch = make_chain(tab, MODE_DPD, cap, ttft_slo=5, tpot_slo=4)
            for n in (1, 2):
                for a in itertools.combinations_with_replacement(range(7), n):
                    for p in itertools.product((1, 2, 3), repeat=n):
                        for o in itertools.product((1, 2, 3), repeat=n):
                            tr = custom_trace(a, p, o)
                            st, ttft, fin = O.simulate_chain(tr, ch)
                            bf = tick_simulate(tr, ch)
                            assert list(fin) == bf["finish"] and st["slo_ok"] == bf["slo_ok"]
                            count += 1
    assert count > 3000


def test_exhaustive_tiny_enumeration_colocated():
    """Co-located modes (R41-R44): all N<=2 traces with arrivals on 0..5, p, o in
    {1,2,3}, cap in {1,2}, Standalone and SpecDecode, against the tick brute force."""
    import itertools
    count = 0
    for cap in (1, 2):
        for mode, gamma, alpha in ((MODE_STANDALONE, 0, 0.0), (MODE_SPEC_COLO, 2, 0.5)):
            tab = make_tables(3, cap, lambda p: 2 * p, lambda p: 0, [0, 3, 5][: cap + 1],
                              e1=lambda p: 7 * p, sbn=[0, 3, 5][: cap + 1], sen=[0, 11, 13][: cap + 1])
            ch = make_chain(tab, mode, cap, gamma, alpha, ttft_slo=5, tpot_slo=4)
            for n in (1, 2):
                for a in itertools.combinations_with_replacement(range(6), n):
                    for p in itertools.product((1, 2, 3), repeat=n):
                        for o in itertools.product((1, 2, 3), repeat=n):
                            tr = custom_trace(a, p, o)
                            st, ttft, fin = O.simulate_chain(tr, ch)
                            bf = tick_simulate(tr, ch)
                            assert list(fin) == bf["finish"] and list(ttft) == bf["ttft"]
                            assert st["slo_ok"] == bf["slo_ok"] and st["e_new_uj"] == bf["e_new_uj"]
                            count += 1
    assert count > 2000


def _colo_chain(mode=MODE_STANDALONE, cap=4, step=None, gamma=0, alpha=0.0):
    step = step or [0] + [8 + b for b in range(1, cap + 1)]
    tab = make_tables(8, cap, lambda p: 10 * p, lambda p: 0, step, e1=lambda p: 7 * p,
                      sbn=step, sen=[0] + [5 * b for b in range(1, cap + 1)])
    return make_chain(tab, mode, cap, gamma, alpha, ttft_slo=10**9, tpot_slo=10**9)


def test_colocated_isolated_request_closed_form():
    """Standalone, one request: TTFT = L_p, finish = a + L_p + (o-1) L_d."""
    for p_, o_ in ((1, 1), (5, 2), (8, 30)):
        ch = _colo_chain()
        st, ttft, fin = O.simulate_chain(custom_trace([1000], [p_], [o_]), ch)
        assert ttft[0] == 10 * p_
        assert fin[0] == 1000 + 10 * p_ + (o_ - 1) * 9
        assert st["busy_new_us"] == 10 * p_ + (o_ - 1) * 9
        assert st["busy_old_us"] == 0 and st["e_old_uj"] == 0


def test_colocated_cap1_is_lindley():
    """cap = 1: one request at a time on the GPU, prefill then decode:
    finish_j = max(finish_prev, a_j) + t1[p_j] + (o_j - 1) S[1] (Lindley)."""
    rng = np.random.default_rng(41)
    for _ in range(50):
        n = int(rng.integers(1, 60))
        a = np.sort(rng.integers(0, 3000, n))
        p = rng.integers(1, 9, n)
        o = rng.integers(1, 12, n)
        ch = _colo_chain(cap=1, step=[0, 13])
        st, ttft, fin = O.simulate_chain(custom_trace(a, p, o), ch)
        prev = -10**18
        for j in range(n):
            start = max(prev, a[j])
            assert ttft[j] == start + 10 * p[j] - a[j]
            prev = start + 10 * p[j] + (o[j] - 1) * 13
            assert fin[j] == prev


def test_colocated_prefill_priority_burst():
    """k simultaneous arrivals, cap >= k, o = 2: all k prefills run first (prefill
    priority), then ONE iteration at batch k finishes everyone (R42)."""
    for k in (1, 2, 5, 8):
        ch = _colo_chain(cap=8)
        p = np.arange(1, k + 1)
        st, ttft, fin = O.simulate_chain(custom_trace(np.zeros(k), p, np.full(k, 2)), ch)
        assert list(ttft) == list(np.cumsum(10 * p))
        assert np.all(fin == 10 * p.sum() + 8 + k)


def test_specdecode_colocated_steps_match_eacc():
    """Isolated SpecDecode requests: (finish - c)/S[1] = K_j steps whose mean
    accepted tokens approach E[acc] = (1 - alpha^(g+1))/(1 - alpha)."""
    n, o_ = 400, 60
    gamma, alpha = 4, 0.8
    ch = _colo_chain(mode=MODE_SPEC_COLO, cap=2, step=[0, 9, 9], gamma=gamma, alpha=alpha)
    a = np.arange(n) * 10**6
    st, ttft, fin = O.simulate_chain(custom_trace(a, np.ones(n), np.full(n, o_)), ch)
    K = (fin - (a + ttft)) / 9
    assert np.all(K == np.round(K))
    eacc = (1 - alpha ** (gamma + 1)) / (1 - alpha)
    assert abs((o_ - 1) / K.mean() - eacc) < 0.25


# ----------------------------------------------------------- invariants
def test_invariants_and_determinism():
    from paper_2412_20322_b200.inputs import build_config
    g = build_config(2, n=2000)
    for ch in g.chains[::7]:
        tr = g.traces[ch.trace_idx]
        st, ttft, fin, r = O.simulate_chain(tr, ch, ready=True)
        st2, ttft2, fin2 = O.simulate_chain(tr, ch)
        assert st == st2 and np.array_equal(fin, fin2)      # determinism
        assert st["tokens"] == int(tr.output_len.astype(np.int64).sum())  # conservation
        dec = tr.output_len > 1
        smin = int(ch.tables.step_us[1:ch.cap + 1].min())
        assert np.all(fin[dec] >= r[dec] + smin)             # causality
        assert np.all(ttft >= ch.tables.t1_us[tr.prompt_len])
        assert st["makespan_us"] == fin.max()


def test_status_bits():
    ch = _const_chain()
    st, _, _ = O.simulate_chain(custom_trace([5, 3], [1, 1], [2, 2]), ch)
    assert st["status"] & O.ST_UNSORTED
    st, _, _ = O.simulate_chain(custom_trace([0, 3], [0, 99], [2, 2]), ch)
    assert st["status"] & O.ST_PROMPT_RANGE
    st, _, _ = O.simulate_chain(custom_trace([0, 3], [1, 1], [0, 2]), ch)
    assert st["status"] & O.ST_OUTPUT_ZERO
    st, _, _ = O.simulate_chain(custom_trace([-4, 3], [1, 1], [1, 2]), ch)
    assert st["status"] & O.ST_NEG_ARRIVAL
