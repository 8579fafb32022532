"""Pins of the oracle's §5 carbon-efficiency analysis (
P:355-414, Eqs. 4-6; readings R48-R49 in DESIGN.md §2).

Pinned against SPEC's hand-worked ratio, the identity case, the algebraic
equivalence of Eq. 5's three lines, the sign of the ratio's derivatives in CI
 and in each lifetime (closed-form sign conditions), Eq. 6's t_B = 0
case, and totals composed from the (separately pinned) carbon function.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_20322_b200.inputs import build_config, savings_pairs

YEAR = 365 * 24 * 3600.0


def st(e_new, e_old, b_new, b_old):
    return dict(n=1, slo_ok=1, tokens=1, busy_new_us=int(b_new), busy_old_us=int(b_old),
                e_new_uj=int(e_new), e_old_uj=int(e_old), makespan_us=0, req_hash=0, status=0,
                capacity_ok=1)


KWH = 3_600_000_000_000  # uJ


def test_spec_worked_ratio_S500():
    # N_A = 1 kWh, N_A' + N_B = 0.7 kWh, E_A = 0.5 g, E_A' + E_B = 0.8 g, alpha = 261
    # -> (0.7*261 + 0.8)/(261 + 0.5) = 183.5/261.5 = 0.70172084 (29.8% savings)
    s = st(KWH, 0, 1e6, 0)                       # (1 s / 1000 s) * 500 g = 0.5 g
    d = st(KWH // 2, KWH // 5, 1e6, 1e6)         # 0.5 g + (1 s / 1000 s) * 300 g = 0.8 g
    r = O.savings(d, (500.0, 300.0), s, (500.0, 0.0), 261.0, 1000.0, 1000.0)
    assert r["ratio"] == pytest.approx(183.5 / 261.5, rel=1e-15)
    assert round(1 - r["ratio"], 3) == 0.298
    assert r["op_saved_g"] == pytest.approx(0.3 * 261, rel=1e-13)
    assert r["emb_saved_g"] == pytest.approx(-0.3, rel=1e-12)
    assert r["eq4"] == 1
    # Eq. 6 as printed: (t_B/T_B * B) / (N_A alpha + t_A'/T_A * A) = 0.3 / (261 + 0.5)
    assert r["eq6_term"] == pytest.approx(0.3 / 261.5, rel=1e-14)


def test_identity_case_S499():
    s = st(123456789, 0, 98765, 0)
    r = O.savings(s, (26340.0, 10300.0), s, (26340.0, 0.0), 261.0, 7 * YEAR, 7 * YEAR)
    assert r["ratio"] == 1.0 and r["op_saved_g"] == 0.0 and r["emb_saved_g"] == 0.0
    assert r["eq4"] == 0 and r["eq6_term"] == 0.0  # t_B = 0: Eq. 6 term vanishes


def _rand(rng):
    s = st(rng.integers(1, 10**12), 0, rng.integers(1, 10**9), 0)
    d = st(rng.integers(1, 10**12), rng.integers(0, 10**12), rng.integers(1, 10**9),
           rng.integers(0, 10**9))
    return d, s


def test_eq5_lines_agree():
    # Eq. 5: first line == (N'/N) + (E_A' + E_B - (N'/N) E_A) / (N alpha + E_A)  (third line)
    rng = np.random.default_rng(1)
    for _ in range(500):
        d, s = _rand(rng)
        ci, ta, tb = rng.uniform(0, 600), rng.uniform(1, 10) * YEAR, rng.uniform(1, 10) * YEAR
        A, B = 26340.0, 10300.0
        r = O.savings(d, (A, B), s, (A, 0.0), ci, ta, tb)
        N = s["e_new_uj"] / 3.6e12
        Np = (d["e_new_uj"] + d["e_old_uj"]) / 3.6e12
        EA = s["busy_new_us"] / 1e6 / ta * A
        EpB = d["busy_new_us"] / 1e6 / ta * A + d["busy_old_us"] / 1e6 / tb * B
        third = Np / N + (EpB - Np / N * EA) / (N * ci + EA)
        assert r["ratio"] == pytest.approx(third, rel=1e-11)
        assert r["eq4"] == int(s["e_new_uj"] > d["e_new_uj"] + d["e_old_uj"])
        # the op/emb split adds up to the difference of the totals
        tot_s = O.carbon(s, A, 0.0, ci, ta, tb)[2]
        tot_d = O.carbon(d, A, B, ci, ta, tb)[2]
        assert r["op_saved_g"] + r["emb_saved_g"] == pytest.approx(tot_s - tot_d, rel=1e-9, abs=1e-9)
        assert r["ratio"] == pytest.approx(tot_d / tot_s, rel=1e-15)


def test_savings_increase_with_ci_S522():
    # N_A' + N_B < N_A and E_A' + E_B > E_A  =>  savings strictly increasing in alpha
    rng = np.random.default_rng(2)
    n = 0
    while n < 1000:
        d, s = _rand(rng)
        A, B, ta, tb = 26340.0, 10300.0, 7 * YEAR, 7 * YEAR
        N = s["e_new_uj"]
        Np = d["e_new_uj"] + d["e_old_uj"]
        EA = s["busy_new_us"] * A / ta
        EpB = d["busy_new_us"] * A / ta + d["busy_old_us"] * B / tb
        if not (Np < N and EpB > EA):
            continue
        n += 1
        sv = [1 - O.savings(d, (A, B), s, (A, 0.0), ci, ta, tb)["ratio"] for ci in (17.0, 261.0, 501.0)]
        assert sv[0] < sv[1] < sv[2]


def test_lifetime_signs_closed_form():
    # R(x) = (a + c x + e)/(b + d x), x = 1/T_A: dR/dx has the sign of c b - d (a + e)
    # (c = t_A' A, d = t_A A, a = N' alpha, b = N alpha, e = E_B); savings rise with T_B
    # whenever t_B > 0.
    rng = np.random.default_rng(3)
    for _ in range(300):
        d, s = _rand(rng)
        A, B, ci = 26340.0, 10300.0, float(rng.uniform(1, 500))
        tb = 7 * YEAR
        sv = [1 - O.savings(d, (A, B), s, (A, 0.0), ci, ta * YEAR, tb)["ratio"]
              for ta in (2.0, 7.0)]
        N, Np = s["e_new_uj"] / 3.6e12, (d["e_new_uj"] + d["e_old_uj"]) / 3.6e12
        c, dd = d["busy_new_us"] / 1e6 * A, s["busy_new_us"] / 1e6 * A
        e = d["busy_old_us"] / 1e6 / tb * B
        sign = c * N * ci - dd * (Np * ci + e)
        if abs(sign) > 1e-6 * (abs(c * N * ci) + abs(dd * (Np * ci + e))):
            # savings(T_A = 2 y) vs savings(T_A = 7 y): larger x = 1/T_A at 2 y
            assert (sv[0] < sv[1]) == (sign > 0)
        if d["busy_old_us"] > 0:
            lo = 1 - O.savings(d, (A, B), s, (A, 0.0), ci, 7 * YEAR, 5 * YEAR)["ratio"]
            hi = 1 - O.savings(d, (A, B), s, (A, 0.0), ci, 7 * YEAR, 10 * YEAR)["ratio"]
            assert hi > lo


def test_cfg6_pairs_and_surface_shape():
    g = build_config(6, n=400)
    pairs = savings_pairs(g)
    assert len(pairs) == 8 * 9
    for d, s in pairs:
        assert g.chains[s].mode == 2 and g.chains[d].trace_idx == g.chains[s].trace_idx
    sub = pairs[:3]
    from paper_2412_20322_b200.inputs.grids import GridSpec
    small = GridSpec(g.name, g.traces, g.chains, g.scenarios[:40], g.row_scenario[:1],
                     g.cell_chain[:10], 1, 10)
    out = O.savings_surface(small, sub)
    assert out["ratio"].shape == (3, 40)
    # DSD/DPD totals over CI rows: the ratio is monotone in CI for fixed lifetimes
    # (Eq. 5: a Moebius function of alpha has no interior extremum)
    for i in range(3):
        for lt in range(16):
            col = out["ratio"][i, lt::16]
            dif = np.diff(col)
            assert (dif >= -1e-15).all() or (dif <= 1e-15).all()
