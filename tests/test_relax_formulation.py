"""R57: the decode stage in the iteration domain has exactly one
solution, the serial simulation's.  Pinned here on the CPU, independently of the CUDA
path: the rules are iterated as a fixed-point map (plain numpy, from J = 0) until
nothing changes, and the resulting finish times tau(J_q + K_q) and per-batch-size
iteration counts must equal the oracle's (the serial, one-iteration-at-a-time DES)
request by request -- on random DPD and DSD chains, sparse and dense arrivals,
caps 1-16, idle periods and saturated stretches.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_20322_b200.inputs import MODE_DPD, MODE_DSD, custom_trace
from tests.helpers import random_case

NEG = -(1 << 62)


def demand(trace, ch, dec):
    """Iterations each decode request needs: o - 1 (DPD) or the speculative steps
    until o - 1 tokens are accepted (DSD, the oracle's own draws, R22)."""
    o = trace.output_len.astype(np.int64)
    if ch.mode == MODE_DPD:
        return o[dec] - 1
    thr = O.thresholds(ch.alpha, ch.gamma)
    k0, k1 = ch.seed & 0xFFFFFFFF, ch.seed >> 32
    K = np.zeros(len(dec), np.int64)
    for i, j in enumerate(dec):
        rem, s = int(o[j]) - 1, 0
        while rem > 0:
            w = O.philox([s // 4, int(j), 0x41434350, 0], k0, k1)[s % 4]
            rem -= O.accept_count(int(w), thr, ch.gamma)
            s += 1
        K[i] = s
    return K


def solve_r57(r, K, step, cap, max_sweeps=100000):
    """Fixed-point iteration of R57's rules (the map k_relax applies, written plainly)."""
    N = len(r)
    ext = lambda b: np.where(b <= cap, step[np.minimum(b, cap)],
                             step[cap] + (b - cap) * max(int(step[cap]) - int(step[cap - 1]) if cap > 1 else int(step[cap]), 0))
    J = np.zeros(N, np.int64)
    for sweep in range(max_sweeps):
        F = J + K
        L = int(F.max())
        GJ = np.cumsum(np.bincount(J, minlength=L + 1)[:L + 1])   # joins at boundaries <= I
        G = np.cumsum(np.bincount(F, minlength=L + 1)[:L + 1])    # leaves at boundaries <= I
        b = GJ - G
        # tau(I+1) = tau(I) + step[b] (b > 0), max(tau(I), r_{GJ(I)}) (b = 0, idle)
        inc = np.where(b > 0, ext(b), 0)
        R = np.where(b > 0, NEG, np.where(GJ < N, r[np.minimum(GJ, N - 1)], NEG))
        Sp = np.concatenate(([0], np.cumsum(inc)))                # prefix of increments
        cand = np.concatenate(([r[0]], R - Sp[1:]))               # resets, shifted by the prefix
        tau = Sp + np.maximum.accumulate(cand)
        A = np.searchsorted(tau, r, side="left")                  # first I with tau(I) >= r
        need = np.arange(N) - cap + 1
        S = np.where(need > 0, np.searchsorted(G, np.maximum(need, 1), side="left"), 0)
        Jn = np.maximum.accumulate(np.maximum(A, S))
        if np.array_equal(Jn, J):
            return J, tau, b, sweep
        J = Jn
    raise AssertionError("no fixed point")


def check_case(trace, ch):
    st, ttft, fin, r_all = O.simulate_chain(trace, ch, per_request=True, ready=True)
    o = trace.output_len.astype(np.int64)
    dec = np.nonzero(o > 1)[0]
    if dec.size == 0:
        return
    r = r_all[dec]
    K = demand(trace, ch, dec)
    step = ch.tables.step_us.astype(np.int64)
    J, tau, b, _ = solve_r57(r, K, step, ch.cap)
    assert np.array_equal(tau[J + K], fin[dec]), "finish times"
    # busy / energy: the oracle's totals minus the stage-1/2 parts (per request, R9-R12)
    # are the decode part, sum over iterations with b > 0 of the batch-indexed tables
    cnt = np.bincount(b[b > 0], minlength=ch.cap + 1)[:ch.cap + 1].astype(np.int64)
    t, p = ch.tables, trace.prompt_len.astype(np.int64)
    d = o > 1
    stage = {"busy_new_us": int(t.t1_us[p].astype(np.int64).sum()),
             "busy_old_us": int(t.b2_old_us[p][d].astype(np.int64).sum()),
             "e_new_uj": int(t.e1_new_uj[p].astype(np.int64).sum()),
             "e_old_uj": int(t.e2_old_uj[p][d].astype(np.int64).sum())}
    per_b = {"busy_new_us": t.step_busy_new_us, "busy_old_us": t.step_busy_old_us,
             "e_new_uj": t.step_e_new_uj, "e_old_uj": t.step_e_old_uj}
    for f, tab in per_b.items():
        assert st[f] - stage[f] == int(np.dot(cnt, tab[:ch.cap + 1].astype(np.int64))), f
    assert np.all(np.diff(J) >= 0)                                # FCFS joins
    assert np.all(b <= ch.cap)                                    # the cap holds at the fixed point
    assert st["makespan_us"] == max(int(tau[int((J + K).max())]), int(fin.max()))


@pytest.mark.parametrize("seed", range(12))
def test_r57_fixed_point_is_the_serial_simulation(seed):
    rng = np.random.default_rng(5700 + seed)
    for mode in (MODE_DPD, MODE_DSD):
        for cap in (1, 2, 4, 16):
            n = int(rng.integers(1, 400))
            tr, ch = random_case(rng, n=n, mode=mode, cap=cap)
            dense = rng.random() < 0.5
            a = np.sort(rng.integers(0, (3 if dense else 60) * n + 1, n))
            check_case(custom_trace(a, tr.prompt_len, tr.output_len), ch)


def test_r57_on_a_workload_chain():
    """A config-4-like chain (chat lengths, A100 pair, DSD gamma 4) at 1,500 requests."""
    from paper_2412_20322_b200.inputs import build_config
    g = build_config(4, n=1500)
    for ci in (33, 46):
        ch = g.chains[ci]
        check_case(g.traces[ch.trace_idx], ch)
