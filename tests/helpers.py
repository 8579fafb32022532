"""Test-case builders: small random traces and integer tables (inputs only)."""
from __future__ import annotations

import numpy as np

from paper_2412_20322_b200.inputs import (MODE_DPD, MODE_DSD, MODE_SPEC_COLO, MODE_STANDALONE,
                                          ChainSpec, ChainTables, custom_trace)


def make_tables(max_prompt, cap, t1, t2, step, b2=None, e1=None, e2=None, sbn=None, sbo=None,
                sen=None, seo=None, label="test"):
    """Tables from callables/arrays: t1(p), t2(p), step(b) etc."""
    P = np.arange(max_prompt + 1)
    B = np.arange(cap + 1)

    def arr(f, idx, dtype, default=0):
        if f is None:
            v = np.full(idx.shape, default, dtype=np.int64)
        elif callable(f):
            v = np.array([f(int(i)) for i in idx], dtype=np.int64)
        else:
            v = np.asarray(f, dtype=np.int64)
        v = v.copy()
        v[0] = 0
        return v.astype(dtype)

    return ChainTables(arr(t1, P, np.int32), arr(e1, P, np.int64), arr(t2, P, np.int32),
                       arr(b2, P, np.int32), arr(e2, P, np.int64), arr(step, B, np.int32),
                       arr(sbn, B, np.int32), arr(sbo, B, np.int32), arr(sen, B, np.int64),
                       arr(seo, B, np.int64), label)


def make_chain(tables, mode=MODE_DPD, cap=None, gamma=0, alpha=0.0, seed=0x1234,
               ttft_slo=10**9, tpot_slo=10**9, ce_new=26340.0, ce_old=10300.0, cap_ok=1,
               trace_idx=0):
    return ChainSpec(mode, trace_idx, tables.cap if cap is None else cap, gamma, alpha, seed,
                     tables, int(ttft_slo), int(tpot_slo), ce_new, ce_old, cap_ok, tables.label)


def random_case(rng: np.random.Generator, n=None, mode=None, cap=None, small=True):
    """A random tiny (trace, chain) pair sized for the 1-us tick brute force."""
    n = int(rng.integers(1, 11)) if n is None else n
    mode = int(rng.integers(0, 4)) if mode is None else mode
    cap = int(rng.integers(1, 5)) if cap is None else cap
    max_prompt = 6
    span = int(rng.integers(0, 150))
    a = np.sort(rng.integers(0, span + 1, n))
    if rng.random() < 0.3:  # bursts of equal arrivals
        a[: n // 2] = a[0]
        a = np.sort(a)
    p = rng.integers(1, max_prompt + 1, n)
    o = rng.integers(1, 9 if mode in (MODE_DPD, MODE_STANDALONE) else 14, n)
    if rng.random() < 0.2:
        o[rng.integers(0, n)] = 1
    t1v = rng.integers(1, 25, max_prompt + 1)
    t2v = rng.integers(0, 25, max_prompt + 1) if rng.random() < 0.8 else np.zeros(max_prompt + 1, int)
    b2v = rng.integers(0, 10, max_prompt + 1)
    e1v = rng.integers(0, 1000, max_prompt + 1)
    e2v = rng.integers(0, 1000, max_prompt + 1)
    stepv = rng.integers(1, 16, cap + 1)
    sbn = rng.integers(0, 16, cap + 1)
    sbo = rng.integers(0, 16, cap + 1)
    sen = rng.integers(0, 5000, cap + 1)
    seo = rng.integers(0, 5000, cap + 1)
    tab = make_tables(max_prompt, cap, t1v, t2v, stepv, b2v, e1v, e2v, sbn, sbo, sen, seo,
                      label="random")
    spec = mode in (MODE_DSD, MODE_SPEC_COLO)
    gamma = int(rng.integers(1, 6)) if spec else 0
    alpha = float(rng.choice([0.0, 0.3, 0.5, 0.8, 0.95, 1.0])) if spec else 0.0
    ttft_slo = int(rng.integers(10, 200))
    tpot_slo = int(rng.integers(5, 40))
    ch = make_chain(tab, mode, cap, gamma, alpha, seed=int(rng.integers(0, 2**63)),
                    ttft_slo=ttft_slo, tpot_slo=tpot_slo)
    return custom_trace(a, p, o), ch
