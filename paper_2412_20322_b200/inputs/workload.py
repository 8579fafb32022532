"""Seeded synthetic request traces shaped like the paper's workloads (inputs only).

Readings (DESIGN.md §3 "Input recipe"):

* Workloads and SLOs are Table 2 (rows P:427-429):
  ShareGPT chat (TTFT 200 ms, TPOT 80 ms), HumanEval code (125 ms / 200 ms),
  LongBench summarisation (15 s / 150 ms), with P25/P50/P75 (input, output)
  request sizes.
* Arrivals are Poisson at rate lambda (the paper gives only QPS; SPEC
  chose Poisson).  gap_i = floor(-ln(U_i) * 1e6 / lambda) microseconds,
  U_i = (w + 0.5) 2^-32 with w = Philox word 0 of counter (i, rate_idx,
  workload_id, 0); a_0 = gap_0, a_i = a_{i-1} + gap_i.
* Lengths follow a piecewise log-linear quantile function through
  (0, lo), (.25, P25), (.5, P50), (.75, P75), (1, hi) with lo = max(1, P25 // 4)
  and hi = 4 * P75, rounded half away from zero; input and output are drawn
  independently from words 0 and 1 of counter (i, 0xFFFF, workload_id, 0), so
  every rate of one workload shares the same length sequence.  The prompt is
  clamped to ctx - output with ctx = 4096 (Llama-2 context).  Mode "fixed"
  gives every request the P50 pair, the paper's truncation methodology.

Everything here is generated once on the host; the CUDA path and the oracle
read the same arrays, so libm differences cannot reach parity.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .philox import key_from_seed, philox4x32_10, uniform_open01

BASE_SEED = 0x0000000241220322  # from the arXiv id 2412.20322
CTX = 4096


@dataclass(frozen=True)
class Workload:
    name: str
    wid: int
    ttft_slo_ms: float
    tpot_slo_ms: float
    p25: tuple
    p50: tuple
    p75: tuple


# Table 2
WORKLOADS = {
    "chat": Workload("ShareGPT", 0, 200.0, 80.0, (24, 24), (160, 140), (510, 357)),
    "code": Workload("HumanEval", 1, 125.0, 200.0, (108, 31), (136, 55), (182, 88)),
    "summ": Workload("LongBench", 2, 15000.0, 150.0, (1134, 201), (1495, 275), (1817, 352)),
}

# R8 of SURVEY.md §8(d): the north star's 0.5-8 req/s
RATES8 = (0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0, 8.0)
# HumanEval's QPS window in the paper's evaluation is [0.5, 11]
RATES_CODE8 = (0.5, 1.0, 2.0, 3.0, 5.0, 7.0, 9.0, 11.0)


def _round_half_away(x: np.ndarray) -> np.ndarray:
    return np.sign(x) * np.floor(np.abs(x) + 0.5)


def quantile_length(u: np.ndarray, p25: int, p50: int, p75: int) -> np.ndarray:
    """Piecewise log-linear quantile function of one length coordinate (R5)."""
    lo = max(1, p25 // 4)
    hi = 4 * p75
    knots_u = np.array([0.0, 0.25, 0.5, 0.75, 1.0])
    knots_l = np.log(np.array([lo, p25, p50, p75, hi], dtype=np.float64))
    v = np.exp(np.interp(u, knots_u, knots_l))
    return np.maximum(1, _round_half_away(v)).astype(np.int64)


def arrivals_us(n: int, rate: float, rate_idx: int, wid: int, seed: int = BASE_SEED) -> np.ndarray:
    """Poisson arrival timestamps in integer microseconds (R4)."""
    k0, k1 = key_from_seed(seed)
    i = np.arange(n, dtype=np.uint64)
    w0, _, _, _ = philox4x32_10(i, rate_idx, wid, 0, k0, k1)
    u = uniform_open01(w0)
    gaps = np.floor(-np.log(u) * 1e6 / float(rate)).astype(np.int64)
    return np.cumsum(gaps, dtype=np.int64)


def lengths(n: int, wl: Workload, mode: str = "dist", seed: int = BASE_SEED):
    """(prompt_len, output_len) as uint32 arrays (R5, R7: both >= 1)."""
    if mode == "fixed":
        p = np.full(n, wl.p50[0], dtype=np.uint32)
        o = np.full(n, wl.p50[1], dtype=np.uint32)
        return p, o
    if mode != "dist":
        raise ValueError(f"unknown length mode {mode!r}")
    k0, k1 = key_from_seed(seed)
    i = np.arange(n, dtype=np.uint64)
    w0, w1, _, _ = philox4x32_10(i, 0xFFFF, wl.wid, 0, k0, k1)
    pin = quantile_length(uniform_open01(w0), wl.p25[0], wl.p50[0], wl.p75[0])
    out = quantile_length(uniform_open01(w1), wl.p25[1], wl.p50[1], wl.p75[1])
    out = np.minimum(out, CTX - 1)
    pin = np.minimum(pin, CTX - out)
    return pin.astype(np.uint32), out.astype(np.uint32)


@dataclass
class Trace:
    """SoA request trace, sorted by arrival: a (int64 us), p, o (uint32)."""
    arrival_us: np.ndarray
    prompt_len: np.ndarray
    output_len: np.ndarray
    workload: str
    rate: float
    label: str = ""

    @property
    def n(self) -> int:
        return int(self.arrival_us.shape[0])


def make_trace(workload: str, n: int, rate: float, rate_idx: int, mode: str = "dist",
               seed: int = BASE_SEED, shared_lengths=None) -> Trace:
    """Build one trace.  ``shared_lengths`` lets all rates of a workload share
    one (p, o) array pair (identical by construction of the length counters)."""
    wl = WORKLOADS[workload]
    a = arrivals_us(n, rate, rate_idx, wl.wid, seed)
    if shared_lengths is None:
        p, o = lengths(n, wl, mode, seed)
    else:
        p, o = shared_lengths
    return Trace(a, p, o, workload, rate, f"{workload}/{mode}/{rate}rps/n{n}")
