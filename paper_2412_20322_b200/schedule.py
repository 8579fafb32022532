"""Launch-order hint for gl_eval_grid_sched / gl_evaluate_host_sched (greenllm.h
`gl_schedule`): which chains to start first.

A step lasts as long as its slowest chain's serial decode walk, and a
walk starts only once the chain's DSD demand and stage scans exist.  Started first,
the slowest chain's trace pays only its own share of that prologue.  Results never
depend on the hint; a wrong guess only moves which chains wait.

Measured (same box, back to back, `scripts/sched_times.py`; profiles/r02i_sched_*.txt):
config 4 16.376 -> 16.338 ms, config 5 112.57 -> 111.83 ms (its one DSD family --
every trace shares the output lengths, hence K -- must finish before any decode, so
the hint only moves the clones), config 3 13.18 -> 13.77 ms (the hinted trace did
not hold the slowest chain).  The Python API therefore leaves the hint off by
default (``api.eval_grid(..., schedule=True)`` turns it on).

The predictor is host logic over host data (the caller's GridSpec).  A chain's decode
load is rho = lambda * E[demand] * step[cap] / cap (arrival rate x mean decode
iterations per request x the iteration time of a full batch / batch slots).  Measured
per-chain walk times (profiles/r01f_chain_times.txt, r02d_cfg5_chain_times.txt) fall
in three regimes:
  * rho < 0.7: the batch empties often; helpers walk the segments between idle points
    in parallel (config 4: 1.3-2.1 ms of a 15.9 ms step);
  * 0.7 <= rho < 1: heavily loaded, not saturated: one busy period over the whole
    trace, walked serially on the light-load path (config 4: 11.7-15.9 ms; config 5:
    94.8-100.7 ms), slowest at the low end of the band and for DSD chains;
  * rho >= 1: saturated; one busy period on the cheaper saturated path (config 4:
    8.8-9.2 ms; config 5: 87.8-94.5 ms).
"""
from __future__ import annotations

import numpy as np

MODE_DSD, MODE_SPEC_COLO = 1, 3


def chain_load(grid, c) -> float:
    """rho of chain c (see the module docstring)."""
    ch = grid.chains[c]
    tr = grid.traces[ch.trace_idx]
    a = np.asarray(tr.arrival_us)
    if tr.n < 2 or a[-1] <= a[0]:
        return 0.0
    lam = (tr.n - 1) / float(a[-1] - a[0])  # requests per us
    d = np.maximum(np.asarray(tr.output_len, dtype=np.float64) - 1.0, 0.0).mean()
    if ch.mode in (MODE_DSD, MODE_SPEC_COLO):  # E[accepted tokens per step] (R22)
        al, g = float(ch.alpha), int(ch.gamma)
        d /= (g + 1.0) if al >= 1.0 else (1.0 - al ** (g + 1)) / (1.0 - al)
    step = float(np.asarray(ch.tables.step_us)[ch.cap])
    return lam * d * step / ch.cap


def chain_cost(grid, c) -> float:
    """Predicted serial walk cost of chain c, in arbitrary units."""
    rho = chain_load(grid, c)
    n = grid.traces[grid.chains[c].trace_idx].n
    if rho < 0.7:
        w = 0.1 * rho
    elif rho < 1.0:
        w = 2.0 - rho
    else:
        w = 0.6
    if grid.chains[c].mode in (MODE_DSD, MODE_SPEC_COLO):
        w *= 1.1
    return n * w


def first_range(grid, lo: int = 0, hi: int | None = None):
    """(first_lo, first_hi), relative to lo: the contiguous run of chains in [lo, hi)
    on the trace of the chain with the largest predicted cost; None when every chain
    is on that run (nothing to reorder)."""
    hi = len(grid.chains) if hi is None else hi
    if hi - lo < 2:
        return None
    costs = [chain_cost(grid, c) for c in range(lo, hi)]
    cstar = lo + int(np.argmax(costs))
    t = grid.chains[cstar].trace_idx
    a = cstar
    while a > lo and grid.chains[a - 1].trace_idx == t:
        a -= 1
    b = cstar + 1
    while b < hi and grid.chains[b].trace_idx == t:
        b += 1
    if a == lo and b == hi:
        return None
    return a - lo, b - lo
