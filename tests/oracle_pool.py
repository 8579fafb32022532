"""The CPU oracle fanned over every host core (test infrastructure).

Each timing chain is one independent, single-threaded oracle_simulate_chain call
in a forked worker process (the oracle itself is unchanged: SURVEY §8(d) runs
"the same single-threaded binary across all host cores as independent
processes").  When the GPU's per-request rows are given, each worker compares its
chain's (ttft, finish) pairs element by element and returns only the mismatches,
so nothing large crosses the process boundary.  The carbon / Alg. 1 epilogue runs
in the parent (oracle.grid_epilogue).
"""
from __future__ import annotations

import multiprocessing as mp
import os
import warnings

import numpy as np

from oracle import oracle as O

_JOB = {}  # set in the parent right before the pool forks


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _chain(ci):
    g = _JOB["grid"]
    ch = g.chains[ci]
    want_pr = _JOB["per_request"]
    st, ttft, fin = O.simulate_chain(g.traces[ch.trace_idx], ch, per_request=want_pr)
    bad = None
    gpu = _JOB["gpu_pr"]
    if want_pr and gpu is not None and st["status"] == 0:
        lo, hi = _JOB["offs"][ci], _JOB["offs"][ci + 1]
        got = gpu[lo:hi]
        idx = np.nonzero((got[:, 0] != ttft) | (got[:, 1] != fin))[0]
        if idx.size:
            k = idx[:5]
            bad = (int(idx.size), k.tolist(), got[k].tolist(), ttft[k].tolist(), fin[k].tolist())
    return ci, st, bad


def _cost(g, ci):
    ch = g.chains[ci]
    n = g.traces[ch.trace_idx].n
    return n * (4 if ch.mode in (1, 3) else 1)  # DSD-like chains draw per member-step


def evaluate_grid(grid, chain_ids=None, gpu_per_request=None, per_request=False, procs=None):
    """Oracle statistics for ``chain_ids`` (default: all) on every host core, plus
    the carbon / Alg. 1 epilogue.  ``gpu_per_request`` = the GPU's [sum n, 2] rows
    (chain-major, chain order) to compare element by element in the workers:
    result["mismatch"] = {chain: (count, first indices, got, want ttft, want finish)}."""
    ids = list(range(len(grid.chains))) if chain_ids is None else list(chain_ids)
    offs = np.concatenate([[0], np.cumsum([grid.traces[c.trace_idx].n for c in grid.chains])])
    _JOB.update(grid=grid, per_request=bool(per_request or gpu_per_request is not None),
                gpu_pr=gpu_per_request, offs=offs)
    O.lib()  # built before forking
    order = sorted(ids, key=lambda ci: -_cost(grid, ci))
    procs = max(1, min(procs or host_cores(), len(order)))
    stats, mism = {}, {}
    try:
        if procs == 1:
            res = map(_chain, order)
            for ci, st, bad in res:
                stats[ci] = st
                if bad:
                    mism[ci] = bad
        else:
            with warnings.catch_warnings():  # the workers never touch CUDA or threads
                warnings.simplefilter("ignore", DeprecationWarning)
                pool = mp.get_context("fork").Pool(procs)
            with pool:
                for ci, st, bad in pool.imap_unordered(_chain, order, chunksize=1):
                    stats[ci] = st
                    if bad:
                        mism[ci] = bad
    finally:
        _JOB.clear()
    out = O.grid_epilogue(grid, stats)
    out["mismatch"] = mism
    return out
