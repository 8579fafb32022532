"""gl_link_demand (NEXT #2: link bandwidth demand, R45-R47) vs the CPU oracle.

Every gl_link_stats field is an integer and must be bit-exact: total bytes,
peak window bytes, the earliest impulse time attaining the peak, the impulse
count.  The chain statistics the leader-only logging launch produces must equal
gl_eval_grid's (the speculative launch) and the oracle's.
"""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_20322_b200 import api
from paper_2412_20322_b200 import native as N
from paper_2412_20322_b200.inputs import (MODE_DPD, MODE_DSD, MODE_SPEC_COLO, MODE_STANDALONE,
                                          build_config, subset_chains)
from tests.helpers import random_case
from tests.test_gpu_parity import INT_FIELDS, grid_of

pytestmark = pytest.mark.gpu

LINK_FIELDS = ("total_bytes", "peak_bytes", "peak_t_us", "n_impulses")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    N.lib()


def link_parity(g, window_us, params=None, chain_ids=None, check_eval=True):
    dg = api.DeviceGrid(g)
    stats, link = api.link_demand(dg, window_us, params=params)
    st_ev = None
    if check_eval:
        st_ev, _ = api.eval_grid(dg)
    torch.cuda.synchronize()
    st = api.stats_numpy(stats)
    lk = api.link_numpy(link)
    ids = range(len(g.chains)) if chain_ids is None else chain_ids
    if st_ev is not None:
        assert np.array_equal(st, api.stats_numpy(st_ev))
    for ci in ids:
        ch = g.chains[ci]
        bpt, pm = params[ci] if params is not None else (None, None)
        want = O.link_demand(g.traces[ch.trace_idx], ch, window_us, bpt, pm)
        for f in LINK_FIELDS:
            assert int(lk[ci][f]) == want[f], (g.name, ci, f, int(lk[ci][f]), want[f])
        for f in INT_FIELDS:
            if f == "capacity_ok":
                continue
            assert int(st[ci][f]) == int(want["stats"][f]), (g.name, ci, f)
    return lk


@pytest.mark.parametrize("window", [1, 7, 40, 1000])
def test_random_tiny_cases(window):
    rng = np.random.default_rng(500 + window)
    pairs, params = [], []
    for i in range(120):
        mode = int(rng.choice([MODE_DPD, MODE_DSD, MODE_STANDALONE, MODE_SPEC_COLO],
                              p=[0.4, 0.4, 0.1, 0.1]))
        tr, ch = random_case(rng, mode=mode, cap=int(rng.choice([1, 2, 3, 4, 7])))
        pairs.append((tr, ch))
        params.append((int(rng.integers(0, 60)), int(rng.integers(0, 90))))
    link_parity(grid_of(pairs), window, params)


@pytest.mark.parametrize("cap", [31, 32, 33, 64, 100, 256])
def test_caps_and_general_loop(cap):
    rng = np.random.default_rng(cap)
    pairs, params = [], []
    for i in range(16):
        tr, ch = random_case(rng, n=int(rng.integers(50, 400)), mode=int(rng.integers(0, 2)),
                             cap=cap)
        pairs.append((tr, ch))
        params.append((int(rng.integers(1, 60)), int(rng.integers(1, 90))))
    link_parity(grid_of(pairs), int(rng.choice([5, 50, 500])), params)


def test_config1_and_colocated_zero():
    for g in (build_config(1), build_config(1, rate=0.5), build_config(1, mode="fixed")):
        link_parity(g, 1_000_000)
    g = subset_chains(build_config(6, n=3000), list(range(64, 80)))
    lk = link_parity(g, 1_000_000, chain_ids=[])
    assert (lk["total_bytes"] == 0).all() and (lk["peak_t_us"] == -1).all()


def test_config2_full():
    link_parity(build_config(2), 1_000_000)


def test_config4_sampled_chains_full_size():
    g = build_config(4)
    ids = list(range(0, 64, 5))
    link_parity(subset_chains(g, ids), 1_000_000, check_eval=False)


def test_window_monotone_and_total_invariant():
    g = build_config(2, n=3000)
    dg = api.DeviceGrid(g)
    prev = None
    for w in (1, 10_000, 1_000_000, 10**7, 10**13):
        _, link = api.link_demand(dg, w)
        lk = api.link_numpy(link)
        if prev is not None:
            assert (lk["peak_bytes"] >= prev["peak_bytes"]).all()
            assert np.array_equal(lk["total_bytes"], prev["total_bytes"])
        prev = lk
    assert np.array_equal(prev["peak_bytes"], prev["total_bytes"])


def test_config5_sampled_chains_full_size():
    # 1M-request LongBench traces (DSD 70B/7B): the largest logs and windows
    g = build_config(5)
    link_parity(subset_chains(g, [0, 319]), 1_000_000, check_eval=False)


def test_config3_bandwidth_axis():
    # config 3 sweeps the link bandwidth (1-100 Gbps) for both modes, incl. the
    # capacity-infeasible 13B DPD chains (still simulated, R38)
    g = build_config(3, n=4000)
    ids = list(range(0, 128, 9))
    lk = link_parity(subset_chains(g, ids), 1_000_000, check_eval=False)
    assert (lk["total_bytes"] > 0).all()


@pytest.mark.parametrize("n_chains,n", [(4, 30000), (60, 3000)])
def test_logged_speculation_stress(n_chains, n):
    # quiet and busy phases: many idle points, long helper runs, aborted runs; the
    # helpers' logs are copied by the leader only for accepted runs
    from tests.test_gpu_parity import _phased_case
    rng = np.random.default_rng(4242 + n_chains)
    pairs, params = [], []
    for i in range(n_chains):
        mode = (MODE_DPD, MODE_DSD)[i % 2]
        pairs.append(_phased_case(rng, n, mode, int(rng.choice([4, 16, 31, 48])),
                                  monotone=(i % 4 < 2)))
        params.append((int(rng.integers(1, 60)), int(rng.integers(1, 90))))
    link_parity(grid_of(pairs), int(rng.choice([1000, 50_000, 1_000_000])), params)
