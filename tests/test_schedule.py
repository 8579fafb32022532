"""The launch-order hint (paper_2412_20322_b200/schedule.py; greenllm.h gl_schedule):
host logic only -- results never depend on it (GPU test: test_gpu_parity.py::
test_schedule_hint_never_changes_results)."""
import numpy as np

from paper_2412_20322_b200 import schedule as S
from paper_2412_20322_b200.inputs import build_config, subset_chains


def test_hint_picks_the_measured_critical_trace():
    # config 4: chain 33 (DSD A100+T4, 3 req/s) is the slowest (profiles/r01f_chain_times.txt)
    g = build_config(4, n=20_000)
    lo, hi = S.first_range(g)
    assert (lo, hi) == (32, 40) and lo <= 33 < hi
    assert {g.chains[c].trace_idx for c in range(lo, hi)} == {g.chains[33].trace_idx}


def test_hint_is_a_maximal_contiguous_run_of_one_trace():
    for k in (3, 4):
        g = build_config(k, n=5_000)
        r = S.first_range(g)
        assert r is not None
        lo, hi = r
        t = g.chains[lo].trace_idx
        assert all(g.chains[c].trace_idx == t for c in range(lo, hi))
        assert lo == 0 or g.chains[lo - 1].trace_idx != t
        assert hi == len(g.chains) or g.chains[hi].trace_idx != t


def test_hint_relative_to_a_shard_and_trivial_cases():
    g = build_config(4, n=5_000)
    r = S.first_range(g, 30, 50)  # relative to the shard start
    assert r is not None and 0 <= r[0] < r[1] <= 20
    assert S.first_range(g, 7, 8) is None          # one chain: nothing to reorder
    g1 = subset_chains(g, list(range(32, 40)))      # one trace: nothing to reorder
    assert S.first_range(g1) is None
    assert S.first_range(build_config(2, n=2_000)) is None  # config 2: one trace


def test_load_regimes_match_the_docstring():
    g = build_config(4, n=20_000)
    rho = np.array([S.chain_load(g, c) for c in range(len(g.chains))])
    assert 0.7 <= rho[33] < 1.0          # heavily loaded, not saturated
    assert rho.min() < 0.7 and rho.max() >= 1.0
