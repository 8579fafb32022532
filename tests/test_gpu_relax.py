"""k_relax (the decode stage as an exact parallel-in-time fixed point, k_relax.cuh)
against the CPU oracle, element by element.

GL_RELAX=solo runs k_relax alone before k_decode, so every chain it solves is
written by k_relax (k_relax_out) and k_decode walks only the chains it gave up on;
GL_RELAX=1 is the production race (both walk the selected chains, the first to
finish owns the statistics).  Either way every integer must match the oracle.
"""
import numpy as np
import pytest

from paper_2412_20322_b200.inputs import (MODE_DPD, MODE_DSD, build_config, custom_trace,
                                          subset_chains)
from tests.helpers import random_case
from tests.test_gpu_parity import _gpu, assert_parity, grid_of  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.fixture
def solo(monkeypatch):
    monkeypatch.setenv("GL_RELAX", "solo")
    yield


def test_relax_solo_random_cases(solo):
    """400 random small chains of every mode; the one-row disaggregated ones go
    through k_relax (any load: saturated ones may exhaust the sweep budget and fall
    back to k_decode)."""
    rng = np.random.default_rng(91)
    pairs = [random_case(rng, n=int(rng.integers(1, 3000))) for _ in range(400)]
    assert_parity(grid_of(pairs))


@pytest.mark.parametrize("cap", [1, 2, 3, 8, 16, 31])
def test_relax_solo_caps_dense(solo, cap):
    """Dense arrivals (long busy periods, saturated stretches, multi-leaves)."""
    rng = np.random.default_rng(1000 + cap)
    pairs = []
    for mode in (MODE_DPD, MODE_DSD):
        for n in (1, 2, 33, 1000, 5000):
            tr, ch = random_case(rng, n=n, mode=mode, cap=cap)
            a = np.sort(rng.integers(0, int(rng.integers(5, 80)) * n, n))
            pairs.append((custom_trace(a, tr.prompt_len, tr.output_len), ch))
    assert_parity(grid_of(pairs))


def test_relax_solo_solves_chains(solo, monkeypatch, capfd):
    """k_relax really owns chains in solo mode (its debug line reports state 3 =
    solved and owned), and the results are the oracle's."""
    monkeypatch.setenv("GL_RELAX_DEBUG", "1")
    g = build_config(4, n=4000)
    assert_parity(subset_chains(g, [33, 51, 46, 6]))
    out = capfd.readouterr().out
    assert "state 3" in out, out[-2000:]


def test_relax_solo_config4_reduced(solo):
    assert_parity(build_config(4, n=8000))


def test_relax_solo_config2_full(solo):
    assert_parity(build_config(2))


def test_relax_race_config4_full_heavy_chains(monkeypatch):
    """The production race at full size: the heavily loaded chains (33, 51, 63, 46,
    26, 21) request by request, every statistic, and the whole grid's Alg. 1."""
    monkeypatch.setenv("GL_RELAX", "1")
    g = build_config(4)
    assert_parity(g, chain_ids=[33, 51, 63, 46, 26, 21])


def test_relax_solo_stage_group_secondaries(solo):
    """Config 5's stage groups: secondary chains share their primary's ready times and
    bring their own DSD demand (k_stage_clone, a DSD family) -- relaxed all the same."""
    g = build_config(5, n=3000)
    assert_parity(subset_chains(g, list(range(0, 80))), per_request=True)
