"""gl_savings_surface (NEXT #3: §5 analysis surfaces, Eqs. 4-6) vs the oracle.

Every fp64 output is computed in the same fixed order with round-to-nearest and
no contraction on both sides, so the surfaces must be bit-identical (compared as
raw 64-bit patterns, NaN included); eq4 is an integer comparison.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_20322_b200 import api
from paper_2412_20322_b200 import native as N
from paper_2412_20322_b200.inputs import build_config, savings_pairs

pytestmark = pytest.mark.gpu
FIELDS = ("ratio", "op_saved_g", "emb_saved_g", "eq6_term")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    N.lib()


def check_surface(got, want):
    for f in FIELDS:
        a = np.ascontiguousarray(got[f]).view(np.int64)
        b = np.ascontiguousarray(want[f]).view(np.int64)
        bad = np.argwhere(a != b)
        assert bad.size == 0, (f, bad[:5], got[f][tuple(bad[0])], want[f][tuple(bad[0])])
    assert np.array_equal(got["eq4_energy_less"], want["eq4"])


@pytest.mark.parametrize("n", [3000, 100_000])
def test_config6_surfaces(n):
    g = build_config(6, n=n)
    pairs = savings_pairs(g)
    dg = api.DeviceGrid(g)
    stats, _ = api.eval_grid(dg)
    out = api.savings_surface(dg, stats)
    torch.cuda.synchronize()
    got = api.savings_numpy(out)
    assert got.shape == (len(pairs), len(g.scenarios))
    want = O.savings_surface(g, pairs)
    check_surface(got, want)


def test_random_stats_and_scenarios():
    rng = np.random.default_rng(11)
    g = build_config(6, n=200)
    k = len(g.chains)
    st = np.zeros(k, N.STATS_DTYPE)
    for f in ("busy_new_us", "busy_old_us", "e_new_uj", "e_old_uj"):
        st[f] = rng.integers(0, 10**13, k)
    st["e_new_uj"][:4] = 0          # zero energies (ratio may be inf / nan on both sides)
    st["busy_new_us"][:2] = 0
    st["e_new_uj"][5] = st["e_new_uj"][6] + st["e_old_uj"][6]  # Eq. 4 equality edge
    scen = np.column_stack([rng.uniform(0, 600, 300), rng.uniform(1e3, 4e8, 300),
                            rng.uniform(1e3, 4e8, 300)])
    scen[:5, 0] = 0.0
    pairs = [(int(a), int(b)) for a, b in rng.integers(0, k, (50, 2))] + [(6, 5), (0, 1), (2, 3)]
    dg = api.DeviceGrid(g)
    dstats = torch.from_numpy(st.view(np.uint8).reshape(k, 80).copy()).to(dg.device)
    out = api.savings_surface(dg, dstats, pairs=pairs, scenarios=scen)
    torch.cuda.synchronize()
    got = api.savings_numpy(out)
    want = {f: np.zeros((len(pairs), len(scen))) for f in FIELDS}
    want["eq4"] = np.zeros((len(pairs), len(scen)), np.int32)
    sd = {i: {f: int(st[i][f]) for f in N.STATS_DTYPE.names} for i in range(k)}
    with np.errstate(all="ignore"):
        for i, (d, s) in enumerate(pairs):
            cd, cs = g.chains[d], g.chains[s]
            for j, sc in enumerate(scen):
                r = O.savings(sd[d], (cd.ce_new_g, cd.ce_old_g), sd[s], (cs.ce_new_g, cs.ce_old_g),
                              *map(float, sc))
                for f in FIELDS:
                    want[f][i, j] = r[f]
                want["eq4"][i, j] = r["eq4"]
    check_surface(got, want)
