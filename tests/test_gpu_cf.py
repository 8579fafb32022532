"""gl_complete_matrices (NEXT #4: collaborative filtering by ALS, R50-R53) vs the
oracle.  Observed entries and status bits must be exact; completed entries and
the factors agree to fp64 rounding (the V-step's parallel row sums reorder the
additions): |gpu - oracle| <= 1e-9 x the matrix RMS scale (R50)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_20322_b200 import api
from paper_2412_20322_b200 import native as N
from paper_2412_20322_b200.inputs import build_config
from paper_2412_20322_b200.inputs.cf import als_init, low_rank_matrix, observation_mask

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    N.lib()


def run_batch(xs, ms, rank, lam, iters, v0s, lo=-np.inf, hi=np.inf):
    dev = torch.device("cuda")
    x = torch.from_numpy(np.stack(xs)).to(dev)
    m = torch.from_numpy(np.stack(ms)).to(dev)
    v0 = torch.from_numpy(np.stack(v0s)).to(dev)
    out, U, V, st = api.complete_matrices(x, m, rank, lam, iters, v0, lo, hi)
    torch.cuda.synchronize()
    return out.cpu().numpy(), U.cpu().numpy(), V.cpu().numpy(), st.cpu().numpy()


def compare(xs, ms, rank, lam, iters, v0s, lo=-np.inf, hi=np.inf):
    out, U, V, st = run_batch(xs, ms, rank, lam, iters, v0s, lo, hi)
    worst = 0.0
    for b, (x, m, v0) in enumerate(zip(xs, ms, v0s)):
        o_out, o_U, o_V, o_st = O.als_complete(x, m, rank, lam, iters, v0, lo, hi)
        assert st[b] == o_st
        assert np.array_equal(out[b][m == 1], x[m == 1])  # verbatim
        scale = max(np.sqrt((x ** 2).mean()), 1e-300)
        err = max(np.abs(out[b] - o_out).max(), np.abs(U[b] @ V[b].T - o_U @ o_V.T).max()) / scale
        worst = max(worst, err)
        assert err <= TOL, (b, err)
        filled = out[b][m == 0]
        assert ((filled >= lo) & (filled <= hi)).all()  # observed entries are kept as given
    return worst


@pytest.mark.parametrize("rank", [1, 2, 3, 4, 8])
def test_random_low_rank_batches(rank):
    xs, ms, vs = [], [], []
    for s in range(12):
        xs.append(low_rank_matrix(57, 11, min(rank, 3), seed=100 * rank + s))
        ms.append(observation_mask(57, 11, 0.3, seed=100 * rank + s))
        vs.append(als_init(11, rank, seed=s))
    compare(xs, ms, rank, 0.1, 60, vs)


@pytest.mark.parametrize("shape", [(1, 1), (1, 5), (9, 1), (300, 16), (200, 17), (64, 40),
                                   (5000, 8), (33, 1024)])
def test_shapes(shape):
    r, c = shape
    k = min(2, r, c)
    x = low_rank_matrix(r, c, k, seed=r * 7 + c)
    m = observation_mask(r, c, 0.25, seed=r + c)
    compare([x], [m], k, 0.1, 40, [als_init(c, k)])


def test_status_bits_and_clamp():
    x = low_rank_matrix(20, 6, 2, seed=3)
    m1 = observation_mask(20, 6, 0.3, seed=3, keep_rows_cols=False)
    m1[4] = 0
    m2 = observation_mask(20, 6, 0.3, seed=4)
    m2[:, 2] = 0
    m3 = observation_mask(20, 6, 0.5, seed=5)
    compare([x, x, x], [m1, m2, m3], 2, 0.1, 30, [als_init(6, 2)] * 3, lo=0.0, hi=2.5)


def test_alg1_matrices_of_config4():
    # the Alg. 1 matrices of a reduced config 4 (carbon, SLO attainment) with 30% of
    # the cells hidden: complete both (independently) on the GPU vs the oracle
    g = build_config(4, n=2000)
    ref = O.evaluate_grid(g)
    carbon = ref["carbon"]
    ok = np.array([[ref["stats"][int(k)]["slo_ok"] / ref["stats"][int(k)]["n"]
                    for k in row] for row in g.cell_chain.reshape(g.rows, g.cols)])
    m = observation_mask(g.rows, g.cols, 0.3, seed=42)
    w = compare([carbon, ok], [m, m], 2, 0.1, 200, [als_init(g.cols, 2)] * 2, lo=0.0,
                hi=np.inf)
    assert w <= TOL
    print(f"config-4 Alg. 1 matrices: max |gpu - oracle| / scale = {w:.3e}")
    out, _, _, _ = run_batch([ok], [m], 2, 0.1, 200, [als_init(g.cols, 2)], 0.0, 1.0)
    assert ((out >= 0) & (out <= 1)).all()


def test_large_batch_one_cta_per_matrix():
    # >= one wave of matrices: the one-CTA-per-matrix kernel (small batches use the
    # cooperative multi-CTA kernel); both must match the oracle
    xs, ms, vs = [], [], []
    for s in range(320):
        xs.append(low_rank_matrix(40, 6, 2, seed=5000 + s))
        ms.append(observation_mask(40, 6, 0.3, seed=5000 + s))
        vs.append(als_init(6, 2, seed=s))
    compare(xs, ms, 2, 0.1, 30, vs)


def test_iters_zero_and_determinism():
    x = low_rank_matrix(3000, 9, 2, seed=8)
    m = observation_mask(3000, 9, 0.3, seed=8)
    compare([x], [m], 2, 0.1, 0, [als_init(9, 2)])
    a = run_batch([x], [m], 2, 0.1, 50, [als_init(9, 2)])
    b = run_batch([x], [m], 2, 0.1, 50, [als_init(9, 2)])
    assert all(np.array_equal(u, v) for u, v in zip(a, b))


def test_argmin_matrices_vs_oracle():
    rng = np.random.default_rng(12)
    dev = torch.device("cuda")
    for rows, cols in ((1, 1), (7, 3), (100, 8), (33, 40), (4096, 10)):
        carbon = rng.choice([1.0, 2.0, 3.0, 2.5], (rows, cols))
        att = rng.choice([0.5, 0.85, 0.9, 0.95, 1.0], (rows, cols))
        present = (rng.random((rows, cols)) < 0.85).astype(np.uint8)
        for prio, dcol in ((0, -1), (1, cols - 1)):
            for pr in (present, None):
                ch, fb = api.argmin_matrices(torch.from_numpy(carbon).to(dev),
                                             torch.from_numpy(att).to(dev),
                                             None if pr is None else torch.from_numpy(pr).to(dev),
                                             0.9, prio, dcol)
                want = O.alg1_matrices(carbon, att, pr, 0.9, prio, dcol)
                assert np.array_equal(ch.cpu().numpy(), want[0])
                assert np.array_equal(fb.cpu().numpy(), want[1])


def test_cf_then_alg1_pipeline_config4():
    # Alg. 1 line 1 then lines 2-9: hide 30% of config 4's (carbon, attainment) cells,
    # complete both on the GPU, choose on the GPU; the same on the oracle side
    g = build_config(4, n=2000)
    ref = O.evaluate_grid(g)
    carbon = ref["carbon"]
    att = np.array([[ref["stats"][int(k)]["slo_ok"] / ref["stats"][int(k)]["n"] for k in row]
                    for row in g.cell_chain.reshape(g.rows, g.cols)])
    m = observation_mask(g.rows, g.cols, 0.3, seed=7)
    v0 = als_init(g.cols, 2)
    out, _, _, st = run_batch([carbon, att], [m, m], 2, 0.1, 200, [v0, v0], lo=0.0)
    c_gpu, a_gpu = out[0], np.minimum(out[1], 1.0)
    dev = torch.device("cuda")
    ch, fb = api.argmin_matrices(torch.from_numpy(c_gpu).to(dev), torch.from_numpy(a_gpu).to(dev),
                                 None, 0.9)
    # the oracle's choice on the GPU-completed matrices (completion parity is tested above)
    want = O.alg1_matrices(c_gpu, a_gpu, None, 0.9)
    assert np.array_equal(ch.cpu().numpy(), want[0]) and np.array_equal(fb.cpu().numpy(), want[1])
    # where no cell was hidden the decision equals Alg. 1 on the simulated matrices
    full_rows = m.all(axis=1)
    assert np.array_equal(ch.cpu().numpy()[full_rows], ref["choice"][full_rows])
