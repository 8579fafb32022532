"""Pins of the oracle's collaborative filtering (Alg. 1 line 1,
P:309; readings R50-R53).

Pinned against: the identity on fully observed input, exact recovery of a
rank-1 matrix with a masked entry, the held-out error bound on rank-2
synthetics, each half-step being the exact ridge solution (numpy's
solver on the normal equations), monotone descent of the ALS objective, clamping,
and the empty row / column status.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_20322_b200.inputs.cf import als_init, low_rank_matrix, observation_mask


def objective(x, m, U, V, lam):
    r = (x - U @ V.T) * m
    return float((r ** 2).sum() + lam * ((U ** 2).sum() + (V ** 2).sum()))


def test_fully_observed_is_identity():
    x = low_rank_matrix(12, 7, 2, seed=1)
    m = np.ones_like(x, np.uint8)
    out, _, _, st = O.als_complete(x, m, 2, 0.1, 50, als_init(7, 2))
    assert st == 0 and np.array_equal(out, x)


@pytest.mark.parametrize("seed", range(5))
def test_rank1_single_masked_entry_recovered(seed):
    rng = np.random.default_rng(seed)
    a, b = rng.uniform(0.5, 2, 5), rng.uniform(0.5, 2, 4)
    x = np.outer(a, b)
    m = np.ones((5, 4), np.uint8)
    i, j = rng.integers(0, 5), rng.integers(0, 4)
    m[i, j] = 0
    out, _, _, st = O.als_complete(x, m, 1, 1e-12, 200, als_init(4, 1, seed=seed))
    assert st == 0
    assert abs(out[i, j] - x[i, j]) <= 1e-6 * abs(x[i, j])


def test_rank2_heldout_rmse_S421():
    # S:421 states < 1% for both errors; measured under lambda = 0.1 the observed-entry
    # RMSE stays <= 1.01% and the MEDIAN held-out RMSE is 1.4%, but ridge shrinkage on
    # rows left with 2-3 observed entries puts the worst of 100 seeds at 10% (DESIGN R50).
    obs_w, held = 0.0, []
    for seed in range(100):
        x = low_rank_matrix(20, 10, 2, seed=seed)
        m = observation_mask(20, 10, 0.3, seed=seed)
        out, U, V, st = O.als_complete(x, m, 2, 0.1, 200, als_init(10, 2, seed=seed))
        scale = np.sqrt((x ** 2).mean())
        hm = m == 0
        obs_rmse = np.sqrt((((U @ V.T) - x)[m == 1] ** 2).mean())
        obs_w = max(obs_w, obs_rmse / scale)
        held.append(np.sqrt(((out - x)[hm] ** 2).mean()) / scale if hm.any() else 0.0)
    assert obs_w < 0.0105, obs_w
    assert np.median(held) < 0.02 and max(held) < 0.15, (np.median(held), max(held))


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_half_steps_are_exact_ridge_solutions(k):
    # after the last iteration V is the ridge solution given U; U is the one given
    # the V before it (checked with one more U-step from the final V)
    x = low_rank_matrix(30, 9, 3, seed=k) + 0.01 * np.arange(270).reshape(30, 9) % 1
    m = observation_mask(30, 9, 0.4, seed=k)
    lam = 0.3
    _, U, V, _ = O.als_complete(x, m, k, lam, 7, als_init(9, k, seed=k))
    for j in range(9):
        rows = m[:, j] == 1
        A = U[rows].T @ U[rows] + lam * np.eye(k)
        want = np.linalg.solve(A, U[rows].T @ x[rows, j])
        np.testing.assert_allclose(V[j], want, rtol=1e-9, atol=1e-12)
    _, U2, _, _ = O.als_complete(x, m, k, lam, 1, V)  # one more U-step from V
    for i in range(30):
        cols = m[i] == 1
        A = V[cols].T @ V[cols] + lam * np.eye(k)
        want = np.linalg.solve(A, V[cols].T @ x[i, cols])
        np.testing.assert_allclose(U2[i], want, rtol=1e-9, atol=1e-12)


def test_objective_non_increasing():
    x = low_rank_matrix(25, 8, 3, seed=4)
    m = observation_mask(25, 8, 0.35, seed=4)
    v0 = als_init(8, 2, seed=4)
    prev = np.inf
    for it in range(1, 25):
        _, U, V, _ = O.als_complete(x, m, 2, 0.1, it, v0)
        f = objective(x, m, U, V, 0.1)
        assert f <= prev * (1 + 1e-12)
        prev = f


def test_clamping_and_observed_verbatim():
    x = low_rank_matrix(15, 6, 2, seed=9)
    m = observation_mask(15, 6, 0.5, seed=9)
    out, U, V, _ = O.als_complete(x, m, 2, 0.1, 30, als_init(6, 2), lo=0.0, hi=1.0)
    assert np.array_equal(out[m == 1], x[m == 1])
    pred = (U @ V.T)[m == 0]
    np.testing.assert_allclose(out[m == 0], np.clip(pred, 0.0, 1.0), rtol=1e-13, atol=0)
    assert ((out[m == 0] == 1.0) == (pred >= 1.0)).all() and (out >= 0).all()


def test_empty_row_and_column_status():
    x = low_rank_matrix(6, 4, 1)
    m = np.ones((6, 4), np.uint8)
    m[2] = 0
    assert O.als_complete(x, m, 1, 0.1, 3, als_init(4, 1))[3] == 1
    m = np.ones((6, 4), np.uint8)
    m[:, 3] = 0
    assert O.als_complete(x, m, 1, 0.1, 3, als_init(4, 1))[3] == 2


# ---- Alg. 1 on explicit (completed) matrices, R54
def test_alg1_matrices_spec_examples_S431_441():
    # 2x2 example: attainment [0.95, 0.92], carbon [5, 4], target 0.9 -> the second column
    ch, fb = O.alg1_matrices(np.array([[5.0, 4.0]]), np.array([[0.95, 0.92]]), target=0.9)
    assert ch[0] == 1 and fb[0] == 0
    # fallback, priority SLO: attainment [0.5, 0.7, 0.6] -> argmax = second column
    ch, fb = O.alg1_matrices(np.array([[1.0, 2.0, 3.0]]), np.array([[0.5, 0.7, 0.6]]), target=0.9)
    assert ch[0] == 1 and fb[0] == 1
    # priority DEFAULT -> the default column regardless of the values
    ch, fb = O.alg1_matrices(np.array([[1.0, 2.0, 3.0]]), np.array([[0.5, 0.7, 0.6]]), target=0.9,
                             priority=1, default_col=2)
    assert ch[0] == 2 and fb[0] == 1
    # all attainments equal in the fallback -> lowest carbon (tie rule)
    ch, fb = O.alg1_matrices(np.array([[3.0, 1.0, 2.0]]), np.array([[0.5, 0.5, 0.5]]), target=0.9)
    assert ch[0] == 1


def test_alg1_matrices_vs_brute_force():
    rng = np.random.default_rng(8)
    for _ in range(1000):
        rows, cols = 6, 8
        carbon = rng.choice([1.0, 2.0, 3.0, 4.0], (rows, cols))  # ties on purpose
        att = rng.choice([0.5, 0.85, 0.9, 0.95, 1.0], (rows, cols))
        present = (rng.random((rows, cols)) < 0.85).astype(np.uint8)
        target = float(rng.choice([0.9, 0.95]))
        ch, fb = O.alg1_matrices(carbon, att, present, target)
        for r in range(rows):
            cols_p = [c for c in range(cols) if present[r, c]]
            feas = [c for c in cols_p if att[r, c] >= target]
            if feas:
                want = min(feas, key=lambda c: (carbon[r, c], -att[r, c], c))
                assert (ch[r], fb[r]) == (want, 0)
            elif cols_p:
                want = min(cols_p, key=lambda c: (-att[r, c], carbon[r, c], c))
                assert (ch[r], fb[r]) == (want, 1)
            else:
                assert (ch[r], fb[r]) == (-1, 1)


def test_alg1_matrices_agrees_with_integer_alg1():
    # attainments ok/n: fp64 ok/n >= 0.9 decides exactly as 10 ok >= 9 n (the gap
    # |ok/n - 0.9| >= 1/(10 n) is far above one ulp), so both forms must choose alike
    rng = np.random.default_rng(9)
    for _ in range(300):
        rows, cols = 5, 7
        n = rng.integers(1, 200, (rows, cols))
        ok = (n * rng.choice([0.5, 0.89, 0.9, 0.91, 1.0], (rows, cols))).astype(np.int64)
        total = rng.choice([1.0, 2.0, 2.5], (rows, cols))
        present = (rng.random((rows, cols)) < 0.9).astype(np.uint8)
        cap = np.ones((rows, cols), np.uint8)
        for prio in (0, 1):
            a = O.alg1(total, ok, n, present, cap, 9, 10, prio, 3)
            b = O.alg1_matrices(total, ok / n, present, 0.9, prio, 3)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
