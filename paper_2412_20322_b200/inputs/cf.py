"""Seeded inputs for collaborative filtering: partially
observed matrices and the ALS initial factor V0 (R51: the method's random draws
are passed in as inputs).  Input generation only -- no ALS arithmetic here.

Philox counters: (i, j, 0xCF00 + stream, 0) with the base seed as key, so every
entry is independent of the matrix shape it is drawn in.
"""
from __future__ import annotations

import numpy as np

from .philox import key_from_seed, philox4x32_10, uniform_open01
from .workload import BASE_SEED

_STREAM = 0xCF00


def _u(shape, stream: int, seed: int) -> np.ndarray:
    k0, k1 = key_from_seed(seed)
    i = np.arange(shape[0], dtype=np.uint64)[:, None]
    j = np.arange(shape[1], dtype=np.uint64)[None, :]
    w = philox4x32_10(i, j, _STREAM + stream, 0, k0, k1)[0]
    return uniform_open01(w)


def als_init(cols: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    """V0 [cols, rank], entries uniform in (0.1, 1.0)."""
    return 0.1 + 0.9 * _u((cols, rank), 0, seed)


def observation_mask(rows: int, cols: int, frac_missing: float, seed: int = BASE_SEED,
                     keep_rows_cols: bool = True) -> np.ndarray:
    """uint8 [rows, cols]: 1 = observed.  Each entry is missing with probability
    frac_missing; with keep_rows_cols every row and column keeps >= 1 entry."""
    m = (_u((rows, cols), 1, seed) >= frac_missing).astype(np.uint8)
    if keep_rows_cols:
        for i in np.nonzero(m.sum(1) == 0)[0]:
            m[i, i % cols] = 1
        for j in np.nonzero(m.sum(0) == 0)[0]:
            m[j % rows, j] = 1
    return m


def low_rank_matrix(rows: int, cols: int, rank: int, seed: int = BASE_SEED,
                    lo: float = 0.5, hi: float = 1.5) -> np.ndarray:
    """A rank-`rank` matrix A B^T with factor entries uniform in (lo, hi)."""
    a = lo + (hi - lo) * _u((rows, rank), 2, seed)
    b = lo + (hi - lo) * _u((cols, rank), 3, seed)
    return a @ b.T
