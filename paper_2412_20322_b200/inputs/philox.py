"""Philox4x32-10 counter-based generator, vectorised in numpy (input generation only).

This module belongs to the seeded *input* generators (SURVEY.md §8(d) "RNG"):
it draws the Poisson arrival gaps and the request lengths that both the CUDA
path and the CPU oracle read.  It holds none of the method's arithmetic.  The
CUDA library and the oracle each carry their own, independent Philox for the
speculative-decoding acceptance draws (R22); all three are pinned to the same
known-answer vectors (tests/golden/philox_kat.txt).

Algorithm (Salmon et al., Random123): per round
    (hi0, lo0) = M0 * c0,  (hi1, lo1) = M1 * c2   (32x32 -> 64-bit products)
    c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
and the key is bumped by the Weyl constants (W0, W1) between rounds.
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Return the four uint32 output words for counters (c0..c3) and key (k0, k1).

    Counters may be numpy arrays (broadcast together) or scalars.
    """
    c0 = np.asarray(c0, dtype=np.uint64) & _MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & _MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & _MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & _MASK32
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    k0 = int(k0) & 0xFFFFFFFF
    k1 = int(k1) & 0xFFFFFFFF
    for rnd in range(10):
        if rnd:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> _S32, p0 & _MASK32
        hi1, lo1 = p1 >> _S32, p1 & _MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0)
    return (c0.astype(np.uint32), c1.astype(np.uint32),
            c2.astype(np.uint32), c3.astype(np.uint32))


def key_from_seed(seed: int):
    """Split a 64-bit seed into the Philox key words (low, high)."""
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & 0xFFFFFFFF, seed >> 32


def uniform_open01(word) -> np.ndarray:
    """Map a uint32 word to (0, 1): U = (w + 0.5) * 2^-32 (never 0 or 1)."""
    return (np.asarray(word, dtype=np.float64) + 0.5) * (2.0 ** -32)
