"""Plain-Python decode-stream builder and event simulator for analysis scripts.

Analysis only (not the product path, not the oracle): rebuilds a config chain's
decode stream (r_q, d_q) with numpy -- stage 1 / stage 2 recurrences, and for DSD
the demand K_j from the same Philox draws (R22) -- and simulates the decode stage
event by event.  Used by scripts/regime.py-style studies of the speculation.
"""
import heapq
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2412_20322_b200.inputs import build_config  # noqa: E402
from paper_2412_20322_b200.inputs.philox import philox4x32_10  # noqa: E402

ACCEPT_STREAM = 0x41434350


def dsd_demand(o, gamma, alpha, seed):
    x, thr = 1.0, []
    for c in range(gamma):
        x *= alpha
        thr.append(int(np.floor(x * 4294967296.0)))
    thr = np.array(thr, dtype=np.uint64)
    n = len(o)
    need = o.astype(np.int64) - 1
    K = np.zeros(n, np.int64)
    tok = np.zeros(n, np.int64)
    active = need > 0
    s = 0
    k0, k1 = seed & 0xFFFFFFFF, seed >> 32
    j = np.arange(n, dtype=np.uint32)
    while active.any():
        idx = np.nonzero(active)[0]
        w = philox4x32_10(np.full(len(idx), s >> 2, np.uint32), j[idx],
                          np.full(len(idx), ACCEPT_STREAM, np.uint32), np.zeros(len(idx), np.uint32),
                          k0, k1)
        word = np.asarray(w[s & 3], dtype=np.uint64)
        acc = 1 + (word[:, None] < thr[None, :]).sum(axis=1)
        tok[idx] += acc
        K[idx] += 1
        active[idx] = tok[idx] < need[idx]
        s += 1
    return K


def chain_stream(cfg, ci, n=None):
    g = build_config(cfg, n=n) if n else build_config(cfg)
    ch = g.chains[ci]
    tr = g.traces[ch.trace_idx]
    a = tr.arrival_us.astype(np.int64)
    p = tr.prompt_len.astype(np.int64)
    o = tr.output_len.astype(np.int64)
    t1, t2 = ch.tables.t1_us.astype(np.int64), ch.tables.t2_us.astype(np.int64)
    step = ch.tables.step_us.astype(np.int64)
    c = np.empty(len(a), np.int64)
    x = -(1 << 62)
    for i in range(len(a)):
        x = max(x, a[i]) + t1[p[i]]
        c[i] = x
    dec = np.nonzero(o > 1)[0]
    r = np.empty(len(dec), np.int64)
    y = -(1 << 62)
    for k, i in enumerate(dec):
        y = max(y, c[i]) + t2[p[i]]
        r[k] = y
    if ch.mode == 0:
        d = o[dec] - 1
    else:
        d = dsd_demand(o, ch.gamma, ch.alpha, ch.seed)[dec]
    return ch, r, d, step, ch.cap


def simulate(r, d, step, cap, q0=0, stops=None, limit=1 << 40):
    """Run from an empty batch at r[q0].  Returns (stop q or None, fin dict, events).
    With ``stops`` (a set of q), stop at the first stop q > q0 where the batch is
    empty when it becomes ready."""
    M = len(r)
    T, I = 0, 0
    heap = []
    q = q0
    maxfin = -(1 << 62)
    fin = {}
    events = 0
    while True:
        if not heap:
            if q >= M:
                return M, fin, events
            if stops is not None and q > q0 and q in stops and maxfin <= r[q]:
                return q, fin, events
            if q - q0 > limit:
                return None, fin, events
            T = max(T, r[q])
        while q < M and len(heap) < cap and r[q] <= T:
            heapq.heappush(heap, (I + d[q], q))
            q += 1
            events += 1
        b = len(heap)
        kL = heap[0][0] - I
        kJ = -(-(r[q] - T) // step[b]) if (q < M and b < cap) else 1 << 62
        k = min(kL, kJ)
        T += k * step[b]
        I += k
        while heap and heap[0][0] == I:
            fin[heapq.heappop(heap)[1]] = T
            maxfin = max(maxfin, T)
            events += 1
