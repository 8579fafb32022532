"""Emulate candidate-hop speculation for one config-4 DPD chain (analysis only).

Candidates: request 0 plus, per window of W decode requests, the request with the
largest slack r_q - max_{q'<q}(r_q' + d_q' * step_min) (only if positive: a
non-positive slack proves the stage busy).  A helper run from candidate k starts
from an empty batch and continues until it reaches a candidate where its own run is
idle (or gives up after LMAX requests).  Prints truly-idle fraction of the
candidates, helper work, and the critical path estimate in requests.

usage: python scripts/spec_sim.py <chain> [W] [LMAX] [H]
"""
import heapq
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2412_20322_b200.inputs import build_config  # noqa: E402

ci = int(sys.argv[1])
W = int(sys.argv[2]) if len(sys.argv) > 2 else 128
LMAX = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
H = int(sys.argv[4]) if len(sys.argv) > 4 else 8
g = build_config(4, n=100_000)
ch = g.chains[ci]
tr = g.traces[ch.trace_idx]
a, p, o = tr.arrival_us.astype(np.int64), tr.prompt_len.astype(np.int64), tr.output_len.astype(np.int64)
t1, t2, step = ch.tables.t1_us.astype(np.int64), ch.tables.t2_us.astype(np.int64), ch.tables.step_us.astype(np.int64)
cap = ch.cap
n = len(a)
c = np.empty(n, np.int64)
x = -(1 << 62)
for i in range(n):
    x = max(x, a[i]) + t1[p[i]]
    c[i] = x
dec = np.nonzero(o > 1)[0]
r = np.empty(len(dec), np.int64)
y = -(1 << 62)
for k, i in enumerate(dec):
    y = max(y, c[i]) + t2[p[i]]
    r[k] = y
d = (o[dec] - 1) if ch.mode == 0 else None
assert d is not None, "DPD only"
M = len(dec)


def run(q0, stop_at, limit):
    """Simulate from an empty batch at r[q0]; stop at the first q in stop_at (q > q0)
    where the run is idle.  Returns (q_stop or None, requests simulated, fin)."""
    T, I = 0, 0
    heap = []
    q = q0
    maxfin = -(1 << 62)
    fin = {}
    while True:
        if q < M and q > q0 and q in stop_at and maxfin <= r[q] and not heap:
            return q, q - q0, fin
        if q - q0 > limit:
            return None, q - q0, fin
        if q >= M and not heap:
            return M, q - q0, fin
        if not heap:
            T = max(T, r[q])
        while q < M and len(heap) < cap and r[q] <= T:
            if q > q0 and q in stop_at and maxfin <= r[q] and not heap:
                break
            heapq.heappush(heap, (I + d[q], q))
            q += 1
        if not heap:
            continue
        b = len(heap)
        kL = heap[0][0] - I
        kJ = -(-(r[q] - T) // step[b]) if (q < M and b < cap) else 1 << 62
        k = min(kL, kJ)
        T += k * step[b]
        I += k
        while heap and heap[0][0] == I:
            fq = heapq.heappop(heap)[1]
            fin[fq] = T
            maxfin = max(maxfin, T)


# true run and idle flags
_, _, fin = run(0, set(), 1 << 40)
finv = np.array([fin[q] for q in range(M)])
prevmax = np.maximum.accumulate(np.concatenate([[-(1 << 62)], finv[:-1]]))
idle = prevmax <= r

smin = int(step[1:].min())
lb = r + d * smin
lbmax = np.maximum.accumulate(np.concatenate([[-(1 << 62)], lb[:-1]]))
slack = r - lbmax
cands = [0]
for w in range(1, (M + W - 1) // W):
    lo, hi = w * W, min(w * W + W, M)
    j = lo + int(np.argmax(slack[lo:hi]))
    if slack[j] > 0:
        cands.append(j)
cset = set(cands)
print(f"chain {ci} {ch.label}: idle requests {idle.sum()}, necessary-condition passes "
      f"{(slack > 0).sum()}, candidates {len(cands)}, truly idle {np.mean([idle[q] for q in cands]):.2f}")
nxt, work = {}, {}
for k in cands:
    e, L, _ = run(k, cset, LMAX)
    nxt[k], work[k] = e, L
tot = sum(work.values())
# leader hops: at a truly idle candidate, jump if the helper closed; else walk to the
# next candidate idle in the true run
hop, q, walked, hops = 0, 0, 0, 0
while q < M:
    if nxt[q] is not None:
        q = nxt[q]
        hops += 1
    else:
        q2 = next((k for k in cands if k > q and idle[k]), M)
        walked += q2 - q
        q = q2
print(f"  helper work {tot} requests ({tot / M:.2f} x M), per helper {tot / H / M:.2f} x M; "
      f"leader hops {hops}, leader walks {walked} requests; longest helper run {max(work.values())}")
