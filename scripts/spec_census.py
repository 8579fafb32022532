"""Speculation census of one chain (analysis only): candidates, helper run lengths,
and a schedule model of k_decode's leader/helper protocol in units of events.

usage: python scripts/spec_census.py <cfg> <chain> [helpers]
"""
import heapq
import sys

import numpy as np

sys.path.insert(0, "scripts")
from chainsim import chain_stream, simulate  # noqa: E402

cfg, ci = int(sys.argv[1]), int(sys.argv[2])
H = int(sys.argv[3]) if len(sys.argv) > 3 else 8
SEG = 256
ch, r, d, step, cap = chain_stream(cfg, ci)
M = len(r)
_, fin, ev_total = simulate(r, d, step, cap)
finv = np.array([fin[q] for q in range(M)])
prevmax = np.maximum.accumulate(np.concatenate([[-(1 << 62)], finv[:-1]]))
idle = prevmax <= r
smin = int(step[1:cap + 1].min())
lb = r + d * smin
lbmax = np.maximum.accumulate(np.concatenate([[-(1 << 62)], lb[:-1]]))
slack = r - lbmax
cands = [0]
for w in range(1, (M + SEG - 1) // SEG):
    lo, hi = w * SEG, min(w * SEG + SEG, M)
    j = lo + int(np.argmax(slack[lo:hi]))
    if slack[j] >= 0:
        cands.append(j)
cset = set(cands)
cidx = {q: i for i, q in enumerate(cands)}
runs = {}
for q in cands:
    e, _, ev = simulate(r, d, step, cap, q, cset)
    runs[q] = (e, ev)
# busy periods (true run)
starts = np.nonzero(idle)[0]
bl = np.diff(np.concatenate([starts, [M]]))
print(f"cfg{cfg} chain {ci} {ch.label}: M={M} events={ev_total} idle={idle.sum()} "
      f"longest busy period={bl.max()} requests")
print(f"  candidates {len(cands)}, truly idle {np.mean([idle[q] for q in cands]):.2f}; "
      f"helper events total {sum(v[1] for v in runs.values())} "
      f"({sum(v[1] for v in runs.values()) / ev_total:.2f} x)")
# schedule model: helpers take candidates in order; leader hops
free = [(0.0, h) for h in range(H)]
heapq.heapify(free)
start, end = {}, {}
for q in cands[1:]:
    t, h = heapq.heappop(free)
    start[q] = t
    end[q] = t + runs[q][1]
    heapq.heappush(free, (end[q], h))
t, q = 0.0, 0
hops = walked = 0
while q < M:
    if q == 0:
        e, ev = runs[0]
        t += ev
        walked += ev
        q = e
        continue
    t = max(t, end[q]) + 10  # wait for the helper, copy
    hops += 1
    q = runs[q][0]
print(f"  model: leader finishes at {t:.0f} events (sequential {ev_total}); "
      f"speedup {ev_total / t:.1f}x; hops {hops}")
longest = max(runs.items(), key=lambda kv: kv[1][1])
print(f"  longest run: from q={longest[0]} ({longest[1][1]} events)")
