"""Event-regime census of a config-4 DPD chain's decode stage (analysis only).

Simulates the decode stage event by event in plain Python (d = o - 1 iterations
per request, step[b] per iteration) and counts, per event, the regime the GPU
loop would be in: saturated (b = cap, head ready), light (b < cap, head not
ready), burst (b < cap, head ready) and idle.  Also reports busy-period lengths
and how many consecutive saturated leave/join events come in runs.

usage: python scripts/regime.py <chain index> [n]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2412_20322_b200.inputs import build_config  # noqa: E402

ci = int(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
g = build_config(4, n=n)
ch = g.chains[ci]
assert ch.mode == 0, "DPD chains only"
tr = g.traces[ch.trace_idx]
a, p, o = tr.arrival_us.astype(np.int64), tr.prompt_len.astype(np.int64), tr.output_len.astype(np.int64)
t1, t2, step = ch.tables.t1_us.astype(np.int64), ch.tables.t2_us.astype(np.int64), ch.tables.step_us.astype(np.int64)
cap = ch.cap
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
d = o[dec] - 1
M = len(dec)

# event loop: iteration counter I, time T, members as finish iterations
import heapq
T, I = 0, 0
heap = []
q = 0
cnt = {"saturated": 0, "light": 0, "burst": 0, "idle": 0}
runs = []  # lengths of runs of consecutive saturated events
run = 0
busy_len, cur_busy = [], 0
while q < M or heap:
    b = len(heap)
    if b == 0:
        cnt["idle"] += 1
        if cur_busy:
            busy_len.append(cur_busy)
        cur_busy = 0
        T = max(T, r[q])
        heapq.heappush(heap, I + d[q])
        q += 1
        cur_busy += 1
        continue
    head_ready = q < M and r[q] <= T
    if head_ready and b < cap:
        cnt["burst"] += 1
        heapq.heappush(heap, I + d[q])
        q += 1
        cur_busy += 1
        if run:
            runs.append(run)
        run = 0
        continue
    fmin = heap[0]
    kL = fmin - I
    if q < M and b < cap:
        kJ = -(-(r[q] - T) // step[b])
    else:
        kJ = 1 << 62
    k = min(kL, kJ)
    T += k * step[b]
    I += k
    if b == cap and head_ready:
        cnt["saturated"] += 1
        run += 1
    else:
        cnt["light"] += 1
        if run:
            runs.append(run)
        run = 0
    while heap and heap[0] == I:
        heapq.heappop(heap)
if cur_busy:
    busy_len.append(cur_busy)
if run:
    runs.append(run)
tot = sum(cnt.values())
print(f"chain {ci} {ch.label}: M={M} events={tot}")
for k_, v in cnt.items():
    print(f"  {k_:10s} {v:8d} {100 * v / tot:5.1f}%")
runs = np.array(runs or [0])
print(f"  saturated runs: {len(runs)}  mean {runs.mean():.1f}  events in runs >= 16: "
      f"{runs[runs >= 16].sum()}")
bl = np.array(busy_len)
print(f"  busy periods: {len(bl)}  max {bl.max()}  mean {bl.mean():.1f}")

# ---- speculation census: true idle flags at the k_segments starts
fin = np.empty(M, np.int64)
T, I = 0, 0
heap = []
q = 0
while q < M or heap:
    b = len(heap)
    if b == 0:
        T = max(T, r[q])
    while q < M and len(heap) < cap and r[q] <= T:
        heapq.heappush(heap, (I + d[q], q))
        q += 1
    b = len(heap)
    fmin = heap[0][0]
    kL = fmin - I
    kJ = -(-(r[q] - T) // step[b]) if (q < M and b < cap) else 1 << 62
    k = min(kL, kJ)
    T += k * step[b]
    I += k
    while heap and heap[0][0] == I:
        fin[heapq.heappop(heap)[1]] = T
prevmax = np.maximum.accumulate(np.concatenate([[-(1 << 62)], fin[:-1]]))
idle = prevmax <= r
SEG = 256
nseg = (M + SEG - 1) // SEG
starts = [0]
for w in range(1, nseg):
    lo, hi = w * SEG, min(w * SEG + SEG, M)
    gaps = r[lo:hi] - r[lo - 1:hi - 1]
    starts.append(lo + int(np.argmax(gaps)))
starts.append(M)
si = np.array([idle[s] for s in starts[:-1]] + [True])
acc = si[:-1] & si[1:]
seglen = np.diff(starts)
win_has_idle = [bool(idle[w * SEG:min(w * SEG + SEG, M)].any()) for w in range(1, nseg)]
print(f"  idle requests {idle.sum()}  segment starts idle {si[:-1].mean():.2f}  "
      f"windows with an idle request {np.mean(win_has_idle):.2f}")
print(f"  accepted segments {acc.mean():.2f} -> leader walks {seglen[~acc].sum() / M:.2f} of the chain")
