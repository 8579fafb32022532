"""Batch-size / queue census of a chain's decode stage (analysis only).
usage: python scripts/regime2.py <cfg> <chain>"""
import heapq
import sys
from collections import Counter

sys.path.insert(0, "scripts")
from chainsim import chain_stream  # noqa: E402

cfg, ci = int(sys.argv[1]), int(sys.argv[2])
ch, r, d, step, cap = chain_stream(cfg, ci)
M = len(r)
T, I, q = 0, 0, 0
heap = []
kinds = Counter()
bhist = Counter()
while q < M or heap:
    if not heap:
        T = max(T, r[q])
    nj = 0
    while q < M and len(heap) < cap and r[q] <= T:
        heapq.heappush(heap, (I + d[q], q))
        q += 1
        nj += 1
    b = len(heap)
    queued = q < M and r[q] <= T
    kL = heap[0][0] - I
    kJ = -(-(r[q] - T) // step[b]) if (q < M and b < cap) else 1 << 62
    k = min(kL, kJ)
    T += k * step[b]
    I += k
    nl = 0
    while heap and heap[0][0] == I:
        heapq.heappop(heap)
        nl += 1
    kind = ("sat" if b == cap and queued else "full" if b == cap else "part") + \
           (f"-L{min(nl, 2)}" if nl else "-J")
    kinds[kind] += 1
    bhist[b] += 1
tot = sum(kinds.values())
print(f"cfg{cfg} chain {ci} {ch.label}: steps {tot}")
for k, v in sorted(kinds.items(), key=lambda kv: -kv[1]):
    print(f"  {k:10s} {v:8d} {100 * v / tot:5.1f}%")
print("  b histogram:", " ".join(f"{b}:{100 * v / tot:.0f}%" for b, v in sorted(bhist.items())))
