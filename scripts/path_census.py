"""Census of the decode-loop paths a chain takes (analysis only): replays the
chain's decode stage event by event with the GPU loop's control structure
(join loop / saturated loop / light loop) and counts loop entries and events."""
import sys
import heapq
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2412_20322_b200.inputs import build_config

ci = int(sys.argv[1])
g = build_config(4)
ch = g.chains[ci]
tr = g.traces[ch.trace_idx]
st, ttft, fin, r = O.simulate_chain(tr, ch, per_request=True, ready=True)
o = tr.output_len.astype(np.int64)
dec = np.nonzero(o > 1)[0]
fin_d = fin[dec]
r_d = r[dec]
# events in time order: joins happen at boundaries; reconstruct b(t) from (join, finish)
# join time = first boundary >= r where a slot is free: not stored -> use counts only
M = len(dec)
# classify leaves: saturated (a head was waiting, ready <= leave time) or not
order = np.argsort(fin_d, kind='stable')
ft = fin_d[order]
# number of requests ready by each leave time
ready_cnt = np.searchsorted(r_d, ft, side='right')
left_cnt = np.arange(1, M + 1)
waiting = ready_cnt - left_cnt  # >= cap means backlog (approx: members = cap)
cap = ch.cap
sat = (ready_cnt - (left_cnt - 1)) > cap  # a ready request waits when this member leaves
print(f"chain {ci} {ch.label}: M={M}")
print(f"  leaves with a waiting ready head (saturated swaps): {sat.mean():.3f}")
runs = np.diff(np.flatnonzero(np.concatenate([[True], ~sat, [True]]))) - 1
runs = runs[runs > 0]
print(f"  saturated runs: {len(runs)}, mean length {runs.mean() if len(runs) else 0:.1f}, "
      f"median {np.median(runs) if len(runs) else 0}")
