"""Busy periods of a chain's decode stage (analysis only): request q (decode order)
starts a busy period iff every earlier decode request finished by r_q.  Prints the
count and the longest periods -- the floor of any exact speculation scheme that
restarts only at idle points."""
import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2412_20322_b200.inputs import build_config

cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = build_config(cfg)
for ci in [int(x) for x in sys.argv[1].split(',')]:
    ch = g.chains[ci]
    tr = g.traces[ch.trace_idx]
    st, ttft, fin, r = O.simulate_chain(tr, ch, per_request=True, ready=True)
    dec = np.nonzero(tr.output_len > 1)[0]
    f, rr = fin[dec], r[dec]
    prevmax = np.maximum.accumulate(np.concatenate([[np.iinfo(np.int64).min], f[:-1]]))
    idle = prevmax <= rr
    starts = np.flatnonzero(idle)
    lens = np.diff(np.concatenate([starts, [len(dec)]]))
    top = np.sort(lens)[::-1][:5]
    print(f"chain {ci} {ch.label}: {len(dec)} decode requests, {len(starts)} busy periods, "
          f"longest {top.tolist()} ({100 * top[0] / len(dec):.1f}% of the chain)")
