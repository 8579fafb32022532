"""Busy periods of a chain's decode stage (analysis only; scripts/chainsim.py, not
the oracle): request q (decode order) starts a busy period iff every earlier decode
request finished by r_q.  Prints the count and the longest periods -- the floor of
any exact speculation scheme that restarts only at idle points.

usage: python scripts/busy_periods.py <chain,chain,...> [config]
"""
import sys

import numpy as np

sys.path.insert(0, '.')
from scripts.chainsim import chain_stream, simulate  # noqa: E402

cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
for ci in [int(x) for x in sys.argv[1].split(',')]:
    ch, r, d, step, cap = chain_stream(cfg, ci)
    _, fin, _ = simulate(r, d, step, cap)
    f = np.array([fin[q] for q in range(len(r))], np.int64)
    prevmax = np.maximum.accumulate(np.concatenate([[np.iinfo(np.int64).min], f[:-1]]))
    starts = np.flatnonzero(prevmax <= r)
    lens = np.diff(np.concatenate([starts, [len(r)]]))
    top = np.sort(lens)[::-1][:5]
    print(f"chain {ci} {ch.label}: {len(r)} decode requests, {len(starts)} busy periods, "
          f"longest {top.tolist()} ({100 * top[0] / len(r):.1f}% of the chain)")
