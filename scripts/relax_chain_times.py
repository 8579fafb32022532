"""Per-chain step of config 4's heavily loaded chains, each evaluated alone (one-chain
grid), with k_relax (default race) and without (GL_RELAX=0): the device time from
the first to the last kernel of the call.  Usage: python scripts/relax_chain_times.py"""
import os
import sys
import torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api, native as N
from paper_2412_20322_b200.inputs import build_config, subset_chains

g = build_config(4)
N.profile_enable(True)
for ci in (33, 51, 63, 46, 26, 41, 38, 21):
    sub = subset_chains(g, [ci])
    dg = api.DeviceGrid(sub)
    row = []
    for mode in ("0", "1"):
        os.environ["GL_RELAX"] = mode
        best = None
        for _ in range(3):
            torch.cuda.synchronize()
            api.eval_grid(dg)
            torch.cuda.synchronize()
            tl = N.kernel_timeline()
            end = max(st + ms for _, st, ms in tl)
            best = end if best is None else min(best, end)
        row.append(best)
    print("chain %2d %-44s serial %6.2f ms   with k_relax %6.2f ms" % (ci, g.chains[ci].label, row[0], row[1]), flush=True)
