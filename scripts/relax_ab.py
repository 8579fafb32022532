"""Step time of one configuration with and without k_relax (GL_RELAX=0), device
timeline per kernel, plus a bit-for-bit comparison of the two results.
Usage: python scripts/relax_ab.py [config] [reps]"""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api, native as N
from paper_2412_20322_b200.inputs import build_config

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = build_config(cfg)
dg = api.DeviceGrid(g)
N.profile_enable(True)
out = {}
for mode in ("0", "1"):
    os.environ["GL_RELAX"] = mode
    best = None
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        stats, pr = api.eval_grid(dg, per_request=True)
        torch.cuda.synchronize()
        tl = N.kernel_timeline()
        end = max(st + ms for _, st, ms in tl)
        if best is None or end < best[0]:
            best = (end, tl)
    out[mode] = (api.stats_numpy(stats), pr.cpu().numpy())
    print("cfg%d GL_RELAX=%s step %.3f ms:" % (cfg, mode, best[0]),
          ", ".join("%s %.2f" % (n, ms) for n, _, ms in best[1] if ms > 0.05), flush=True)
print("identical:", np.array_equal(out["0"][0], out["1"][0]) and np.array_equal(out["0"][1], out["1"][1]))
