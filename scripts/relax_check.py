"""k_relax A/B on one configuration: per-request rows and statistics with the
relaxation (default) against the serial k_decode (GL_RELAX=0), bit for bit, and the
kernel times of both.  Usage: python scripts/relax_check.py [config] [n]"""
import os
import sys
import time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api, native as N
from paper_2412_20322_b200.inputs import build_config

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
kw = {"n": int(sys.argv[2])} if len(sys.argv) > 2 else {}
g = build_config(cfg, **kw)
dg = api.DeviceGrid(g)
N.profile_enable(True)
res = {}
for it, mode in enumerate(("0", "1", "1", "1", "0")):
    os.environ["GL_RELAX"] = mode
    os.environ["GL_RELAX_DEBUG"] = os.environ.get("DBG", "1") if it == 2 else "0"
    torch.cuda.synchronize()
    stats, pr = api.eval_grid(dg, per_request=True)
    torch.cuda.synchronize()
    tlist = N.kernel_timeline()
    tl = {}
    for name, st, ms in tlist:
        tl[name] = tl.get(name, 0.0) + ms
        if it == 3:
            print("   %-14s start %8.3f ms  dur %8.3f ms" % (name, st, ms))
    res[mode] = (api.stats_numpy(stats), pr.cpu().numpy())
    print("GL_RELAX=%s" % mode, {k: round(v, 3) for k, v in tl.items()}, flush=True)
s0, p0 = res["0"]
s1, p1 = res["1"]
print("stats identical:", np.array_equal(s0, s1), " rows identical:", np.array_equal(p0, p1))
if not np.array_equal(p0, p1):
    bad = np.nonzero((p0 != p1).any(axis=1))[0]
    print("differing rows:", bad.size, bad[:10])
