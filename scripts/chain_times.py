"""Per-chain k_decode time of config 4 (one launch per chain)."""
import sys, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api, native as N
from paper_2412_20322_b200.inputs import build_config
from oracle import oracle as O
g = build_config(4)
dg = api.DeviceGrid(g)
N.profile_enable(True)
out = []
stats, _ = api.eval_grid(dg)
torch.cuda.synchronize(); N.kernel_times()
for ci in range(len(g.chains)):
    st = torch.empty((1, 80), dtype=torch.uint8, device='cuda')
    api.eval_grid(dg, ci, ci + 1, stats=st)
    torch.cuda.synchronize()
    kt = dict(N.kernel_times())
    s = api.stats_numpy(st)[0]
    ch = g.chains[ci]
    out.append((kt['k_decode'], ci, ch.label, int(s['slo_ok']), int(s['makespan_us']), kt['k_stages']))
out.sort(reverse=True)
for r in out: print("%.2f ms  chain %2d  %-50s ok=%d makespan=%.0fs  (k_stages %.2f ms)" % (r[0], r[1], r[2], r[3], r[4]/1e6, r[5]))
