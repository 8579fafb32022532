"""Per-chain decode time of a config (default 4), one launch per chain: the speculative
k_decode (gl_eval_grid) and the leader-only serial walk k_decode_log
(gl_link_demand), plus the request count of the chain's decode stream."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api, native as N
from paper_2412_20322_b200.inputs import build_config
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
walk_too = "--no-walk" not in sys.argv
g = build_config(cfg)
dg = api.DeviceGrid(g)
N.profile_enable(True)
stats, _ = api.eval_grid(dg)
torch.cuda.synchronize(); N.kernel_times()
out = []
for ci in range(len(g.chains)):
    st = torch.empty((1, 80), dtype=torch.uint8, device='cuda')
    api.eval_grid(dg, ci, ci + 1, stats=st)
    torch.cuda.synchronize()
    kt = dict(N.kernel_times())
    kl = {}
    if walk_too:
        api.link_demand(dg, chain_lo=ci, chain_hi=ci + 1)
        torch.cuda.synchronize()
        kl = dict(N.kernel_times())
    ch = g.chains[ci]
    M = int((g.traces[ch.trace_idx].output_len > 1).sum())
    dec = kt.get('k_decode', kt.get('k_decode_colo', 0.0))
    walk = kl.get('k_decode_log', 0.0)
    out.append((dec, walk, ci, ch.label, M))
out.sort(reverse=True)
for dec, walk, ci, lab, M in out:
    print("%6.2f ms spec  %6.2f ms walk (%5.1f ns/request)  chain %2d  %s" % (dec, walk, 1e6 * walk / max(M, 1), ci, lab))
