"""Per-chain decode time (spec + leader-only walk) for a few config-4 chains."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api, native as N
from paper_2412_20322_b200.inputs import build_config
ids = [int(x) for x in sys.argv[1].split(',')] if len(sys.argv) > 1 else [33, 51, 46, 26, 8, 54, 2, 31]
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = build_config(cfg)
dg = api.DeviceGrid(g)
N.profile_enable(True)
api.eval_grid(dg); torch.cuda.synchronize(); N.kernel_times()
for _ in range(2):
    api.eval_grid(dg); torch.cuda.synchronize()
    kt = dict(N.kernel_times())
print(f"all {len(g.chains)} chains: " + ", ".join(f"{k} {v:.2f} ms" for k, v in kt.items() if 'decode' in k))
for ci in ids:
    st = torch.empty((1, 80), dtype=torch.uint8, device='cuda')
    api.eval_grid(dg, ci, ci + 1, stats=st); torch.cuda.synchronize()
    kt = dict(N.kernel_times())
    dec = kt.get('k_decode', kt.get('k_decode_colo', 0.0))
    api.link_demand(dg, chain_lo=ci, chain_hi=ci + 1); torch.cuda.synchronize()
    walk = dict(N.kernel_times()).get('k_decode_log', 0.0)
    M = int((g.traces[g.chains[ci].trace_idx].output_len > 1).sum())
    print(f"{dec:6.2f} ms spec {walk:6.2f} ms walk ({1e6 * walk / M:5.1f} ns/req) chain {ci:2d} {g.chains[ci].label}")
