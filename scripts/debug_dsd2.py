import dataclasses, sys
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2412_20322_b200 import api
from paper_2412_20322_b200.inputs import build_config, subset_chains
from tests.helpers import random_case
from tests.test_gpu_parity import grid_of

def run(g, label):
    dg = api.DeviceGrid(g)
    stats, pr = api.eval_grid(dg, per_request=False)
    torch.cuda.synchronize()
    st = api.stats_numpy(stats)
    for i, ch in enumerate(g.chains):
        ref, _, _ = O.simulate_chain(g.traces[ch.trace_idx], ch, False)
        bad = [k for k in ref if int(st[i][k]) != int(ref[k])]
        print(label, i, "mode", ch.mode, "g", ch.gamma, "a", ch.alpha, "BAD" if bad else "ok", bad[:3],
              [int(st[i][k]) for k in bad[:2]], [ref[k] for k in bad[:2]])

rng = np.random.default_rng(20322)
tr, ch = random_case(rng)
run(grid_of([(tr, ch), (tr, dataclasses.replace(ch, alpha=0.8))]), "same-trace-2")
tr2, ch2 = random_case(rng)
run(grid_of([(tr, ch), (tr2, ch2)]), "two-traces")
g2 = build_config(2, n=300)
for k in (1, 2, 3, 8):
    run(subset_chains(g2, range(k)), f"cfg2-first{k}")
run(subset_chains(g2, [5]), "cfg2-only5")
