import dataclasses, sys
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2412_20322_b200 import api
from paper_2412_20322_b200.inputs import build_config, subset_chains
from tests.helpers import random_case
from tests.test_gpu_parity import grid_of

def run(g, label, pr_on):
    dg = api.DeviceGrid(g)
    stats, pr = api.eval_grid(dg, per_request=pr_on)
    torch.cuda.synchronize()
    st = api.stats_numpy(stats)
    nbad = 0
    first = None
    for i, ch in enumerate(g.chains):
        ref, _, _ = O.simulate_chain(g.traces[ch.trace_idx], ch, False)
        bad = [k for k in ref if int(st[i][k]) != int(ref[k])]
        if bad:
            nbad += 1
            if first is None: first = (i, ch.mode, ch.gamma, ch.alpha, bad[:3])
    print(label, "per_request", pr_on, "chains", len(g.chains), "bad", nbad, first, flush=True)

g2 = build_config(2, n=300)
for k in (16, 32, 40):
    for pr_on in (False, True):
        run(subset_chains(g2, range(k)), f"cfg2-first{k}", pr_on)
rng = np.random.default_rng(20322)
pairs = [random_case(rng) for _ in range(400)]
for k in (10, 50, 400):
    for pr_on in (False, True):
        run(grid_of(pairs[:k]), f"rand{k}", pr_on)
