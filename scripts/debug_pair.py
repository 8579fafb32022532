import sys
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2412_20322_b200 import api
from tests.helpers import random_case
from tests.test_gpu_parity import grid_of
rng = np.random.default_rng(20322)
pairs = [random_case(rng) for _ in range(50)]
ref0, _, _ = O.simulate_chain(*pairs[0], False)
print("chain0", pairs[0][1].mode, pairs[0][1].gamma, pairs[0][1].alpha, hex(pairs[0][1].seed), pairs[0][0].n)
for j in range(1, 50):
    g = grid_of([pairs[0], pairs[j]])
    dg = api.DeviceGrid(g)
    stats, pr = api.eval_grid(dg, per_request=False)
    torch.cuda.synchronize()
    st = api.stats_numpy(stats)
    bad = [f for f in ref0 if int(st[0][f]) != int(ref0[f])]
    ch = pairs[j][1]
    if bad:
        print("partner", j, "mode", ch.mode, "gamma", ch.gamma, "alpha", ch.alpha, "seed", hex(ch.seed), "n", pairs[j][0].n, "BAD", bad)
print("done")
