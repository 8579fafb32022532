import sys
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2412_20322_b200 import api
from tests.helpers import random_case
from tests.test_gpu_parity import grid_of
k = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rng = np.random.default_rng(20322)
pairs = [random_case(rng) for _ in range(400)][:k]
g = grid_of(pairs)
dg = api.DeviceGrid(g)
stats, pr = api.eval_grid(dg, per_request=True)
torch.cuda.synchronize()
st = api.stats_numpy(stats)
nbad = 0
for i, ch in enumerate(g.chains):
    ref, _, _ = O.simulate_chain(g.traces[ch.trace_idx], ch, False)
    bad = [f for f in ref if int(st[i][f]) != int(ref[f])]
    nbad += bool(bad)
print("bad", nbad)
