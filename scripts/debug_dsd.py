"""Ad-hoc GPU debugging of DSD chains (prints GPU vs oracle per-request)."""
import dataclasses, sys
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2412_20322_b200 import api
from tests.helpers import random_case
from tests.test_gpu_parity import grid_of

rng = np.random.default_rng(20322)
tr, ch = random_case(rng)
for alpha in (0.0, 0.5, 1.0):
    c2 = dataclasses.replace(ch, alpha=alpha)
    g = grid_of([(tr, c2)])
    dg = api.DeviceGrid(g)
    stats, pr = api.eval_grid(dg, per_request=True)
    torch.cuda.synchronize()
    st = api.stats_numpy(stats)[0]
    ref, ttft, fin = O.simulate_chain(tr, c2)
    print("alpha", alpha, "gpu", {k: int(st[k]) for k in st.dtype.names})
    print("   ref", ref)
    print("   gpu ttft", pr[:, 0].tolist(), "ref", ttft.tolist())
    print("   gpu fin ", pr[:, 1].tolist(), "ref", fin.tolist())
