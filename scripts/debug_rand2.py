import sys, math
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2412_20322_b200 import api
from paper_2412_20322_b200.inputs.philox import philox4x32_10, key_from_seed
from tests.helpers import random_case
from tests.test_gpu_parity import grid_of
rng = np.random.default_rng(20322)
pairs = [random_case(rng) for _ in range(400)][:50]
g = grid_of(pairs)
dg = api.DeviceGrid(g)
stats, pr = api.eval_grid(dg, per_request=True)
torch.cuda.synchronize()
st = api.stats_numpy(stats)
pr = pr.cpu().numpy()
off = 0
for i, ch in enumerate(g.chains):
    tr = g.traces[ch.trace_idx]
    ref, ttft, fin = O.simulate_chain(tr, ch)
    bad = [f for f in ref if int(st[i][f]) != int(ref[f])]
    if bad:
        print("chain", i, "mode", ch.mode, "cap", ch.cap, "gamma", ch.gamma, "alpha", ch.alpha, "n", tr.n, bad)
        print(" o", tr.output_len.tolist())
        print(" gpu ttft", pr[off:off+tr.n, 0].tolist(), "\n ref ttft", ttft.tolist())
        print(" gpu fin", pr[off:off+tr.n, 1].tolist(), "\n ref fin", fin.tolist())
        print(" gpu", {f: int(st[i][f]) for f in ref}, "\n ref", ref)
        # K per request
        k0, k1 = key_from_seed(ch.seed)
        thr = []; x = 1.0
        for c in range(ch.gamma): x *= ch.alpha; thr.append(math.floor(x * 2**32))
        Ks = []
        for j, o in enumerate(tr.output_len.tolist()):
            need, tok, s = o - 1, 0, 0
            while need > 0 and tok < need:
                u = int(philox4x32_10(s // 4, j, 0x41434350, 0, k0, k1)[s % 4]); tok += 1 + sum(u < t for t in thr); s += 1
            Ks.append(s)
        print(" K", Ks)
    off += tr.n
