"""Run a config-4 chain subset through a different libgreenllm build (A/B comparisons)."""
import sys
sys.path.insert(0, '.')
from paper_2412_20322_b200 import native
native.LIB_PATH = sys.argv[2]
import torch
from paper_2412_20322_b200 import api
from paper_2412_20322_b200.inputs import build_config, subset_chains
ids = [int(x) for x in sys.argv[1].split(',')]
g = subset_chains(build_config(4), ids)
dg = api.DeviceGrid(g)
native.profile_enable(True)
for _ in range(3):
    api.eval_grid(dg)
torch.cuda.synchronize()
print(native.kernel_times())
kt = {}
for _ in range(3):
    api.eval_grid(dg)
torch.cuda.synchronize()
for name, ms in native.kernel_times():
    kt.setdefault(name, []).append(ms)
print("RESULT", " ".join(f"{k}={sum(v) / len(v):.3f}" for k, v in kt.items()))
