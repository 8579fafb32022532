"""Launch the decode pipeline on a subset of config-4 chains (for ncu)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api
from paper_2412_20322_b200.inputs import build_config, subset_chains
ids = [int(x) for x in sys.argv[1].split(',')] if len(sys.argv) > 1 else list(range(64))
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = subset_chains(build_config(cfg), ids)
dg = api.DeviceGrid(g)
for _ in range(3):
    api.eval_grid(dg)
torch.cuda.synchronize()
