"""Launch the decode pipeline on a subset of chains of one configuration (for ncu):
python scripts/prof_cfg.py <cfg> <chain,chain,...> [n]"""
import sys
import torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api
from paper_2412_20322_b200.inputs import build_config, subset_chains
cfg = int(sys.argv[1])
ids = [int(x) for x in sys.argv[2].split(',')]
kw = {"n": int(sys.argv[3])} if len(sys.argv) > 3 else {}
g = subset_chains(build_config(cfg, **kw), ids)
dg = api.DeviceGrid(g)
for _ in range(3):
    api.eval_grid(dg)
torch.cuda.synchronize()
