"""One config-4 evaluation with k_relax in solo mode on the chains with rho in the
given range (for ncu captures of k_relax).  Usage: python scripts/relax_one.py lo,hi"""
import os
import sys
import torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api
from paper_2412_20322_b200.inputs import build_config

os.environ["GL_RELAX"] = "solo"
os.environ["GL_RELAX_RHO"] = sys.argv[1] if len(sys.argv) > 1 else "0.86,0.87"
g = build_config(4)
dg = api.DeviceGrid(g)
for _ in range(2):
    api.eval_grid(dg)
    torch.cuda.synchronize()
