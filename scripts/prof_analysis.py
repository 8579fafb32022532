"""Launch the NEXT-row entry points once each on their full-size workloads (for ncu):
gl_link_demand on config 4, gl_savings_surface on config 6, gl_complete_matrices on
config 4's Alg. 1 matrices (carbon and attainment, 30% hidden)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api
from paper_2412_20322_b200.inputs import build_config
from paper_2412_20322_b200.inputs.cf import als_init, observation_mask

g4 = build_config(4)
dg4 = api.DeviceGrid(g4)
for _ in range(2):
    api.link_demand(dg4)
g6 = build_config(6)
dg6 = api.DeviceGrid(g6)
stats6, _ = api.eval_grid(dg6)
for _ in range(2):
    api.savings_surface(dg6, stats6)
stats4, _ = api.eval_grid(dg4)
carbon, choice, fb = api.argmin_feasible(dg4, stats4)
st = api.stats_numpy(stats4)
att = torch.from_numpy((st["slo_ok"] / st["n"])[g4.cell_chain].reshape(g4.rows, g4.cols)).cuda()
m = torch.from_numpy(observation_mask(g4.rows, g4.cols, 0.3, seed=42)).cuda()
x = torch.stack([carbon, att])
mm = torch.stack([m, m])
for _ in range(2):
    api.complete_matrices(x, mm, 2, 0.1, 200, lo=0.0)
torch.cuda.synchronize()
print("ok")
