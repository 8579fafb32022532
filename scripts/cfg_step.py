"""One full step (gl_eval_grid + gl_argmin_feasible) of a BASELINE config on one GPU,
with per-kernel times (analysis only)."""
import sys
import time
import torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api, native as N
from paper_2412_20322_b200.inputs import build_config
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
t0 = time.time()
g = build_config(cfg)
print(f"cfg{cfg}: {len(g.chains)} chains, {g.rows}x{g.cols} grid, inputs built in {time.time() - t0:.1f} s")
dg = api.DeviceGrid(g)
for _ in range(2):
    st, _ = api.eval_grid(dg)
    api.argmin_feasible(dg, st)
torch.cuda.synchronize()
N.profile_enable(True)
N.kernel_times()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
st, _ = api.eval_grid(dg)
api.argmin_feasible(dg, st)
e1.record()
torch.cuda.synchronize()
print(f"step {e0.elapsed_time(e1):.2f} ms;", ", ".join(f"{k} {v:.2f}" for k, v in N.kernel_times()))
