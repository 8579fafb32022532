"""Device timeline of one gl_evaluate_host call (torch.profiler / CUPTI; analysis only)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api
from paper_2412_20322_b200.inputs import build_config
g = build_config(4)
dg = api.DeviceGrid(g)
host = dg.pinned_traces()
res = api.evaluate_host(dg, host)
for _ in range(3):
    api.evaluate_host(dg, host, out=res)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    api.evaluate_host(dg, host, out=res)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs:
    print(f"{(e.time_range.start - t0) / 1e3:9.3f} ms  {(e.time_range.end - e.time_range.start) / 1e3:8.3f} ms  {e.name[:70]}")
