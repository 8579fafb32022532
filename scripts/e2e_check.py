import os, sys, torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api
from paper_2412_20322_b200.inputs import build_config
g = build_config(4)
dg = api.DeviceGrid(g)
host = dg.pinned_traces()
res = api.evaluate_host(dg, host)
s = torch.cuda.current_stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
for mode in ("0", "1"):
    os.environ["GL_RELAX"] = mode
    for name, fn in (("eval_grid", lambda: api.eval_grid(dg)), ("evaluate_host", lambda: api.evaluate_host(dg, host, out=res))):
        ts = []
        for i in range(12):
            flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); fn(); b.record(s); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts = ts[2:]
        print(mode, name, "min %.3f mean %.3f max %.3f" % (min(ts), sum(ts) / len(ts), max(ts)), flush=True)
