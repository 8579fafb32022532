"""e2e breakdown on config 4: H2D copies alone, the device step, gl_evaluate_host (analysis only)."""
import sys, torch, time
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api
from paper_2412_20322_b200.inputs import build_config
g = build_config(4); dg = api.DeviceGrid(g)
host = dg.pinned_traces()
uniq = {}
for arrs in host:
    for x in arrs: uniq[x.data_ptr()] = x
dev = {k: torch.empty_like(v, device='cuda') for k, v in uniq.items()}
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
def timed(fn, n=6):
    out = []
    for i in range(n):
        flush.fill_(i); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); out.append(e0.elapsed_time(e1))
    return sorted(out)[len(out)//2]
res = api.evaluate_host(dg, host)
print("bytes", sum(v.numel()*v.element_size() for v in uniq.values()), "arrays", len(uniq))
print("h2d copies only  %.3f ms" % timed(lambda: [dev[k].copy_(v, non_blocking=True) for k, v in uniq.items()]))
def dev_step():
    st, _ = api.eval_grid(dg); api.argmin_feasible(dg, st, want_carbon=False)
print("device step      %.3f ms" % timed(dev_step))
print("evaluate_host    %.3f ms" % timed(lambda: api.evaluate_host(dg, host, out=res)))
t0 = time.perf_counter()
for _ in range(5): api.evaluate_host(dg, host, out=res)
print("evaluate_host wall %.3f ms" % ((time.perf_counter() - t0) / 5 * 1e3))
