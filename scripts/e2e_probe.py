"""Where the end-to-end time goes (analysis only): pinned H2D of the config-4
traces alone, the device-resident step, and gl_evaluate_host, each with CUDA events."""
import sys
import time
import torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api
from paper_2412_20322_b200.inputs import build_config
g = build_config(4)
dg = api.DeviceGrid(g)
host = dg.pinned_traces()
dev = [tuple(torch.empty_like(x, device='cuda') for x in t) for t in host]
s = torch.cuda.current_stream()


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s); fn(); e1.record(s); torch.cuda.synchronize()
        ms.append((e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0)))
    return min(m[0] for m in ms), min(m[1] for m in ms)


def h2d():
    for d, h in zip(dev, host):
        for a, b in zip(d, h):
            a.copy_(b, non_blocking=True)


def step():
    st, _ = api.eval_grid(dg)
    api.argmin_feasible(dg, st)


res = api.evaluate_host(dg, host)
nbytes = sum(x.numel() * x.element_size() for t in host for x in t)
print("H2D %.1f MB: %.3f ms device (%.3f ms wall)" % ((nbytes / 1e6,) + timed(h2d)))
print("device step: %.3f ms device (%.3f ms wall)" % timed(step))
print("evaluate_host: %.3f ms device (%.3f ms wall)" % timed(lambda: api.evaluate_host(dg, host, out=res)))

from paper_2412_20322_b200 import native as N
N.profile_enable(True)
N.kernel_times()
step(); torch.cuda.synchronize()
print("device step kernels:", ", ".join(f"{k} {v:.3f}" for k, v in N.kernel_times()))
api.evaluate_host(dg, host, out=res); torch.cuda.synchronize()
print("evaluate_host kernels:", ", ".join(f"{k} {v:.3f}" for k, v in N.kernel_times()))
