"""Device time of one gl_eval_grid call with and without the launch-order hint
(greenllm.h gl_schedule), same box, back to back; L2 flushed between calls.
usage: python scripts/sched_times.py [config ...]"""
import sys

import torch

sys.path.insert(0, '.')
from paper_2412_20322_b200 import api, native as N  # noqa: E402
from paper_2412_20322_b200.inputs import build_config  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
for cfg in [int(x) for x in sys.argv[1:]] or [4, 5]:
    g = build_config(cfg)
    dg = api.DeviceGrid(g)
    N.profile_enable(True)
    out = {}
    for mode in (False, True, False, True):
        ms = []
        for i in range(4 if cfg != 5 else 3):
            flush.fill_(i)
            s = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            api.eval_grid(dg, schedule=mode)
            e1.record(s)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        kt = dict(N.kernel_times())
        out.setdefault(mode, []).append(min(ms[1:]))
        print(f"cfg{cfg} schedule={mode} hint={dg.first_range() if mode else None} "
              f"step {min(ms[1:]):.3f} ms (all {', '.join('%.3f' % m for m in ms)}) "
              f"launches {dg.last_launches}", flush=True)
    print(f"cfg{cfg} best: no hint {min(out[False]):.3f} ms, hint {min(out[True]):.3f} ms")

# one step's launch timeline per mode (start offset, duration) for the last config
for mode in (False, True):
    flush.fill_(7)
    torch.cuda.synchronize()
    N.kernel_times()
    api.eval_grid(dg, schedule=mode)
    torch.cuda.synchronize()
    print(f"timeline cfg{cfg} schedule={mode}:")
    for name, t0, ms in N.kernel_timeline():
        print(f"   {name:16s} start {t0:9.3f} ms  dur {ms:9.3f} ms  end {t0 + ms:9.3f}")
