"""k_relax on config 5 (1M-request chains, normally excluded by RX_MAX_N): serial vs race
vs solo, with GL_RELAX_MAXN lifting the cap.  Result (profiles/r02zf_cfg5_relax.txt): its
heavily loaded chains are saturated ones and do not converge within 160 sweeps."""
import os, sys, torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api, native as N
from paper_2412_20322_b200.inputs import build_config
g = build_config(5)
dg = api.DeviceGrid(g)
N.profile_enable(True)
for it, (mode, rho) in enumerate((("0", None), ("1", "0.5,1.2"), ("solo", "0.5,1.2"))):
    os.environ["GL_RELAX"] = mode
    os.environ["GL_RELAX_MAXN"] = "2000000"
    if rho: os.environ["GL_RELAX_RHO"] = rho
    os.environ["GL_RELAX_DEBUG"] = "1" if mode != "0" else "0"
    torch.cuda.synchronize(); api.eval_grid(dg); torch.cuda.synchronize()
    tl = N.kernel_timeline()
    print(mode, "step %.2f ms" % max(st + ms for _, st, ms in tl), [(n, round(ms, 2)) for n, _, ms in tl if ms > 0.5], flush=True)
