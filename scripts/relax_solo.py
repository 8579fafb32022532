"""k_relax alone (GL_RELAX=solo: it runs before k_decode) on config 4's heavily
loaded chains: sweeps and time per chain set, and the serial k_decode that follows.
Usage: python scripts/relax_solo.py [rho_lo,rho_hi] [--quiet]
(--quiet: two evaluations and no output, for ncu captures of k_relax)"""
import os
import sys
import torch
sys.path.insert(0, '.')
from paper_2412_20322_b200 import api, native as N
from paper_2412_20322_b200.inputs import build_config

os.environ["GL_RELAX"] = "solo"
args = [a for a in sys.argv[1:] if not a.startswith("--")]
quiet = "--quiet" in sys.argv
if args:
    os.environ["GL_RELAX_RHO"] = args[0]
g = build_config(4)
dg = api.DeviceGrid(g)
N.profile_enable(not quiet)
for it in range(2 if quiet else 3):
    os.environ["GL_RELAX_DEBUG"] = "1" if it == 2 and not quiet else "0"
    torch.cuda.synchronize()
    api.eval_grid(dg)
    torch.cuda.synchronize()
    if quiet:
        continue
    tl = N.kernel_timeline()
    if it == 2:
        for name, st, ms in tl:
            print("   %-14s start %8.3f ms  dur %8.3f ms" % (name, st, ms), flush=True)
