"""Per-path event census of the leader's decode loop for one chain, from the A/B
build with debug counters (python scripts/ab_build.py census --patch
scripts/census_patch.py; GL_LIB_PATH=build/ab/census.so).
usage: python scripts/census_run.py cfg chain [chain ...]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, '.')
from paper_2412_20322_b200 import api, native as N  # noqa: E402
from paper_2412_20322_b200.inputs import build_config  # noqa: E402

NAMES = ["top join", "outer loop trips", "saturated leave+join", "saturated exits",
         "light join", "light join exit: batch full", "light join exit: next head ready",
         "light leave", "light leave exit: multi-leave", "light leave exit: batch empty",
         "light leave exit: head ready", "light join exit: ring refill", "light slow exit",
         "general events", "saturated exit: multi-leave", "saturated exit: head not ready",
         "saturated exit: ring refill", "saturated exit: other", "  (multi-leave, head ready)"]
cfg = int(sys.argv[1])
g = build_config(cfg)
dg = api.DeviceGrid(g)
lib = N.lib()
lib.gl_census_read.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 32)()
for ci in [int(x) for x in sys.argv[2:]]:
    lib.gl_census_read(buf, 1)
    api.eval_grid(dg, ci, ci + 1)
    torch.cuda.synchronize()
    lib.gl_census_read(buf, 1)
    M = int((g.traces[g.chains[ci].trace_idx].output_len > 1).sum())
    print(f"cfg{cfg} chain {ci} ({g.chains[ci].label}), {M} decode requests:")
    for i, nm in enumerate(NAMES):
        print(f"   {nm:36s} {buf[i]:9d}")
