"""Every C-ABI entry point once at small sizes, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Product path only: no oracle.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_run.py
Exercises: gl_eval_grid (DPD, DSD, Standalone, co-located SpecDecode chains; caps
<= 31 and > 31; k_stages split widths 1-4; side-stream fork; deferred DSD demand with
k_stages on a side stream and the fill pass; DSD families; the two-phase launch
order of gl_eval_grid_sched / gl_evaluate_host_sched), gl_argmin_feasible,
gl_link_demand, gl_savings_surface, gl_complete_matrices (cooperative and
one-CTA paths), gl_argmin_matrices, gl_evaluate_host, and k_relax alone and racing k_decode.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_20322_b200 import api  # noqa: E402
from paper_2412_20322_b200.inputs import build_config, subset_chains  # noqa: E402
from paper_2412_20322_b200.inputs.cf import low_rank_matrix, observation_mask  # noqa: E402


def main():
    torch.cuda.set_device(0)
    grids = [build_config(1), build_config(2, n=800), build_config(6, n=1500),
             subset_chains(build_config(3, n=1200), list(range(0, 128, 16))),
             build_config(1, cap=40), build_config(1, cap=200)]
    for g in grids:
        dg = api.DeviceGrid(g)
        stats, rows = api.eval_grid(dg, per_request=True)
        api.argmin_feasible(dg, stats)
        _, link = api.link_demand(dg, 50_000)
        torch.cuda.synchronize()
        api.check_status(api.stats_numpy(stats))
        print(g.name, "chains", len(g.chains), "ok", flush=True)
    # deferred DSD demand (solo groups and a family) and the two-phase launch order
    for g, hints in ((build_config(4, n=1000), [(32, 40), (3, 17)]),
                     (subset_chains(build_config(5, n=600), list(range(0, 120))), [(0, 40), (45, 50)])):
        dg = api.DeviceGrid(g)
        base, _ = api.eval_grid(dg, per_request=True)
        for h in hints:
            st, _ = api.eval_grid(dg, per_request=True, schedule=h)
            torch.cuda.synchronize()
            assert torch.equal(st, base), (g.name, h)
        host = api.evaluate_host(dg, dg.pinned_traces(), schedule=hints[0])
        print(g.name, "deferred demand + hints", hints, "ok", flush=True)
    g6 = build_config(6, n=1500)
    dg6 = api.DeviceGrid(g6)
    st6, _ = api.eval_grid(dg6)
    sav = api.savings_surface(dg6, st6)
    host = api.evaluate_host(dg6, dg6.pinned_traces(), want_carbon=True)
    torch.cuda.synchronize()
    print("savings", tuple(sav.shape), "evaluate_host choice[0]", int(host.choice[0]), flush=True)
    for (B, R, C, k) in ((2, 300, 8, 2), (1, 33, 64, 3), (5, 40, 6, 1)):
        x = np.stack([low_rank_matrix(R, C, k, seed=7 + b) for b in range(B)])
        m = np.stack([observation_mask(R, C, 0.3, seed=11 + b) for b in range(B)])
        out, U, V, status = api.complete_matrices(torch.from_numpy(x).cuda(),
                                                  torch.from_numpy(m).cuda(), rank=k, iters=20)
        choice, fb = api.argmin_matrices(out[0], out[0].clamp(0, 1))
        torch.cuda.synchronize()
        print("als", (B, R, C, k), "status", status.cpu().tolist()[:3], flush=True)
    # k_relax: alone (solo: it owns what it solves, k_decode walks the rest) and racing
    import os
    for mode, g in (("solo", build_config(4, n=1500)), ("solo", build_config(2, n=800)),
                    ("1", build_config(4, n=9000))):
        os.environ["GL_RELAX"] = mode
        if mode == "1":
            os.environ["GL_RELAX_RHO"] = "0.0,10.0"
        dg = api.DeviceGrid(g)
        stats, rows = api.eval_grid(dg, per_request=True)
        torch.cuda.synchronize()
        print("relax", mode, g.name, "ok", flush=True)
    os.environ.pop("GL_RELAX", None)
    os.environ.pop("GL_RELAX_RHO", None)
    print("sanitize_run done")


if __name__ == "__main__":
    main()
