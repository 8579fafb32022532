"""One rank of tests/test_gpu_nccl.py (launched by torchrun): the sharded
evaluation of config 6 at 4k requests over NCCL; saves what this rank got."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2412_20322_b200 import api  # noqa: E402
from paper_2412_20322_b200.dist import chain_costs, evaluate_sharded  # noqa: E402
from paper_2412_20322_b200.inputs import build_config  # noqa: E402


def main(out_dir):
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    g = build_config(6, n=4000)
    dg = api.DeviceGrid(g, f"cuda:{local}")
    held = {}

    def compute(lo, hi, out):
        api.eval_grid(dg, lo, hi, stats=out)

    def argmin(full):
        held["stats"] = api.stats_numpy(full)
        _, choice, fb = api.argmin_feasible(dg, full)
        return choice.cpu().numpy(), fb.cpu().numpy()

    choice, fb = evaluate_sharded(dg.n_chains, compute, argmin, torch.device("cuda", local),
                                  costs=chain_costs(g))
    np.savez(os.path.join(out_dir, f"r{dist.get_rank()}.npz"), stats=held["stats"].view(np.uint8),
             choice=choice, fb=fb)
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
