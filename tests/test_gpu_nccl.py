"""The multi-GPU path over NCCL: chains sharded in cost-balanced
contiguous blocks over 2 ranks (one process per GPU, torchrun), one
all_gather_into_tensor of the 80-B records, Alg. 1 on every rank.  Every rank's
statistics, choices and fallback flags must be byte-identical to one process
evaluating the whole grid.  Skipped on boxes with fewer than 2 GPUs."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs 2 GPUs")
def test_nccl_two_ranks_equal_one_process(tmp_path):
    from paper_2412_20322_b200 import api
    from paper_2412_20322_b200.inputs import build_config
    g = build_config(6, n=4000)
    dg = api.DeviceGrid(g)
    stats, _ = api.eval_grid(dg)
    _, choice, fb = api.argmin_feasible(dg, stats)
    torch.cuda.synchronize()
    want = (api.stats_numpy(stats).tobytes(), choice.cpu().numpy(), fb.cpu().numpy())
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr=127.0.0.1", "--master-port=29533",
                          os.path.join(ROOT, "tests", "nccl_worker.py"), str(tmp_path)],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    for r in range(2):
        z = np.load(tmp_path / f"r{r}.npz")
        assert z["stats"].tobytes() == want[0]
        assert np.array_equal(z["choice"], want[1]) and np.array_equal(z["fb"], want[2])
