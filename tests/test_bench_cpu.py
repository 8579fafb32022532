"""bench.py contract checks that need no GPU: the reference arm (the oracle on a
bounded sample) prints one JSON line with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--n", "2000"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert "workload" in d["config"]


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--n", "500"], cwd=ROOT, capture_output=True,
                         text=True, timeout=300, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_reference_arm_other_configs():
    """--config 5 / 7 select BASELINE configs[4] and the HumanEval grid."""
    for cfg in (5, 7):
        out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                              "--warmup", "3", "--n", "800", "--config", str(cfg)], cwd=ROOT,
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        d = json.loads(out.stdout.strip().splitlines()[-1])
        assert d["config"]["workload"].startswith(f"cfg{cfg}:") and d["value"] > 0


def test_bench_helpers_roofline_units():
    """The roofline's algorithmic bytes are SURVEY §8(d)'s 16 B per (timing chain,
    request); shards are cost-balanced and cover every chain."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2412_20322_b200.inputs import build_config
    g = build_config(4, n=1000)
    assert bench.algorithmic_bytes(g, 0, 64) == 16 * 64 * 1000
    assert bench.algorithmic_bytes(g, 3, 5) == 16 * 2 * 1000
    for w in (1, 2, 4, 8):
        b = bench.shard_bounds(g, w)
        assert b[0][0] == 0 and b[-1][1] == 64 and len(b) == w
