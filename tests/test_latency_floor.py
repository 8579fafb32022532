"""The latency roofline's floor (profiles/k_decode_latency.json, bench.py
roofline.latency) is reproducible from committed inputs: scripts/latency_floor.py on
the built libgreenllm.so and the committed B200 latency measurements must give the
committed numbers (a change to the decode loop's SASS makes this fail until the
profile is regenerated)."""
import json
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2412_20322_b200", "libgreenllm.so")
PROFILE = os.path.join(ROOT, "profiles", "k_decode_latency.json")


@pytest.mark.skipif(not (os.path.exists(SO) and shutil.which("cuobjdump") and shutil.which("nvcc")),
                    reason="needs the built library and the CUDA toolkit")
def test_latency_floor_reproduces_the_committed_profile():
    committed = json.load(open(PROFILE))
    args = committed["command"].split()[2:]  # after "python scripts/latency_floor.py"
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "latency_floor.py"), *args],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    now = json.loads(out.stdout)
    assert now["paths"]["J"]["sass"] == committed["paths"]["J"]["sass"]
    assert now["paths"]["L"]["sass"] == committed["paths"]["L"]["sass"]
    assert now["min_cycles_per_event"] == pytest.approx(committed["min_cycles_per_event"], abs=0.05)
    assert now["issue_bound_cycles_per_event"] == pytest.approx(
        committed["issue_bound_cycles_per_event"], abs=0.05)
    # the floor is a floor: below the in-order model, below what the B200 measured
    assert now["min_cycles_per_event"] <= now["issue_bound_cycles_per_event"]
    for crit in committed.get("critical_chain", {}).values():
        assert now["min_cycles_per_event"] < crit["cycles_per_event"]
