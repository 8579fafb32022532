"""The all-cores oracle fan-out used by the GPU parity tests equals the serial
oracle, and its in-worker per-request comparison reports mismatches."""
import numpy as np

from oracle import oracle as O
from paper_2412_20322_b200.inputs import build_config
from tests import oracle_pool


def test_pool_equals_serial_oracle_and_flags_mismatches():
    g = build_config(4, n=700)
    want = O.evaluate_grid(g, per_request=True)
    rows = np.concatenate([np.stack(want["per_request"][ci], axis=1) for ci in range(len(g.chains))])
    got = oracle_pool.evaluate_grid(g, gpu_per_request=rows, procs=4)
    assert got["mismatch"] == {}
    for ci in range(len(g.chains)):
        assert got["stats"][ci] == want["stats"][ci]
    assert np.array_equal(got["carbon"], want["carbon"])
    assert np.array_equal(got["choice"], want["choice"])
    assert np.array_equal(got["via_fallback"], want["via_fallback"])
    bad = rows.copy()
    bad[700 * 5 + 17, 1] += 1  # chain 5, request 17: finish off by one
    got = oracle_pool.evaluate_grid(g, gpu_per_request=bad, procs=3)
    assert list(got["mismatch"]) == [5] and got["mismatch"][5][0] == 1 and got["mismatch"][5][1] == [17]
