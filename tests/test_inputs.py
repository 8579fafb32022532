"""The seeded input generators: Philox KAT, trace shape, table-generator pins."""
import os

import numpy as np
import pytest

from paper_2412_20322_b200.inputs import WORKLOADS, build_config
from paper_2412_20322_b200.inputs.philox import philox4x32_10
from paper_2412_20322_b200.inputs.tables import (GPUS, MODELS, dpd_tables, dsd_tables, link_us,
                                                 roofline)
from paper_2412_20322_b200.inputs.workload import arrivals_us, lengths

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_numpy_philox_kat():
    for line in open(os.path.join(GOLD, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        out = philox4x32_10(*v[:4], *v[4:6])
        assert [int(x) for x in out] == v[6:10]


def test_poisson_arrivals():
    a = arrivals_us(200_000, 2.0, 3, 0)
    gaps = np.diff(np.concatenate([[0], a]))
    assert np.all(gaps >= 0) and np.all(np.diff(a) >= 0)
    assert abs(gaps.mean() / 5e5 - 1) < 0.01          # mean 1/lambda (1% at 2e5 samples)
    assert abs(gaps.std() / gaps.mean() - 1) < 0.02   # exponential: CV = 1
    assert np.array_equal(a, arrivals_us(200_000, 2.0, 3, 0))   # determinism


@pytest.mark.parametrize("wl", ["chat", "code", "summ"])
def test_lengths_follow_table2_quantiles(wl):
    w = WORKLOADS[wl]
    p, o = lengths(200_000, w)
    assert p.min() >= 1 and o.min() >= 1 and np.all(p.astype(int) + o <= 4096)
    for q, (pin, pout) in ((25, w.p25), (50, w.p50), (75, w.p75)):
        if wl != "summ":  # summ prompts are clamped by the 4096 context
            assert abs(np.percentile(p, q) / pin - 1) < 0.03
        assert abs(np.percentile(o, q) / pout - 1) < 0.03
    pf, of = lengths(10, w, "fixed")
    assert set(pf) == {w.p50[0]} and set(of) == {w.p50[1]}


def test_kv_bytes_and_link_pins():
    """Appendix B KV bytes/token; R2: 160-token 7B KV at 16 Gbps = 41,943.04 us -> 41,944."""
    want = {"7B": 524_288, "13B": 819_200, "70B": 327_680, "1B": 22_528, "68M": 6_144}
    for m, b in want.items():
        assert MODELS[m].kv_bytes_per_token == b
    assert 160 * 524_288 == 83_886_080
    assert int(link_us(83_886_080, 16.0)) == 41_944
    t = dpd_tables("A100", "T4", "7B", 4)
    assert t.t2_us[159] == int(link_us(160 * 524_288, 16.0))  # KV of p+1 tokens


def test_roofline_sanity_spec_examples():
    """SPEC S:124-125 with eta = 1: prefill 7B/160 tok/A100 ~ 7.18 ms; decode 9.0 ms."""
    import paper_2412_20322_b200.inputs.tables as T
    old = T.ETA_C, T.ETA_M
    try:
        T.ETA_C = T.ETA_M = 1.0
        # compute term 7.18 ms is below the 9.0 ms weight-streaming term
        lat, _ = roofline(GPUS["A100"], MODELS["7B"], 1000)
        assert abs(float(lat) - 2 * 7e9 * 1000 / 312e12) < 1e-12
        assert abs(2 * 7e9 * 160 / 312e12 * 1e3 - 7.18) < 0.01
        lat, e = roofline(GPUS["A100"], MODELS["7B"], 160)
        assert abs(float(lat) * 1e3 - 9.0) < 0.01
        lat, e = roofline(GPUS["A100"], MODELS["7B"], 1)
        assert abs(float(lat) * 1e3 - 9.0) < 0.01
    finally:
        T.ETA_C, T.ETA_M = old


def test_dsd_step_overlap_rule():
    """Per step S_overlap = S_serial - min(V, t_probs); probs hidden iff t_probs <= V
    (Fig. 7; SURVEY G6 corrects SPEC's equality claim)."""
    for bw in (1.0, 16.0, 100.0):
        t = dsd_tables("A100", "T4", "7B", "1B", 4, 8, bw)
        for b in range(1, 9):
            v = int(t.step_busy_new_us[b])
            probs = int(link_us(4 * 32000 * 2 * b, bw))
            serial = int(t.step_busy_old_us[b]) + int(link_us(16 * b, bw)) + v + probs + \
                int(link_us(20 * b, bw))
            assert t.step_us[b] == serial - min(v, probs)


def test_trend_checks_vs_figs_2_3():
    """Synthetic tables follow the paper's qualitative trends: old GPUs are
    slower per step (Fig. 2) and energy per step grows with batch (Fig. 3 shape)."""
    a = dpd_tables("A100", "A100", "7B", 16)
    t = dpd_tables("A100", "T4", "7B", 16)
    assert np.all(t.step_us[1:] > a.step_us[1:])
    assert np.all(np.diff(t.step_e_old_uj[1:]) >= 0)
    assert np.all(np.diff(t.t1_us[1:]) >= 0)


def test_grid_shapes():
    g4 = build_config(4, n=1000)
    assert (len(g4.chains), g4.rows, g4.cols, g4.grid_points) == (64, 8192, 8, 65536)
    g5 = build_config(5, n=1000)
    assert (len(g5.chains), g5.rows, g5.cols) == (320, 40, 8)
    assert all(c.capacity_ok == 0 for c in g5.chains)     # 70B does not fit A100-40GB (R38)
    g3 = build_config(3, n=1000)
    assert {c.capacity_ok for c in g3.chains if c.mode == 0} == {0}   # 13B DPD on V100
    g2 = build_config(2, n=1000)
    assert (len(g2.chains), g2.rows, g2.cols) == (40, 5, 8)
    # every rate of one workload shares one length sequence (R5)
    assert g4.traces[0].output_len is g4.traces[5].output_len


def test_config7_humaneval_grid():
    """Config 7: HumanEval lengths and SLOs (Table 2) at rates spanning the
    paper's QPS window [0.5, 11], config 6's candidate set."""
    g = build_config(7, n=2000)
    assert (len(g.chains), g.rows, g.cols, g.grid_points) == (80, 8192, 10, 81920)
    rates = sorted({t.rate for t in g.traces})
    assert rates[0] == 0.5 and rates[-1] == 11.0 and len(rates) == 8
    wl = WORKLOADS["code"]
    assert all(t.workload == "code" for t in g.traces)
    assert all((c.ttft_slo_us, c.tpot_slo_us) == (125_000, 200_000) for c in g.chains)
    o = g.traces[0].output_len
    assert abs(np.median(o) - wl.p50[1]) <= 2
    assert {c.mode for c in g.chains} == {0, 1, 2, 3}
    # arrivals differ from config 6's chat traces (own workload id in the counter)
    assert not np.array_equal(g.traces[0].arrival_us, build_config(6, n=2000).traces[0].arrival_us)
