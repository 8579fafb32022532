"""The five BASELINE.json configurations as (traces, timing chains, scenarios, grid).

Vocabulary: a *timing chain* is one (trace, GPU pair, mode,
gamma, alpha, batch cap, link) combination -- everything that changes timing.
A *scenario* is one (CI, LT_new, LT_old) point -- it changes only carbon
(Eqs. 1-3).  Alg. 1's matrices (Fig. 8) have
rows = workloads/scenarios and columns = candidate configurations; each cell
names the chain it is scored on (R35).

Axis values: rates R8 = {0.5..8} req/s; CI64 = 17 + k*484/63
(NCSW 17 ... MISO 501); LT16 = T_A in {2, 11/3, 16/3, 7} y x T_B in
{5, 20/3, 25/3, 10} y; default CI 261 (CISO) and LT 7 y;
link 16 Gbps; batch cap 16; 365-day years.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .tables import (GPUS, ChainTables, capacity_ok, dpd_tables, dsd_tables, spec_colo_tables,
                     standalone_tables)
from .workload import BASE_SEED, RATES8, RATES_CODE8, WORKLOADS, Trace, lengths, make_trace

MODE_DPD = 0
MODE_DSD = 1
MODE_STANDALONE = 2   # co-located on one GPU: target only
MODE_SPEC_COLO = 3    # co-located on one GPU: draft + target
PRIORITY_SLO = 0
PRIORITY_DEFAULT = 1
YEAR_S = 365 * 24 * 3600  # 31,536,000 s
CI_DEFAULT = 261.0
LT_DEFAULT_Y = 7.0
ALPHAS5 = (0.5, 0.6, 0.7, 0.8, 0.9)
PAIRS4 = (("A100", "T4"), ("A100", "V100"), ("V100", "T4"), ("A100", "A100"))
BW8 = (1.0, 2.0, 4.0, 8.0, 16.0, 25.0, 50.0, 100.0)


@dataclass
class ChainSpec:
    mode: int
    trace_idx: int
    cap: int
    gamma: int
    alpha: float
    seed: int
    tables: ChainTables
    ttft_slo_us: int
    tpot_slo_us: int
    ce_new_g: float
    ce_old_g: float
    capacity_ok: int
    label: str = ""


@dataclass
class GridSpec:
    name: str
    traces: list
    chains: list
    scenarios: np.ndarray          # float64 [S, 3]: ci_g_per_kwh, lt_new_s, lt_old_s
    row_scenario: np.ndarray       # int32 [rows]
    cell_chain: np.ndarray         # int32 [rows * cols], -1 = absent
    rows: int
    cols: int
    slo_num: int = 9
    slo_den: int = 10
    priority: int = PRIORITY_SLO
    default_col: int = -1
    row_labels: list = field(default_factory=list)
    col_labels: list = field(default_factory=list)
    workload: str = ""

    @property
    def n_requests_total(self) -> int:
        return sum(self.traces[c.trace_idx].n for c in self.chains)

    @property
    def grid_points(self) -> int:
        return int((self.cell_chain >= 0).sum())


def ci64() -> np.ndarray:
    return np.array([17.0 + k * 484.0 / 63.0 for k in range(64)])


def lt16_years():
    ta = (2.0, 11.0 / 3.0, 16.0 / 3.0, 7.0)
    tb = (5.0, 20.0 / 3.0, 25.0 / 3.0, 10.0)
    return [(a, b) for a in ta for b in tb]


def _slo_us(workload: str):
    wl = WORKLOADS[workload]
    return int(round(wl.ttft_slo_ms * 1000)), int(round(wl.tpot_slo_ms * 1000))


def _chain(mode, trace_idx, cap, tables, workload, new, old, target, draft,
           gamma=0, alpha=0.0, seed=BASE_SEED, label=""):
    ttft, tpot = _slo_us(workload)
    kind = {MODE_DPD: "dpd", MODE_DSD: "dsd", MODE_STANDALONE: "standalone",
            MODE_SPEC_COLO: "spec_colo"}[mode]
    cap_ok = capacity_ok(kind, new, old, target, draft, cap, WORKLOADS[workload].p50)
    ce_old = GPUS[old].embodied_g if old is not None else 0.0  # co-located: one GPU
    return ChainSpec(mode, trace_idx, cap, gamma, float(alpha), seed, tables, ttft, tpot,
                     GPUS[new].embodied_g, ce_old, cap_ok, label)


def _default_scenario():
    lt = LT_DEFAULT_Y * YEAR_S
    return np.array([[CI_DEFAULT, lt, lt]], dtype=np.float64)


def config1(n: int = 100, rate: float = 1.0, mode: str = "dist", cap: int = 16) -> GridSpec:
    """Llama-7B DPD, A100 prefill + T4 decode, 100 Poisson requests at 1 req/s,
    1 CI, 1 lifetime."""
    tr = make_trace("chat", n, rate, RATES8.index(rate) if rate in RATES8 else 0, mode)
    tab = dpd_tables("A100", "T4", "7B", cap)
    ch = _chain(MODE_DPD, 0, cap, tab, "chat", "A100", "T4", "7B", None, label=tab.label)
    return GridSpec(f"cfg1/{mode}/{rate}", [tr], [ch], _default_scenario(),
                    np.zeros(1, np.int32), np.zeros(1, np.int32), 1, 1,
                    row_labels=[f"chat@{rate}"], col_labels=["DPD A100+T4"], workload="chat")


def config2(n: int = 10_000, rate: float = 2.0, cap: int = 16) -> GridSpec:
    """Llama-7B DSD: 68M draft on T4, target on A100; gamma 1..8 (cols) x
    alpha 0.5..0.9 (rows); 10k chat requests."""
    tr = make_trace("chat", n, rate, RATES8.index(rate))
    chains, cells = [], []
    tabs = {g: dsd_tables("A100", "T4", "7B", "68M", g, cap) for g in range(1, 9)}
    for ai, a in enumerate(ALPHAS5):
        for g in range(1, 9):
            cells.append(len(chains))
            chains.append(_chain(MODE_DSD, 0, cap, tabs[g], "chat", "A100", "T4", "7B", "68M",
                                 g, a, label=f"DSD g{g} a{a}"))
    return GridSpec("cfg2", [tr], chains, _default_scenario(),
                    np.zeros(5, np.int32), np.array(cells, np.int32), 5, 8,
                    row_labels=[f"alpha={a}" for a in ALPHAS5],
                    col_labels=[f"gamma={g}" for g in range(1, 9)], workload="chat")


def _rate_traces(workload: str, n: int, rates):
    wl = WORKLOADS[workload]
    shared = lengths(n, wl)
    return [make_trace(workload, n, r, i, shared_lengths=shared) for i, r in enumerate(rates)]


def config3(n: int = 100_000, cap: int = 16, rates=RATES8, bws=BW8) -> GridSpec:
    """Llama-13B both modes on (A100, V100), KV-link bandwidth sweep 1-100 Gbps,
    0.5-8 req/s.  DSD drafts with 1B, gamma 4, alpha 0.8."""
    traces = _rate_traces("chat", n, rates)
    chains, cells, rl = [], [], []
    for ri, r in enumerate(rates):
        for bw in bws:
            rl.append(f"{r}rps/{bw}Gbps")
            dpd = dpd_tables("A100", "V100", "13B", cap, bw)
            dsd = dsd_tables("A100", "V100", "13B", "1B", 4, cap, bw)
            cells.append(len(chains))
            chains.append(_chain(MODE_DPD, ri, cap, dpd, "chat", "A100", "V100", "13B", None,
                                 label=dpd.label + f" {r}rps"))
            cells.append(len(chains))
            chains.append(_chain(MODE_DSD, ri, cap, dsd, "chat", "A100", "V100", "13B", "1B",
                                 4, 0.8, label=dsd.label + f" {r}rps"))
    rows = len(rates) * len(bws)
    return GridSpec("cfg3", traces, chains, _default_scenario(),
                    np.zeros(rows, np.int32), np.array(cells, np.int32), rows, 2,
                    row_labels=rl, col_labels=["DPD", "DSD"], workload="chat")


def config4(n: int = 100_000, cap: int = 16, rates=RATES8, workload: str = "chat",
            name: str = "cfg4") -> GridSpec:
    """Full grid: 4 GPU pairs x 2 modes x 64 CI x 16 lifetimes x 8 rates.
    64 timing chains (rate x pair x mode) score 8,192 rows x 8 columns."""
    traces = _rate_traces(workload, n, rates)
    chains = []
    chain_of = {}
    tabs = {}
    for pi, (new, old) in enumerate(PAIRS4):
        tabs[(pi, 0)] = dpd_tables(new, old, "7B", cap)
        tabs[(pi, 1)] = dsd_tables(new, old, "7B", "1B", 4, cap)
    for ri, r in enumerate(rates):
        for pi, (new, old) in enumerate(PAIRS4):
            for mode in (MODE_DPD, MODE_DSD):
                chain_of[(ri, pi, mode)] = len(chains)
                chains.append(_chain(mode, ri, cap, tabs[(pi, mode)], workload, new, old, "7B",
                                     "1B" if mode == MODE_DSD else None,
                                     4 if mode == MODE_DSD else 0,
                                     0.8 if mode == MODE_DSD else 0.0,
                                     label=f"{tabs[(pi, mode)].label} {r}rps"))
    cis = ci64()
    lts = lt16_years()
    scen = np.array([[ci, ta * YEAR_S, tb * YEAR_S] for ci in cis for (ta, tb) in lts],
                    dtype=np.float64)
    row_scen, cells, rl = [], [], []
    for ri, r in enumerate(rates):
        for si in range(len(scen)):
            row_scen.append(si)
            rl.append(f"{r}rps/ci{scen[si, 0]:.2f}/lt{scen[si, 1] / YEAR_S:.3g},{scen[si, 2] / YEAR_S:.3g}")
            for pi in range(len(PAIRS4)):
                for mode in (MODE_DPD, MODE_DSD):
                    cells.append(chain_of[(ri, pi, mode)])
    cols = [f"{'DPD' if m == 0 else 'DSD'} {a}+{b}" for (a, b) in PAIRS4 for m in (0, 1)]
    return GridSpec(name, traces, chains, scen, np.array(row_scen, np.int32),
                    np.array(cells, np.int32), len(row_scen), 8,
                    row_labels=rl, col_labels=cols, workload=workload)


def config5(n: int = 1_000_000, cap: int = 16, rates=RATES8) -> GridSpec:
    """Llama-70B DSD with a 7B draft (A100 + T4), LongBench lengths, gamma 1..8
    (cols) x alpha 0.5..0.9 x rate (rows), 1M-request traces."""
    traces = _rate_traces("summ", n, rates)
    tabs = {g: dsd_tables("A100", "T4", "70B", "7B", g, cap) for g in range(1, 9)}
    chains, cells, rl = [], [], []
    for ri, r in enumerate(rates):
        for a in ALPHAS5:
            rl.append(f"{r}rps/alpha={a}")
            for g in range(1, 9):
                cells.append(len(chains))
                chains.append(_chain(MODE_DSD, ri, cap, tabs[g], "summ", "A100", "T4", "70B",
                                     "7B", g, a, label=f"DSD 70B/7B g{g} a{a} {r}rps"))
    rows = len(rates) * len(ALPHAS5)
    return GridSpec("cfg5", traces, chains, _default_scenario(),
                    np.zeros(rows, np.int32), np.array(cells, np.int32), rows, 8,
                    row_labels=rl, col_labels=[f"gamma={g}" for g in range(1, 9)],
                    workload="summ")


def config6(n: int = 100_000, cap: int = 16, rates=RATES8, workload: str = "chat",
            name: str = "cfg6") -> GridSpec:
    """config 4 plus the paper's two single-GPU columns
     -- Standalone 7B on an A100 (the paper's baseline) and
    SpecDecode 7B/1B (gamma 4, alpha 0.8) co-located on an A100 -- so Alg. 1
    chooses among all four configuration families.  80 timing chains score
    8,192 rows x 10 columns."""
    g4 = config4(n, cap, rates, workload, name)
    chains = list(g4.chains)
    st = standalone_tables("A100", "7B", cap)
    sc = spec_colo_tables("A100", "7B", "1B", 4, cap)
    extra = {}
    for ri, r in enumerate(rates):
        extra[(ri, 0)] = len(chains)
        chains.append(_chain(MODE_STANDALONE, ri, cap, st, workload, "A100", None, "7B", None,
                             label=f"{st.label} {r}rps"))
        extra[(ri, 1)] = len(chains)
        chains.append(_chain(MODE_SPEC_COLO, ri, cap, sc, workload, "A100", None, "7B", "1B", 4,
                             0.8, label=f"{sc.label} {r}rps"))
    cells4 = g4.cell_chain.reshape(g4.rows, g4.cols)
    n_scen = len(g4.scenarios)
    cells = []
    for row in range(g4.rows):
        ri = row // n_scen
        cells.extend(list(cells4[row]) + [extra[(ri, 0)], extra[(ri, 1)]])
    return GridSpec(name, g4.traces, chains, g4.scenarios, g4.row_scenario,
                    np.array(cells, np.int32), g4.rows, g4.cols + 2, row_labels=g4.row_labels,
                    col_labels=g4.col_labels + ["Standalone A100", "SpecDecode A100"],
                    workload=workload)


def config7(n: int = 100_000, cap: int = 16, rates=RATES_CODE8) -> GridSpec:
    """The paper's third workload (§6): HumanEval code requests (Table 2,
    P:428: TTFT 125 ms / TPOT 200 ms SLOs, sizes 108/136/182 in, 31/55/88 out) at
    rates covering its QPS window [0.5, 11], on config 6's candidate set:
    7B DPD and DSD (1B, gamma 4, alpha 0.8) on the four GPU pairs, plus Standalone
    and SpecDecode on an A100.  80 timing chains score 8,192 (rate x CI64 x LT16)
    rows x 10 columns."""
    return config6(n, cap, rates, workload="code", name="cfg7")


def savings_pairs(grid: GridSpec):
    """§5 analysis pairs (NEXT #3): every non-Standalone chain (Case 2) with the
    Standalone chain on the same trace (Case 1)."""
    base = {c.trace_idx: i for i, c in enumerate(grid.chains) if c.mode == MODE_STANDALONE}
    return [(i, base[c.trace_idx]) for i, c in enumerate(grid.chains)
            if c.mode != MODE_STANDALONE and c.trace_idx in base]


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5, 6: config6,
           7: config7}


def build_config(k: int, **kw) -> GridSpec:
    return CONFIGS[int(k)](**kw)


def subset_chains(grid: GridSpec, chain_ids) -> GridSpec:
    """Keep only the given chains (cells naming others become absent, -1)."""
    chain_ids = list(chain_ids)
    remap = {c: i for i, c in enumerate(chain_ids)}
    cells = np.array([remap.get(int(c), -1) for c in grid.cell_chain], np.int32)
    return GridSpec(grid.name + "/subset", grid.traces, [grid.chains[c] for c in chain_ids],
                    grid.scenarios, grid.row_scenario, cells, grid.rows, grid.cols,
                    grid.slo_num, grid.slo_den, grid.priority, grid.default_col,
                    grid.row_labels, grid.col_labels, grid.workload)


def custom_trace(a, p, o, label="custom") -> Trace:
    return Trace(np.asarray(a, np.int64), np.asarray(p, np.uint32), np.asarray(o, np.uint32),
                 "custom", 0.0, label)
