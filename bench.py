"""Benchmark: the full config-4 grid (BASELINE.json configs[3]) per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 4|5|7]

One step = the whole hot path over the grid: gl_eval_grid on this rank's
shard of timing chains (k_dsd_demand, k_stages, k_segments, k_decode, k_finalize), one NCCL all_gather of the
80-byte chain statistics (N > 1), gl_argmin_feasible (k_argmin) over all
8,192 rows x 8 columns.  Inputs are resident in HBM; L2 is flushed (512 MiB
write) between timed steps, outside the timed events.  Rank 0 prints one JSON
line.  ``--impl reference`` times the CPU oracle (oracle/) on a bounded
sample of the same workload instead (the reference arm of this tier).
``--config 5`` times BASELINE configs[4] instead (320 chains x 1M LongBench
requests, the configuration BASELINE states "at 1/2/4/8 GPUs"); ``--config 7``
the HumanEval grid.  Chains are sharded over ranks in
cost-balanced contiguous blocks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "config×request evals/sec at 1/2/4/8 B200; % HBM roofline; speedup vs CPU oracle"
UNIT = "config×request evals/s"
WORKLOADS = {
    4: ("cfg4: full grid, Llama-7B DPD + DSD(1B draft, gamma 4, alpha 0.8) x 4 GPU pairs "
        "x 8 rates (0.5-8 req/s) x 64 CI x 16 lifetimes, 100k chat requests per trace"),
    5: ("cfg5: Llama-70B DSD with a 7B draft (A100 + T4), gamma 1..8 x alpha 0.5..0.9 x 8 "
        "rates (0.5-8 req/s), 1M LongBench requests per trace"),
    7: ("cfg7: HumanEval code requests, 7B DPD + DSD(1B, gamma 4, alpha 0.8) x 4 GPU pairs + "
        "Standalone + SpecDecode (A100) x 8 rates (0.5-11 req/s) x 64 CI x 16 lifetimes, "
        "100k requests per trace"),
}
WORKLOAD = WORKLOADS[4]
DEFAULT_N = {4: 100_000, 5: 1_000_000, 7: 100_000}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=sorted(WORKLOADS))
    ap.add_argument("--n", type=int, default=None, help="requests per trace (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-analysis", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


# 16 B of input per (timing chain, request) -- arrival i64 + prompt u32
# + output u32 -- is the path's algorithmic traffic
BYTES_PER_CHAIN_REQUEST = 16
# the build's own intermediate: k_decode reads the decode stream k_stages wrote (r i64 +
# (demand, j) 2 x u32) and writes each finish time (i64) -- a secondary view
DECODE_BYTES_PER_REQUEST = 24


def decode_requests(grid, lo, hi):
    """Decode requests (o > 1) per chain of the shard: the units k_decode processes."""
    import numpy as np
    per_trace = {}
    out = []
    for ch in grid.chains[lo:hi]:
        if ch.trace_idx not in per_trace:
            per_trace[ch.trace_idx] = int(np.count_nonzero(np.asarray(grid.traces[ch.trace_idx].output_len) > 1))
        out.append(per_trace[ch.trace_idx])
    return out


def algorithmic_bytes(grid, lo, hi):
    """SURVEY §8(d)'s algorithmic bytes of one launch over chains [lo, hi): 16 B per
    (timing chain, request) -- the request's arrival (i64), prompt and output
    lengths (2 x u32); tables amortise to < 1 B/request and CI x lifetime scenarios
    add 0 B per request."""
    return BYTES_PER_CHAIN_REQUEST * sum(grid.traces[c.trace_idx].n for c in grid.chains[lo:hi])


def stream_bytes(grid, lo, hi):
    """The build's decode-stream view: 24 B per decode request read
    and written by k_decode."""
    return DECODE_BYTES_PER_REQUEST * sum(decode_requests(grid, lo, hi))


def shard_bounds(grid, world):
    """Cost-balanced contiguous blocks of chains, N (1 + w_DSD) per chain."""
    from paper_2412_20322_b200.dist import chain_costs, shard_bounds_cost
    return shard_bounds_cost(chain_costs(grid), world)


# --------------------------------------------------------------- clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,utilization.gpu,"
              "clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = []
        for ts, line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm, smax = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            rows.append((ts, sm, smax, parts[3], parts[4:8]))
        inside = [r for r in rows if t0 <= r[0] <= t1] or rows
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        reasons = sorted({names[i] for r in inside for i, v in enumerate(r[4]) if v == "Active"})
        return {"sm_mhz": statistics.median(r[1] for r in inside),
                "sm_max_mhz": max(r[2] for r in inside), "reasons": reasons,
                "samples": len(inside)}


# ------------------------------------------------------------------ CPU oracle
def cpu_baseline(grid, budget_s, chain_order=None):
    """Time the oracle as it stands (single thread) on a bounded sample of the
    workload: whole chains (simulation + carbon + Alg. 1 over their cells)."""
    from oracle import oracle as O
    O.lib()
    order = chain_order if chain_order is not None else list(range(len(grid.chains)))
    # size the sample to the budget from one probe chain of each mode
    t0 = time.perf_counter()
    for ci in order[:2]:
        O.simulate_chain(grid.traces[grid.chains[ci].trace_idx], grid.chains[ci], False)
    per_chain = (time.perf_counter() - t0) / 2
    k = int(max(2, min(len(order), budget_s / max(per_chain, 1e-6))))
    step = max(1, len(order) // k)
    done = order[::step][:k]
    sub = _subset(grid, done)
    t1 = time.perf_counter()
    O.evaluate_grid(sub)  # simulation + carbon + Alg. 1 over the sample's cells
    t_all = time.perf_counter() - t1
    cells = int(np.isin(grid.cell_chain, done).sum())
    reqs = grid.traces[0].n
    evals = cells * reqs
    return dict(value=evals / t_all, cells=cells, chains=len(done), seconds=t_all,
                chain_request_sims_per_s=len(done) * reqs / t_all)


def _oracle_chain_worker(args):
    """One whole chain through the oracle in a worker process (all-cores baseline)."""
    cfg, n, ci = args
    from oracle import oracle as O
    g = _worker_grid(cfg, n)
    ch = g.chains[ci]
    t0 = time.perf_counter()
    O.simulate_chain(g.traces[ch.trace_idx], ch, per_request=False)
    return time.perf_counter() - t0


_WORKER_GRID = {}


def _worker_grid(cfg, n):
    from paper_2412_20322_b200.inputs import build_config
    if (cfg, n) not in _WORKER_GRID:
        _WORKER_GRID[(cfg, n)] = build_config(cfg, n=n)
    return _WORKER_GRID[(cfg, n)]


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def host_cpu_model():
    """The host CPU model (lscpu's "Model name"), SURVEY 8(d)."""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline_all_cores(grid, cfg, n, max_rounds=2):
    """The same single-threaded oracle, one chain per process across every host core
    (per-core rate, aggregate, nproc).  Timing chains only (the
    carbon/Alg. 1 epilogue is < 1% of the oracle's time); wall clock of the pool.
    A bounded sample (at most ``max_rounds`` chains per core, spread over the grid)
    when the workload has more chains than that (config 5: ~5 s per chain)."""
    import multiprocessing as mp
    cores = host_cores()
    all_ids = list(range(len(grid.chains)))
    k = min(len(all_ids), max_rounds * cores)
    ids = all_ids[::max(1, len(all_ids) // k)][:k]
    jobs = [(cfg, n, ci) for ci in ids]
    procs = min(cores, len(jobs))
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_worker_grid, initargs=(cfg, n)) as pool:
        t0 = time.perf_counter()
        per = pool.map(_oracle_chain_worker, jobs, chunksize=1)
        wall = time.perf_counter() - t0
    reqs = grid.traces[0].n
    cells = int(np.isin(grid.cell_chain, ids).sum())
    return {"value": cells * reqs / wall, "unit": UNIT, "cores": procs,
            "kind": "oracle", "sample": f"{len(jobs)} of {len(all_ids)} timing chains x {reqs} "
            f"requests (all {cells} of their grid cells), one process per chain on {procs} of "
            f"{cores} host cores, {wall:.1f} s wall",
            "cpu_model": host_cpu_model(),
            "chain_request_sims_per_s": len(jobs) * reqs / wall,
            "per_core_chain_request_sims_per_s": reqs / (sum(per) / len(per))}


def _subset(grid, chain_ids):
    from paper_2412_20322_b200.inputs import subset_chains
    return subset_chains(grid, chain_ids)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_2412_20322_b200.inputs import build_config
    O.lib()
    grid = build_config(args.config, n=args.n)
    per_step_chains = 1 if args.config == 5 else 2  # a config-5 chain is ~5 s of oracle
    times, evals = [], []
    for step in range(args.warmup + args.steps):
        ids = [(step * per_step_chains + k) % len(grid.chains) for k in range(per_step_chains)]
        t0 = time.perf_counter()
        sub = _subset(grid, ids)
        ref = O.evaluate_grid(sub)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
            evals.append(int(ref["present"].sum()) * grid.traces[0].n)
    value = sum(evals) / sum(times)
    cells_per_chain = grid.grid_points // len(grid.chains)
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
           "config": {"workload": WORKLOADS[args.config],
                      "sample": f"{per_step_chains} timing chain(s) (each {grid.traces[0].n} "
                      f"requests, all {cells_per_chain} of its grid cells) per step, rotating"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": f"{per_step_chains} of {len(grid.chains)} chains per step"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def load_profile_json(name, cfg):
    """A committed ncu summary under profiles/: the entry for this config
    ("cfg5": {...}) or, for config 4, the top-level fields."""
    path = os.path.join(ROOT, "profiles", name)
    try:
        pj = json.load(open(path))
    except (OSError, ValueError):
        return {}
    if f"cfg{cfg}" in pj:
        return pj[f"cfg{cfg}"]
    return pj if cfg == 4 else {}


# --------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2412_20322_b200 import api
    from paper_2412_20322_b200 import native as N
    from paper_2412_20322_b200.dist import all_gather_stats
    from paper_2412_20322_b200.inputs import build_config

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    grid = build_config(args.config, n=args.n)
    dg = api.DeviceGrid(grid, dev)
    bounds = shard_bounds(grid, world)
    lo, hi = bounds[rank]
    max_shard = max(h - l for l, h in bounds)
    local_stats = torch.zeros((max_shard, 80), dtype=torch.uint8, device=dev)
    gathered = torch.empty((world * max_shard, 80), dtype=torch.uint8, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        launches = 0
        if hi > lo:
            api.eval_grid(dg, lo, hi, stats=local_stats[: hi - lo])
            launches += dg.last_launches
        if world > 1:
            full = all_gather_stats(local_stats, gathered, bounds, dg.n_chains)
        else:
            full = local_stats
        api.argmin_feasible(dg, full, want_carbon=True)
        launches += dg.last_launches
        return launches

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st = api.stats_numpy(local_stats[: hi - lo]) if hi > lo else None
    if st is not None:
        api.check_status(st)

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    N.profile_enable(True)
    N.kernel_times()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    launches = 0
    kt = {}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.time()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        evs[i][0].record(stream)
        launches += step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_wall1 = time.time()
    for name, ms in N.kernel_times():
        kt.setdefault(name, []).append(ms)
    N.profile_enable(False)
    sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    ms_per_step = float(total_ms.item()) / args.steps

    # end to end: pinned host traces -> gl_evaluate_host (H2D, kernels, D2H)
    e2e = None
    if world == 1:
        host = dg.pinned_traces()
        res = api.evaluate_host(dg, host)
        for _ in range(2):
            api.evaluate_host(dg, host, out=res)
        e_ms = []
        for i in range(max(3, args.steps // 2)):
            flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            api.evaluate_host(dg, host, out=res)
            e1.record(stream)
            torch.cuda.synchronize()
            e_ms.append(e0.elapsed_time(e1))
        e2e_ms = sum(e_ms) / len(e_ms)
        e2e = {"value": grid.grid_points * grid.traces[0].n / (e2e_ms / 1e3), "unit": UNIT,
               "ms_per_step": e2e_ms, "h2d_bytes_per_step": res.h2d_bytes,
               "d2h_bytes_per_step": res.d2h_bytes,
               "path": "gl_evaluate_host (pinned host traces, cudaMemcpyAsync in, results out)"}
    else:
        e2e = e2e_distributed(args, dg, grid, bounds, lo, hi, local_stats, gathered, flush, dev)

    analysis = None
    if world == 1 and not args.no_analysis and args.config == 4:
        analysis = {"link_demand": link_demand_bench(dg, grid, flush),
                    **analysis_bench(dg, grid)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    reqs = grid.traces[0].n
    evals = grid.grid_points * reqs
    value = evals / (ms_per_step / 1e3)
    chain_req = dg.chain_n.sum() / (ms_per_step / 1e3)
    kname = "k_decode" if "k_decode" in kt else max(kt, key=lambda k: sum(kt[k]), default="k_decode")
    kdec = kt.get(kname, [])
    kdec_ms = sum(kdec) / max(1, len(kdec))
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm_peak = peaks.get("hbm_gbs")
    peak_src = "MEASURED_PEAKS.json hbm_gbs (burst copy bandwidth)"
    if hbm_peak is None:
        hbm_peak, peak_src = 7700.0, "B200_PROFILING.md fallback (no MEASURED_PEAKS.json)"
    alg_bytes = algorithmic_bytes(grid, lo, hi)
    achieved = alg_bytes / (kdec_ms / 1e3) / 1e9 if kdec_ms > 0 else 0.0
    sbytes = stream_bytes(grid, lo, hi)
    prof = load_profile_json("k_decode_dram_bytes.json", args.config)
    traffic = prof.get("dram_bytes_per_launch")
    l2_traffic = prof.get("l2_bytes_per_launch")
    winst = prof.get("warp_inst_per_launch")
    step_total = {k: sum(v) / max(1, len(v)) for k, v in kt.items()}
    cpu = None
    if not args.no_cpu_baseline:
        cb = cpu_baseline(grid, args.cpu_budget_s)
        cpu = {"value": cb["value"], "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{cb['chains']} of {len(grid.chains)} timing chains x {reqs} requests "
                         f"(all {cb['cells']} of their grid cells), single-threaded, "
                         f"{cb['seconds']:.1f} s",
               "chain_request_sims_per_s": cb["chain_request_sims_per_s"]}
        try:
            cpu["all_cores"] = cpu_baseline_all_cores(grid, args.config, args.n)
        except Exception as exc:  # a host without fork / enough memory: report why
            cpu["all_cores"] = {"unavailable": repr(exc)[:200]}
    clocks = sampler.summary(t_wall0, t_wall1)
    sm_mhz = (clocks or {}).get("sm_mhz") or 1965.0
    latency = latency_view(grid, lo, hi, kdec_ms, sm_mhz, args.config)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "grid_points": grid.grid_points,
                   "timing_chains": len(grid.chains), "requests_per_trace": reqs,
                   "l2": "flushed between timed steps (512 MiB device write, outside the events)",
                   "parallelism": f"chains sharded over {world} GPU(s) in cost-balanced "
                                  "contiguous blocks, one NCCL all_gather of 80-B chain stats"
                                  if world > 1 else "1 GPU",
                   "grid_point_factorisation": "each timing chain is simulated once and scores "
                                               f"its {grid.grid_points // len(grid.chains)} grid "
                                               "cells (CI x lifetime rows share it; SURVEY F2)"},
        "chain_request_sims_per_s": chain_req,
        "kernel_ms_per_step": step_total,
        "roofline": {"bound": "latency", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "l2_traffic": l2_traffic,
                     "peak_source": peak_src,
                     "kernel": kname, "algorithmic_bytes_per_launch": alg_bytes,
                     "bytes_per_unit": BYTES_PER_CHAIN_REQUEST,
                     "unit_name": "(timing chain, request): arrival i64 + prompt u32 + output u32 "
                                  "(SURVEY §8(d))",
                     "units_per_launch": alg_bytes // BYTES_PER_CHAIN_REQUEST,
                     "kernel_ms": kdec_ms,
                     "stream_view": {"bytes_per_decode_request": DECODE_BYTES_PER_REQUEST,
                                     "bytes_per_launch": sbytes,
                                     "achieved_gbs": sbytes / (kdec_ms / 1e3) / 1e9 if kdec_ms else 0.0,
                                     "note": "the decode stream k_stages writes and k_decode reads "
                                             "(r, demand, index) plus the finish times written"},
                     "latency": latency,
                     "alu_view": alu_view(winst, kdec_ms, sm_mhz, grid, lo, hi),
                     "note": "bound = latency: k_decode runs one serial event loop per timing "
                             "chain, so the step lasts as long as the slowest chain it walks; "
                             "k_relax (the decode stage as an exact parallel fixed point) races it "
                             "on the heavily loaded chains and takes those it solves first; HBM "
                             "and the issue rate are both far from saturated (DESIGN.md §4)"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
        "analysis": analysis,
    }
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


def latency_view(grid, lo, hi, kernel_ms, sm_mhz, cfg):
    """The latency roofline of k_decode.  Every decode request
    is one join and one leave event of its chain's serial loop; the launch lasts as
    long as its slowest chain, so the achieved cycles per event of the critical
    chain are at most kernel cycles / (2 x its decode requests).  The floor is the
    loop's minimal dependent-instruction cycles per event from the committed
    analysis (profiles/k_decode_latency.json: measured instruction latencies,
    scripts/ubench/lat.cu, along the SASS of the loop body); frac = floor / achieved."""
    m_max = max(decode_requests(grid, lo, hi) or [0])
    achieved = (kernel_ms * 1e-3 * sm_mhz * 1e6 / (2 * m_max)) if m_max and kernel_ms else None
    lat = load_profile_json("k_decode_latency.json", 4)
    floor = lat.get("min_cycles_per_event")
    out = {"max_decode_requests_per_chain": m_max, "events_per_chain": 2 * m_max,
           "cycles_per_event": achieved, "sm_mhz": sm_mhz,
           "min_cycles_per_event": floor,
           "frac": (floor / achieved) if (floor and achieved) else None,
           "floor_source": lat.get("source")}
    crit = lat.get("critical_chain", {}).get(f"cfg{cfg}")
    if crit:
        out["critical_chain"] = crit
    return out


def alu_view(warp_inst, kernel_ms, sm_mhz, grid, lo, hi):
    """The issue-rate view of k_decode: warp-instructions per
    launch (ncu smsp__inst_executed.sum, profiles/k_decode_dram_bytes.json) over the
    live kernel time, against 148 SMs x 4 schedulers x 1 warp-instruction per cycle
    at the sampled SM clock."""
    if not warp_inst or kernel_ms <= 0:
        return None
    peak = 148 * 4 * sm_mhz * 1e6
    achieved = warp_inst / (kernel_ms / 1e3)
    reqs = sum(g.n for g in [grid.traces[c.trace_idx] for c in grid.chains[lo:hi]])
    return {"achieved": achieved, "peak": peak, "unit": "warp-inst/s", "frac": achieved / peak,
            "warp_inst_per_chain_request": warp_inst / max(reqs, 1),
            "note": "instruction count from the committed ncu capture; the kernel is bound by "
                    "the slowest chain's dependent latency, so most SMs idle (warps_active ~3%)"}


def link_demand_bench(dg, grid, flush, reps=3):
    """NEXT #2 (not part of the timed step): gl_link_demand over all chains of the
    workload -- the same speculative simulation recording batch-size logs, then the
    1 s sliding-window peak (k_link_*).  Device time with CUDA events; per-kernel
    times from gl_kernel_times."""
    import torch

    from paper_2412_20322_b200 import api
    from paper_2412_20322_b200 import native as N
    stream = torch.cuda.current_stream()
    api.link_demand(dg)
    torch.cuda.synchronize()
    N.profile_enable(True)
    N.kernel_times()
    ms = []
    for i in range(reps):
        flush.fill_(i & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, link = api.link_demand(dg)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    kt = {}
    for name, t in N.kernel_times():
        kt.setdefault(name, []).append(t)
    N.profile_enable(False)
    lk = api.link_numpy(link)
    gbps = {}
    for ci, ch in enumerate(grid.chains):
        kind = {0: "dpd", 1: "dsd"}.get(ch.mode)
        if kind:
            gbps.setdefault(kind, []).append(float(lk[ci]["peak_bytes"]) * 8 / 1e9)
    # Fig. 4's view: DPD / DSD peak-demand ratio per GPU pair and rate.
    # config 4's chain order is rate x pair x (DPD, DSD): chains 2k and 2k + 1 pair up.
    fig4 = {}
    for ci in range(0, len(grid.chains) - 1, 2):
        a, b = grid.chains[ci], grid.chains[ci + 1]
        if a.mode == 0 and b.mode == 1 and a.trace_idx == b.trace_idx:
            pair = a.label.split(" ")[2]
            rate = a.label.split(" ")[-1]
            dpd, dsd = float(lk[ci]["peak_bytes"]), float(lk[ci + 1]["peak_bytes"])
            fig4.setdefault(pair, {})[rate] = round(dpd / dsd, 1) if dsd > 0 else None
    return {"ms": sum(ms) / len(ms), "window_us": 1_000_000,
            "kernel_ms": {k: sum(v) / len(v) for k, v in kt.items()},
            "peak_gbps_range": {k: [min(v), max(v)] for k, v in gbps.items()},
            "dpd_over_dsd_peak_ratio": fig4,
            "note": "peak link demand of every chain (R45-R47); logging decode + "
                    "k_link_scan/window/reduce; outside the timed step"}


def analysis_bench(dg, grid, reps=3):
    """NEXT #3 / #4 (not part of the timed step), device time with CUDA events:
    gl_savings_surface over config 6 (72 pairs x 1,024 scenarios) and
    gl_complete_matrices on this workload's Alg. 1 matrices (carbon, attainment;
    30% of the cells hidden; rank 2, lambda 0.1, 200 iterations)."""
    import torch

    from paper_2412_20322_b200 import api
    from paper_2412_20322_b200 import native as N
    from paper_2412_20322_b200.inputs import build_config
    from paper_2412_20322_b200.inputs.cf import observation_mask

    def timed(fn, reps=reps):
        fn()
        torch.cuda.synchronize()
        ms = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return sum(ms) / len(ms)

    g6 = build_config(6, n=grid.traces[0].n)
    dg6 = api.DeviceGrid(g6, dg.device)
    stats6, _ = api.eval_grid(dg6)
    sav_ms = timed(lambda: api.savings_surface(dg6, stats6))
    # the §5 view (Eq. 5): carbon savings 1 - ratio of each Case-2 family against
    # Standalone over the (rate, CI, T_A, T_B) surface -- the paper's headline is
    # 31.3-40.6% (measured on GCP; context, not a target)
    sv = api.savings_numpy(api.savings_surface(dg6, stats6))
    pairs6 = api_pairs(g6)
    fam = {}
    for i, (d, _) in enumerate(pairs6):
        lab = g6.chains[d].label
        key = " ".join(lab.split(" ")[:3]) if g6.chains[d].mode < 2 else " ".join(lab.split(" ")[:2])
        fam.setdefault(key, []).append(1.0 - sv["ratio"][i])
    savings_summary = {k: {"max_pct": round(100 * float(np.max(v)), 1),
                           "median_pct": round(100 * float(np.median(v)), 1),
                           "cells_saving_pct": round(100 * float(np.mean(np.concatenate(v) > 0)), 1)}
                       for k, v in fam.items()}
    # NEXT #1: the whole config-6 step (cfg 4 + the Standalone and SpecDecode columns)
    N.profile_enable(True)
    N.kernel_times()
    cfg6_ms = timed(lambda: (api.eval_grid(dg6), api.argmin_feasible(dg6, stats6)))
    kt6 = {}
    for name, t in N.kernel_times():
        kt6.setdefault(name, []).append(t)
    N.profile_enable(False)
    # the paper's headline view: Alg. 1's choice per workload row vs the
    # Standalone column, over config 6's 8,192 rows (rate x CI x lifetimes)
    c6, ch6, fb6 = api.argmin_feasible(dg6, stats6)
    c6, ch6, fb6 = c6.cpu().numpy(), ch6.cpu().numpy(), fb6.cpu().numpy()
    sa_col = g6.col_labels.index("Standalone A100")
    picked = c6[np.arange(g6.rows), ch6]
    red = 1.0 - picked / c6[:, sa_col]
    feas = fb6 == 0
    chosen = {g6.col_labels[c]: int(np.sum(ch6 == c)) for c in np.unique(ch6)}
    alg1_summary = {"rows": int(g6.rows), "rows_feasible": int(feas.sum()),
                    "carbon_reduction_vs_standalone_pct": {
                        "median": round(100 * float(np.median(red[feas])), 1) if feas.any() else None,
                        "max": round(100 * float(np.max(red[feas])), 1) if feas.any() else None},
                    "chosen_columns": chosen}
    stats, _ = api.eval_grid(dg)
    carbon, _, _ = api.argmin_feasible(dg, stats)
    st = api.stats_numpy(stats)
    att = torch.from_numpy((st["slo_ok"] / st["n"])[grid.cell_chain]
                           .reshape(grid.rows, grid.cols)).to(dg.device)
    m = torch.from_numpy(observation_mask(grid.rows, grid.cols, 0.3, seed=42)).to(dg.device)
    x, mm = torch.stack([carbon, att]), torch.stack([m, m])
    cf_ms = timed(lambda: api.complete_matrices(x, mm, 2, 0.1, 200, lo=0.0))
    # the other BASELINE configurations, one device-timed step each (inputs resident)
    others = {}
    for k in (1, 2, 3, 5, 7):
        gk = build_config(k)
        dk = api.DeviceGrid(gk, dg.device)
        sk, _ = api.eval_grid(dk)
        N.profile_enable(True)
        N.kernel_times()
        ms_k = timed(lambda: api.argmin_feasible(dk, api.eval_grid(dk, stats=sk)[0]), reps=2)
        ktk = {}
        for name, t in N.kernel_times():
            ktk.setdefault(name, []).append(t)
        N.profile_enable(False)
        others[f"cfg{k}"] = {"ms": ms_k, "timing_chains": len(gk.chains),
                             "requests_per_trace": gk.traces[0].n, "grid": [gk.rows, gk.cols],
                             "kernel_ms": {n: sum(v) / len(v) for n, v in ktk.items()}}
        del dk, sk
    return {"other_configs": others,
            "cfg6_step": {"ms": cfg6_ms, "timing_chains": len(g6.chains),
                          "grid": [g6.rows, g6.cols],
                          "kernel_ms": {k: sum(v) / len(v) for k, v in kt6.items()},
                          "workload": "cfg6: cfg4 + Standalone and SpecDecode (A100) columns, "
                                      "8,192 x 10 cells, 80 timing chains",
                          "alg1_vs_standalone": alg1_summary},
            "savings_surface": {"ms": sav_ms, "cells": len(api_pairs(g6)) * len(g6.scenarios),
                                "workload": "cfg6: 72 (Case 2, Standalone) pairs x 1,024 (CI, T_A, T_B)",
                                "savings_vs_standalone": savings_summary},
            "complete_matrices": {"ms": cf_ms, "matrices": 2, "shape": [grid.rows, grid.cols],
                                  "rank": 2, "iters": 200, "hidden": 0.3}}


def api_pairs(g):
    from paper_2412_20322_b200.inputs import savings_pairs
    return savings_pairs(g)


def e2e_distributed(args, dg, grid, bounds, lo, hi, local_stats, gathered, flush, dev):
    """N > 1, end to end per rank: pinned host -> device copies of its shard's traces
    (each distinct host array once), gl_eval_grid ON THOSE COPIES, the NCCL
    all_gather of the 80-B records, gl_argmin_feasible on every row, and the
    device -> host read of the choices; CUDA events on the launching stream, max
    over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2412_20322_b200 import api
    from paper_2412_20322_b200.dist import all_gather_stats
    host = dg.pinned_traces()
    needed = sorted({grid.chains[c].trace_idx for c in range(lo, hi)})
    dev_of = {}  # one device buffer per distinct host array
    for t in needed:
        for x in host[t]:
            if x.data_ptr() not in dev_of:
                dev_of[x.data_ptr()] = (x, torch.empty_like(x, device=dev))
    # the shard's traces point at the copies; traces outside the shard are never read
    traces = [tuple(dev_of[x.data_ptr()][1] for x in host[t]) if t in needed
              else dg.trace_tensors[t] for t in range(len(grid.traces))]
    stream = torch.cuda.current_stream()
    h2d = sum(h.numel() * h.element_size() for h, _ in dev_of.values())
    times, d2h = [], 0
    c_h = torch.empty(grid.rows, dtype=torch.int32, pin_memory=True)
    f_h = torch.empty(grid.rows, dtype=torch.uint8, pin_memory=True)
    for i in range(args.warmup + max(3, args.steps // 2)):
        flush.fill_(i & 0xFF)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for h, d in dev_of.values():
            d.copy_(h, non_blocking=True)
        if hi > lo:
            api.eval_grid(dg, lo, hi, stats=local_stats[: hi - lo], traces=traces)
        full = all_gather_stats(local_stats, gathered, bounds, dg.n_chains)
        _, choice, fb = api.argmin_feasible(dg, full, want_carbon=False)
        c_h.copy_(choice, non_blocking=True)
        f_h.copy_(fb, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        d2h = c_h.numel() * 4 + f_h.numel()
        if i >= args.warmup:
            times.append(e0.elapsed_time(e1))
    t = torch.tensor([sum(times) / len(times)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": grid.grid_points * grid.traces[0].n / (ms / 1e3), "unit": UNIT,
            "ms_per_step": ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": "per rank: pinned H2D of its shard's traces, gl_eval_grid on the copies, "
                    "NCCL all_gather, gl_argmin_feasible, D2H of choices (max over ranks)"}


def main():
    args = parse()
    if args.warmup < 3:
        args.warmup = 3
    if args.n is None:
        args.n = DEFAULT_N[args.config]
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
