"""Public Python API: resident device grids, gl_eval_grid / gl_argmin_feasible /
gl_evaluate_host through the C ABI.  PyTorch provides device memory and
streams only; every step of the path runs in libgreenllm.so's kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import native as N
from . import schedule as S
from .inputs.grids import GridSpec


def _dev_tensor(x: np.ndarray, device) -> torch.Tensor:
    x = np.ascontiguousarray(x)
    if x.dtype == np.uint32:
        x = x.view(np.int32)  # same bits; the kernels read uint32
    return torch.from_numpy(x).to(device)


def _pinned(x: np.ndarray) -> torch.Tensor:
    x = np.ascontiguousarray(x)
    if x.dtype == np.uint32:
        x = x.view(np.int32)
    return torch.from_numpy(x).pin_memory()


class DeviceGrid:
    """A GridSpec resident in device memory: traces (SoA) and integer tables,
    plus the host descriptor arrays the C ABI consumes."""

    def __init__(self, grid: GridSpec, device="cuda", chain_ids=None):
        self.grid = grid
        self.device = torch.device(device)
        self._keep = []
        arr_cache = self._dev_cache = {}  # device tensors must outlive every ABI call

        def up(x):
            k = id(x)
            if k not in arr_cache:
                arr_cache[k] = _dev_tensor(x, self.device)
                self._keep.append(x)  # keep id() stable
            return arr_cache[k]

        self.trace_tensors = []
        self.gl_traces = []
        for tr in grid.traces:
            a, p, o = up(tr.arrival_us), up(tr.prompt_len), up(tr.output_len)
            self.trace_tensors.append((a, p, o))
            self.gl_traces.append(N.GlTrace(a.data_ptr(), p.data_ptr(), o.data_ptr(), tr.n))
        self.gl_chains = []
        for ch in grid.chains:
            t = ch.tables
            tabs = [up(getattr(t, f)) for f in ("t1_us", "e1_new_uj", "t2_us", "b2_old_us",
                                                 "e2_old_uj", "step_us", "step_busy_new_us",
                                                 "step_busy_old_us", "step_e_new_uj",
                                                 "step_e_old_uj")]
            self.gl_chains.append(N.GlChain(
                ch.mode, ch.trace_idx, ch.cap, ch.gamma if ch.mode in (N.GL_MODE_DSD, N.GL_MODE_SPEC_COLO) else 0,
                t.max_prompt, int(ch.capacity_ok), float(ch.alpha), int(ch.seed) & (2**64 - 1),
                *[x.data_ptr() for x in tabs], int(ch.ttft_slo_us), int(ch.tpot_slo_us),
                float(ch.ce_new_g), float(ch.ce_old_g)))
        self.n_chains = len(self.gl_chains)
        self._arr_cache = {}  # ctypes descriptor arrays, built once per (kind, lo, hi)
        self.chain_n = np.array([grid.traces[c.trace_idx].n for c in grid.chains], np.int64)
        self.last_launches = 0
        self._sched = {}

    def first_range(self, lo: int = 0, hi: int | None = None):
        """The launch-order hint for chains [lo, hi) (schedule.first_range), cached."""
        hi = self.n_chains if hi is None else hi
        if (lo, hi) not in self._sched:
            self._sched[(lo, hi)] = S.first_range(self.grid, lo, hi)
        return self._sched[(lo, hi)]

    def chain_arr(self, lo: int = 0, hi: int | None = None):
        """gl_chain[lo:hi] as a cached ctypes array (the descriptors never change)."""
        hi = self.n_chains if hi is None else hi
        key = ("c", lo, hi)
        if key not in self._arr_cache:
            items = self.gl_chains[lo:hi]
            self._arr_cache[key] = (N.GlChain * len(items))(*items)
        return self._arr_cache[key]

    def trace_arr(self):
        if "t" not in self._arr_cache:
            self._arr_cache["t"] = (N.GlTrace * len(self.gl_traces))(*self.gl_traces)
        return self._arr_cache["t"]

    # ------------------------------------------------------------ host copies
    def pinned_traces(self):
        """Pinned host copies of the traces (inputs of the end-to-end path)."""
        out = []
        cache = {}
        for tr in self.grid.traces:
            arrs = []
            for x in (tr.arrival_us, tr.prompt_len, tr.output_len):
                if id(x) not in cache:
                    cache[id(x)] = _pinned(x)
                arrs.append(cache[id(x)])
            out.append(tuple(arrs))
        return out


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def eval_grid(dg: DeviceGrid, chain_lo: int = 0, chain_hi: int | None = None, stats=None,
              per_request: bool = False, stream=None, traces=None, schedule=False):
    """Simulate chains [chain_lo, chain_hi) -> (stats uint8 tensor [k, 80], per-request
    int64 tensor [sum n, 2] or None).  ``stats`` may be a preallocated view.
    ``traces`` = [(arrival, prompt, output) device tensors] per trace replaces the
    grid's resident copies (e.g. buffers just copied from the host).  ``schedule``:
    False = no launch-order hint (the default: measured no faster, see schedule.py),
    True = the predicted hint (schedule.first_range), or an explicit (first_lo,
    first_hi) relative to chain_lo; results never depend on it."""
    hi = dg.n_chains if chain_hi is None else chain_hi
    chains = dg.chain_arr(chain_lo, hi)
    k = len(chains)
    if stats is None:
        stats = torch.empty((k, N.STATS_DTYPE.itemsize), dtype=torch.uint8, device=dg.device)
    pr = None
    if per_request:
        tot = int(dg.chain_n[chain_lo:hi].sum())
        pr = torch.empty((tot, 2), dtype=torch.int64, device=dg.device)
    if traces is None:
        tr = dg.trace_arr()
    else:
        assert len(traces) == len(dg.gl_traces)
        for (a, p, o), g in zip(traces, dg.gl_traces):
            assert a.numel() == g.n and p.numel() == g.n and o.numel() == g.n
            assert a.is_cuda and p.is_cuda and o.is_cuda
        tr = [N.GlTrace(a.data_ptr(), p.data_ptr(), o.data_ptr(), a.numel())
              for (a, p, o) in traces]
    sched = dg.first_range(chain_lo, hi) if schedule is True else (schedule or None)
    dg.last_launches = N.eval_grid(tr, chains, stats.data_ptr(),
                                   pr.data_ptr() if pr is not None else None, _stream_ptr(stream),
                                   sched=sched)
    return stats, pr


def link_demand(dg: DeviceGrid, window_us: int = 1_000_000, chain_lo: int = 0,
                chain_hi: int | None = None, params=None, stream=None):
    """Link bandwidth demand of chains [chain_lo, chain_hi) (gl_link_demand; NEXT #2)
    -> (stats uint8 tensor [k, 80], link uint8 tensor [k, 32]).  ``params`` =
    [(bytes_per_token, bytes_per_member_step)] per chain, default the chain tables'."""
    hi = dg.n_chains if chain_hi is None else chain_hi
    chains = dg.gl_chains[chain_lo:hi]
    k = len(chains)
    if params is None:
        params = [(c.tables.link_bytes_per_token, c.tables.link_bytes_per_member_step)
                  for c in dg.grid.chains[chain_lo:hi]]
    stats = torch.empty((k, N.STATS_DTYPE.itemsize), dtype=torch.uint8, device=dg.device)
    link = torch.empty((k, N.LINK_DTYPE.itemsize), dtype=torch.uint8, device=dg.device)
    dg.last_launches = N.link_demand(dg.gl_traces, chains, params, window_us, stats.data_ptr(),
                                     link.data_ptr(), _stream_ptr(stream))
    return stats, link


def savings_surface(dg: DeviceGrid, stats: torch.Tensor, pairs=None, scenarios=None,
                    stream=None):
    """§5 analysis surfaces (gl_savings_surface; NEXT #3) over (pair, scenario):
    uint8 tensor [P, S, 40] of gl_savings records.  ``pairs`` defaults to every
    non-Standalone chain against the Standalone chain on its trace."""
    from .inputs import savings_pairs
    pairs = savings_pairs(dg.grid) if pairs is None else pairs
    scen = dg.grid.scenarios if scenarios is None else scenarios
    S = len(np.asarray(scen).reshape(-1, 3))
    out = torch.empty((len(pairs), S, N.SAVINGS_DTYPE.itemsize), dtype=torch.uint8,
                      device=dg.device)
    dg.last_launches = N.savings_surface(stats.data_ptr(), dg.gl_chains, pairs, scen,
                                         out.data_ptr(), _stream_ptr(stream))
    return out


def savings_numpy(out: torch.Tensor) -> np.ndarray:
    """Device savings tensor [P, S, 40] -> numpy structured array [P, S]."""
    x = out.detach().cpu().numpy()
    return x.reshape(x.shape[0], -1).view(N.SAVINGS_DTYPE).reshape(x.shape[0], x.shape[1])


def complete_matrices(x: torch.Tensor, observed: torch.Tensor, rank: int = 2,
                      lam: float = 0.1, iters: int = 200, v0: torch.Tensor | None = None,
                      lo: float = float("-inf"), hi: float = float("inf"), stream=None):
    """Collaborative filtering (gl_complete_matrices; NEXT #4) of a batch of
    partially observed matrices x [batch, rows, cols] (fp64, device) with mask
    ``observed`` (uint8) -> (out, U, V, status) device tensors.  ``v0`` [batch, cols,
    rank] defaults to the seeded inputs.cf.als_init draw for every matrix."""
    if x.dim() == 2:
        x, observed = x[None], observed[None]
        if v0 is not None and v0.dim() == 2:
            v0 = v0[None]
    x = x.contiguous().to(torch.float64)
    observed = observed.contiguous().to(torch.uint8)
    B, R, Cc = x.shape
    if v0 is None:
        from .inputs.cf import als_init
        v0 = torch.from_numpy(np.broadcast_to(als_init(Cc, rank), (B, Cc, rank)).copy())
    v0 = v0.to(x.device, torch.float64).contiguous()
    out = torch.empty_like(x)
    U = torch.empty((B, R, rank), dtype=torch.float64, device=x.device)
    V = torch.empty((B, Cc, rank), dtype=torch.float64, device=x.device)
    status = torch.empty(B, dtype=torch.int32, device=x.device)
    N.complete_matrices(x.data_ptr(), observed.data_ptr(), B, R, Cc, rank, lam, iters,
                        v0.data_ptr(), lo, hi, out.data_ptr(), U.data_ptr(), V.data_ptr(),
                        status.data_ptr(), _stream_ptr(stream))
    return out, U, V, status


def argmin_matrices(carbon: torch.Tensor, att: torch.Tensor, present: torch.Tensor | None = None,
                    target: float = 0.9, priority: int = 0, default_col: int = -1, stream=None):
    """Alg. 1 on explicit [rows, cols] matrices (gl_argmin_matrices), e.g. the ones
    complete_matrices filled -> (choice int32 [rows], via_fallback uint8 [rows])."""
    carbon = carbon.contiguous().to(torch.float64)
    att = att.contiguous().to(torch.float64)
    rows, cols = carbon.shape
    pr = None if present is None else present.contiguous().to(torch.uint8)
    choice = torch.empty(rows, dtype=torch.int32, device=carbon.device)
    fb = torch.empty(rows, dtype=torch.uint8, device=carbon.device)
    N.argmin_matrices(carbon.data_ptr(), att.data_ptr(), None if pr is None else pr.data_ptr(),
                      rows, cols, target, priority, default_col, choice.data_ptr(), fb.data_ptr(),
                      _stream_ptr(stream))
    return choice, fb


def link_numpy(link: torch.Tensor) -> np.ndarray:
    """Device link tensor -> numpy structured array (gl_link_stats fields)."""
    return link.detach().cpu().numpy().view(N.LINK_DTYPE).reshape(-1)


def argmin_feasible(dg: DeviceGrid, stats: torch.Tensor, want_carbon: bool = True, stream=None,
                    per_token_out: torch.Tensor | None = None):
    """Alg. 1 over the grid -> (carbon f64 [rows, cols] or None, choice int32 [rows],
    via_fallback uint8 [rows]) as device tensors.  ``per_token_out`` (f64 [rows,
    cols], device), when given, receives the carbon per token."""
    g = dg.grid
    carbon = torch.empty((g.rows, g.cols), dtype=torch.float64, device=dg.device) \
        if want_carbon else None
    choice = torch.empty(g.rows, dtype=torch.int32, device=dg.device)
    fb = torch.empty(g.rows, dtype=torch.uint8, device=dg.device)
    if per_token_out is not None:
        assert per_token_out.dtype == torch.float64 and per_token_out.is_contiguous()
        assert per_token_out.numel() == g.rows * g.cols
    dg.last_launches = N.argmin_feasible(
        stats.data_ptr(), dg.chain_arr(), g.scenarios, g.rows, g.cols, g.row_scenario,
        g.cell_chain, g.slo_num, g.slo_den, g.priority, g.default_col,
        carbon.data_ptr() if carbon is not None else None, choice.data_ptr(), fb.data_ptr(),
        _stream_ptr(stream),
        per_token_ptr=per_token_out.data_ptr() if per_token_out is not None else None)
    return carbon, choice, fb


@dataclass
class HostResult:
    stats: np.ndarray
    carbon: np.ndarray | None
    choice: np.ndarray
    via_fallback: np.ndarray
    launches: int
    h2d_bytes: int
    d2h_bytes: int
    carbon_per_token: np.ndarray | None = None


def evaluate_host(dg: DeviceGrid, host_traces, want_carbon: bool = False, stream=None,
                  out: HostResult | None = None, want_per_token: bool = False,
                  schedule=False) -> HostResult:
    """End to end through gl_evaluate_host_sched: pinned host traces in, host results
    out (``schedule`` as for eval_grid)."""
    g = dg.grid
    gl_tr = [N.GlTrace(a.data_ptr(), p.data_ptr(), o.data_ptr(), a.shape[0])
             for (a, p, o) in host_traces]
    if out is None:  # pinned host results: the device->host copies stay asynchronous
        def pinned(nbytes):
            return torch.empty(nbytes, dtype=torch.uint8, pin_memory=True).numpy()
        out = HostResult(pinned(dg.n_chains * N.STATS_DTYPE.itemsize).view(N.STATS_DTYPE),
                         pinned(g.rows * g.cols * 8).view(np.float64).reshape(g.rows, g.cols)
                         if want_carbon else None,
                         pinned(g.rows * 4).view(np.int32), pinned(g.rows), 0, 0, 0,
                         pinned(g.rows * g.cols * 8).view(np.float64).reshape(g.rows, g.cols)
                         if want_per_token else None)
    out.launches = N.evaluate_host(gl_tr, dg.chain_arr(), g.scenarios, g.rows, g.cols,
                                   g.row_scenario, g.cell_chain, g.slo_num, g.slo_den, g.priority,
                                   g.default_col, out.stats, out.carbon, out.choice,
                                   out.via_fallback, _stream_ptr(stream),
                                   per_token_out=out.carbon_per_token,
                                   sched=dg.first_range() if schedule is True else (schedule or None))
    seen = set()
    h2d = 0
    for arrs in host_traces:
        for x in arrs:
            key = (x.data_ptr(), x.numel() * x.element_size())
            if key not in seen:  # the ABI copies each distinct host array once
                seen.add(key)
                h2d += key[1]
    out.h2d_bytes = h2d
    out.d2h_bytes = out.stats.nbytes + (out.carbon.nbytes if out.carbon is not None else 0) + \
        (out.carbon_per_token.nbytes if out.carbon_per_token is not None else 0) + \
        out.choice.nbytes + out.via_fallback.nbytes
    return out


def stats_numpy(stats: torch.Tensor) -> np.ndarray:
    """Device stats tensor -> numpy structured array (gl_chain_stats fields)."""
    return stats.detach().cpu().numpy().view(N.STATS_DTYPE).reshape(-1)


def check_status(stats_np: np.ndarray):
    bad = np.nonzero(stats_np["status"])[0]
    if bad.size:
        raise N.GreenLLMError(N.GL_E_INVALID, f"device status bits {stats_np['status'][bad]} "
                                              f"on chains {bad.tolist()}")
