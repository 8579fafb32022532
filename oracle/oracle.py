"""ctypes wrapper of the C oracle (oracle/greenllm_oracle.c).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  The product
path (paper_2412_20322_b200) never imports it and has no CPU fallback.

The wrapper only marshals numpy arrays; every step of the evaluated method
runs in the C file, which cites the passage each step follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "greenllm_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC"]
# the same source under AddressSanitizer + UndefinedBehaviorSanitizer
# (any report aborts); tests/test_oracle_sanitizers.py runs the pin suite against it
SAN_LIB = os.path.join(HERE, "liboracle_san.so")
SAN_CFLAGS = ["-O1", "-g", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-shared",
              "-fPIC", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
              "-fno-omit-frame-pointer"]

ST_UNSORTED, ST_PROMPT_RANGE, ST_OUTPUT_ZERO, ST_OVERFLOW, ST_NEG_ARRIVAL = 1, 2, 4, 8, 16
STAT_FIELDS = ("n", "slo_ok", "tokens", "busy_new_us", "busy_old_us", "e_new_uj", "e_old_uj",
               "makespan_us", "req_hash", "status", "capacity_ok")


class OrChain(C.Structure):
    _fields_ = [("mode", C.c_int32), ("cap", C.c_int32), ("gamma", C.c_int32),
                ("max_prompt", C.c_int32), ("alpha", C.c_double), ("seed", C.c_uint64),
                ("t1_us", C.c_void_p), ("e1_new_uj", C.c_void_p), ("t2_us", C.c_void_p),
                ("b2_old_us", C.c_void_p), ("e2_old_uj", C.c_void_p), ("step_us", C.c_void_p),
                ("step_busy_new_us", C.c_void_p), ("step_busy_old_us", C.c_void_p),
                ("step_e_new_uj", C.c_void_p), ("step_e_old_uj", C.c_void_p),
                ("ttft_slo_us", C.c_int64), ("tpot_slo_us", C.c_int64)]


class OrStats(C.Structure):
    _fields_ = [("n", C.c_int64), ("slo_ok", C.c_int64), ("tokens", C.c_int64),
                ("busy_new_us", C.c_int64), ("busy_old_us", C.c_int64),
                ("e_new_uj", C.c_int64), ("e_old_uj", C.c_int64), ("makespan_us", C.c_int64),
                ("req_hash", C.c_uint64), ("status", C.c_uint32), ("capacity_ok", C.c_uint32)]


_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, single-threaded, no FP contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


def build_sanitized(force: bool = False) -> str:
    """Compile liboracle_san.so (ASan + UBSan; load it under LD_PRELOAD=libasan)."""
    if force or not os.path.exists(SAN_LIB) or os.path.getmtime(SAN_LIB) < os.path.getmtime(SRC):
        tmp = SAN_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *SAN_CFLAGS, "-o", tmp, SRC, "-lm"])
        os.replace(tmp, SAN_LIB)
    return SAN_LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            # GREENLLM_ORACLE_SANITIZED=1: the ASan/UBSan build (test_oracle_sanitizers)
            if os.environ.get("GREENLLM_ORACLE_SANITIZED") == "1":
                L = C.CDLL(build_sanitized())
            else:
                build()
                L = C.CDLL(LIB)
            L.oracle_simulate_chain.restype = C.c_uint32
            L.oracle_simulate_chain.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                                C.POINTER(OrChain), C.POINTER(OrStats),
                                                C.c_void_p, C.c_void_p, C.c_void_p]
            L.oracle_link_demand.restype = C.c_uint32
            L.oracle_link_demand.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                             C.POINTER(OrChain), C.c_int64, C.c_int64,
                                             C.c_int64, C.POINTER(OrStats),
                                             C.POINTER(C.c_int64)]
            L.oracle_carbon.restype = None
            L.oracle_carbon.argtypes = [C.POINTER(OrStats), C.c_double, C.c_double, C.c_double,
                                        C.c_double, C.c_double, C.POINTER(C.c_double)]
            L.oracle_carbon_per_token.restype = C.c_double
            L.oracle_carbon_per_token.argtypes = [C.POINTER(OrStats), C.c_double]
            L.oracle_savings.restype = None
            L.oracle_savings.argtypes = [C.POINTER(OrStats), C.c_double, C.c_double,
                                         C.POINTER(OrStats), C.c_double, C.c_double,
                                         C.c_double, C.c_double, C.c_double,
                                         C.POINTER(C.c_double), C.POINTER(C.c_int32)]
            L.oracle_als_complete.restype = C.c_int32
            L.oracle_als_complete.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                              C.c_int32, C.c_double, C.c_int32, C.c_void_p,
                                              C.c_double, C.c_double, C.c_void_p, C.c_void_p,
                                              C.c_void_p]
            L.oracle_alg1_matrices.restype = None
            L.oracle_alg1_matrices.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                               C.c_void_p, C.c_double, C.c_int32, C.c_int32,
                                               C.c_void_p, C.c_void_p]
            L.oracle_alg1.restype = None
            L.oracle_alg1.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_void_p, C.c_void_p]
            L.oracle_philox4x32_10.restype = None
            L.oracle_philox4x32_10.argtypes = [C.POINTER(C.c_uint32), C.c_uint32, C.c_uint32,
                                               C.POINTER(C.c_uint32)]
            L.oracle_thresholds.restype = None
            L.oracle_thresholds.argtypes = [C.c_double, C.c_int32, C.POINTER(C.c_uint64)]
            L.oracle_accept_count.restype = C.c_int32
            L.oracle_accept_count.argtypes = [C.c_uint32, C.POINTER(C.c_uint64), C.c_int32]
            L.oracle_mix64.restype = C.c_uint64
            L.oracle_mix64.argtypes = [C.c_uint64, C.c_int64, C.c_int64]
            _lib = L
    return _lib


def _ptr(x: np.ndarray):
    return x.ctypes.data_as(C.c_void_p)


def _c(x, dtype):
    return np.ascontiguousarray(x, dtype=dtype)


def make_chain(ch) -> tuple:
    """OrChain from an inputs.ChainSpec (returns the struct and the arrays it
    points into, which must stay alive)."""
    t = ch.tables
    arrs = dict(t1_us=_c(t.t1_us, np.int32), e1_new_uj=_c(t.e1_new_uj, np.int64),
                t2_us=_c(t.t2_us, np.int32), b2_old_us=_c(t.b2_old_us, np.int32),
                e2_old_uj=_c(t.e2_old_uj, np.int64), step_us=_c(t.step_us, np.int32),
                step_busy_new_us=_c(t.step_busy_new_us, np.int32),
                step_busy_old_us=_c(t.step_busy_old_us, np.int32),
                step_e_new_uj=_c(t.step_e_new_uj, np.int64),
                step_e_old_uj=_c(t.step_e_old_uj, np.int64))
    if arrs["step_us"].shape[0] < ch.cap + 1:
        raise ValueError("step tables shorter than batch_cap + 1")
    s = OrChain(ch.mode, ch.cap, ch.gamma, t.t1_us.shape[0] - 1, ch.alpha, ch.seed,
                *[_ptr(arrs[k]) for k in ("t1_us", "e1_new_uj", "t2_us", "b2_old_us",
                                           "e2_old_uj", "step_us", "step_busy_new_us",
                                           "step_busy_old_us", "step_e_new_uj",
                                           "step_e_old_uj")],
                ch.ttft_slo_us, ch.tpot_slo_us)
    return s, arrs


def simulate_chain(trace, ch, per_request: bool = True, ready: bool = False):
    """Return (stats dict, ttft[n], finish[n]) for one timing chain (plus the
    stage-2 completion times r[n] when ``ready``)."""
    L = lib()
    a = _c(trace.arrival_us, np.int64)
    p = _c(trace.prompt_len, np.uint32)
    o = _c(trace.output_len, np.uint32)
    n = a.shape[0]
    s, keep = make_chain(ch)
    st = OrStats()
    ttft = np.zeros(n, np.int64) if per_request else None
    fin = np.zeros(n, np.int64) if per_request else None
    r = np.zeros(n, np.int64) if ready else None
    L.oracle_simulate_chain(_ptr(a), _ptr(p), _ptr(o), n, C.byref(s), C.byref(st),
                            _ptr(ttft) if per_request else None,
                            _ptr(fin) if per_request else None,
                            _ptr(r) if ready else None)
    d = {f: getattr(st, f) for f in STAT_FIELDS}
    d["capacity_ok"] = int(ch.capacity_ok)
    del keep
    if ready:
        return d, ttft, fin, r
    return d, ttft, fin


LINK_FIELDS = ("total_bytes", "peak_bytes", "peak_t_us", "n_impulses")


def link_demand(trace, ch, window_us: int = 1_000_000, bytes_per_token=None,
                bytes_per_member_step=None):
    """Peak link bandwidth demand of one chain (oracle_link_demand): dict with
    total_bytes, peak_bytes (max bytes issued in any [t, t + window_us)),
    peak_t_us (earliest impulse time attaining it, -1 if none), n_impulses, and
    the chain's stats under "stats".  Payload sizes default to the chain tables'."""
    L = lib()
    a = _c(trace.arrival_us, np.int64)
    p = _c(trace.prompt_len, np.uint32)
    o = _c(trace.output_len, np.uint32)
    s, keep = make_chain(ch)
    bpt = ch.tables.link_bytes_per_token if bytes_per_token is None else bytes_per_token
    pm = ch.tables.link_bytes_per_member_step if bytes_per_member_step is None \
        else bytes_per_member_step
    st = OrStats()
    out = (C.c_int64 * 4)()
    status = L.oracle_link_demand(_ptr(a), _ptr(p), _ptr(o), a.shape[0], C.byref(s), int(bpt),
                                  int(pm), int(window_us), C.byref(st), out)
    del keep
    d = {f: int(out[i]) for i, f in enumerate(LINK_FIELDS)}
    d["stats"] = {f: getattr(st, f) for f in STAT_FIELDS}
    d["status"] = int(status)
    return d


def _stats_struct(d) -> OrStats:
    return OrStats(*[int(d[f]) for f in STAT_FIELDS])


def carbon(stats: dict, ce_new_g: float, ce_old_g: float, ci: float, lt_new_s: float,
           lt_old_s: float):
    """(operational, embodied, total) grams -- Eqs. 1-3."""
    out = (C.c_double * 3)()
    lib().oracle_carbon(C.byref(_stats_struct(stats)), ce_new_g, ce_old_g, ci, lt_new_s,
                        lt_old_s, out)
    return out[0], out[1], out[2]


def carbon_per_token(stats: dict, total: float) -> float:
    """gCO2 per generated token (R33): total / tokens."""
    return lib().oracle_carbon_per_token(C.byref(_stats_struct(stats)), float(total))


def savings(stats_d: dict, ce_d, stats_s: dict, ce_s, ci: float, lt_new_s: float,
            lt_old_s: float):
    """§5 analysis for one (disaggregated d, Standalone s) pair and scenario:
    dict(ratio, op_saved_g, emb_saved_g, eq6_term, eq4).  ce_d / ce_s = (ce_new, ce_old)."""
    out = (C.c_double * 4)()
    eq4 = C.c_int32()
    lib().oracle_savings(C.byref(_stats_struct(stats_d)), ce_d[0], ce_d[1],
                         C.byref(_stats_struct(stats_s)), ce_s[0], ce_s[1], ci, lt_new_s,
                         lt_old_s, out, C.byref(eq4))
    return dict(ratio=out[0], op_saved_g=out[1], emb_saved_g=out[2], eq6_term=out[3],
                eq4=int(eq4.value))


def savings_surface(grid, pairs, stats=None):
    """Oracle surfaces over (pair, scenario): arrays [P, S] of ratio, op_saved_g,
    emb_saved_g, eq6_term (f64) and eq4 (int32).  ``stats`` = {chain: stats dict}
    (simulated here when absent)."""
    need = sorted({c for pr in pairs for c in pr})
    if stats is None:
        stats = {}
    for ci in need:
        if ci not in stats:
            ch = grid.chains[ci]
            stats[ci] = simulate_chain(grid.traces[ch.trace_idx], ch, per_request=False)[0]
    P, S = len(pairs), len(grid.scenarios)
    out = {k: np.zeros((P, S)) for k in ("ratio", "op_saved_g", "emb_saved_g", "eq6_term")}
    out["eq4"] = np.zeros((P, S), np.int32)
    for i, (d, s) in enumerate(pairs):
        cd, cs = grid.chains[d], grid.chains[s]
        for j, sc in enumerate(grid.scenarios):
            r = savings(stats[d], (cd.ce_new_g, cd.ce_old_g), stats[s], (cs.ce_new_g, cs.ce_old_g),
                        float(sc[0]), float(sc[1]), float(sc[2]))
            for k in out:
                out[k][i, j] = r[k]
    return out


def als_complete(x, observed, rank, lam, iters, v0, lo=-np.inf, hi=np.inf):
    """Collaborative filtering by ALS (oracle_als_complete): returns
    (completed [rows, cols], U [rows, rank], V [cols, rank], status)."""
    x = _c(x, np.float64)
    rows, cols = x.shape
    m = _c(observed, np.uint8)
    v = _c(v0, np.float64).reshape(cols, rank)
    out = np.zeros_like(x)
    U = np.zeros((rows, rank))
    V = np.zeros((cols, rank))
    st = lib().oracle_als_complete(_ptr(x), _ptr(m), rows, cols, rank, float(lam), int(iters),
                                   _ptr(v), float(lo), float(hi), _ptr(out), _ptr(U), _ptr(V))
    return out, U, V, int(st)


def alg1_matrices(carbon, att, present=None, target=0.9, priority=0, default_col=-1):
    """Alg. 1 on explicit [rows, cols] matrices with fractional attainment
    (oracle_alg1_matrices) -> (choice int32[rows], via_fallback uint8[rows])."""
    carbon = _c(carbon, np.float64)
    att = _c(att, np.float64)
    rows, cols = carbon.shape
    pr = None if present is None else _c(present, np.uint8)
    choice = np.zeros(rows, np.int32)
    fb = np.zeros(rows, np.uint8)
    lib().oracle_alg1_matrices(rows, cols, _ptr(carbon), _ptr(att),
                               None if pr is None else _ptr(pr), float(target), priority,
                               default_col, _ptr(choice), _ptr(fb))
    return choice, fb


def alg1(total, ok, n, present, cap_ok, slo_num=9, slo_den=10, priority=0, default_col=-1):
    """Alg. 1 on [rows, cols] matrices -> (choice int32[rows], via_fallback uint8[rows])."""
    total = _c(total, np.float64)
    rows, cols = total.shape
    ok = _c(ok, np.int64)
    n = _c(n, np.int64)
    present = _c(present, np.uint8)
    cap_ok = _c(cap_ok, np.uint8)
    choice = np.zeros(rows, np.int32)
    fb = np.zeros(rows, np.uint8)
    lib().oracle_alg1(rows, cols, _ptr(present), _ptr(total), _ptr(ok), _ptr(n), _ptr(cap_ok),
                      slo_num, slo_den, priority, default_col, _ptr(choice), _ptr(fb))
    return choice, fb


def philox(ctr, k0, k1):
    c = (C.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    out = (C.c_uint32 * 4)()
    lib().oracle_philox4x32_10(c, int(k0) & 0xFFFFFFFF, int(k1) & 0xFFFFFFFF, out)
    return tuple(out)


def thresholds(alpha: float, gamma: int):
    out = (C.c_uint64 * max(gamma, 1))()
    lib().oracle_thresholds(alpha, gamma, out)
    return [out[i] for i in range(gamma)]


def accept_count(u: int, thr, gamma: int) -> int:
    arr = (C.c_uint64 * max(gamma, 1))(*thr)
    return lib().oracle_accept_count(u, arr, gamma)


def mix64(j: int, ttft: int, finish: int) -> int:
    return lib().oracle_mix64(j, ttft, finish)


def evaluate_grid(grid, chain_ids=None, per_request=False):
    """Oracle for a whole GridSpec: per-chain stats, carbon [rows, cols] (g),
    Alg. 1 choice / via_fallback.  ``chain_ids`` restricts the simulated chains
    (the others must then be absent from the grid)."""
    ids = range(len(grid.chains)) if chain_ids is None else chain_ids
    stats = {}
    per = {}
    for ci in ids:
        ch = grid.chains[ci]
        st, ttft, fin = simulate_chain(grid.traces[ch.trace_idx], ch, per_request)
        stats[ci] = st
        if per_request:
            per[ci] = (ttft, fin)
    out = grid_epilogue(grid, stats)
    out["per_request"] = per
    return out


def grid_epilogue(grid, stats):
    """Carbon (Eqs. 1-3) per present cell and Alg. 1 per row from per-chain oracle
    statistics ``stats`` = {chain: stats dict}; cells of chains not in ``stats``
    are treated as absent."""
    rows, cols = grid.rows, grid.cols
    total = np.zeros((rows, cols))
    per_token = np.zeros((rows, cols))
    ok = np.zeros((rows, cols), np.int64)
    n = np.ones((rows, cols), np.int64)
    present = np.zeros((rows, cols), np.uint8)
    cap = np.zeros((rows, cols), np.uint8)
    cells = grid.cell_chain.reshape(rows, cols)
    for r in range(rows):
        sc = grid.scenarios[grid.row_scenario[r]]
        for c in range(cols):
            k = int(cells[r, c])
            if k < 0 or k not in stats:
                continue
            ch = grid.chains[k]
            st = stats[k]
            total[r, c] = carbon(st, ch.ce_new_g, ch.ce_old_g, sc[0], sc[1], sc[2])[2]
            per_token[r, c] = carbon_per_token(st, total[r, c])
            ok[r, c], n[r, c] = st["slo_ok"], st["n"]
            present[r, c] = 1
            # R55: a chain with invalid input (status bits) is never feasible; like a
            # capacity-infeasible one it counts as ok = 0, total = +inf in the fallback
            cap[r, c] = 1 if (ch.capacity_ok and st["status"] == 0) else 0
    choice, fb = alg1(total, ok, n, present, cap, grid.slo_num, grid.slo_den, grid.priority,
                      grid.default_col)
    return dict(stats=stats, carbon=total, carbon_per_token=per_token, choice=choice,
                via_fallback=fb, present=present)
