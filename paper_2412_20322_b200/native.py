"""ctypes binding of libgreenllm.so (include/greenllm.h) -- marshalling only.

Every step of the evaluated path runs in the CUDA kernels behind these entry
points.  There is no CPU fallback: if the shared library is missing or the
device is not sm_100 the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# GL_LIB_PATH selects another build of the same library (A/B kernel experiments,
# scripts/ab_build.py); the default is the in-tree build of __graft_entry__.build()
LIB_PATH = os.environ.get("GL_LIB_PATH") or os.path.join(HERE, "libgreenllm.so")

GL_OK, GL_E_INVALID, GL_E_DOMAIN, GL_E_LOOKUP, GL_E_CUDA, GL_E_UNSUPPORTED = 0, -1, -2, -3, -4, -5
GL_MODE_DPD, GL_MODE_DSD, GL_MODE_STANDALONE, GL_MODE_SPEC_COLO = 0, 1, 2, 3
GL_PRIORITY_SLO, GL_PRIORITY_DEFAULT = 0, 1
GL_MAX_CAP, GL_MAX_GAMMA, GL_MAX_PROMPT = 256, 16, 16384
ST_UNSORTED, ST_PROMPT_RANGE, ST_OUTPUT_ZERO, ST_OVERFLOW, ST_NEG_ARRIVAL, ST_TABLE = \
    1, 2, 4, 8, 16, 32


class GlTrace(C.Structure):
    _fields_ = [("arrival_us", C.c_void_p), ("prompt_len", C.c_void_p),
                ("output_len", C.c_void_p), ("n", C.c_int64)]


class GlChain(C.Structure):
    _fields_ = [("mode", C.c_int32), ("trace_idx", C.c_int32), ("batch_cap", C.c_int32),
                ("gamma", C.c_int32), ("max_prompt", C.c_int32), ("capacity_ok", C.c_int32),
                ("alpha", C.c_double), ("seed", C.c_uint64),
                ("t1_us", C.c_void_p), ("e1_new_uj", C.c_void_p), ("t2_us", C.c_void_p),
                ("b2_old_us", C.c_void_p), ("e2_old_uj", C.c_void_p), ("step_us", C.c_void_p),
                ("step_busy_new_us", C.c_void_p), ("step_busy_old_us", C.c_void_p),
                ("step_e_new_uj", C.c_void_p), ("step_e_old_uj", C.c_void_p),
                ("ttft_slo_us", C.c_int64), ("tpot_slo_us", C.c_int64),
                ("ce_new_g", C.c_double), ("ce_old_g", C.c_double)]


class GlScenario(C.Structure):
    _fields_ = [("ci_g_per_kwh", C.c_double), ("lt_new_s", C.c_double), ("lt_old_s", C.c_double)]


class GlGrid(C.Structure):
    _fields_ = [("rows", C.c_int32), ("cols", C.c_int32), ("row_scenario", C.c_void_p),
                ("cell_chain", C.c_void_p)]


# gl_chain_stats (80 B) as a numpy structured dtype
STATS_DTYPE = np.dtype([("n", "<i8"), ("slo_ok", "<i8"), ("tokens", "<i8"),
                        ("busy_new_us", "<i8"), ("busy_old_us", "<i8"), ("e_new_uj", "<i8"),
                        ("e_old_uj", "<i8"), ("makespan_us", "<i8"), ("req_hash", "<u8"),
                        ("status", "<u4"), ("capacity_ok", "<u4")])
assert STATS_DTYPE.itemsize == 80
# gl_link_stats (32 B)
LINK_DTYPE = np.dtype([("total_bytes", "<i8"), ("peak_bytes", "<i8"), ("peak_t_us", "<i8"),
                       ("n_impulses", "<i8")])
assert LINK_DTYPE.itemsize == 32


class GlLinkParams(C.Structure):
    _fields_ = [("bytes_per_token", C.c_int64), ("bytes_per_member_step", C.c_int64)]


# gl_savings (40 B) and gl_savings_pair
SAVINGS_DTYPE = np.dtype([("ratio", "<f8"), ("op_saved_g", "<f8"), ("emb_saved_g", "<f8"),
                          ("eq6_term", "<f8"), ("eq4_energy_less", "<i4"), ("pad", "<i4")])
assert SAVINGS_DTYPE.itemsize == 40


class GlSavingsPair(C.Structure):
    _fields_ = [("disagg_chain", C.c_int32), ("standalone_chain", C.c_int32)]


SCEN_DTYPE = np.dtype([("ci", "<f8"), ("lt_new", "<f8"), ("lt_old", "<f8")])


class GlSchedule(C.Structure):
    """Launch-order hint (greenllm.h gl_schedule): chains [first_lo, first_hi) first."""
    _fields_ = [("first_lo", C.c_int32), ("first_hi", C.c_int32)]

EXPORTS = ("gl_eval_grid", "gl_eval_grid_sched", "gl_argmin_feasible", "gl_evaluate_host",
           "gl_evaluate_host_sched", "gl_link_demand",
           "gl_savings_surface", "gl_complete_matrices", "gl_argmin_matrices", "gl_last_launch_count",
           "gl_profile_enable", "gl_kernel_times", "gl_kernel_timeline", "gl_strerror",
           "gl_version")

_lib = None


class GreenLLMError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib().gl_strerror(status).decode() if _lib is not None else str(status)
        super().__init__(f"{where}: {msg} (status {status})")
        self.status = status


def lib():
    """Load libgreenllm.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA extension missing: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        vp, i32 = C.c_void_p, C.c_int32
        L.gl_eval_grid.restype = i32
        L.gl_eval_grid.argtypes = [C.POINTER(GlTrace), i32, C.POINTER(GlChain), i32, vp, vp, vp]
        L.gl_eval_grid_sched.restype = i32
        L.gl_eval_grid_sched.argtypes = [C.POINTER(GlTrace), i32, C.POINTER(GlChain), i32, vp, vp,
                                         C.POINTER(GlSchedule), vp]
        L.gl_argmin_feasible.restype = i32
        L.gl_argmin_feasible.argtypes = [vp, i32, C.POINTER(GlChain), C.POINTER(GlScenario), i32,
                                         C.POINTER(GlGrid), i32, i32, i32, i32, vp, vp, vp, vp,
                                         vp]
        L.gl_evaluate_host.restype = i32
        L.gl_evaluate_host.argtypes = [C.POINTER(GlTrace), i32, C.POINTER(GlChain), i32,
                                       C.POINTER(GlScenario), i32, C.POINTER(GlGrid), i32, i32,
                                       i32, i32, vp, vp, vp, vp, vp, vp]
        L.gl_evaluate_host_sched.restype = i32
        L.gl_evaluate_host_sched.argtypes = [C.POINTER(GlTrace), i32, C.POINTER(GlChain), i32,
                                             C.POINTER(GlScenario), i32, C.POINTER(GlGrid), i32,
                                             i32, i32, i32, vp, vp, vp, vp, vp,
                                             C.POINTER(GlSchedule), vp]
        L.gl_link_demand.restype = i32
        L.gl_link_demand.argtypes = [C.POINTER(GlTrace), i32, C.POINTER(GlChain), i32,
                                     C.POINTER(GlLinkParams), C.c_int64, vp, vp, vp]
        L.gl_savings_surface.restype = i32
        L.gl_savings_surface.argtypes = [vp, i32, C.POINTER(GlChain), C.POINTER(GlSavingsPair),
                                         i32, C.POINTER(GlScenario), i32, vp, vp]
        L.gl_complete_matrices.restype = i32
        L.gl_complete_matrices.argtypes = [vp, vp, i32, i32, i32, i32, C.c_double, i32, vp,
                                           C.c_double, C.c_double, vp, vp, vp, vp, vp]
        L.gl_argmin_matrices.restype = i32
        L.gl_argmin_matrices.argtypes = [vp, vp, vp, i32, i32, C.c_double, i32, i32, vp, vp, vp]
        L.gl_last_launch_count.restype = i32
        L.gl_last_launch_count.argtypes = []
        L.gl_profile_enable.restype = i32
        L.gl_profile_enable.argtypes = [i32]
        L.gl_kernel_times.restype = i32
        L.gl_kernel_times.argtypes = [C.POINTER(C.c_char_p), C.POINTER(C.c_float), i32]
        L.gl_kernel_timeline.restype = i32
        L.gl_kernel_timeline.argtypes = [C.POINTER(C.c_char_p), C.POINTER(C.c_float),
                                         C.POINTER(C.c_float), i32]
        L.gl_strerror.restype = C.c_char_p
        L.gl_strerror.argtypes = [i32]
        L.gl_version.restype = i32
        L.gl_version.argtypes = []
        _lib = L
    return _lib


def check(status: int, where: str):
    if status != GL_OK:
        raise GreenLLMError(status, where)


def _arr(kind, items):
    """ctypes array of `kind` from a list (or a prebuilt array, passed through)."""
    return items if isinstance(items, C.Array) else (kind * len(items))(*items)


def _scen_arr(scen):
    """[S, 3] float64 scenarios viewed in place as gl_scenario[S] (same layout)."""
    s = np.ascontiguousarray(scen, dtype=np.float64).reshape(-1, 3)
    return s, s.ctypes.data_as(C.POINTER(GlScenario))


def eval_grid(traces, chains, stats_ptr: int, per_request_ptr: int | None, stream: int,
              sched=None):
    """sched: (first_lo, first_hi) launch-order hint (gl_eval_grid_sched) or None."""
    t_arr = _arr(GlTrace, traces)
    c_arr = _arr(GlChain, chains)
    if sched is None:
        check(lib().gl_eval_grid(t_arr, len(traces), c_arr, len(chains), stats_ptr,
                                 per_request_ptr or None, stream or None), "gl_eval_grid")
    else:
        sc = GlSchedule(int(sched[0]), int(sched[1]))
        check(lib().gl_eval_grid_sched(t_arr, len(traces), c_arr, len(chains), stats_ptr,
                                       per_request_ptr or None, C.byref(sc), stream or None),
              "gl_eval_grid_sched")
    return lib().gl_last_launch_count()


def link_demand(traces, chains, params, window_us: int, stats_ptr: int | None, link_ptr: int,
                stream: int):
    """params: [(bytes_per_token, bytes_per_member_step)] per chain."""
    t_arr = _arr(GlTrace, traces)
    c_arr = _arr(GlChain, chains)
    p_arr = (GlLinkParams * len(chains))(*[GlLinkParams(int(a), int(b)) for a, b in params])
    check(lib().gl_link_demand(t_arr, len(traces), c_arr, len(chains), p_arr, int(window_us),
                               stats_ptr or None, link_ptr, stream or None), "gl_link_demand")
    return lib().gl_last_launch_count()


def savings_surface(stats_ptr: int, chains, pairs, scen: np.ndarray, out_ptr: int, stream: int):
    c_arr = _arr(GlChain, chains)
    p_arr = (GlSavingsPair * len(pairs))(*[GlSavingsPair(int(d), int(s)) for d, s in pairs])
    sc, s_arr = _scen_arr(scen)
    check(lib().gl_savings_surface(stats_ptr, len(chains), c_arr, p_arr, len(pairs), s_arr,
                                   len(sc), out_ptr, stream or None), "gl_savings_surface")
    return lib().gl_last_launch_count()


def complete_matrices(x_ptr: int, obs_ptr: int, batch: int, rows: int, cols: int, rank: int,
                      lam: float, iters: int, v0_ptr: int, lo: float, hi: float, out_ptr: int,
                      u_ptr: int | None, v_ptr: int | None, status_ptr: int, stream: int):
    check(lib().gl_complete_matrices(x_ptr, obs_ptr, batch, rows, cols, rank, float(lam),
                                     int(iters), v0_ptr, float(lo), float(hi), out_ptr,
                                     u_ptr or None, v_ptr or None, status_ptr, stream or None),
          "gl_complete_matrices")
    return lib().gl_last_launch_count()


def argmin_matrices(carbon_ptr: int, att_ptr: int, present_ptr: int | None, rows: int, cols: int,
                    target: float, priority: int, default_col: int, choice_ptr: int, fb_ptr: int,
                    stream: int):
    check(lib().gl_argmin_matrices(carbon_ptr, att_ptr, present_ptr or None, rows, cols,
                                   float(target), priority, default_col, choice_ptr, fb_ptr,
                                   stream or None), "gl_argmin_matrices")
    return lib().gl_last_launch_count()


def argmin_feasible(stats_ptr: int, chains, scen: np.ndarray, rows: int, cols: int,
                    row_scenario: np.ndarray, cell_chain: np.ndarray, slo_num: int, slo_den: int,
                    priority: int, default_col: int, carbon_ptr: int | None, choice_ptr: int,
                    fb_ptr: int, stream: int, per_token_ptr: int | None = None):
    c_arr = _arr(GlChain, chains)
    s, s_arr = _scen_arr(scen)
    rs = np.ascontiguousarray(row_scenario, dtype=np.int32)
    cc = np.ascontiguousarray(cell_chain, dtype=np.int32)
    g = GlGrid(rows, cols, rs.ctypes.data, cc.ctypes.data)
    check(lib().gl_argmin_feasible(stats_ptr, len(chains), c_arr, s_arr, len(s), C.byref(g),
                                   slo_num, slo_den, priority, default_col, carbon_ptr or None,
                                   per_token_ptr or None, choice_ptr, fb_ptr, stream or None),
          "gl_argmin_feasible")
    return lib().gl_last_launch_count()


def evaluate_host(host_traces, chains, scen, rows, cols, row_scenario, cell_chain, slo_num,
                  slo_den, priority, default_col, stats_out: np.ndarray, carbon_out,
                  choice_out: np.ndarray, fb_out: np.ndarray, stream: int,
                  per_token_out: np.ndarray | None = None, sched=None):
    t_arr = _arr(GlTrace, host_traces)
    c_arr = _arr(GlChain, chains)
    s, s_arr = _scen_arr(scen)
    rs = np.ascontiguousarray(row_scenario, dtype=np.int32)
    cc = np.ascontiguousarray(cell_chain, dtype=np.int32)
    g = GlGrid(rows, cols, rs.ctypes.data, cc.ctypes.data)
    sc = None if sched is None else GlSchedule(int(sched[0]), int(sched[1]))
    check(lib().gl_evaluate_host_sched(t_arr, len(host_traces), c_arr, len(chains), s_arr,
                                       len(s), C.byref(g), slo_num, slo_den, priority,
                                       default_col, stats_out.ctypes.data,
                                       None if carbon_out is None else carbon_out.ctypes.data,
                                       None if per_token_out is None else per_token_out.ctypes.data,
                                       choice_out.ctypes.data, fb_out.ctypes.data,
                                       None if sc is None else C.byref(sc), stream or None),
          "gl_evaluate_host_sched")
    return lib().gl_last_launch_count()


def profile_enable(on: bool):
    check(lib().gl_profile_enable(1 if on else 0), "gl_profile_enable")


def kernel_timeline(max_n: int = 256):
    """[(kernel name, start ms after the first, ms)] since the last read (synchronised)."""
    names = (C.c_char_p * max_n)()
    t0 = (C.c_float * max_n)()
    ms = (C.c_float * max_n)()
    k = lib().gl_kernel_timeline(names, t0, ms, max_n)
    return [(names[i].decode(), float(t0[i]), float(ms[i])) for i in range(k)]


def kernel_times(max_n: int = 256):
    """[(kernel name, ms)] recorded since the last read (stream must be synchronised)."""
    names = (C.c_char_p * max_n)()
    ms = (C.c_float * max_n)()
    k = lib().gl_kernel_times(names, ms, max_n)
    return [(names[i].decode(), float(ms[i])) for i in range(k)]
