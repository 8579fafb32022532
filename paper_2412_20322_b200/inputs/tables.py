"""Integer latency / energy tables: the stand-in for the paper's profiling database.

The paper's scheduler consumes a *profiled* database D (§4.2;
Alg. 1 input).  There are no profiles here, so -- like SPEC's
hardware_model -- a roofline surrogate produces them once on the
host.  These tables are INPUTS of the evaluated method (they replace D); both
the CUDA path and the oracle read the same integer arrays.  Parity therefore
does not depend on anything in this file; the tables' realism is only
trend-checked against Figs. 2-3 ("parity unpinned" w.r.t. the paper's
measurements).

Surrogate (SURVEY.md §8(d) "Tables"):
    compute_s = 2 * params * tokens / (fp16_tflops * 1e12 * eta_c)
    memory_s  = (params * bytes_per_param + kv_read_bytes) / (bw_gbs * 1e9 * eta_m)
    latency_s = max(compute_s, memory_s)
    util      = compute_s / latency_s
    power_w   = idle + util * (max_power - idle),  idle = 15% of max power
    energy_j  = latency_s * power_w
Latencies are rounded UP to integer microseconds and energies half-up to
integer microjoules (R2).  Link transfers cost base_us + ceil(bits*1e6/bw_bps)
microseconds (R2) and no GPU time or energy (assumption A.2).
KV bytes/token = 2 * layers * kv_heads * head_dim * 2 (R39, GQA-aware).
"""
from __future__ import annotations

from dataclasses import dataclass

import functools

import numpy as np

ETA_C = 0.6
ETA_M = 0.8
IDLE_FRAC = 0.15
BYTES_PER_PARAM = 2
BYTES_PER_PROB = 2
VOCAB = 32000
GIB = 1 << 30
# Decode / verify steps also stream each member's KV cache; the surrogate uses a
# nominal resident context of KV_CTX tokens per member so that step latency
# grows with the batch size b (ours; S:121 has the weights term only).
KV_CTX = 256


@dataclass(frozen=True)
class GpuSpec:
    name: str
    vram_gb: float
    bw_gbs: float
    area_mm2: float
    max_power_w: float
    node_nm: int
    fp16_tflops: float
    year: int
    embodied_kg: float

    @property
    def idle_w(self) -> float:
        return IDLE_FRAC * self.max_power_w

    @property
    def embodied_g(self) -> float:
        return self.embodied_kg * 1000.0


# Table 1, printed values as-is (SURVEY G4 notes the mixed
# FP16 bases; kept verbatim).
GPUS = {
    "T4": GpuSpec("T4", 16, 320, 545, 70, 12, 65.0, 2018, 10.3),
    "V100": GpuSpec("V100", 16, 900, 815, 300, 12, 28.26, 2017, 20.0),
    "A100": GpuSpec("A100", 40, 1555, 826, 400, 7, 312.0, 2020, 26.34),
}


@dataclass(frozen=True)
class ModelSpec:
    name: str
    params: float
    layers: int
    kv_heads: int
    head_dim: int

    @property
    def kv_bytes_per_token(self) -> int:
        return 2 * self.layers * self.kv_heads * self.head_dim * BYTES_PER_PARAM

    @property
    def weight_bytes(self) -> float:
        return self.params * BYTES_PER_PARAM


MODELS = {
    "7B": ModelSpec("Llama-7B", 7e9, 32, 32, 128),
    "13B": ModelSpec("Llama-13B", 13e9, 40, 40, 128),
    "70B": ModelSpec("Llama-70B", 70e9, 80, 8, 128),
    "1B": ModelSpec("Llama-1B", 1.1e9, 22, 4, 64),
    "300M": ModelSpec("Llama-300M", 3e8, 16, 16, 64),
    "68M": ModelSpec("Llama-68M", 6.8e7, 2, 12, 64),
}


def ceil_us(seconds) -> np.ndarray:
    return np.ceil(np.asarray(seconds, dtype=np.float64) * 1e6).astype(np.int64)


def round_uj(joules) -> np.ndarray:
    return np.floor(np.asarray(joules, dtype=np.float64) * 1e6 + 0.5).astype(np.int64)


def roofline(gpu: GpuSpec, model: ModelSpec, tokens, kv_read_tokens=0):
    """(latency_s, energy_j) of one forward pass processing ``tokens`` tokens
    that also reads ``kv_read_tokens`` tokens of KV cache."""
    tokens = np.asarray(tokens, dtype=np.float64)
    kv = np.asarray(kv_read_tokens, dtype=np.float64) * model.kv_bytes_per_token
    compute = 2.0 * model.params * tokens / (gpu.fp16_tflops * 1e12 * ETA_C)
    memory = (model.weight_bytes + kv) / (gpu.bw_gbs * 1e9 * ETA_M)
    lat = np.maximum(compute, memory)
    util = np.where(lat > 0, compute / np.where(lat > 0, lat, 1.0), 0.0)
    power = gpu.idle_w + util * (gpu.max_power_w - gpu.idle_w)
    return lat, lat * power


def link_us(nbytes, bw_gbps: float, base_us: int = 0) -> np.ndarray:
    """base + ceil(bits * 1e6 / bw) in exact integer arithmetic (R2)."""
    bw_bps = int(round(bw_gbps * 1e9))
    nb = np.asarray(nbytes, dtype=object)
    out = np.vectorize(lambda b: base_us + (-(-(int(b) * 8 * 1_000_000) // bw_bps)),
                       otypes=[np.int64])(nb)
    return out.astype(np.int64)


@dataclass
class ChainTables:
    """Prompt-indexed [max_prompt+1] and batch-indexed [cap+1] integer tables."""
    t1_us: np.ndarray        # int32, prefill on the new GPU
    e1_new_uj: np.ndarray    # int64
    t2_us: np.ndarray        # int32, stage-2 service (DPD: KV link; DSD: handoff + draft prefill)
    b2_old_us: np.ndarray    # int32, stage-2 busy time on the old GPU
    e2_old_uj: np.ndarray    # int64
    step_us: np.ndarray      # int32, decode iteration / DSD step latency at batch b
    step_busy_new_us: np.ndarray
    step_busy_old_us: np.ndarray
    step_e_new_uj: np.ndarray    # int64
    step_e_old_uj: np.ndarray    # int64
    label: str = ""
    # GPU-GPU link payloads (bandwidth demand, NEXT #2, R45-R47): a request's
    # stage-2 payload is link_bytes_per_token * (p + 1) bytes (DPD: its KV, R11;
    # DSD: its prompt IDs, R12); a decode iteration at batch b puts
    # b * link_bytes_per_member_step bytes on the link (DSD: draft IDs, probs and
    # accepted IDs of every member, R21).  Zero where nothing crosses the link.
    link_bytes_per_token: int = 0
    link_bytes_per_member_step: int = 0

    @property
    def max_prompt(self) -> int:
        return int(self.t1_us.shape[0]) - 1

    @property
    def cap(self) -> int:
        return int(self.step_us.shape[0]) - 1


def _i32(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.int64)
    if x.size and (x.min() < 0 or x.max() >= 2**31):
        raise OverflowError("table latency does not fit int32 microseconds")
    return x.astype(np.int32)


def dpd_tables(new: str, old: str, model: str, cap: int, bw_gbps: float = 16.0,
               max_prompt: int = 4096, base_us: int = 0) -> ChainTables:
    """Disg-Pref-Decode: prefill on the new GPU, KV of p+1
    tokens over one FIFO link, decode on the old GPU."""
    g_new, g_old, m = GPUS[new], GPUS[old], MODELS[model]
    p = np.arange(max_prompt + 1)
    lat1, en1 = roofline(g_new, m, p)
    t1 = ceil_us(lat1)
    e1 = round_uj(en1)
    t1[0] = 0
    e1[0] = 0
    t2 = link_us(m.kv_bytes_per_token * (p + 1), bw_gbps, base_us)
    t2[0] = 0
    zero_p = np.zeros(max_prompt + 1, dtype=np.int64)
    b = np.arange(cap + 1)
    latd, end = roofline(g_old, m, b, b * KV_CTX)
    step = ceil_us(latd)
    ed = round_uj(end)
    step[0] = 0
    ed[0] = 0
    zero_b = np.zeros(cap + 1, dtype=np.int64)
    return ChainTables(_i32(t1), e1, _i32(t2), _i32(zero_p), zero_p.copy(),
                       _i32(step), _i32(zero_b), _i32(step), zero_b.copy(), ed,
                       f"DPD {model} {new}->{old} {bw_gbps}Gbps cap{cap}",
                       link_bytes_per_token=m.kv_bytes_per_token, link_bytes_per_member_step=0)


def dsd_member_step_bytes(gamma: int) -> int:
    """Link bytes one member puts on the link per speculative step (R21, Fig. 7):
    gamma draft token IDs (4 B), gamma probability vectors (VOCAB fp16), and the
    gamma+1 accepted / bonus token IDs returned."""
    return 4 * gamma + gamma * VOCAB * BYTES_PER_PROB + 4 * (gamma + 1)


@functools.lru_cache(maxsize=None)
def _dsd_prompt_tables(new: str, old: str, target: str, draft: str, bw_gbps: float,
                       max_prompt: int, base_us: int):
    """DSD's prompt-indexed tables (independent of gamma and the batch cap): one set of
    arrays per (GPU pair, models, link), shared by every chain that uses them, so the
    library sees equal tables as equal pointers (stage groups).  The
    arrays are never written after this."""
    g_new, g_old = GPUS[new], GPUS[old]
    mt, md = MODELS[target], MODELS[draft]
    p = np.arange(max_prompt + 1)
    lat1, en1 = roofline(g_new, mt, p)
    t1, e1 = ceil_us(lat1), round_uj(en1)
    t1[0] = 0
    e1[0] = 0
    latdp, endp = roofline(g_old, md, p)
    b2, e2 = ceil_us(latdp), round_uj(endp)
    b2[0] = 0
    e2[0] = 0
    t2 = link_us(4 * (p + 1), bw_gbps, base_us) + b2
    t2[0] = 0
    return (_i32(t1), e1, _i32(t2), _i32(b2), e2)


def dsd_tables(new: str, old: str, target: str, draft: str, gamma: int, cap: int,
               bw_gbps: float = 16.0, max_prompt: int = 4096, base_us: int = 0) -> ChainTables:
    """Disg-Spec-Decode (Fig. 7): draft on the old GPU, target
    + verifier on the new GPU.  Stage 2 = prompt-ID handoff (4(p+1) B) + draft
    prefill on the old GPU (R12).  Step latency (R21):
        S[b] = gamma*D_old[b] + t_link(4*gamma*b) + max(V_new[b], t_link(probs))
               + t_link(4*(gamma+1)*b),   probs = gamma*VOCAB*2*b bytes,
    i.e. ID send, then verify overlapped with the async probs send,
    then the accepted-ID return."""
    g_new, g_old = GPUS[new], GPUS[old]
    mt, md = MODELS[target], MODELS[draft]
    t1, e1, t2, b2, e2 = _dsd_prompt_tables(new, old, target, draft, bw_gbps, max_prompt, base_us)
    b = np.arange(cap + 1)
    latd, end = roofline(g_old, md, b, b * KV_CTX)  # one draft pass at batch b
    d_old, e_d = ceil_us(latd), round_uj(end)
    latv, env = roofline(g_new, mt, b * (gamma + 1), b * KV_CTX)  # verify gamma+1 tokens/seq
    v_new, e_v = ceil_us(latv), round_uj(env)
    ids = link_us(4 * gamma * b, bw_gbps, base_us)
    probs = link_us(gamma * VOCAB * BYTES_PER_PROB * b, bw_gbps, base_us)
    ret = link_us(4 * (gamma + 1) * b, bw_gbps, base_us)
    step = gamma * d_old + ids + np.maximum(v_new, probs) + ret
    busy_old = gamma * d_old
    busy_new = v_new.copy()
    se_old = gamma * e_d
    se_new = e_v.copy()
    for arr in (step, busy_old, busy_new, se_old, se_new):
        arr[0] = 0
    return ChainTables(t1, e1, t2, b2, e2,
                       _i32(step), _i32(busy_new), _i32(busy_old), se_new, se_old,
                       f"DSD {target}/{draft} {new}+{old} g{gamma} {bw_gbps}Gbps cap{cap}",
                       link_bytes_per_token=4,
                       link_bytes_per_member_step=dsd_member_step_bytes(gamma))


def standalone_tables(gpu: str, model: str, cap: int, max_prompt: int = 4096) -> ChainTables:
    """Standalone: the target alone on one GPU.  Prefill t1[p] and
    decode iterations step[b] run on that GPU one at a time (R41-R43); no link,
    no old GPU (old-GPU tables zero)."""
    g, m = GPUS[gpu], MODELS[model]
    p = np.arange(max_prompt + 1)
    lat1, en1 = roofline(g, m, p)
    t1, e1 = ceil_us(lat1), round_uj(en1)
    t1[0] = 0
    e1[0] = 0
    zero_p = np.zeros(max_prompt + 1, dtype=np.int64)
    b = np.arange(cap + 1)
    latd, end = roofline(g, m, b, b * KV_CTX)
    step, ed = ceil_us(latd), round_uj(end)
    step[0] = 0
    ed[0] = 0
    zero_b = np.zeros(cap + 1, dtype=np.int64)
    return ChainTables(_i32(t1), e1, _i32(zero_p), _i32(zero_p), zero_p.copy(),
                       _i32(step), _i32(step), _i32(zero_b), ed, zero_b.copy(),
                       f"Standalone {model} {gpu} cap{cap}")


def spec_colo_tables(gpu: str, target: str, draft: str, gamma: int, cap: int,
                     max_prompt: int = 4096) -> ChainTables:
    """SpecDecode: draft and target co-located on one GPU.  The
    prefill runs both models' prompt passes back to back; a step is gamma draft
    passes then the target's verification of gamma+1 tokens per sequence, all on
    the same GPU (no transfers): S[b] = gamma*D[b] + V[b] (R43)."""
    g, mt, md = GPUS[gpu], MODELS[target], MODELS[draft]
    p = np.arange(max_prompt + 1)
    lat_t, en_t = roofline(g, mt, p)
    lat_d, en_d = roofline(g, md, p)
    t1 = ceil_us(lat_t) + ceil_us(lat_d)
    e1 = round_uj(en_t) + round_uj(en_d)
    t1[0] = 0
    e1[0] = 0
    zero_p = np.zeros(max_prompt + 1, dtype=np.int64)
    b = np.arange(cap + 1)
    latd, end = roofline(g, md, b, b * KV_CTX)
    d_pass, e_d = ceil_us(latd), round_uj(end)
    latv, env = roofline(g, mt, b * (gamma + 1), b * KV_CTX)
    v_pass, e_v = ceil_us(latv), round_uj(env)
    step = gamma * d_pass + v_pass
    se = gamma * e_d + e_v
    step[0] = 0
    se[0] = 0
    zero_b = np.zeros(cap + 1, dtype=np.int64)
    return ChainTables(_i32(t1), e1, _i32(zero_p), _i32(zero_p), zero_p.copy(),
                       _i32(step), _i32(step), _i32(zero_b), se, zero_b.copy(),
                       f"SpecDecode {target}/{draft} {gpu} g{gamma} cap{cap}")


def capacity_ok(mode: str, new: str, old: str, target: str, draft, cap: int,
                p50: tuple) -> int:
    """R38: weights + cap * (P50 in + P50 out) * kv <= VRAM.
    Capacity-infeasible chains are still simulated; only Alg. 1 excludes them."""
    g_new, mt = GPUS[new], MODELS[target]
    seq = p50[0] + p50[1]
    if mode in ("standalone", "spec_colo"):  # everything on the one GPU
        need = mt.weight_bytes + cap * seq * mt.kv_bytes_per_token
        if mode == "spec_colo":
            md = MODELS[draft]
            need += md.weight_bytes + cap * seq * md.kv_bytes_per_token
        return int(need <= g_new.vram_gb * GIB)
    g_old = GPUS[old]
    if mode == "dpd":
        ok_new = mt.weight_bytes + (p50[0] + 1) * mt.kv_bytes_per_token <= g_new.vram_gb * GIB
        ok_old = mt.weight_bytes + cap * seq * mt.kv_bytes_per_token <= g_old.vram_gb * GIB
    else:
        md = MODELS[draft]
        ok_new = mt.weight_bytes + cap * seq * mt.kv_bytes_per_token <= g_new.vram_gb * GIB
        ok_old = md.weight_bytes + cap * seq * md.kv_bytes_per_token <= g_old.vram_gb * GIB
    return int(bool(ok_new and ok_old))
