/*
 * greenllm.cu -- libgreenllm.so: the C ABI of include/greenllm.h over sm_100a kernels.
 *
 * The evaluated method (each step with the paper passage it follows):
 *   stage 1  prefill FCFS on the new GPU      c_i = max(c_{i-1}, a_i) + t1[p_i]
 *            (TTFT = c - a)
 *   stage 2  KV link (DPD) / handoff + draft prefill (DSD)
 *                                              r_i = max(r_{i-1}, c_i) + t2[p_i]
 *   decode   continuous batching on the old GPU (DPD) or speculative steps across
 *            both GPUs (DSD, Fig. 7), batch <= cap, FCFS joins at
 *            iteration boundaries (R15-R18)
 *   SLO      TTFT <= SLO_ttft and finish - c <= SLO_tpot (o - 1) (Table 2)
 *   carbon   Eqs. 1-3;   Alg. 1 feasible argmin
 *
 * Kernels, in launch order:
 *   k_dsd_demand  (k_dsd_demand.cuh) one thread per (DSD demand group, request)
 *   k_stages      (k_stages.cuh)     S 16-warp blocks per chain: TMA-staged tables,
 *                                    128-bit loads, max-plus scans with decoupled
 *                                    look-back between blocks -> decode stream
 *   k_segments    (k_stages.cuh)     idle-point candidates for the decode speculation
 *   k_decode      (k_decode.cuh)     leader + helper warps per chain: exact
 *                                    speculative decode event loops
 *   k_finalize    (k_decode.cuh)     whole GPU over (chain, request): SLO, hash
 *   k_argmin      (k_argmin.cuh)     one warp per Alg. 1 row
 * gl_link_demand (NEXT #2) runs the same simulation with a
 * k_decode<.., LOG> that records batch-size changes, then
 *   k_link_scan / k_link_window / k_link_reduce (k_link.cuh).
 * No tensor cores: nothing on this path is a contraction.
 */
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "greenllm.h"
#include "k_argmin.cuh"
#include "k_decode.cuh"
#include "k_stages.cuh"
#include "k_dsd_demand.cuh"
#include "k_link.cuh"
#include "k_savings.cuh"
#include "k_als.cuh"
#include "k_relax.cuh"

namespace {

using gl::DCarbon;
using gl::DChain;
using gl::DGroup;

thread_local int32_t g_last_launches = 0;

// benchmark instrumentation: CUDA events around each kernel (gl_profile_enable)
constexpr int PROF_MAX = 256;
struct ProfState {
    bool on = false;
    int used = 0;
    std::vector<cudaEvent_t> ev;
    const char *names[PROF_MAX];
};
thread_local ProfState g_prof;

void prof_begin(const char *name, cudaStream_t s)
{
    if (!g_prof.on || g_prof.used >= PROF_MAX) return;
    while ((int)g_prof.ev.size() < 2 * (g_prof.used + 1)) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        g_prof.ev.push_back(e);
    }
    g_prof.names[g_prof.used] = name;
    cudaEventRecord(g_prof.ev[2 * g_prof.used], s);
}

void prof_end(cudaStream_t s)
{
    if (!g_prof.on || g_prof.used >= PROF_MAX || (int)g_prof.ev.size() < 2 * (g_prof.used + 1))
        return;
    cudaEventRecord(g_prof.ev[2 * g_prof.used + 1], s);
    ++g_prof.used;
}

// Per device (ordinal < 64): the compute-capability verdict, cached in an atomic
// once known (a failed query is retried next call); the pool setup it does is
// idempotent, so two threads racing on the first call are harmless.  Devices
// beyond 64 are checked every call.
constexpr int MAX_DEV = 64;
std::atomic<int> g_dev_ok[MAX_DEV];  // 0 = unknown, 1 = sm_100, 2 = unsupported

int query_device(int dev)
{
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
        cudaGetLastError();
        return 3;
    }
    if (major != 10 || minor != 0) return 2;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;  // keep stream-ordered scratch cached in the pool
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    return 1;
}

gl_status device_check()
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return GL_E_CUDA;
    }
    int v = (dev >= 0 && dev < MAX_DEV) ? g_dev_ok[dev].load() : 0;
    if (v == 0) {
        v = query_device(dev);  // 3 = the query failed: not cached
        if (v != 3 && dev >= 0 && dev < MAX_DEV) g_dev_ok[dev].store(v);
    }
    return v == 1 ? GL_OK : (v == 2 ? GL_E_UNSUPPORTED : GL_E_CUDA);
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// thresholds of R22: thr_c = floor(alpha^c * 2^32), alpha^c by repeated products
void accept_thresholds(double alpha, int gamma, uint64_t *thr)
{
    double x = 1.0;
    for (int c = 1; c <= GL_MAX_GAMMA; ++c) {
        if (c <= gamma) {
            x = x * alpha;
            thr[c - 1] = (uint64_t)std::floor(x * 4294967296.0);
        } else {
            thr[c - 1] = 0;
        }
    }
}

gl_status validate_traces(const gl_trace *traces, int32_t n_traces)
{
    if (!traces || n_traces <= 0) return GL_E_INVALID;
    for (int32_t t = 0; t < n_traces; ++t) {
        const gl_trace &tr = traces[t];
        if (!tr.arrival_us || !tr.prompt_len || !tr.output_len) return GL_E_INVALID;
        if (tr.n <= 0 || tr.n >= (int64_t)1 << 31) return GL_E_INVALID;
        if (!aligned16(tr.arrival_us) || !aligned16(tr.prompt_len) || !aligned16(tr.output_len))
            return GL_E_INVALID;
    }
    return GL_OK;
}

gl_status validate_chain(const gl_chain &c, int32_t n_traces)
{
    if (c.mode < GL_MODE_DPD || c.mode > GL_MODE_SPEC_COLO) return GL_E_INVALID;
    const bool spec = c.mode == GL_MODE_DSD || c.mode == GL_MODE_SPEC_COLO;
    if (c.trace_idx < 0 || c.trace_idx >= n_traces) return GL_E_LOOKUP;
    if (c.batch_cap < 1 || c.batch_cap > GL_MAX_CAP) return GL_E_INVALID;
    if (c.max_prompt < 1 || c.max_prompt > GL_MAX_PROMPT) return GL_E_INVALID;
    if (spec && (c.gamma < 1 || c.gamma > GL_MAX_GAMMA)) return GL_E_INVALID;
    if (!c.t1_us || !c.e1_new_uj || !c.t2_us || !c.b2_old_us || !c.e2_old_uj || !c.step_us ||
        !c.step_busy_new_us || !c.step_busy_old_us || !c.step_e_new_uj || !c.step_e_old_uj)
        return GL_E_INVALID;
    if (spec && !(c.alpha >= 0.0 && c.alpha <= 1.0)) return GL_E_DOMAIN;
    if (c.ttft_slo_us < 0 || c.tpot_slo_us < 0) return GL_E_DOMAIN;
    if (c.tpot_slo_us > ((int64_t)1 << 32)) return GL_E_DOMAIN;  // keeps deadlines in int64
    return GL_OK;
}

gl_status cuda_status(cudaError_t e) { return e == cudaSuccess ? GL_OK : GL_E_CUDA; }

// A side stream forked from `from` (its work starts after everything enqueued on
// `from` so far), with an event for joining it back.  One per (host thread, device,
// slot), created on first use and kept: creating a stream per call costs more than
// the overlap it buys.  Returns false (and nothing to join) if CUDA refuses.
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
bool side_fork(int slot, cudaStream_t from, cudaStream_t &side, cudaEvent_t &join)
{
    thread_local SideStream tl[16][6];  // [device][slot]
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) {
        cudaGetLastError();
        return false;
    }
    SideStream &ss = tl[dev][slot];
    if (!ss.s) {
        SideStream n;
        // slot 4 carries short kernels that must not queue behind a whole-GPU kernel
        // on `from` (k_stages beside the DSD demand): the highest stream priority
        int least = 0, greatest = 0;
        if (slot != 4 || cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) {
            cudaGetLastError();
            greatest = 0;
        }
        if (cudaStreamCreateWithPriority(&n.s, cudaStreamNonBlocking, greatest) == cudaSuccess &&
            cudaEventCreateWithFlags(&n.fork, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&n.join, cudaEventDisableTiming) == cudaSuccess) {
            ss = n;
        } else {
            cudaGetLastError();
            if (n.s) cudaStreamDestroy(n.s);
            if (n.fork) cudaEventDestroy(n.fork);
            return false;
        }
    }
    if (cudaEventRecord(ss.fork, from) != cudaSuccess ||
        cudaStreamWaitEvent(ss.s, ss.fork, 0) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    side = ss.s;
    join = ss.join;
    return true;
}

// the extra work of gl_link_demand
struct LinkReq {
    const gl_link_params *params;  // host [n_chains]
    int64_t window;
    gl_link_stats *out;            // device [n_chains]
};

gl_status eval_impl(const gl_trace *traces, int32_t n_traces, const gl_chain *chains,
                    int32_t n_chains, gl_chain_stats *stats_out, int64_t *per_request_out,
                    cudaStream_t stream, const LinkReq *lk,
                    cudaEvent_t stages_wait = nullptr,  // k_stages waits for it (host path)
                    const gl_schedule *sched = nullptr)
{
    gl_status st = validate_traces(traces, n_traces);
    if (st) return st;
    if (!chains || n_chains <= 0 || (!stats_out && !lk)) return GL_E_INVALID;
    for (int32_t i = 0; i < n_chains; ++i)
        if ((st = validate_chain(chains[i], n_traces))) return st;
    if (lk) {
        if (!lk->params || !lk->out || lk->window < 1) return GL_E_INVALID;
        for (int32_t i = 0; i < n_chains; ++i)
            if (lk->params[i].bytes_per_token < 0 || lk->params[i].bytes_per_member_step < 0)
                return GL_E_DOMAIN;
    }
    if ((st = device_check())) return st;

    // DSD demand groups: equal (output_len, n, gamma, thresholds, seed) share K
    std::vector<DGroup> groups;
    std::map<std::tuple<const uint32_t *, int64_t, int32_t, uint64_t, std::vector<uint64_t>>, int> gid;
    std::vector<int> chain_group(n_chains, -1);
    std::vector<double> group_alpha;
    int max_cap = 1;
    size_t smem_st = 0;
    int64_t rows_total = 0, maxn = 0;
    bool has_colo = false, has_disg = false;
    for (int32_t i = 0; i < n_chains; ++i) {
        const gl_chain &c = chains[i];
        max_cap = std::max(max_cap, (int)c.batch_cap);
        smem_st = std::max(smem_st, (size_t)8 * gl::round_up4(c.max_prompt + 1) + 16);
        rows_total += traces[c.trace_idx].n;
        maxn = std::max(maxn, traces[c.trace_idx].n);
        if (c.mode == GL_MODE_STANDALONE || c.mode == GL_MODE_SPEC_COLO) has_colo = true;
        else has_disg = true;
        if (c.mode != GL_MODE_DSD && c.mode != GL_MODE_SPEC_COLO) continue;
        DGroup g{};
        g.o = traces[c.trace_idx].output_len;
        g.n = traces[c.trace_idx].n;
        g.seed = c.seed;
        g.gamma = c.gamma;
        accept_thresholds(c.alpha, c.gamma, g.thr);
        auto key = std::make_tuple(g.o, g.n, g.gamma, g.seed,
                                   std::vector<uint64_t>(g.thr, g.thr + GL_MAX_GAMMA));
        auto it = gid.find(key);
        if (it == gid.end()) {
            it = gid.emplace(key, (int)groups.size()).first;
            groups.push_back(g);
            group_alpha.push_back(c.alpha);
        }
        chain_group[i] = it->second;
    }
    // Families: groups drawing the same acceptance words (equal output lengths, n and
    // seed), differing in (alpha, gamma); one kernel pass evaluates each word once for
    // all of them (k_dsd_family).  Up to FAM_NA alphas and gamma <= FAM_GM; any other
    // group (and a family of one) keeps the per-group kernel.
    std::vector<gl::DFamily> fams;
    std::vector<std::vector<std::pair<int, int>>> fam_slots;  // (group, slot a * GM + g)
    std::vector<int> solo;
    {
        std::map<std::tuple<const uint32_t *, int64_t, uint64_t>, std::vector<int>> fam_of;
        for (size_t g = 0; g < groups.size(); ++g)
            fam_of[std::make_tuple(groups[g].o, groups[g].n, groups[g].seed)].push_back((int)g);
        for (auto &kv : fam_of) {
            const std::vector<int> &L = kv.second;
            // alpha-sets: the threshold sequence up to FAM_GM (repeated products, R22)
            std::map<std::vector<uint64_t>, int> aset;
            bool ok = L.size() >= 2;
            for (int g : L) {
                if (groups[g].gamma > gl::FAM_GM) ok = false;
                uint64_t t[GL_MAX_GAMMA];
                accept_thresholds(group_alpha[g], GL_MAX_GAMMA, t);
                aset.emplace(std::vector<uint64_t>(t, t + gl::FAM_GM), 0);
            }
            if (aset.size() > (size_t)gl::FAM_NA) ok = false;
            if (!ok) {
                solo.insert(solo.end(), L.begin(), L.end());
                continue;
            }
            gl::DFamily f{};
            f.o = groups[L[0]].o;
            f.n = groups[L[0]].n;
            f.seed = groups[L[0]].seed;
            f.na = (int32_t)aset.size();
            int a = 0;  // std::map orders the sequences ascending: smallest alpha first
            for (auto &av : aset) {
                av.second = a;
                const bool one = av.first[0] == (uint64_t)1 << 32;
                f.all[a] = one ? 1u : 0u;
                for (int c = 0; c < gl::FAM_GM; ++c) f.thr[a][c] = one ? 0u : (uint32_t)av.first[c];
                ++a;
            }
            std::vector<std::pair<int, int>> slots;
            for (int g : L) {
                uint64_t t[GL_MAX_GAMMA];
                accept_thresholds(group_alpha[g], GL_MAX_GAMMA, t);
                const int ai = aset[std::vector<uint64_t>(t, t + gl::FAM_GM)];
                slots.emplace_back(g, ai * gl::FAM_GM + (groups[g].gamma - 1));
            }
            fams.push_back(f);
            fam_slots.push_back(slots);
        }
    }
    const size_t smem_dec = gl::decode_smem_bytes(max_cap);
    int dev = 0, n_sm = 0, smem_optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (smem_st > (size_t)smem_optin || smem_dec > (size_t)smem_optin) return GL_E_UNSUPPORTED;

    // Stream-ordered scratch: [chains][groups][K arrays][per-request rows if not
    // given][decode stream r, (d, j): n + 512 per chain][helpers' finish-time
    // buffers: helpers x (n + 512) per chain][candidates]
    // [segment results][per-chain bookkeeping].  The last two are zeroed.
    const size_t off_groups = align256(sizeof(DChain) * n_chains);
    const size_t off_fams = off_groups + align256(sizeof(DGroup) * groups.size());
    size_t total = off_fams + align256(sizeof(gl::DFamily) * fams.size());
    std::vector<size_t> k_off(groups.size());
    for (size_t g = 0; g < groups.size(); ++g) {
        k_off[g] = total;
        total += align256(sizeof(uint32_t) * (size_t)groups[g].n);
    }
    const size_t off_rows = total;
    if (!per_request_out) total += align256(sizeof(int64_t) * 2 * (size_t)rows_total);
    std::vector<int64_t> dec_off(n_chains), seg_off(n_chains);
    int64_t dec_total = 0, seg_total = 0;
    for (int32_t i = 0; i < n_chains; ++i) {
        const int64_t n = traces[chains[i].trace_idx].n;
        dec_off[i] = dec_total;
        dec_total += (n + 512 + 31) & ~(int64_t)31;
        seg_off[i] = seg_total;
        seg_total += (n + gl::SEG_LEN - 1) / gl::SEG_LEN + 2;
    }
    const size_t off_dec_r = total;
    total += align256(sizeof(int64_t) * (size_t)dec_total);
    const size_t off_dec_dj = total;
    total += align256(sizeof(uint2) * (size_t)dec_total);
    const size_t off_dec_pf = total;
    total += align256(sizeof(int32_t) * (size_t)dec_total);
    // k_decode: one leader warp per chain plus helper warps, about four warps per
    // SM in total; each helper keeps its finish times in a buffer of its own
    // (capped at 8 GiB of scratch)
    int extra = std::max(0, std::min(15, (4 * n_sm) / std::max(1, (int)n_chains) - 1));
    // helpers' buffers per decode-stream entry: finish times (co-located chains keep
    // two columns, finish and TTFT) and, for gl_link_demand, batch-size logs (2
    // entries x 16 B per request); none at all when there are no helpers
    const int spec_mult = has_colo ? 2 : 1;
    const size_t per_helper_req = spec_mult * sizeof(int64_t) + (lk ? 2 * sizeof(longlong2) : 0);
    while (extra > 0 && (size_t)dec_total * per_helper_req * extra > ((size_t)8 << 30)) --extra;
    const size_t off_spec = total;
    total += align256(sizeof(int64_t) * (size_t)dec_total * spec_mult * (size_t)extra);
    const size_t off_segs = total;
    total += align256(sizeof(int32_t) * (size_t)seg_total);
    const size_t off_segwc = total;
    total += align256(sizeof(int32_t) * (size_t)seg_total);
    // gl_link_demand: batch-size logs [2 n + 8], prefix sums, per-block partials, stats
    std::vector<int64_t> ev_off(n_chains, 0), rq_off(n_chains, 0), evs_off(n_chains, 0);
    int64_t ev_total = 0, rq_total = 0, evs_total = 0;
    size_t off_ev = 0, off_itpre = 0, off_rqpre = 0, off_links = 0, off_part = 0, off_lstats = 0;
    size_t off_evd = 0, off_evs = 0;
    if (lk) {
        for (int32_t i = 0; i < n_chains; ++i) {
            const int64_t n = traces[chains[i].trace_idx].n;
            ev_off[i] = ev_total;
            ev_total += 2 * n + 16;
            rq_off[i] = rq_total;
            rq_total += n + 8;
            evs_off[i] = evs_total;
            evs_total += (2 * n + 16) * extra;
        }
        off_ev = total;
        total += align256(sizeof(longlong2) * (size_t)ev_total);
        off_evd = total;  // compacted logs
        total += align256(sizeof(longlong2) * (size_t)ev_total);
        off_evs = total;  // helpers' logs
        total += align256(sizeof(longlong2) * (size_t)evs_total);
        off_itpre = total;
        total += align256(sizeof(int64_t) * (size_t)ev_total);
        off_rqpre = total;
        total += align256(sizeof(int64_t) * (size_t)rq_total);
        off_links = total;
        total += align256(sizeof(gl::DLink) * (size_t)n_chains);
        off_part = total;
        total += align256(sizeof(longlong2) * (gl::LINK_BLOCKS + 1) * (size_t)n_chains);
        off_lstats = total;
        if (!stats_out) total += align256(sizeof(gl_chain_stats) * (size_t)n_chains);
    }
    const size_t off_zero = total;
    const size_t off_segout = total;
    total += align256(sizeof(gl::DSegOut) * (size_t)seg_total);
    const size_t off_x = total;
    total += align256(sizeof(gl::DChainX) * (size_t)n_chains);
    // Stage groups: disaggregated chains of one mode on the same trace with the same
    // prompt-indexed tables run identical stage-1/2 scans; the first (primary) runs
    // k_stages, the others (secondaries) take its results in k_stage_clone.
    std::vector<int32_t> prim_of(n_chains), prim_ids, sec_ids;
    {
        std::map<std::tuple<int32_t, int32_t, const void *, const void *, const void *,
                            const void *, const void *, int32_t>, int32_t> first;
        for (int32_t i = 0; i < n_chains; ++i) {
            const gl_chain &c = chains[i];
            prim_of[i] = i;
            if (c.mode == GL_MODE_DPD || c.mode == GL_MODE_DSD) {
                auto key = std::make_tuple(c.trace_idx, c.mode, (const void *)c.t1_us,
                                           (const void *)c.t2_us, (const void *)c.b2_old_us,
                                           (const void *)c.e1_new_uj, (const void *)c.e2_old_uj,
                                           c.max_prompt);
                auto it = first.find(key);
                if (it == first.end()) first.emplace(key, i);
                else prim_of[i] = it->second;
            }
            if (prim_of[i] == i) prim_ids.push_back(i);
            else sec_ids.push_back(i);
        }
    }
    const int32_t n_prim = (int32_t)prim_ids.size(), n_sec = (int32_t)sec_ids.size();
    // Two-phase launch order (gl_schedule): phase A = the hinted chain range
    // [s_lo, s_hi) for the decode, plus, for the prologue, the primaries its
    // secondaries copy from and every DSD group / family those chains use.  Not for
    // co-located chains (their decode overlaps on a side stream already) or the link
    // analysis; an empty or full range is one phase.
    const int32_t s_lo = sched ? sched->first_lo : 0, s_hi = sched ? sched->first_hi : 0;
    const bool phased = sched && !lk && !has_colo && s_lo < s_hi && !(s_lo == 0 && s_hi == n_chains);
    int32_t fam_a = 0, solo_a = 0, prim_a = 0, sec_a = 0;
    if (phased) {
        std::vector<char> stage_a(n_chains, 0), group_a(groups.size(), 0);
        for (int32_t c = s_lo; c < s_hi; ++c) stage_a[c] = stage_a[prim_of[c]] = 1;
        for (int32_t c = 0; c < n_chains; ++c)
            if (stage_a[c] && chain_group[c] >= 0) group_a[chain_group[c]] = 1;
        auto is_a = [&](int32_t c) { return stage_a[c] != 0; };
        prim_a = (int32_t)(std::stable_partition(prim_ids.begin(), prim_ids.end(), is_a) - prim_ids.begin());
        sec_a = (int32_t)(std::stable_partition(sec_ids.begin(), sec_ids.end(), is_a) - sec_ids.begin());
        solo_a = (int32_t)(std::stable_partition(solo.begin(), solo.end(),
                                                 [&](int g) { return group_a[g] != 0; }) - solo.begin());
        std::vector<size_t> order(fams.size());
        for (size_t f = 0; f < fams.size(); ++f) order[f] = f;
        auto fam_in_a = [&](size_t f) {
            for (auto &gs : fam_slots[f])
                if (group_a[gs.first]) return true;
            return false;
        };
        fam_a = (int32_t)(std::stable_partition(order.begin(), order.end(), fam_in_a) - order.begin());
        std::vector<gl::DFamily> f2;
        std::vector<std::vector<std::pair<int, int>>> s2;
        for (size_t f : order) {
            f2.push_back(fams[f]);
            s2.push_back(fam_slots[f]);
        }
        fams.swap(f2);
        fam_slots.swap(s2);
    }
    // Deferred DSD demand: when DSD demand kernels run, k_stages of the disaggregated
    // DSD primaries does not wait for them -- it runs on a side stream alongside, with
    // demand 0 in their decode streams, and k_stage_clone's fill pass writes K_j there
    // once both are done (the stage scans never read K).  The primaries to fill, by phase.
    std::vector<int32_t> fill_ids;
    int32_t fill_a = 0;
    // (co-located SpecDecode chains read K inside k_stages: no deferral with them)
    bool any_spec_colo = false;
    for (int32_t i = 0; i < n_chains; ++i) any_spec_colo |= chains[i].mode == GL_MODE_SPEC_COLO;
    const bool defer = (!fams.empty() || !solo.empty()) && !any_spec_colo;
    if (defer) {
        for (int32_t i = 0; i < n_prim; ++i)
            if (chains[prim_ids[i]].mode == GL_MODE_DSD) {
                fill_ids.push_back(prim_ids[i]);
                if (i < prim_a) ++fill_a;  // prim_ids holds phase A's primaries first
            }
    }
    const int32_t n_fill = (int32_t)fill_ids.size();
    const bool use_ids = phased || n_sec > 0 || n_fill > 0;  // kernels read chain id lists
    // k_stages: S blocks per chain (decoupled look-back between them), S <= 4 chosen
    // to minimise the waves per chain's work, ceil(chains S / resident) / S (ties to
    // the smaller S): 2 on config 4's 64 chains, 3 on config 6's 80, 4 on config 5's 320
    int stage_split = 1;
    {
        int per_sm = 0;
        if (cudaFuncSetAttribute(gl::k_stages, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem_st) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gl::k_stages, 32 * gl::ST_WARPS,
                                                          smem_st) == cudaSuccess &&
            per_sm > 0) {
            const int64_t slots = (int64_t)per_sm * n_sm;
            int64_t best_w = (n_prim + slots - 1) / slots;
            for (int S = 2; S <= gl::ST_MAX_SPLIT; ++S) {
                const int64_t w = ((int64_t)n_prim * S + slots - 1) / slots;
                if (w * stage_split < best_w * S) {
                    best_w = w;
                    stage_split = S;
                }
            }
        }
        cudaGetLastError();
    }
    const size_t off_stp = total;
    total += align256(sizeof(gl::DStagePart) * (size_t)n_chains * stage_split);
    const size_t off_ticket = total;
    total += 256;
    const size_t off_ids = total;  // primaries, secondaries, primary of each chain, fills
    total += align256(sizeof(int32_t) * ((size_t)n_chains * 3 + 2));
    // k_relax (exact parallel decode of heavily loaded chains, k_relax.cuh): slots for
    // the chains k_relax_pick selects on the device by load factor.  Not with the link
    // analysis (it needs the batch-size log) or a launch-order hint, and by default not
    // beside co-located chains (their decode shares the SMs' issue slots with it:
    // config 6 +5%, config 7 +1.6%; config 4 -5.8%).  GL_RELAX=0 turns
    // it off, GL_RELAX=1 on; GL_RELAX=force (tests) makes every one-row chain eligible
    // at any load.
    const char *rx_env = std::getenv("GL_RELAX");
    const bool rx_off = rx_env ? (rx_env[0] != '1' && rx_env[0] != 'f' && rx_env[0] != 's') : has_colo;
    const bool rx_force = rx_env && (rx_env[0] == 'f' || rx_env[0] == 's');
    // GL_RELAX=solo (tests): k_relax runs first on `stream`, so it wins every chain it
    // solves and k_decode walks only the rest
    const bool rx_solo = rx_env && rx_env[0] == 's';
    int64_t rx_ncap = 0;
    int32_t rx_elig = 0;
    int64_t rx_max_n = gl::RX_MAX_N;  // GL_RELAX_MAXN: experiments
    if (const char *mn = std::getenv("GL_RELAX_MAXN")) rx_max_n = std::atoll(mn);
    if (!lk && !phased && !rx_off)
        for (int32_t i = 0; i < n_chains; ++i) {
            const gl_chain &c = chains[i];
            const int64_t n = traces[c.trace_idx].n;
            // (by default not on 1M-request traces: their heavy chains are saturated ones
            // that do not relax in time, and the slots would take ~4 GiB of scratch)
            if ((c.mode == GL_MODE_DPD || c.mode == GL_MODE_DSD) && c.batch_cap <= gl::RX_MAXCAP &&
                n >= (rx_force ? 1 : gl::RX_MIN_M) && (rx_force || n <= rx_max_n)) {
                ++rx_elig;
                rx_ncap = std::max(rx_ncap, n);
            }
        }
    const int64_t rx_lcap = std::min<int64_t>((int64_t)gl::RX_LFACTOR * rx_ncap + 64, ((int64_t)1 << 31) - 64) & ~(int64_t)7;
    const int32_t rx_nsegcap = (int32_t)((rx_ncap + gl::RX_SEG - 1) / gl::RX_SEG);
    const size_t rx_b_j = align256(sizeof(int32_t) * (size_t)rx_ncap);
    const size_t rx_b_seg = align256(sizeof(int32_t) * 2 * (size_t)rx_nsegcap);
    const size_t rx_b_l = align256(sizeof(int64_t) * (size_t)(rx_lcap + 1));   // tau
    const size_t rx_b_h = align256(sizeof(uint32_t) * (size_t)rx_lcap);        // histogram
    const size_t rx_b_blk = align256(sizeof(gl::RxBlk) * (size_t)n_sm * gl::RX_BPS);
    int32_t rx_slots = 0;
    if (rx_elig > 0) {
        const size_t per = 3 * rx_b_j + rx_b_seg + rx_b_l + rx_b_h + rx_b_blk;
        rx_slots = (int32_t)std::min<int64_t>(std::min<int64_t>(rx_elig, rx_force ? gl::RX_MAX_SLOTS : gl::RX_DEF_SLOTS),
                                              (int64_t)(((size_t)4 << 30) / per));
    }
    const size_t off_rx_blk = total;
    total += rx_b_blk * rx_slots;
    const size_t zero_bytes = total - off_zero;
    // (not zeroed) slot descriptors, load factors, iterates and iteration arrays
    const size_t off_rx_slots = total;
    total += align256(sizeof(gl::DRelax) * (size_t)rx_slots);
    const size_t off_rx_rho = total;
    total += rx_slots ? align256(sizeof(double) * (size_t)n_chains) : 0;
    const size_t off_rx_buf = total;
    total += (3 * rx_b_j + rx_b_seg + rx_b_l + rx_b_h) * rx_slots;
    unsigned char *scratch = nullptr;
    if ((st = cuda_status(cudaMallocAsync(reinterpret_cast<void **>(&scratch), total, stream))))
        return st;
    int64_t *rows = per_request_out ? per_request_out : reinterpret_cast<int64_t *>(scratch + off_rows);
    if (!stats_out) stats_out = reinterpret_cast<gl_chain_stats *>(scratch + off_lstats);
    std::vector<gl::DLink> dl(lk ? n_chains : 0);
    for (size_t g = 0; g < groups.size(); ++g)
        groups[g].K = reinterpret_cast<uint32_t *>(scratch + k_off[g]);
    for (size_t fi = 0; fi < fams.size(); ++fi)
        for (auto &gs : fam_slots[fi])
            fams[fi].K[gs.second / gl::FAM_GM][gs.second % gl::FAM_GM] = groups[gs.first].K;
    std::vector<DGroup> solo_groups;  // the per-group kernel's share
    for (int g : solo) solo_groups.push_back(groups[g]);

    std::vector<DChain> dch(n_chains);
    int64_t out_off = 0;
    for (int32_t i = 0; i < n_chains; ++i) {
        const gl_chain &c = chains[i];
        const gl_trace &tr = traces[c.trace_idx];
        DChain &d = dch[i];
        d.a = tr.arrival_us;
        d.p = tr.prompt_len;
        d.o = tr.output_len;
        d.K = chain_group[i] >= 0 ? groups[chain_group[i]].K : nullptr;
        d.t1 = c.t1_us;
        d.t2 = c.t2_us;
        d.b2 = c.b2_old_us;
        d.e1 = c.e1_new_uj;
        d.e2 = c.e2_old_uj;
        d.step = c.step_us;
        d.sbn = c.step_busy_new_us;
        d.sbo = c.step_busy_old_us;
        d.sen = c.step_e_new_uj;
        d.seo = c.step_e_old_uj;
        d.dec_r = reinterpret_cast<int64_t *>(scratch + off_dec_r) + dec_off[i];
        d.dec_dj = reinterpret_cast<uint2 *>(scratch + off_dec_dj) + dec_off[i];
        d.dec_pf = reinterpret_cast<int32_t *>(scratch + off_dec_pf) + dec_off[i];
        d.spec_fin = reinterpret_cast<int64_t *>(scratch + off_spec) + dec_off[i] * spec_mult * extra;
        d.spec_stride = ((tr.n + 512 + 31) & ~(int64_t)31) *
                        ((c.mode == GL_MODE_STANDALONE || c.mode == GL_MODE_SPEC_COLO) ? 2 : 1);
        d.seg_start = reinterpret_cast<int32_t *>(scratch + off_segs) + seg_off[i];
        d.seg_out = reinterpret_cast<gl::DSegOut *>(scratch + off_segout) + seg_off[i];
        d.x = reinterpret_cast<gl::DChainX *>(scratch + off_x) + i;
        d.stp = reinterpret_cast<gl::DStagePart *>(scratch + off_stp) + (size_t)stage_split * i;
        d.ev = lk ? reinterpret_cast<longlong2 *>(scratch + off_ev) + ev_off[i] : nullptr;
        d.ev_spec = lk ? reinterpret_cast<longlong2 *>(scratch + off_evs) + evs_off[i] : nullptr;
        d.ev_stride = 2 * tr.n + 16;
        if (lk) {
            gl::DLink &L = dl[i];
            L.bpt = lk->params[i].bytes_per_token;
            L.pm = lk->params[i].bytes_per_member_step;
            L.it_pre = reinterpret_cast<int64_t *>(scratch + off_itpre) + ev_off[i];
            L.req_pre = reinterpret_cast<int64_t *>(scratch + off_rqpre) + rq_off[i];
            L.part = reinterpret_cast<longlong2 *>(scratch + off_part) + (size_t)(gl::LINK_BLOCKS + 1) * i;
            L.ev_cap = 2 * tr.n + 16;
            L.ev = reinterpret_cast<longlong2 *>(scratch + off_evd) + ev_off[i];
        }
        d.n = tr.n;
        d.ttft_slo = c.ttft_slo_us;
        d.tpot_slo = c.tpot_slo_us;
        d.out_off = out_off;
        out_off += tr.n;
        d.mode = c.mode;
        d.cap = c.batch_cap;
        d.max_prompt = c.max_prompt;
        d.capacity_ok = c.capacity_ok ? 1 : 0;
    }
    for (int32_t i : sec_ids) dch[i].dec_r = dch[prim_of[i]].dec_r;  // shared ready times
    const DChain *dc = reinterpret_cast<const DChain *>(scratch);
    int32_t *d_prim_ids = reinterpret_cast<int32_t *>(scratch + off_ids);
    int32_t *d_sec_ids = d_prim_ids + n_prim;
    int32_t *d_prim_of = d_sec_ids + n_sec;
    int32_t *d_fill_ids = d_prim_of + n_chains;
    cudaError_t e = cudaMemcpyAsync(scratch, dch.data(), sizeof(DChain) * n_chains,
                                    cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess && !solo_groups.empty())
        e = cudaMemcpyAsync(scratch + off_groups, solo_groups.data(),
                            sizeof(DGroup) * solo_groups.size(), cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess && !fams.empty())
        e = cudaMemcpyAsync(scratch + off_fams, fams.data(), sizeof(gl::DFamily) * fams.size(),
                            cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess && lk)
        e = cudaMemcpyAsync(scratch + off_links, dl.data(), sizeof(gl::DLink) * n_chains,
                            cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(scratch + off_zero, 0, zero_bytes, stream);
    std::vector<int32_t> idv;  // (kept alive until the copy is enqueued: pageable, synchronous staging)
    if (e == cudaSuccess && use_ids) {  // after the memset: the ids live in the zeroed region
        idv = prim_ids;
        idv.insert(idv.end(), sec_ids.begin(), sec_ids.end());
        idv.insert(idv.end(), prim_of.begin(), prim_of.end());
        idv.insert(idv.end(), fill_ids.begin(), fill_ids.end());
        e = cudaMemcpyAsync(d_prim_ids, idv.data(), sizeof(int32_t) * idv.size(),
                            cudaMemcpyHostToDevice, stream);
    }
    std::vector<gl::DRelax> rxv(rx_slots);
    for (int32_t k = 0; k < rx_slots; ++k) {
        gl::DRelax &R = rxv[k];
        std::memset(&R, 0, sizeof R);
        unsigned char *b = scratch + off_rx_buf + (3 * rx_b_j + rx_b_seg + rx_b_l + rx_b_h) * k;
        R.J = reinterpret_cast<int32_t *>(b);
        R.A = reinterpret_cast<int32_t *>(b + rx_b_j);
        R.Sq = reinterpret_cast<int32_t *>(b + 2 * rx_b_j);
        R.seg = reinterpret_cast<int32_t *>(b + 3 * rx_b_j);
        R.tau = reinterpret_cast<int64_t *>(b + 3 * rx_b_j + rx_b_seg);
        R.h = reinterpret_cast<uint32_t *>(b + 3 * rx_b_j + rx_b_seg + rx_b_l);
        R.blk = reinterpret_cast<gl::RxBlk *>(scratch + off_rx_blk + rx_b_blk * k);
        R.lcap = rx_lcap;
        R.ncap = (int32_t)rx_ncap;
        R.nsegcap = rx_nsegcap;
        R.chain = -1;
    }
    if (e == cudaSuccess && rx_slots)
        e = cudaMemcpyAsync(scratch + off_rx_slots, rxv.data(), sizeof(gl::DRelax) * rx_slots,
                            cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess && lk)  // log sentinels: every byte 0xFF -> (T, b) = (-1, -1)
        e = cudaMemsetAsync(scratch + off_ev, 0xFF, sizeof(longlong2) * (size_t)ev_total, stream);
    int launches = 0;
    // ---- kernels over a phase: families [f0, f1), solo groups [g0, g1), primaries
    // [p0, p1) and secondaries [s0, s1) of the device id lists, chains [c0, c1)
    auto launch_family = [&](int32_t f0, int32_t f1) {
        if (e != cudaSuccess || f1 <= f0) return;
        // persistent threads: about 8 blocks of 128 threads per SM in total (two waves
        // at the register limit of 4 resident; one wave measured the same), spread
        // over the families, never more than one thread per request
        int64_t fmax = 0;
        for (int32_t f = f0; f < f1; ++f) fmax = std::max(fmax, fams[f].n);
        const int64_t want = std::max<int64_t>(1, (8 * (int64_t)n_sm) / (int64_t)(f1 - f0));
        const int64_t need_b = (fmax + 127) / 128;
        dim3 grid((unsigned)std::max<int64_t>(1, std::min(want, need_b)), (unsigned)(f1 - f0));
        prof_begin("k_dsd_family", stream);
        gl::k_dsd_family<<<grid, 128, 0, stream>>>(
            reinterpret_cast<const gl::DFamily *>(scratch + off_fams) + f0);
        e = cudaGetLastError();
        prof_end(stream);
        ++launches;
    };
    auto launch_solo = [&](int32_t g0, int32_t g1) {
        if (e != cudaSuccess || g1 <= g0) return;
        // persistent quads: about 16 resident blocks of 256 threads per SM in total,
        // spread over the groups, never more than one quad per request
        int64_t gmax = 0;
        for (int32_t g = g0; g < g1; ++g) gmax = std::max(gmax, solo_groups[g].n);
        const int64_t want = std::max<int64_t>(1, (16 * (int64_t)n_sm) / (int64_t)(g1 - g0));
        const int64_t need_b = (gmax * gl::DSD_QL + 255) / 256;
        dim3 grid((unsigned)std::max<int64_t>(1, std::min(want, need_b)), (unsigned)(g1 - g0));
        prof_begin("k_dsd_demand", stream);
        gl::k_dsd_demand<<<grid, 256, 0, stream>>>(
            reinterpret_cast<const DGroup *>(scratch + off_groups) + g0);
        e = cudaGetLastError();
        prof_end(stream);
        ++launches;
    };
    bool waited = false;  // gl_evaluate_host: the arrival arrays may still be in flight
    auto launch_stages = [&](int32_t p0, int32_t p1, int32_t ticket_slot, cudaStream_t ss) {
        if (e == cudaSuccess && stages_wait && !waited) {
            e = cudaStreamWaitEvent(ss, stages_wait, 0);
            waited = true;
        }
        if (e != cudaSuccess || p1 <= p0) return;
        e = cudaFuncSetAttribute(gl::k_stages, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem_st);
        if (e != cudaSuccess) return;
        prof_begin("k_stages", ss);
        gl::k_stages<<<(p1 - p0) * stage_split, 32 * gl::ST_WARPS, smem_st, ss>>>(
            dc, stats_out, rows, stage_split,
            reinterpret_cast<int32_t *>(scratch + off_ticket) + ticket_slot,
            use_ids ? d_prim_ids + p0 : nullptr, defer ? 1 : 0);
        e = cudaGetLastError();
        prof_end(ss);
        ++launches;
    };
    // rows are an output (or feed the link analysis): secondaries get full copies
    const bool copy_rows = per_request_out != nullptr || lk != nullptr;
    // secondaries [s0, s1) of d_sec_ids, or (fill) DSD primaries [s0, s1) of d_fill_ids
    auto launch_clone = [&](int32_t s0, int32_t s1, bool fill) {
        if (e != cudaSuccess || s1 <= s0) return;
        const int32_t ns = s1 - s0;
        const int bpc = (int)std::max<int64_t>(1, std::min<int64_t>(64, (8 * (int64_t)n_sm + ns - 1) / ns));
        prof_begin(fill ? "k_stage_fill" : "k_stage_clone", stream);
        gl::k_stage_clone<<<dim3((unsigned)bpc, (unsigned)ns), 256, 0, stream>>>(
            dc, stats_out, rows, (fill ? d_fill_ids : d_sec_ids) + s0, d_prim_of, stage_split,
            copy_rows ? 1 : 0, fill ? 1 : 0);
        e = cudaGetLastError();
        prof_end(stream);
        ++launches;
    };
    // a phase's prologue: with deferred demand, k_stages on a side stream (slot 4)
    // alongside the DSD demand kernels, joined before the fill and the clones
    auto prologue = [&](int32_t f0, int32_t f1, int32_t g0, int32_t g1, int32_t p0, int32_t p1,
                        int32_t l0, int32_t l1, int32_t s0, int32_t s1, int32_t ticket_slot) {
        cudaStream_t ss = nullptr;
        cudaEvent_t js = nullptr;
        if (e == cudaSuccess && defer && p1 > p0 && (f1 > f0 || g1 > g0) &&
            !side_fork(4, stream, ss, js))
            ss = nullptr;
        if (defer) launch_stages(p0, p1, ticket_slot, ss ? ss : stream);
        launch_family(f0, f1);
        launch_solo(g0, g1);
        if (!defer) launch_stages(p0, p1, ticket_slot, stream);  // it reads K
        if (ss) {
            cudaError_t r = cudaEventRecord(js, ss);
            if (r == cudaSuccess) r = cudaStreamWaitEvent(stream, js, 0);
            if (e == cudaSuccess) e = r;
        }
        launch_clone(l0, l1, true);
        launch_clone(s0, s1, false);
    };
    auto launch_segments = [&](int32_t c0, int32_t c1) {
        if (e != cudaSuccess || c1 <= c0) return;
        prof_begin("k_segments", stream);
        if (extra == 0) {
            // no helper warps (many chains): each leader walks its chain alone, one segment
            gl::k_segments_single<<<(unsigned)((c1 - c0 + 127) / 128), 128, 0, stream>>>(dc + c0, c1 - c0);
        } else {
            // 1024-thread blocks, one per SM; S per chain while they fit in a wave
            const int seg_split = std::max(1, std::min(4, n_sm / std::max(1, (int)n_chains)));
            gl::k_segments<<<(c1 - c0) * seg_split, 1024, 0, stream>>>(
                dc + c0, seg_split, (int64_t)((off_segwc - off_segs) / sizeof(int32_t)));
        }
        e = cudaGetLastError();
        prof_end(stream);
        ++launches;
    };
    // decode launches over chains [c0, c1) on `dstream`: disaggregated chains, then
    // co-located ones (each launch skips the other family's chains)
    auto launch_decode = [&](int32_t c0, int32_t c1, cudaStream_t dstream, cudaStream_t colo_stream,
                             int32_t rxpass = -1) {
        if (e != cudaSuccess || c1 <= c0) return;
        const int32_t nc = c1 - c0;
        const unsigned blocks = (unsigned)(nc * (1 + extra));
        cudaStream_t ds = dstream;
        auto launch = [&](auto kern, const char *name) {
            cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem_dec);
            if (r != cudaSuccess) return r;
            prof_begin(name, ds);
            kern<<<blocks, 32 * gl::DEC_WARPS, smem_dec, ds>>>(dc + c0, stats_out + c0, rows, nc, rxpass);
            r = cudaGetLastError();
            prof_end(ds);
            ++launches;
            return r;
        };
        if (has_disg && lk) {  // runs that also log the batch size
            if (max_cap <= 31)
                e = launch(gl::k_decode<1, false, true>, "k_decode_log");
            else if (max_cap <= 64)
                e = launch(gl::k_decode<2, false, true>, "k_decode_log");
            else if (max_cap <= 128)
                e = launch(gl::k_decode<4, false, true>, "k_decode_log");
            else
                e = launch(gl::k_decode<8, false, true>, "k_decode_log");
        } else if (has_disg) {
            if (max_cap <= 31)  // the one-row fast paths need b < 32
                e = launch(gl::k_decode<1, false>, "k_decode");
            else if (max_cap <= 64)
                e = launch(gl::k_decode<2, false>, "k_decode");
            else if (max_cap <= 128)
                e = launch(gl::k_decode<4, false>, "k_decode");
            else
                e = launch(gl::k_decode<8, false>, "k_decode");
        }
        if (has_colo && e == cudaSuccess) {
            ds = colo_stream;
            if (max_cap <= 31)  // the one-row fast paths need b < 32
                e = launch(gl::k_decode<1, true>, "k_decode_colo");
            else if (max_cap <= 64)
                e = launch(gl::k_decode<2, true>, "k_decode_colo");
            else if (max_cap <= 128)
                e = launch(gl::k_decode<4, true>, "k_decode_colo");
            else
                e = launch(gl::k_decode<8, true>, "k_decode_colo");
        }
    };
    auto join = [&](cudaStream_t side, cudaEvent_t ev) {
        if (!side) return;
        cudaError_t r = cudaEventRecord(ev, side);
        if (r == cudaSuccess) r = cudaStreamWaitEvent(stream, ev, 0);
        if (e == cudaSuccess) e = r;
    };
    if (!phased) {
        prologue(0, (int32_t)fams.size(), 0, (int32_t)solo_groups.size(), 0, n_prim, 0, n_fill,
                 0, n_sec, 0);
        launch_segments(0, n_chains);
        // k_relax: pick the heavily loaded chains, then (side stream) guess and relax
        // them while k_decode walks every chain on `stream`; each chain goes to
        // whichever finishes it first (k_relax.cuh)
        cudaStream_t rxs = nullptr;
        cudaEvent_t rxj = nullptr;
        const bool relax = rx_slots > 0 && e == cudaSuccess;
        if (relax) {
            gl::DRelax *d_slots = reinterpret_cast<gl::DRelax *>(scratch + off_rx_slots);
            double *d_rho = reinterpret_cast<double *>(scratch + off_rx_rho);
            double rx_ipr = gl::RX_MAX_IPR;  // GL_RELAX_IPR: experiments
            if (const char *ip = std::getenv("GL_RELAX_IPR")) rx_ipr = std::atof(ip);
            prof_begin("k_relax_pick", stream);
            gl::k_relax_rho<<<(unsigned)n_chains, 256, 0, stream>>>(dc, stats_out, d_rho,
                                                                   rx_force ? 1 : gl::RX_MIN_M,
                                                                   rx_force ? 1e300 : rx_ipr);
            double rlo = rx_force ? 0.0 : gl::RX_RHO_LO, rhi = rx_force ? 1e300 : gl::RX_RHO_HI;
            if (const char *rr = std::getenv("GL_RELAX_RHO")) std::sscanf(rr, "%lf,%lf", &rlo, &rhi);
            gl::k_relax_pick<<<1, 32, 0, stream>>>(dc, n_chains, d_rho, d_slots, rx_slots, rlo, rhi);
            e = cudaGetLastError();
            prof_end(stream);
            launches += 2;
            if (e == cudaSuccess && !rx_solo && !side_fork(5, stream, rxs, rxj)) rxs = nullptr;
        }
        auto launch_relax = [&]() {
            if (!relax) return;
            gl::DRelax *d_slots = reinterpret_cast<gl::DRelax *>(scratch + off_rx_slots);
            cudaStream_t xs = rxs ? rxs : stream;
            const int32_t segs = rx_nsegcap;
            const int64_t warps = (int64_t)rx_slots * segs;
            if (e == cudaSuccess) {
                prof_begin("k_relax_guess", xs);
                gl::k_relax_guess<<<(unsigned)((warps + gl::RX_GWARPS - 1) / gl::RX_GWARPS),
                                    32 * gl::RX_GWARPS, 0, xs>>>(d_slots, rx_slots, segs, dc);
                e = cudaGetLastError();
                prof_end(xs);
                ++launches;
            }
            if (e == cudaSuccess) {
                // one block per SM: room beside k_decode's warps (registers), all resident
                int per_sm = 0;
                const size_t rx_smem = (size_t)rx_slots * gl::RX_THREADS * 24;  // lane carries and maps
                e = cudaFuncSetAttribute(gl::k_relax, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rx_smem);
                if (e == cudaSuccess)
                    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gl::k_relax, gl::RX_THREADS, rx_smem);
                if (e == cudaSuccess && per_sm < 1) e = cudaErrorCooperativeLaunchTooLarge;
                if (e == cudaSuccess) {
                    int32_t ns = rx_slots;
                    const char *dbg_env = std::getenv("GL_RELAX_DEBUG");
                    int32_t dbg = dbg_env ? std::atoi(dbg_env) : 0;
                    void *args[] = {&d_slots, &ns, (void *)&dc, &dbg};
                    prof_begin("k_relax", xs);
                    int rx_blocks = n_sm * std::min(gl::RX_BPS, per_sm);  // GL_RELAX_BLOCKS: experiments
                    if (const char *rb = std::getenv("GL_RELAX_BLOCKS"))
                        rx_blocks = std::max(1, std::min(n_sm * std::min(gl::RX_BPS, per_sm), std::atoi(rb)));
                    e = cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(gl::k_relax),
                                                    dim3((unsigned)rx_blocks), dim3(gl::RX_THREADS), args, rx_smem, xs);
                    prof_end(xs);
                    ++launches;
                }
                // k_relax is an accelerator: without it k_decode walks every chain (no slot
                // is ever marked solved, k_relax_out writes nothing)
                if (e != cudaSuccess) {
                    cudaGetLastError();
                    e = cudaSuccess;
                }
            }
        };
        if (rx_solo) launch_relax();
        // Both families present (configurations 6 and 7): the co-located launch goes
        // to a side stream forked from `stream` and joined back, so the two launches
        // (disjoint chains) overlap; the call stays stream-ordered on `stream`.
        cudaStream_t side = nullptr;
        cudaEvent_t ev_join = nullptr;
        if (e == cudaSuccess && has_disg && has_colo && !lk && !side_fork(0, stream, side, ev_join))
            side = nullptr;  // no fork: both launches stay on `stream` (serialised)
        launch_decode(0, n_chains, stream, side ? side : stream, relax ? 1 : -1);
        // (enqueued after k_decode, so that k_decode's blocks are placed first)
        if (!rx_solo) launch_relax();
        join(side, ev_join);
        join(rxs, rxj);
        if (relax && e == cudaSuccess) {  // the chains k_relax solved first
            prof_begin("k_relax_out", stream);
            gl::k_relax_out<<<dim3(32, (unsigned)rx_slots), 256, 0, stream>>>(
                reinterpret_cast<gl::DRelax *>(scratch + off_rx_slots), dc, stats_out, rows);
            e = cudaGetLastError();
            prof_end(stream);
            ++launches;
        }
    } else {
        // Phase A (the hinted chains and the primaries they copy from): DSD demand,
        // stage scans, clones, segments, then its decode on a side stream; phase B's
        // prologue runs on `stream` meanwhile, its decodes on `stream` and a second
        // side stream; both joined before k_finalize.
        prologue(0, fam_a, 0, solo_a, 0, prim_a, 0, fill_a, 0, sec_a, 0);
        launch_segments(s_lo, s_hi);
        cudaStream_t sa = nullptr, sb = nullptr;
        cudaEvent_t ja = nullptr, jb = nullptr;
        if (e == cudaSuccess && !side_fork(2, stream, sa, ja)) sa = nullptr;
        launch_decode(s_lo, s_hi, sa ? sa : stream, nullptr);
        prologue(fam_a, (int32_t)fams.size(), solo_a, (int32_t)solo_groups.size(), prim_a, n_prim,
                 fill_a, n_fill, sec_a, n_sec, 1);
        launch_segments(0, s_lo);
        launch_segments(s_hi, n_chains);
        if (e == cudaSuccess && s_hi < n_chains && s_lo > 0 && !side_fork(3, stream, sb, jb))
            sb = nullptr;
        launch_decode(s_hi, n_chains, sb ? sb : stream, nullptr);
        launch_decode(0, s_lo, stream, nullptr);
        join(sa, ja);
        join(sb, jb);
    }
    if (e == cudaSuccess) {
        const int per_thread = 8;
        dim3 grid((unsigned)((maxn + 256 * per_thread - 1) / (256 * per_thread)), (unsigned)n_chains);
        prof_begin("k_finalize", stream);
        gl::k_finalize<<<grid, 256, 0, stream>>>(dc, stats_out, rows, per_thread,
                                                 (n_sec > 0 && !copy_rows) ? d_prim_of : nullptr);
        e = cudaGetLastError();
        prof_end(stream);
        ++launches;
    }
    if (e == cudaSuccess && lk) {
        const gl::DLink *dlk = reinterpret_cast<const gl::DLink *>(scratch + off_links);
        prof_begin("k_link_scan", stream);
        gl::k_link_scan<<<dim3((unsigned)n_chains, 2), 1024, 0, stream>>>(dc, dlk);
        e = cudaGetLastError();
        prof_end(stream);
        ++launches;
        if (e == cudaSuccess) {
            prof_begin("k_link_window", stream);
            gl::k_link_window<<<dim3(gl::LINK_BLOCKS, (unsigned)n_chains), gl::LINK_THREADS, 0,
                                stream>>>(dc, dlk, rows, lk->window);
            e = cudaGetLastError();
            prof_end(stream);
            ++launches;
        }
        if (e == cudaSuccess) {
            prof_begin("k_link_reduce", stream);
            gl::k_link_reduce<<<(unsigned)n_chains, 32, 0, stream>>>(dc, dlk, lk->out, n_chains);
            e = cudaGetLastError();
            prof_end(stream);
            ++launches;
        }
    }
    cudaError_t ef = cudaFreeAsync(scratch, stream);
    if (e == cudaSuccess) e = ef;
    if (e != cudaSuccess) return GL_E_CUDA;
    g_last_launches = launches;
    return GL_OK;
}

}  // namespace

// ---------------------------------------------------------------- C ABI
extern "C" {

gl_status gl_eval_grid(const gl_trace *traces, int32_t n_traces, const gl_chain *chains,
                       int32_t n_chains, gl_chain_stats *stats_out, int64_t *per_request_out,
                       void *stream_)
{
    return gl_eval_grid_sched(traces, n_traces, chains, n_chains, stats_out, per_request_out,
                              nullptr, stream_);
}

gl_status gl_eval_grid_sched(const gl_trace *traces, int32_t n_traces, const gl_chain *chains,
                             int32_t n_chains, gl_chain_stats *stats_out,
                             int64_t *per_request_out, const gl_schedule *sched, void *stream_)
{
    g_last_launches = 0;
    if (!stats_out) return GL_E_INVALID;
    if (sched && (sched->first_lo < 0 || sched->first_lo > sched->first_hi ||
                  sched->first_hi > n_chains))
        return GL_E_INVALID;
    return eval_impl(traces, n_traces, chains, n_chains, stats_out, per_request_out,
                     static_cast<cudaStream_t>(stream_), nullptr, nullptr, sched);
}

gl_status gl_link_demand(const gl_trace *traces, int32_t n_traces, const gl_chain *chains,
                         int32_t n_chains, const gl_link_params *params, int64_t window_us,
                         gl_chain_stats *stats_out, gl_link_stats *link_out, void *stream_)
{
    g_last_launches = 0;
    const LinkReq lk{params, window_us, link_out};
    return eval_impl(traces, n_traces, chains, n_chains, stats_out, nullptr,
                     static_cast<cudaStream_t>(stream_), &lk);
}

gl_status gl_argmin_feasible(const gl_chain_stats *stats, int32_t n_chains, const gl_chain *chains,
                             const gl_scenario *scen, int32_t n_scen, const gl_grid *grid,
                             int32_t slo_num, int32_t slo_den, int32_t priority,
                             int32_t default_col, double *carbon_out, double *per_token_out,
                             int32_t *choice_out, uint8_t *via_fallback_out, void *stream_)
{
    g_last_launches = 0;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    if (!stats || n_chains <= 0 || !chains || !scen || n_scen <= 0 || !grid || !choice_out ||
        !via_fallback_out)
        return GL_E_INVALID;
    if (grid->rows <= 0 || grid->cols <= 0 || !grid->row_scenario || !grid->cell_chain)
        return GL_E_INVALID;
    if (slo_den <= 0 || slo_num < 0 || slo_num > slo_den) return GL_E_INVALID;
    if (priority != GL_PRIORITY_SLO && priority != GL_PRIORITY_DEFAULT) return GL_E_INVALID;
    if (priority == GL_PRIORITY_DEFAULT && (default_col < -1 || default_col >= grid->cols))
        return GL_E_LOOKUP;
    for (int32_t i = 0; i < n_scen; ++i) {
        const gl_scenario &s = scen[i];
        if (!(std::isfinite(s.ci_g_per_kwh) && s.ci_g_per_kwh >= 0.0)) return GL_E_DOMAIN;
        if (!(std::isfinite(s.lt_new_s) && s.lt_new_s > 0.0)) return GL_E_DOMAIN;
        if (!(std::isfinite(s.lt_old_s) && s.lt_old_s > 0.0)) return GL_E_DOMAIN;
    }
    std::vector<DCarbon> cp(n_chains);
    for (int32_t i = 0; i < n_chains; ++i) {
        if (!(std::isfinite(chains[i].ce_new_g) && chains[i].ce_new_g > 0.0)) return GL_E_DOMAIN;
        if (!(std::isfinite(chains[i].ce_old_g) && chains[i].ce_old_g >= 0.0)) return GL_E_DOMAIN;
        cp[i] = DCarbon{chains[i].ce_new_g, chains[i].ce_old_g, chains[i].capacity_ok ? 1 : 0, 0};
    }
    const int64_t rows = grid->rows, cols = grid->cols;
    for (int64_t r = 0; r < rows; ++r)
        if (grid->row_scenario[r] < 0 || grid->row_scenario[r] >= n_scen) return GL_E_LOOKUP;
    for (int64_t k = 0; k < rows * cols; ++k)
        if (grid->cell_chain[k] < -1 || grid->cell_chain[k] >= n_chains) return GL_E_LOOKUP;
    gl_status st = device_check();
    if (st) return st;

    const size_t o_scen = align256(sizeof(DCarbon) * n_chains);
    const size_t o_rows = o_scen + align256(sizeof(gl_scenario) * n_scen);
    const size_t o_cells = o_rows + align256(sizeof(int32_t) * rows);
    const size_t total = o_cells + align256(sizeof(int32_t) * rows * cols);
    unsigned char *scratch = nullptr;
    if ((st = cuda_status(cudaMallocAsync(reinterpret_cast<void **>(&scratch), total, stream))))
        return st;
    cudaError_t e = cudaMemcpyAsync(scratch, cp.data(), sizeof(DCarbon) * n_chains,
                                    cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(scratch + o_scen, scen, sizeof(gl_scenario) * n_scen,
                            cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(scratch + o_rows, grid->row_scenario, sizeof(int32_t) * rows,
                            cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(scratch + o_cells, grid->cell_chain, sizeof(int32_t) * rows * cols,
                            cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) {
        const int warps = 8;
        const unsigned blocks = (unsigned)((rows + warps - 1) / warps);
        prof_begin("k_argmin", stream);
        gl::k_argmin<<<blocks, 32 * warps, 0, stream>>>(
            stats, reinterpret_cast<const DCarbon *>(scratch),
            reinterpret_cast<const gl_scenario *>(scratch + o_scen),
            reinterpret_cast<const int32_t *>(scratch + o_rows),
            reinterpret_cast<const int32_t *>(scratch + o_cells), (int32_t)rows, (int32_t)cols,
            slo_num, slo_den, priority, default_col, carbon_out, per_token_out, choice_out,
            via_fallback_out);
        e = cudaGetLastError();
        prof_end(stream);
    }
    cudaError_t ef = cudaFreeAsync(scratch, stream);
    if (e == cudaSuccess) e = ef;
    if (e != cudaSuccess) return GL_E_CUDA;
    g_last_launches = 1;
    return GL_OK;
}

gl_status gl_savings_surface(const gl_chain_stats *stats, int32_t n_chains,
                             const gl_chain *chains, const gl_savings_pair *pairs,
                             int32_t n_pairs, const gl_scenario *scen, int32_t n_scen,
                             gl_savings *out, void *stream_)
{
    g_last_launches = 0;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    if (!stats || n_chains <= 0 || !chains || !pairs || n_pairs <= 0 || !scen || n_scen <= 0 ||
        !out)
        return GL_E_INVALID;
    for (int32_t i = 0; i < n_scen; ++i) {
        const gl_scenario &s = scen[i];
        if (!(std::isfinite(s.ci_g_per_kwh) && s.ci_g_per_kwh >= 0.0)) return GL_E_DOMAIN;
        if (!(std::isfinite(s.lt_new_s) && s.lt_new_s > 0.0)) return GL_E_DOMAIN;
        if (!(std::isfinite(s.lt_old_s) && s.lt_old_s > 0.0)) return GL_E_DOMAIN;
    }
    std::vector<gl::DPairC> pc(n_pairs);
    for (int32_t i = 0; i < n_pairs; ++i) {
        const int32_t d = pairs[i].disagg_chain, sa = pairs[i].standalone_chain;
        if (d < 0 || d >= n_chains || sa < 0 || sa >= n_chains) return GL_E_LOOKUP;
        for (int32_t c : {d, sa}) {
            if (!(std::isfinite(chains[c].ce_new_g) && chains[c].ce_new_g > 0.0)) return GL_E_DOMAIN;
            if (!(std::isfinite(chains[c].ce_old_g) && chains[c].ce_old_g >= 0.0)) return GL_E_DOMAIN;
        }
        pc[i] = gl::DPairC{d, sa, chains[d].ce_new_g, chains[d].ce_old_g, chains[sa].ce_new_g,
                           chains[sa].ce_old_g};
    }
    gl_status st = device_check();
    if (st) return st;
    const size_t o_scen = align256(sizeof(gl::DPairC) * n_pairs);
    const size_t total = o_scen + align256(sizeof(gl_scenario) * n_scen);
    unsigned char *scratch = nullptr;
    if ((st = cuda_status(cudaMallocAsync(reinterpret_cast<void **>(&scratch), total, stream))))
        return st;
    cudaError_t e = cudaMemcpyAsync(scratch, pc.data(), sizeof(gl::DPairC) * n_pairs,
                                    cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(scratch + o_scen, scen, sizeof(gl_scenario) * n_scen,
                            cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) {
        const int64_t cells = (int64_t)n_pairs * n_scen;
        prof_begin("k_savings", stream);
        gl::k_savings<<<(unsigned)((cells + 255) / 256), 256, 0, stream>>>(
            stats, reinterpret_cast<const gl::DPairC *>(scratch),
            reinterpret_cast<const gl_scenario *>(scratch + o_scen), n_pairs, n_scen, out);
        e = cudaGetLastError();
        prof_end(stream);
    }
    cudaError_t ef = cudaFreeAsync(scratch, stream);
    if (e == cudaSuccess) e = ef;
    if (e != cudaSuccess) return GL_E_CUDA;
    g_last_launches = 1;
    return GL_OK;
}

gl_status gl_complete_matrices(const double *x, const uint8_t *observed, int32_t batch,
                               int32_t rows, int32_t cols, int32_t rank, double lambda,
                               int32_t iters, const double *v0, double lo, double hi,
                               double *out, double *u_out, double *v_out, int32_t *status_out,
                               void *stream_)
{
    g_last_launches = 0;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    if (!x || !observed || !v0 || !out || !status_out) return GL_E_INVALID;
    if (batch <= 0 || rows <= 0 || cols <= 0 || cols > 1024 || iters < 0) return GL_E_INVALID;
    if (rank < 1 || rank > GL_MAX_RANK || rank > rows || rank > cols) return GL_E_INVALID;
    if (!(std::isfinite(lambda) && lambda >= 0.0) || std::isnan(lo) || std::isnan(hi) || lo > hi)
        return GL_E_DOMAIN;
    gl_status st = device_check();
    if (st) return st;
    double *u = u_out;
    if (!u) {
        if ((st = cuda_status(cudaMallocAsync(reinterpret_cast<void **>(&u),
                                              sizeof(double) * (size_t)batch * rows * rank, stream))))
            return st;
    }
    const gl::DAls p{x, observed, v0, u, v_out, out, status_out, (int64_t)rows, cols, iters,
                     lambda, lo, hi};
    const size_t smem = gl::als_smem_bytes(cols, rank);
    cudaError_t e = cudaSuccess;
    // small batches: P CTAs per matrix with a grid-wide barrier per iteration
    // (cooperative launch), so the whole GPU works on a handful of matrices
    int dev = 0, n_sm = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    const size_t smem_c = sizeof(double) * (size_t)cols * rank;
    auto launch_coop = [&](auto kern) -> cudaError_t {
        int per_sm = 0;
        cudaError_t r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern,
                                                                      gl::ALSC_THREADS, smem_c);
        if (r != cudaSuccess) return r;
        const int64_t fit = (int64_t)per_sm * n_sm;
        int P = (int)std::min<int64_t>(fit / batch, (rows + 63) / 64);
        P = std::min(P, 2 * n_sm);
        if (P < 2) return cudaErrorNotSupported;  // the one-CTA kernel below
        const int ns = rank * (rank + 1) / 2 + rank;
        const int cw = (cols + 31) / 32;
        const size_t part_b = sizeof(double) * 2 * (size_t)batch * P * cols * ns;
        const size_t mask_b = sizeof(uint32_t) * (size_t)batch * cw + sizeof(int32_t) * batch;
        unsigned char *scr = nullptr;
        r = cudaMallocAsync(reinterpret_cast<void **>(&scr), align256(part_b) + mask_b, stream);
        if (r != cudaSuccess) return r;
        double *part = reinterpret_cast<double *>(scr);
        uint32_t *cmask = reinterpret_cast<uint32_t *>(scr + align256(part_b));
        int32_t *rflag = reinterpret_cast<int32_t *>(cmask + (size_t)batch * cw);
        r = cudaMemsetAsync(cmask, 0, mask_b, stream);
        if (r == cudaSuccess) {
            gl::DAls pp = p;
            int Pv = P;
            void *args[] = {&pp, &part, &cmask, &rflag, &Pv};
            prof_begin("k_als", stream);
            r = cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(kern),
                                            dim3((unsigned)(batch * P)), dim3(gl::ALSC_THREADS),
                                            args, smem_c, stream);
            prof_end(stream);
        }
        cudaError_t rf = cudaFreeAsync(scr, stream);
        return r != cudaSuccess ? r : rf;
    };
    bool done = false;
    if (coop && smem_c <= 48 * 1024) {
        cudaError_t r;
        switch (rank) {
            case 1: r = launch_coop(gl::k_als_coop<1>); break;
            case 2: r = launch_coop(gl::k_als_coop<2>); break;
            case 3: r = launch_coop(gl::k_als_coop<3>); break;
            case 4: r = launch_coop(gl::k_als_coop<4>); break;
            case 5: r = launch_coop(gl::k_als_coop<5>); break;
            case 6: r = launch_coop(gl::k_als_coop<6>); break;
            case 7: r = launch_coop(gl::k_als_coop<7>); break;
            default: r = launch_coop(gl::k_als_coop<8>); break;
        }
        if (r == cudaSuccess) done = true;
        else if (r != cudaErrorNotSupported) e = r;
        cudaGetLastError();  // clear a NotSupported marker
    }
    auto launch = [&](auto kern) {
        cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (r != cudaSuccess) return r;
        prof_begin("k_als", stream);
        kern<<<(unsigned)batch, gl::ALS_THREADS, smem, stream>>>(p);
        r = cudaGetLastError();
        prof_end(stream);
        return r;
    };
    if (!done && e == cudaSuccess) switch (rank) {
        case 1: e = launch(gl::k_als<1>); break;
        case 2: e = launch(gl::k_als<2>); break;
        case 3: e = launch(gl::k_als<3>); break;
        case 4: e = launch(gl::k_als<4>); break;
        case 5: e = launch(gl::k_als<5>); break;
        case 6: e = launch(gl::k_als<6>); break;
        case 7: e = launch(gl::k_als<7>); break;
        default: e = launch(gl::k_als<8>); break;
    }
    if (!u_out) {
        cudaError_t ef = cudaFreeAsync(u, stream);
        if (e == cudaSuccess) e = ef;
    }
    if (e != cudaSuccess) return GL_E_CUDA;
    g_last_launches = 1;
    return GL_OK;
}

gl_status gl_argmin_matrices(const double *carbon, const double *att, const uint8_t *present,
                             int32_t rows, int32_t cols, double slo_target, int32_t priority,
                             int32_t default_col, int32_t *choice_out, uint8_t *via_fallback_out,
                             void *stream_)
{
    g_last_launches = 0;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    if (!carbon || !att || !choice_out || !via_fallback_out || rows <= 0 || cols <= 0)
        return GL_E_INVALID;
    if (priority != GL_PRIORITY_SLO && priority != GL_PRIORITY_DEFAULT) return GL_E_INVALID;
    if (!(std::isfinite(slo_target) && slo_target >= 0.0 && slo_target <= 1.0)) return GL_E_DOMAIN;
    if (priority == GL_PRIORITY_DEFAULT && (default_col < -1 || default_col >= cols))
        return GL_E_LOOKUP;
    gl_status st = device_check();
    if (st) return st;
    const int warps = 8;
    prof_begin("k_argmin_matrices", stream);
    gl::k_argmin_matrices<<<(unsigned)((rows + warps - 1) / warps), 32 * warps, 0, stream>>>(
        carbon, att, present, rows, cols, slo_target, priority, default_col, choice_out,
        via_fallback_out);
    const cudaError_t e = cudaGetLastError();
    prof_end(stream);
    if (e != cudaSuccess) return GL_E_CUDA;
    g_last_launches = 1;
    return GL_OK;
}

gl_status gl_evaluate_host(const gl_trace *host_traces, int32_t n_traces, const gl_chain *chains,
                           int32_t n_chains, const gl_scenario *scen, int32_t n_scen,
                           const gl_grid *grid, int32_t slo_num, int32_t slo_den,
                           int32_t priority, int32_t default_col, gl_chain_stats *stats_host,
                           double *carbon_host, double *per_token_host, int32_t *choice_host,
                           uint8_t *via_fallback_host, void *stream_)
{
    return gl_evaluate_host_sched(host_traces, n_traces, chains, n_chains, scen, n_scen, grid,
                                  slo_num, slo_den, priority, default_col, stats_host,
                                  carbon_host, per_token_host, choice_host, via_fallback_host,
                                  nullptr, stream_);
}

gl_status gl_evaluate_host_sched(const gl_trace *host_traces, int32_t n_traces,
                                 const gl_chain *chains, int32_t n_chains,
                                 const gl_scenario *scen, int32_t n_scen, const gl_grid *grid,
                                 int32_t slo_num, int32_t slo_den, int32_t priority,
                                 int32_t default_col, gl_chain_stats *stats_host,
                                 double *carbon_host, double *per_token_host,
                                 int32_t *choice_host, uint8_t *via_fallback_host,
                                 const gl_schedule *sched, void *stream_)
{
    if (sched && (sched->first_lo < 0 || sched->first_lo > sched->first_hi ||
                  sched->first_hi > n_chains))
        return GL_E_INVALID;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    gl_status st = validate_traces(host_traces, n_traces);
    if (st) return st;
    if (!grid || grid->rows <= 0 || grid->cols <= 0 || !stats_host || !choice_host ||
        !via_fallback_host || n_chains <= 0)
        return GL_E_INVALID;
    if ((st = device_check())) return st;
    const int64_t rows = grid->rows, cols = grid->cols;
    // Each distinct host array is copied once: traces that share a host array
    // (e.g. rate-independent lengths) share the device copy, and with it their DSD
    // demand group in gl_eval_grid.
    std::map<std::pair<const void *, size_t>, size_t> arr_off;  // (host ptr, bytes) -> offset
    std::vector<std::pair<const void *, size_t>> arr_list;
    size_t total = 0;
    auto place = [&](const void *h, size_t bytes) {
        auto key = std::make_pair(h, bytes);
        if (arr_off.find(key) == arr_off.end()) {
            arr_off[key] = total;
            arr_list.push_back(key);
            total += align256(bytes);
        }
    };
    for (int32_t t = 0; t < n_traces; ++t) {
        const size_t n = (size_t)host_traces[t].n;
        place(host_traces[t].arrival_us, 8 * n);
        place(host_traces[t].prompt_len, 4 * n);
        place(host_traces[t].output_len, 4 * n);
    }
    const size_t o_stats = total;
    total += align256(sizeof(gl_chain_stats) * n_chains);
    const size_t o_carbon = total;
    total += carbon_host ? align256(sizeof(double) * rows * cols) : 0;
    const size_t o_ptok = total;
    total += per_token_host ? align256(sizeof(double) * rows * cols) : 0;
    const size_t o_choice = total;
    total += align256(sizeof(int32_t) * rows);
    const size_t o_fb = total;
    total += align256(rows);
    unsigned char *dev = nullptr;
    if ((st = cuda_status(cudaMallocAsync(reinterpret_cast<void **>(&dev), total, stream)))) return st;
    std::vector<gl_trace> dtr(n_traces);
    cudaError_t e = cudaSuccess;
    // Arrival arrays go on a side stream forked from `stream`, so their copy overlaps
    // k_dsd_demand (which needs only the output lengths, copied first on `stream`);
    // k_stages waits for the side stream's event.  No fork: everything on `stream`.
    std::set<const void *> arrivals;
    for (int32_t t = 0; t < n_traces; ++t) arrivals.insert(host_traces[t].arrival_us);
    cudaStream_t side = nullptr;
    cudaEvent_t ev_arr = nullptr;
    if (!side_fork(1, stream, side, ev_arr)) side = nullptr;
    for (int pass = 0; pass < 2; ++pass)  // lengths first, then arrivals
        for (size_t k = 0; k < arr_list.size() && e == cudaSuccess; ++k) {
            const bool arr = arrivals.count(arr_list[k].first) != 0;
            if (arr != (pass == 1)) continue;
            e = cudaMemcpyAsync(dev + arr_off[arr_list[k]], arr_list[k].first, arr_list[k].second,
                                cudaMemcpyHostToDevice, (arr && side) ? side : stream);
        }
    if (side) {  // recorded whatever happened above, so the joins below never wait
                 // on a stale record while copies queued on `side` are in flight
        const cudaError_t r = cudaEventRecord(ev_arr, side);
        if (e == cudaSuccess) e = r;
    }
    for (int32_t t = 0; t < n_traces; ++t) {
        const gl_trace &h = host_traces[t];
        const size_t n = (size_t)h.n;
        dtr[t].arrival_us = reinterpret_cast<int64_t *>(dev + arr_off[{h.arrival_us, 8 * n}]);
        dtr[t].prompt_len = reinterpret_cast<uint32_t *>(dev + arr_off[{h.prompt_len, 4 * n}]);
        dtr[t].output_len = reinterpret_cast<uint32_t *>(dev + arr_off[{h.output_len, 4 * n}]);
        dtr[t].n = h.n;
    }
    int launches = 0;
    if (e == cudaSuccess) {
        gl_chain_stats *dstats = reinterpret_cast<gl_chain_stats *>(dev + o_stats);
        g_last_launches = 0;
        st = eval_impl(dtr.data(), n_traces, chains, n_chains, dstats, nullptr, stream, nullptr,
                       side ? ev_arr : nullptr, sched);
        launches += g_last_launches;
        if (st == GL_OK) {
            st = gl_argmin_feasible(dstats, n_chains, chains, scen, n_scen, grid, slo_num, slo_den,
                                    priority, default_col,
                                    carbon_host ? reinterpret_cast<double *>(dev + o_carbon) : nullptr,
                                    per_token_host ? reinterpret_cast<double *>(dev + o_ptok) : nullptr,
                                    reinterpret_cast<int32_t *>(dev + o_choice),
                                    reinterpret_cast<uint8_t *>(dev + o_fb), stream_);
            launches += g_last_launches;
        }
        if (st == GL_OK) {
            e = cudaMemcpyAsync(stats_host, dstats, sizeof(gl_chain_stats) * n_chains,
                                cudaMemcpyDeviceToHost, stream);
            if (e == cudaSuccess && carbon_host)
                e = cudaMemcpyAsync(carbon_host, dev + o_carbon, sizeof(double) * rows * cols,
                                    cudaMemcpyDeviceToHost, stream);
            if (e == cudaSuccess && per_token_host)
                e = cudaMemcpyAsync(per_token_host, dev + o_ptok, sizeof(double) * rows * cols,
                                    cudaMemcpyDeviceToHost, stream);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(choice_host, dev + o_choice, sizeof(int32_t) * rows,
                                    cudaMemcpyDeviceToHost, stream);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(via_fallback_host, dev + o_fb, rows, cudaMemcpyDeviceToHost,
                                    stream);
        }
    }
    if (side) {  // join the side stream (a no-op when k_stages already waited on it)
        cudaError_t r = cudaStreamWaitEvent(stream, ev_arr, 0);
        // on any error the join may not cover the copies queued on `side`: wait for
        // them before the scratch they write is freed
        if (r != cudaSuccess || e != cudaSuccess || st != GL_OK) cudaStreamSynchronize(side);
        if (e == cudaSuccess) e = r;
    }
    cudaError_t ef = cudaFreeAsync(dev, stream);
    cudaError_t es = cudaStreamSynchronize(stream);
    if (st != GL_OK) return st;
    if (e == cudaSuccess) e = ef;
    if (e == cudaSuccess) e = es;
    if (e != cudaSuccess) return GL_E_CUDA;
    g_last_launches = launches;
    return GL_OK;
}

int32_t gl_last_launch_count(void) { return g_last_launches; }

gl_status gl_profile_enable(int32_t on)
{
    g_prof.on = on != 0;
    g_prof.used = 0;
    return GL_OK;
}

int32_t gl_kernel_timeline(const char **names_out, float *start_ms_out, float *ms_out,
                           int32_t max)
{
    int32_t k = 0;
    for (int i = 0; i < g_prof.used && k < max; ++i) {
        float ms = 0.f, t0 = 0.f;
        if (cudaEventElapsedTime(&ms, g_prof.ev[2 * i], g_prof.ev[2 * i + 1]) != cudaSuccess)
            ms = -1.f;
        if (i > 0 && cudaEventElapsedTime(&t0, g_prof.ev[0], g_prof.ev[2 * i]) != cudaSuccess)
            t0 = -1.f;
        if (names_out) names_out[k] = g_prof.names[i];
        if (start_ms_out) start_ms_out[k] = t0;
        if (ms_out) ms_out[k] = ms;
        ++k;
    }
    cudaGetLastError();
    g_prof.used = 0;
    return k;
}

int32_t gl_kernel_times(const char **names_out, float *ms_out, int32_t max)
{
    return gl_kernel_timeline(names_out, nullptr, ms_out, max);
}

const char *gl_strerror(gl_status s)
{
    switch (s) {
        case GL_OK: return "ok";
        case GL_E_INVALID: return "invalid argument";
        case GL_E_DOMAIN: return "value outside its domain";
        case GL_E_LOOKUP: return "index out of range";
        case GL_E_CUDA: return "CUDA runtime error";
        case GL_E_UNSUPPORTED: return "unsupported device or size (needs sm_100)";
        default: return "unknown status";
    }
}

int32_t gl_version(void) { return GL_VERSION; }

}  // extern "C"
