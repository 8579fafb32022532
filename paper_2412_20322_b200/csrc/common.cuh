// common.cuh -- device descriptors and warp / PTX helpers shared by the kernels
// of libgreenllm.so (sm_100a).  Part of the CUDA path only.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "greenllm.h"

namespace gl {

constexpr int RING = 256;       // decode-request ring per chain (shared memory)
constexpr int RING_MASK = RING - 1;
constexpr int CHUNK = 128;      // requests per produce step: 4 per lane, 128-bit loads
constexpr int LOOKAHEAD = 64;   // decode candidates kept staged ahead of the ring head
constexpr uint32_t ACCEPT_STREAM = 0x41434350u;  // "ACCP": third Philox counter word (R22)
constexpr int64_t NEG_INF = INT64_MIN / 4;
constexpr uint32_t F_EMPTY = 0xFFFFFFFFu;
constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr uint32_t O_LIMIT = 1u << 30;

constexpr int SEG_LEN = 256;  // decode requests per candidate window (k_segments)

// per-candidate result of a speculative run (k_decode)
struct DSegOut {
    int64_t maxfin;   // last finish time of the run
    int64_t sums[4];  // decode busy_new, busy_old, e_new, e_old of that run
    int32_t state;    // 0 unclaimed, 1 claimed, 2 published (release)
    int32_t next;     // candidate index at which the run stopped (idle there)
    int32_t helper;   // whose finish-time buffer holds the run
    int32_t nev;      // LOG launches: batch-size log entries of the run (from 2 q0)
};
constexpr int32_t SEG_FREE = 0, SEG_CLAIMED = 1, SEG_DONE = 2;

// per-chain decode bookkeeping (stream-ordered scratch, zeroed by the host)
struct DChainX {
    int32_t M;           // decode requests (o > 1), set by k_stages
    int32_t nseg;        // idle-point candidates, set by k_segments
    int32_t leader_pos;  // candidate the leader is at (helpers skip and abort below)
    int32_t next_seg;    // helper work counter
    int32_t n_ev;        // LOG launches: batch-size log entries written
    int32_t stage_done;  // k_stages CTAs of this chain that have finished
    int32_t seg_done;    // k_segments CTAs of this chain that have finished
    int32_t pad;         // k_relax race: slot + 1 (RX_SLOT_MASK), RX_SERIAL, RX_RELAXED
};
constexpr int32_t RX_SLOT_MASK = 0xFFFF;
constexpr int32_t RX_SERIAL = 1 << 16;   // k_decode's leader finished the chain first
constexpr int32_t RX_RELAXED = 1 << 17;  // k_relax solved the chain first

// one k_stages CTA's share of a chain (k_stages splits a chain over S CTAs): its
// aggregates are published with release flags for the CTAs after it, its partial
// statistics are combined by the chain's last CTA (stream-ordered scratch, zeroed)
struct DStagePart {
    int64_t agg1_A, agg1_B;  // stage-1 max-plus map of the CTA's requests
    int64_t agg2_A, agg2_B;  // stage-2 map
    int64_t sums[6];         // busy_new, busy_old, e_new, e_old, tokens, max finish (o = 1)
    int32_t dcount;          // decode requests of the CTA
    uint32_t status;
    int32_t flag1, flag2;    // release flags of the two aggregates
};

// one timing chain as the kernels see it (built by the host from gl_chain + gl_trace)
struct DChain {
    const int64_t *a;
    const uint32_t *p;
    const uint32_t *o;
    const uint32_t *K;  // DSD: speculative steps per request (k_dsd_demand); DPD: null
    const int32_t *t1, *t2, *b2;
    const int64_t *e1, *e2;
    const int32_t *step, *sbn, *sbo;
    const int64_t *sen, *seo;
    // decode stream written by k_stages: ready time r and (demand, request index)
    // per decode request q, in FCFS order, with two INT64_MAX sentinels after M.
    // Co-located modes: every request, r = arrival, plus its prefill time.
    int64_t *dec_r;
    uint2 *dec_dj;
    int32_t *dec_pf;    // co-located modes: prefill time t1[p] per stream entry
    int64_t *spec_fin;  // helper h's speculative finish times: spec_fin[h * spec_stride + q]
    int64_t spec_stride;
    int32_t *seg_start; // [nseg + 1] candidate starts (q), seg_start[nseg] = M
    DSegOut *seg_out;   // [nseg]
    DChainX *x;
    DStagePart *stp;    // [stage_split] k_stages partials of this chain
    longlong2 *ev;      // LOG launches: batch-size log [2 n + 16] of (T, b) (k_link.cuh);
                        // a run from decode request q0 writes from position 2 q0, unused
                        // positions keep the sentinel b = -1 (removed by k_link_scan)
    longlong2 *ev_spec; // LOG launches: helpers' logs, helper h at ev_spec + h * ev_stride
    int64_t ev_stride;
    int64_t n;
    int64_t ttft_slo, tpot_slo;
    int64_t out_off;  // first row of this chain in the per-request (ttft, finish) array
    int32_t mode, cap, max_prompt, capacity_ok;
};
// A size that is a multiple of 16 B keeps every chains[i] 16-B aligned, which k_decode's
// schedule depends on: an 8-B pad field made k_decode 2.6% slower.
static_assert(sizeof(DChain) % 16 == 0, "DChain: keep the size a multiple of 16 bytes");

// ceil(gap / st) for 0 < gap < 2^31, 1 <= st < 2^31 without a division:
// Lemire, Kaser & Kurz (2019): with M = floor((2^64 - 1) / d) + 1, floor(x / d) =
// mulhi64(M, x) for every 32-bit x.  (d = 1 is stored as M = 0 and handled apart.)
__device__ __forceinline__ uint32_t ceil_div_magic(uint32_t gap, uint32_t st, uint64_t M)
{
    const uint32_t x = gap + st - 1u;
    const uint64_t hi = (uint64_t)(uint32_t)(M >> 32) * x + __umulhi((uint32_t)M, x);
    return st == 1u ? gap : (uint32_t)(hi >> 32);
}

// one DSD demand group: requests sharing (output lengths, gamma, alpha, seed)
struct DGroup {
    const uint32_t *o;
    uint32_t *K;
    int64_t n;
    uint64_t seed;
    int32_t gamma, pad;
    uint64_t thr[GL_MAX_GAMMA];
};

// A DSD demand FAMILY: the groups that share (output lengths, n, seed) -- so the same
// acceptance draws u(j, s) -- and differ in (alpha, gamma).  Laid out as a table of
// alpha-sets (distinct threshold sequences, ascending alpha) x gamma = 1..FAM_GM;
// K[a][g] is the K array of group (a, gamma = g + 1), null if no chain uses it.
constexpr int FAM_NA = 5;  // alpha-sets per family (a family with more goes per group)
constexpr int FAM_GM = 8;  // largest gamma in a family
struct DFamily {
    const uint32_t *o;
    int64_t n;
    uint64_t seed;
    uint32_t thr[FAM_NA][FAM_GM];  // floor(alpha^c 2^32) < 2^32 (alpha < 1)
    uint32_t all[FAM_NA];          // alpha = 1: every draft token accepted
    int32_t na, pad;
    uint32_t *K[FAM_NA][FAM_GM];
};

struct DCarbon {
    double ce_new, ce_old;
    int32_t cap_ok, pad;
};

// Philox4x32-10 (Salmon et al. 2011), the CUDA path's own implementation
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

// SplitMix64 finaliser; the per-request hash is mix(j ^ rotl(ttft,21) ^ rotl(finish,42))
__device__ __forceinline__ uint64_t splitmix_fin(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ int64_t shfl_i64(int64_t v, int src) { return __shfl_sync(FULL, v, src); }
__device__ __forceinline__ int64_t shfl_up_i64(int64_t v, int d) { return __shfl_up_sync(FULL, v, d); }

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v)
{
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

__device__ __forceinline__ int64_t warp_max_i64(int64_t v)
{
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, (int64_t)__shfl_xor_sync(FULL, v, o));
    return v;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// The retry loop lives inside the PTX: a C++ spin loop would make the compiler
// add forward-progress YIELDs to every enclosing loop (the decode loops).
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase)
{
    asm volatile(
        "{\n .reg .pred p;\n"
        "GL_MBAR_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra GL_MBAR_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// TMA bulk copy global -> shared; completion is signalled on the mbarrier's tx count
__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__host__ __device__ __forceinline__ int round_up4(int x) { return (x + 3) & ~3; }

// Predicated forms (the predicate lives inside the PTX, so a warp-uniform caller
// needs no divergent branch and no reconvergence barrier around them).
__device__ __forceinline__ void mbar_arrive_expect_tx_if(bool p, uint64_t *bar, uint32_t bytes)
{
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n"
        " @q mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
        "r"(bytes), "r"((uint32_t)p)
        : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s_if(bool p, void *dst, const void *src, uint32_t bytes,
                                                uint64_t *bar)
{
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.u32 q, %4, 0;\n"
        " @q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "r"((uint32_t)p)
        : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu_if(bool p, int32_t *ptr, int32_t v)
{
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.relaxed.gpu.global.s32 [%0], %1;\n}\n" ::"l"(ptr),
        "r"(v), "r"((uint32_t)p)
        : "memory");
}

// Stage a [count] int32 table into shared memory: the 16-B aligned bulk by TMA
// (lane 0 issues), the ragged tail by plain loads.  Returns the TMA byte count.
__device__ __forceinline__ uint32_t stage_table(int32_t *dst, const int32_t *src, int count,
                                                uint64_t *bar, int lane)
{
    uint32_t bulk = 0;
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) bulk = (uint32_t)(count * 4) & ~15u;
    if (bulk && lane == 0) tma_bulk_g2s(dst, src, bulk, bar);
    for (int i = bulk / 4 + lane; i < count; i += 32) dst[i] = __ldg(src + i);
    return bulk;
}

// GPU-scope release store / acquire load (helper -> leader publication in k_decode)
__device__ __forceinline__ void st_release_gpu(int32_t *p, int32_t v)
{
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_acquire_gpu(const int32_t *p)
{
    int32_t v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int32_t ld_relaxed_gpu(const int32_t *p)
{
    int32_t v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu(int32_t *p, int32_t v)
{
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace gl
