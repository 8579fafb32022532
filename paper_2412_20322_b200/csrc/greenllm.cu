/*
 * greenllm.cu -- libgreenllm.so: sm_100a kernels + the C ABI of include/greenllm.h.
 *
 * The evaluated method (with the paper passages each step follows):
 *   stage 1  prefill FCFS on the new GPU      c_i = max(c_{i-1}, a_i) + t1[p_i]
 *            (TTFT = c - a)
 *   stage 2  KV link (DPD) / handoff + draft prefill (DSD)
 *                                              r_i = max(r_{i-1}, c_i) + t2[p_i]
 *   decode   continuous batching on the old GPU (DPD) or speculative steps
 *            across both (DSD, Fig. 7), batch <= cap, FCFS joins at
 *            iteration boundaries (R15-R18)
 *   SLO      TTFT <= SLO_ttft and finish - c <= SLO_tpot (o - 1) (Table 2)
 *   carbon   Eqs. 1-3;   Alg. 1 feasible argmin
 *
 * B200 design:
 *   k_dsd_demand  one thread per (DSD demand group, request): K_j = number of
 *                 speculative steps request j needs.  Draws are keyed by
 *                 (request, its own step), so K_j is independent of batching
 *                 and chains with equal (lengths, gamma, alpha, seed) share it.
 *   k_chain       one warp per timing chain.  TMA bulk copies (cp.async.bulk +
 *                 mbarrier) stage the prompt-indexed stage tables and the
 *                 batch-indexed step table into shared memory; 128-request
 *                 chunks are read with 128-bit loads (4 requests per lane);
 *                 stages 1-2 are warp max-plus scans on int64 (A, B) pairs;
 *                 decode requests are compacted into a shared-memory ring and
 *                 consumed by a warp-uniform event loop that jumps whole runs
 *                 of iterations (REDUX min of the members' finish iterations,
 *                 ballot/popc for leaves, SLO counts and FCFS joins).
 *   k_argmin      one warp per Alg. 1 row: fp64 carbon per cell in the fixed
 *                 R34 order with explicit round-to-nearest intrinsics (never
 *                 contracted to FMA), feasibility by integer cross-products,
 *                 lexicographic warp-shuffle argmin.
 * No tensor cores: nothing here is a contraction.
 */
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <tuple>
#include <vector>

#include "greenllm.h"

namespace {

constexpr int RING = 256;                 // decode-request ring per warp (shared memory)
constexpr int RING_MASK = RING - 1;
constexpr int CHUNK = 128;                // requests per produce step: 4 per lane
constexpr int LOOKAHEAD = 64;             // decode candidates kept ahead of the head
constexpr uint32_t ACCEPT_STREAM = 0x41434350u;  // "ACCP"
constexpr int64_t NEG_INF = INT64_MIN / 4;
constexpr uint32_t F_EMPTY = 0xFFFFFFFFu;
constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr uint32_t O_LIMIT = 1u << 30;

struct DChain {
    const int64_t *a;
    const uint32_t *p;
    const uint32_t *o;
    const uint32_t *K;  // DSD: steps per request (k_dsd_demand); DPD: null
    const int32_t *t1, *t2, *b2;
    const int64_t *e1, *e2;
    const int32_t *step, *sbn, *sbo;
    const int64_t *sen, *seo;
    int64_t n;
    int64_t ttft_slo, tpot_slo;
    int64_t out_off;
    int32_t mode, cap, max_prompt, capacity_ok;
};

struct DGroup {
    const uint32_t *o;
    uint32_t *K;
    int64_t n;
    uint64_t seed;
    int32_t gamma, pad;
    uint64_t thr[GL_MAX_GAMMA];
};

struct DCarbon {
    double ce_new, ce_old;
    int32_t cap_ok, pad;
};

// ------------------------------------------------------------------ helpers
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

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase)
{
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}

// TMA bulk copy global -> shared, completion tracked by the mbarrier's tx count
__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__host__ __device__ __forceinline__ int round_up4(int x) { return (x + 3) & ~3; }

// ------------------------------------------------------- k_dsd_demand
__global__ void __launch_bounds__(256) k_dsd_demand(const DGroup *__restrict__ groups)
{
    __shared__ uint64_t thr[GL_MAX_GAMMA];
    __shared__ int32_t gamma_s;
    __shared__ uint64_t seed_s;
    const DGroup *g = groups + blockIdx.y;
    if (threadIdx.x < GL_MAX_GAMMA) thr[threadIdx.x] = g->thr[threadIdx.x];
    if (threadIdx.x == 0) {
        gamma_s = g->gamma;
        seed_s = g->seed;
    }
    __syncthreads();
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= g->n) return;
    uint32_t o = __ldg(g->o + j);
    if (o >= O_LIMIT) o = O_LIMIT - 1;
    const int64_t need = (int64_t)o - 1;
    uint32_t s = 0;
    if (need > 0) {
        const uint32_t k0 = (uint32_t)seed_s, k1 = (uint32_t)(seed_s >> 32);
        const int gam = gamma_s;
        int64_t tok = 0;
        for (;;) {
            const uint4 w = philox4x32_10(make_uint4(s >> 2, (uint32_t)j, ACCEPT_STREAM, 0u), k0, k1);
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
            bool done = false;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (!done) {
                    int acc = 1;
                    for (int c = 0; c < gam; ++c) acc += ((uint64_t)ws[q] < thr[c]) ? 1 : 0;
                    tok += acc;
                    ++s;
                    done = tok >= need;
                }
            }
            if (done) break;
        }
    }
    g->K[j] = s;
}

// ------------------------------------------------------------ k_chain
struct SmemLayout {
    int p1pad, cappad;
    size_t off_t1, off_t2, off_step, off_r, off_D, off_h, off_dj, off_bar, total;
    __host__ __device__ SmemLayout(int max_prompt, int cap)
    {
        p1pad = round_up4(max_prompt + 1);
        cappad = round_up4(cap + 1);
        off_t1 = 0;
        off_t2 = off_t1 + 4 * (size_t)p1pad;
        off_step = off_t2 + 4 * (size_t)p1pad;
        off_r = (off_step + 4 * (size_t)cappad + 15) & ~(size_t)15;
        off_D = off_r + 8 * RING;
        off_h = off_D + 8 * RING;
        off_dj = off_h + 8 * RING;
        off_bar = off_dj + 8 * RING;
        total = off_bar + 16;
    }
};

// stage a [count] int32 table into shared memory: 16-B aligned bulk part by
// TMA (lane 0 issues), the ragged tail by plain loads.  Returns TMA bytes.
__device__ __forceinline__ uint32_t stage_table(int32_t *dst, const int32_t *src, int count,
                                                uint64_t *bar, int lane)
{
    uint32_t bulk = 0;
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) bulk = (uint32_t)(count * 4) & ~15u;
    if (bulk && lane == 0) tma_bulk_g2s(dst, src, bulk, bar);
    for (int i = bulk / 4 + lane; i < count; i += 32) dst[i] = __ldg(src + i);
    return bulk;
}

template <int SPL>
__global__ void __launch_bounds__(32, 1)
    k_chain(const DChain *__restrict__ chains, gl_chain_stats *__restrict__ stats,
            int64_t *__restrict__ perreq)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x;
    const DChain ch = chains[blockIdx.x];
    const SmemLayout L(ch.max_prompt, ch.cap);
    int32_t *t1s = reinterpret_cast<int32_t *>(smem + L.off_t1);
    int32_t *t2s = reinterpret_cast<int32_t *>(smem + L.off_t2);
    int32_t *steps = reinterpret_cast<int32_t *>(smem + L.off_step);
    int64_t *ring_r = reinterpret_cast<int64_t *>(smem + L.off_r);
    int64_t *ring_D = reinterpret_cast<int64_t *>(smem + L.off_D);
    uint64_t *ring_h = reinterpret_cast<uint64_t *>(smem + L.off_h);
    uint2 *ring_dj = reinterpret_cast<uint2 *>(smem + L.off_dj);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L.off_bar);

    // ---- S0: stage tables (TMA bulk copies + mbarrier) ----------------------
    if (lane == 0) mbar_init(bar, 1);
    __syncwarp();
    const int P = ch.max_prompt, cap = ch.cap;
    uint32_t tx = 0;
    tx += stage_table(t1s, ch.t1, P + 1, bar, lane);
    tx += stage_table(t2s, ch.t2, P + 1, bar, lane);
    tx += stage_table(steps, ch.step, cap + 1, bar, lane);
    if (lane == 0) mbar_arrive_expect_tx(bar, tx);
    mbar_wait(bar, 0);
    __syncwarp();

    uint32_t status = 0;
    {
        bool bad = false;
        for (int i = 1 + lane; i <= P; i += 32) bad |= (t1s[i] < 0) | (t2s[i] < 0);
        for (int b = 1 + lane; b <= cap; b += 32) bad |= steps[b] < 1;
        if (__any_sync(FULL, bad)) status |= GL_ST_TABLE;
    }

    // lane-local accumulators
    int64_t acc_busy_new = 0, acc_busy_old = 0, acc_e_new = 0, acc_e_old = 0, acc_tokens = 0;
    int64_t acc_ok = 0, acc_mk = 0;
    uint64_t acc_hash = 0;
    uint64_t iters[SPL + 1];
#pragma unroll
    for (int s = 0; s <= SPL; ++s) iters[s] = 0;

    const int64_t n = ch.n;
    const bool dsd = ch.mode == GL_MODE_DSD;
    const bool dump = perreq != nullptr;
    int64_t chunk_next = 0, produced = 0;
    int64_t carry_c = NEG_INF, carry_r = NEG_INF, carry_a = INT64_MIN;

    // ---- S1-S4: one 128-request chunk -> scans -> compacted decode ring -----
    auto produce = [&]() {
        const int64_t i0 = chunk_next + 4 * lane;
        int64_t av[4];
        uint32_t pv[4], ov[4], kv[4];
        if (i0 + 3 < n) {  // 128-bit loads: 2 x (2 x int64), 1 x (4 x u32) per stream
            const longlong2 x0 = __ldg(reinterpret_cast<const longlong2 *>(ch.a + i0));
            const longlong2 x1 = __ldg(reinterpret_cast<const longlong2 *>(ch.a + i0) + 1);
            const uint4 pp = __ldg(reinterpret_cast<const uint4 *>(ch.p + i0));
            const uint4 oo = __ldg(reinterpret_cast<const uint4 *>(ch.o + i0));
            av[0] = x0.x; av[1] = x0.y; av[2] = x1.x; av[3] = x1.y;
            pv[0] = pp.x; pv[1] = pp.y; pv[2] = pp.z; pv[3] = pp.w;
            ov[0] = oo.x; ov[1] = oo.y; ov[2] = oo.z; ov[3] = oo.w;
            if (dsd) {
                const uint4 kk = __ldg(reinterpret_cast<const uint4 *>(ch.K + i0));
                kv[0] = kk.x; kv[1] = kk.y; kv[2] = kk.z; kv[3] = kk.w;
            } else {
                kv[0] = kv[1] = kv[2] = kv[3] = 0;
            }
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const bool v = i0 + q < n;
                av[q] = v ? __ldg(ch.a + i0 + q) : 0;
                pv[q] = v ? __ldg(ch.p + i0 + q) : 1;
                ov[q] = v ? __ldg(ch.o + i0 + q) : 1;
                kv[q] = (v && dsd) ? __ldg(ch.K + i0 + q) : 0;
            }
        }
        bool valid[4], dec[4];
        int64_t s1[4], s2[4], x_a[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            valid[q] = i0 + q < n;
            uint32_t pc = pv[q], oc = ov[q];
            if (valid[q]) {
                if (av[q] < 0) status |= GL_ST_NEG_ARRIVAL;
                if (pc < 1 || pc > (uint32_t)P) status |= GL_ST_PROMPT_RANGE;
                if (oc == 0) status |= GL_ST_OUTPUT_ZERO;
                if (oc >= O_LIMIT) status |= GL_ST_OVERFLOW;
            }
            pc = min(max(pc, 1u), (uint32_t)P);
            oc = min(max(oc, 1u), O_LIMIT - 1);
            pv[q] = pc;
            ov[q] = oc;
            dec[q] = valid[q] && oc > 1;
            s1[q] = valid[q] ? t1s[pc] : 0;
            s2[q] = dec[q] ? t2s[pc] : 0;
            x_a[q] = valid[q] ? av[q] : NEG_INF;
            if (valid[q]) {
                acc_busy_new += s1[q];
                acc_e_new += __ldg(ch.e1 + pc);
                acc_tokens += oc;
            }
            if (dec[q]) {
                acc_busy_old += __ldg(ch.b2 + pc);
                acc_e_old += __ldg(ch.e2 + pc);
            }
        }
        // sortedness across the lane boundary and the chunk boundary
        {
            int64_t prev = shfl_up_i64(av[3], 1);
            if (lane == 0) prev = carry_a;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (valid[q] && av[q] < prev) status |= GL_ST_UNSORTED;
                if (valid[q]) prev = av[q];
            }
            const int64_t last = shfl_i64(prev, 31);
            carry_a = last;
        }
        // S3: prefill FCFS max-plus scan, element = (A = s1, B = a + s1)
        int64_t c[4];
        {
            int64_t A = 0, B = NEG_INF;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                A += s1[q];
                B = max(B + s1[q], x_a[q] + s1[q]);
            }
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int64_t Ap = shfl_up_i64(A, off), Bp = shfl_up_i64(B, off);
                if (lane >= off) {
                    B = max(Bp + A, B);
                    A = Ap + A;
                }
            }
            int64_t Ax = shfl_up_i64(A, 1), Bx = shfl_up_i64(B, 1);
            if (lane == 0) {
                Ax = 0;
                Bx = NEG_INF;
            }
            int64_t x = max(carry_c + Ax, Bx);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                x = max(x, x_a[q]) + s1[q];
                c[q] = valid[q] ? x : NEG_INF;
            }
            carry_c = shfl_i64(x, 31);
        }
        // S4: stage-2 FIFO max-plus scan, element = (A = s2, B = c + s2)
        int64_t r[4];
        {
            int64_t A = 0, B = NEG_INF;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                A += s2[q];
                B = max(B + s2[q], c[q] + s2[q]);
            }
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int64_t Ap = shfl_up_i64(A, off), Bp = shfl_up_i64(B, off);
                if (lane >= off) {
                    B = max(Bp + A, B);
                    A = Ap + A;
                }
            }
            int64_t Ax = shfl_up_i64(A, 1), Bx = shfl_up_i64(B, 1);
            if (lane == 0) {
                Ax = 0;
                Bx = NEG_INF;
            }
            int64_t y = max(carry_r + Ax, Bx);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                y = max(y, c[q]) + s2[q];
                r[q] = y;
            }
            carry_r = shfl_i64(y, 31);
        }
        // per request: TTFT, single-token requests finish at c, others -> ring
        int cnt = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) cnt += dec[q] ? 1 : 0;
        const unsigned b0 = __ballot_sync(FULL, cnt & 1), b1 = __ballot_sync(FULL, cnt & 2),
                       b2 = __ballot_sync(FULL, cnt & 4);
        const unsigned lt = (1u << lane) - 1u;
        int pos = __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
        const int total = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (!valid[q]) continue;
            const int64_t j = i0 + q;
            const int64_t ttft = c[q] - av[q];
            const bool ok_t = ttft <= ch.ttft_slo;
            if (dump) perreq[2 * (ch.out_off + j)] = ttft;
            if (!dec[q]) {
                acc_ok += ok_t ? 1 : 0;
                acc_hash += splitmix_fin((uint64_t)j ^ rotl64((uint64_t)ttft, 21) ^
                                         rotl64((uint64_t)c[q], 42));
                acc_mk = max(acc_mk, c[q]);
                if (dump) perreq[2 * (ch.out_off + j) + 1] = c[q];
            } else {
                const int e = (int)((produced + pos) & RING_MASK);
                ring_r[e] = r[q];
                ring_D[e] = ok_t ? c[q] + ch.tpot_slo * (int64_t)(ov[q] - 1) : INT64_MIN;
                ring_h[e] = (uint64_t)j ^ rotl64((uint64_t)ttft, 21);
                ring_dj[e] = make_uint2(dsd ? kv[q] : ov[q] - 1, (uint32_t)j);
                ++pos;
            }
        }
        produced += total;
        chunk_next += CHUNK;
        __syncwarp();
    };

    if (status & GL_ST_TABLE) chunk_next = n;  // nothing to simulate

    // ---- S5-S6: continuous-batching decode event loop ------------------------
    uint32_t F[SPL];
    int64_t Dl[SPL];
    uint64_t hl[SPL];
    uint32_t jl[SPL];
#pragma unroll
    for (int s = 0; s < SPL; ++s) {
        F[s] = F_EMPTY;
        Dl[s] = 0;
        hl[s] = 0;
        jl[s] = 0;
    }
    int64_t T = 0, mk_dec = 0;
    uint32_t I = 0;
    int b = 0;
    int64_t nxt = 0;
    auto ensure = [&]() {
        while (chunk_next < n && produced - nxt < LOOKAHEAD) produce();
    };
    ensure();
    for (;;) {
        // FCFS joins at boundary T (r <= T), while the batch has room (R16, R18)
        while (b < cap) {
            const int64_t avail = produced - nxt;
            if (avail <= 0) break;
            const bool rdy = (lane < avail) && ring_r[(nxt + lane) & RING_MASK] <= T;
            int m = __popc(__ballot_sync(FULL, rdy));  // a prefix: r is non-decreasing
            if (m == 0) break;
            m = min(m, cap - b);
            int q0 = 0;
#pragma unroll
            for (int s = 0; s < SPL; ++s) {
                if (q0 < m) {
                    const bool fr = (F[s] == F_EMPTY) && (s * 32 + lane < cap);
                    const unsigned fm = __ballot_sync(FULL, fr);
                    const int q = q0 + __popc(fm & ((1u << lane) - 1u));
                    if (fr && q < m) {
                        const int e = (int)((nxt + q) & RING_MASK);
                        const uint2 dj = ring_dj[e];
                        F[s] = I + dj.x;
                        Dl[s] = ring_D[e];
                        hl[s] = ring_h[e];
                        jl[s] = dj.y;
                    }
                    q0 += __popc(fm);
                }
            }
            nxt += m;
            b += m;
            ensure();
        }
        if (b == 0) {  // idle until the next decode request is ready (R17)
            if (nxt >= produced) break;
            T = ring_r[nxt & RING_MASK];
            continue;
        }
        // next event: first member leave, or the boundary at which the head joins
        const int64_t st = steps[b];
        uint32_t fmin = F[0];
#pragma unroll
        for (int s = 1; s < SPL; ++s) fmin = min(fmin, F[s]);
        fmin = __reduce_min_sync(FULL, fmin);
        const uint32_t kL = fmin - I;
        uint32_t k = kL;
        if (b < cap && nxt < produced) {
            const int64_t gap = ring_r[nxt & RING_MASK] - T;  // > 0: not admitted at T
            if (gap <= (int64_t)(kL - 1) * st) {
                if (gap < 0x80000000ll)
                    k = ((uint32_t)gap + (uint32_t)st - 1u) / (uint32_t)st;
                else
                    k = (uint32_t)((gap + st - 1) / st);
            }
        }
        T += (int64_t)k * st;
        I += k;
#pragma unroll
        for (int s = 0; s <= SPL; ++s)
            if (s == (b >> 5) && lane == (b & 31)) iters[s] += k;
        if (k == kL) {  // leaves at boundary T (R16): finish = T, SLO via deadline
            int nl = 0;
#pragma unroll
            for (int s = 0; s < SPL; ++s) {
                const bool lv = F[s] == I;
                const unsigned lm = __ballot_sync(FULL, lv);
                if (lm) {
                    if (lv) {
                        acc_ok += (T <= Dl[s]) ? 1 : 0;
                        acc_hash += splitmix_fin(hl[s] ^ rotl64((uint64_t)T, 42));
                        if (dump) perreq[2 * (ch.out_off + jl[s]) + 1] = T;
                        F[s] = F_EMPTY;
                    }
                    nl += __popc(lm);
                }
            }
            b -= nl;
            mk_dec = T;
        }
        if (I >= 0x80000000u) {  // rebase the 32-bit iteration counter
#pragma unroll
            for (int s = 0; s < SPL; ++s)
                if (F[s] != F_EMPTY) F[s] -= I;
            I = 0;
        }
    }

    // ---- S7: chain reductions -------------------------------------------------
#pragma unroll
    for (int s = 0; s <= SPL; ++s) {
        const int bb = s * 32 + lane;
        if (bb >= 1 && bb <= cap && iters[s]) {
            const int64_t it = (int64_t)iters[s];
            acc_busy_new += it * __ldg(ch.sbn + bb);
            acc_busy_old += it * __ldg(ch.sbo + bb);
            acc_e_new += it * __ldg(ch.sen + bb);
            acc_e_old += it * __ldg(ch.seo + bb);
        }
    }
    const int64_t busy_new = warp_sum_i64(acc_busy_new), busy_old = warp_sum_i64(acc_busy_old);
    const int64_t e_new = warp_sum_i64(acc_e_new), e_old = warp_sum_i64(acc_e_old);
    const int64_t tokens = warp_sum_i64(acc_tokens), ok = warp_sum_i64(acc_ok);
    const int64_t mk = max(warp_max_i64(acc_mk), mk_dec);
    const uint64_t hash = (uint64_t)warp_sum_i64((int64_t)acc_hash);
    status = __reduce_or_sync(FULL, status);
    if (lane == 0) {
        gl_chain_stats out;
        out.n = n;
        out.slo_ok = ok;
        out.tokens = tokens;
        out.busy_new_us = busy_new;
        out.busy_old_us = busy_old;
        out.e_new_uj = e_new;
        out.e_old_uj = e_old;
        out.makespan_us = mk;
        out.req_hash = hash;
        out.status = status;
        out.capacity_ok = (uint32_t)ch.capacity_ok;
        stats[blockIdx.x] = out;
    }
}

// ----------------------------------------------------------- k_argmin
// Eqs. 1-3 in the fixed R34 order; _rn intrinsics are never contracted to FMA.
__device__ __forceinline__ double carbon_total(const gl_chain_stats &s, const DCarbon &cp,
                                               const gl_scenario &sc)
{
    const double kwh_new = __ddiv_rn((double)s.e_new_uj, 3.6e12);
    const double kwh_old = __ddiv_rn((double)s.e_old_uj, 3.6e12);
    const double op = __dmul_rn(__dadd_rn(kwh_new, kwh_old), sc.ci_g_per_kwh);
    const double emb_new =
        __dmul_rn(__ddiv_rn(__ddiv_rn((double)s.busy_new_us, 1e6), sc.lt_new_s), cp.ce_new);
    const double emb_old =
        __dmul_rn(__ddiv_rn(__ddiv_rn((double)s.busy_old_us, 1e6), sc.lt_old_s), cp.ce_old);
    return __dadd_rn(op, __dadd_rn(emb_new, emb_old));
}

struct Cand {
    double total;
    int64_t ok, n;
    int32_t col;   // -1 = none
    int32_t feas;  // 1 = feasible
};

__device__ __forceinline__ int cmp_att(int64_t ok1, int64_t n1, int64_t ok2, int64_t n2)
{
    const int64_t l = ok1 * n2, r = ok2 * n1;  // n < 2^31 => no overflow
    return (l > r) - (l < r);
}

// feasible phase: lower total, then higher attainment, then lower column
__device__ __forceinline__ bool better_feasible(const Cand &x, const Cand &y)
{
    if (x.col < 0) return false;
    if (y.col < 0) return true;
    if (x.total != y.total) return x.total < y.total;
    const int c = cmp_att(x.ok, x.n, y.ok, y.n);
    if (c) return c > 0;
    return x.col < y.col;
}

// fallback (priority SLO): higher attainment, then lower total, then lower column
__device__ __forceinline__ bool better_fallback(const Cand &x, const Cand &y)
{
    if (x.col < 0) return false;
    if (y.col < 0) return true;
    const int c = cmp_att(x.ok, x.n, y.ok, y.n);
    if (c) return c > 0;
    if (x.total != y.total) return x.total < y.total;
    return x.col < y.col;
}

__device__ __forceinline__ Cand shfl_cand(const Cand &c, int src)
{
    Cand o;
    o.total = __shfl_xor_sync(FULL, c.total, src);
    o.ok = __shfl_xor_sync(FULL, c.ok, src);
    o.n = __shfl_xor_sync(FULL, c.n, src);
    o.col = __shfl_xor_sync(FULL, c.col, src);
    o.feas = __shfl_xor_sync(FULL, c.feas, src);
    return o;
}

__global__ void __launch_bounds__(256)
    k_argmin(const gl_chain_stats *__restrict__ stats, const DCarbon *__restrict__ cpar,
             const gl_scenario *__restrict__ scen, const int32_t *__restrict__ row_scen,
             const int32_t *__restrict__ cells, int32_t rows, int32_t cols, int32_t slo_num,
             int32_t slo_den, int32_t priority, int32_t default_col, double *__restrict__ carbon_out,
             int32_t *__restrict__ choice_out, uint8_t *__restrict__ fb_out)
{
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (row >= rows) return;  // warp-uniform
    const gl_scenario sc = scen[row_scen[row]];
    Cand bf{0.0, 0, 1, -1, 0}, bb{0.0, 0, 1, -1, 0};
    for (int col = lane; col < cols; col += 32) {
        const int32_t k = cells[row * cols + col];
        if (k < 0) {
            if (carbon_out) carbon_out[row * cols + col] = __longlong_as_double(0x7ff8000000000000ll);
            continue;
        }
        const gl_chain_stats s = stats[k];
        const DCarbon cp = cpar[k];
        const double total = carbon_total(s, cp, sc);
        if (carbon_out) carbon_out[row * cols + col] = total;
        const bool cap_ok = cp.cap_ok != 0;
        const bool feas = cap_ok && (int64_t)slo_den * s.slo_ok >= (int64_t)slo_num * s.n;
        const Cand cf{total, s.slo_ok, s.n, col, 1};
        if (feas && better_feasible(cf, bf)) bf = cf;
        const Cand cb{cap_ok ? total : __longlong_as_double(0x7ff0000000000000ll),
                      cap_ok ? s.slo_ok : 0, s.n, col, 0};
        if (better_fallback(cb, bb)) bb = cb;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        const Cand of = shfl_cand(bf, off), ob = shfl_cand(bb, off);
        if (better_feasible(of, bf)) bf = of;
        if (better_fallback(ob, bb)) bb = ob;
    }
    if (lane == 0) {
        if (bf.col >= 0) {
            choice_out[row] = bf.col;
            fb_out[row] = 0;
        } else {
            choice_out[row] = (priority == GL_PRIORITY_SLO) ? bb.col : default_col;
            fb_out[row] = 1;
        }
    }
}

// ================================================================ host side
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

gl_status device_check()
{
    static int cached = -1;  // 1 = ok, 0 = unsupported
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return GL_E_CUDA;
    if (cached < 0) {
        int major = 0, minor = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
            return GL_E_CUDA;
        cached = (major == 10 && minor == 0) ? 1 : 0;
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;  // keep stream-ordered scratch cached in the pool
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    return cached ? GL_OK : GL_E_UNSUPPORTED;
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
    if (c.mode != GL_MODE_DPD && c.mode != GL_MODE_DSD) return GL_E_INVALID;
    if (c.trace_idx < 0 || c.trace_idx >= n_traces) return GL_E_LOOKUP;
    if (c.batch_cap < 1 || c.batch_cap > GL_MAX_CAP) return GL_E_INVALID;
    if (c.max_prompt < 1 || c.max_prompt > GL_MAX_PROMPT) return GL_E_INVALID;
    if (c.mode == GL_MODE_DSD && (c.gamma < 1 || c.gamma > GL_MAX_GAMMA)) return GL_E_INVALID;
    if (!c.t1_us || !c.e1_new_uj || !c.t2_us || !c.b2_old_us || !c.e2_old_uj || !c.step_us ||
        !c.step_busy_new_us || !c.step_busy_old_us || !c.step_e_new_uj || !c.step_e_old_uj)
        return GL_E_INVALID;
    if (c.mode == GL_MODE_DSD && !(c.alpha >= 0.0 && c.alpha <= 1.0)) return GL_E_DOMAIN;
    if (c.ttft_slo_us < 0 || c.tpot_slo_us < 0) return GL_E_DOMAIN;
    if (c.tpot_slo_us > ((int64_t)1 << 32)) return GL_E_DOMAIN;  // keeps deadlines in int64
    return GL_OK;
}

gl_status cuda_status(cudaError_t e) { return e == cudaSuccess ? GL_OK : GL_E_CUDA; }

}  // namespace

// ---------------------------------------------------------------- C ABI
extern "C" {

gl_status gl_eval_grid(const gl_trace *traces, int32_t n_traces, const gl_chain *chains,
                       int32_t n_chains, gl_chain_stats *stats_out, int64_t *per_request_out,
                       void *stream_)
{
    g_last_launches = 0;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    gl_status st = validate_traces(traces, n_traces);
    if (st) return st;
    if (!chains || n_chains <= 0 || !stats_out) return GL_E_INVALID;
    for (int32_t i = 0; i < n_chains; ++i)
        if ((st = validate_chain(chains[i], n_traces))) return st;
    if ((st = device_check())) return st;

    // DSD demand groups: equal (output_len, n, gamma, thresholds, seed) share K
    std::vector<DGroup> groups;
    std::map<std::tuple<const uint32_t *, int64_t, int32_t, uint64_t, std::vector<uint64_t>>, int> gid;
    std::vector<int> chain_group(n_chains, -1);
    int max_cap = 1;
    size_t smem = 0;
    for (int32_t i = 0; i < n_chains; ++i) {
        const gl_chain &c = chains[i];
        max_cap = std::max(max_cap, (int)c.batch_cap);
        smem = std::max(smem, SmemLayout(c.max_prompt, c.batch_cap).total);
        if (c.mode != GL_MODE_DSD) continue;
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
        }
        chain_group[i] = it->second;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (smem > (size_t)smem_optin) return GL_E_UNSUPPORTED;

    // stream-ordered scratch: [chain descriptors][group descriptors][K arrays]
    const size_t off_groups = align256(sizeof(DChain) * n_chains);
    size_t off_k = off_groups + align256(sizeof(DGroup) * groups.size());
    std::vector<size_t> k_off(groups.size());
    size_t total = off_k;
    for (size_t g = 0; g < groups.size(); ++g) {
        k_off[g] = total;
        total += align256(sizeof(uint32_t) * (size_t)groups[g].n);
    }
    unsigned char *scratch = nullptr;
    if ((st = cuda_status(cudaMallocAsync(reinterpret_cast<void **>(&scratch), total, stream))))
        return st;
    for (size_t g = 0; g < groups.size(); ++g)
        groups[g].K = reinterpret_cast<uint32_t *>(scratch + k_off[g]);

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
    cudaError_t e = cudaMemcpyAsync(scratch, dch.data(), sizeof(DChain) * n_chains,
                                    cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess && !groups.empty())
        e = cudaMemcpyAsync(scratch + off_groups, groups.data(), sizeof(DGroup) * groups.size(),
                            cudaMemcpyHostToDevice, stream);
    int launches = 0;
    if (e == cudaSuccess && !groups.empty()) {
        int64_t maxn = 0;
        for (auto &g : groups) maxn = std::max(maxn, g.n);
        dim3 grid((unsigned)((maxn + 255) / 256), (unsigned)groups.size());
        prof_begin("k_dsd_demand", stream);
        k_dsd_demand<<<grid, 256, 0, stream>>>(reinterpret_cast<const DGroup *>(scratch + off_groups));
        e = cudaGetLastError();
        prof_end(stream);
        ++launches;
    }
    if (e == cudaSuccess) {
        const DChain *dc = reinterpret_cast<const DChain *>(scratch);
        auto launch = [&](auto kern) {
            cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (r != cudaSuccess) return r;
            prof_begin("k_chain", stream);
            kern<<<n_chains, 32, smem, stream>>>(dc, stats_out, per_request_out);
            r = cudaGetLastError();
            prof_end(stream);
            return r;
        };
        if (max_cap <= 32)
            e = launch(k_chain<1>);
        else if (max_cap <= 64)
            e = launch(k_chain<2>);
        else if (max_cap <= 128)
            e = launch(k_chain<4>);
        else
            e = launch(k_chain<8>);
        ++launches;
    }
    cudaError_t ef = cudaFreeAsync(scratch, stream);
    if (e == cudaSuccess) e = ef;
    if (e != cudaSuccess) return GL_E_CUDA;
    g_last_launches = launches;
    return GL_OK;
}

gl_status gl_argmin_feasible(const gl_chain_stats *stats, int32_t n_chains, const gl_chain *chains,
                             const gl_scenario *scen, int32_t n_scen, const gl_grid *grid,
                             int32_t slo_num, int32_t slo_den, int32_t priority,
                             int32_t default_col, double *carbon_out, int32_t *choice_out,
                             uint8_t *via_fallback_out, void *stream_)
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
        if (!(std::isfinite(chains[i].ce_old_g) && chains[i].ce_old_g > 0.0)) return GL_E_DOMAIN;
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
        k_argmin<<<blocks, 32 * warps, 0, stream>>>(
            stats, reinterpret_cast<const DCarbon *>(scratch),
            reinterpret_cast<const gl_scenario *>(scratch + o_scen),
            reinterpret_cast<const int32_t *>(scratch + o_rows),
            reinterpret_cast<const int32_t *>(scratch + o_cells), (int32_t)rows, (int32_t)cols,
            slo_num, slo_den, priority, default_col, carbon_out, choice_out, via_fallback_out);
        e = cudaGetLastError();
        prof_end(stream);
    }
    cudaError_t ef = cudaFreeAsync(scratch, stream);
    if (e == cudaSuccess) e = ef;
    if (e != cudaSuccess) return GL_E_CUDA;
    g_last_launches = 1;
    return GL_OK;
}

gl_status gl_evaluate_host(const gl_trace *host_traces, int32_t n_traces, const gl_chain *chains,
                           int32_t n_chains, const gl_scenario *scen, int32_t n_scen,
                           const gl_grid *grid, int32_t slo_num, int32_t slo_den,
                           int32_t priority, int32_t default_col, gl_chain_stats *stats_host,
                           double *carbon_host, int32_t *choice_host, uint8_t *via_fallback_host,
                           void *stream_)
{
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    gl_status st = validate_traces(host_traces, n_traces);
    if (st) return st;
    if (!grid || grid->rows <= 0 || grid->cols <= 0 || !stats_host || !choice_host ||
        !via_fallback_host || n_chains <= 0)
        return GL_E_INVALID;
    if ((st = device_check())) return st;
    const int64_t rows = grid->rows, cols = grid->cols;
    std::vector<size_t> off(n_traces);
    size_t total = 0;
    for (int32_t t = 0; t < n_traces; ++t) {
        off[t] = total;
        const size_t n = (size_t)host_traces[t].n;
        total += align256(8 * n) + 2 * align256(4 * n);
    }
    const size_t o_stats = total;
    total += align256(sizeof(gl_chain_stats) * n_chains);
    const size_t o_carbon = total;
    total += carbon_host ? align256(sizeof(double) * rows * cols) : 0;
    const size_t o_choice = total;
    total += align256(sizeof(int32_t) * rows);
    const size_t o_fb = total;
    total += align256(rows);
    unsigned char *dev = nullptr;
    if ((st = cuda_status(cudaMallocAsync(reinterpret_cast<void **>(&dev), total, stream)))) return st;
    std::vector<gl_trace> dtr(n_traces);
    cudaError_t e = cudaSuccess;
    for (int32_t t = 0; t < n_traces && e == cudaSuccess; ++t) {
        const gl_trace &h = host_traces[t];
        const size_t n = (size_t)h.n;
        unsigned char *base = dev + off[t];
        dtr[t].arrival_us = reinterpret_cast<int64_t *>(base);
        dtr[t].prompt_len = reinterpret_cast<uint32_t *>(base + align256(8 * n));
        dtr[t].output_len = reinterpret_cast<uint32_t *>(base + align256(8 * n) + align256(4 * n));
        dtr[t].n = h.n;
        e = cudaMemcpyAsync((void *)dtr[t].arrival_us, h.arrival_us, 8 * n, cudaMemcpyHostToDevice,
                            stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync((void *)dtr[t].prompt_len, h.prompt_len, 4 * n,
                                cudaMemcpyHostToDevice, stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync((void *)dtr[t].output_len, h.output_len, 4 * n,
                                cudaMemcpyHostToDevice, stream);
    }
    int launches = 0;
    if (e == cudaSuccess) {
        gl_chain_stats *dstats = reinterpret_cast<gl_chain_stats *>(dev + o_stats);
        st = gl_eval_grid(dtr.data(), n_traces, chains, n_chains, dstats, nullptr, stream_);
        launches += g_last_launches;
        if (st == GL_OK) {
            st = gl_argmin_feasible(dstats, n_chains, chains, scen, n_scen, grid, slo_num, slo_den,
                                    priority, default_col,
                                    carbon_host ? reinterpret_cast<double *>(dev + o_carbon) : nullptr,
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
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(choice_host, dev + o_choice, sizeof(int32_t) * rows,
                                    cudaMemcpyDeviceToHost, stream);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(via_fallback_host, dev + o_fb, rows, cudaMemcpyDeviceToHost,
                                    stream);
        }
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

int32_t gl_kernel_times(const char **names_out, float *ms_out, int32_t max)
{
    int32_t k = 0;
    for (int i = 0; i < g_prof.used && k < max; ++i) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, g_prof.ev[2 * i], g_prof.ev[2 * i + 1]) != cudaSuccess)
            ms = -1.f;
        if (names_out) names_out[k] = g_prof.names[i];
        if (ms_out) ms_out[k] = ms;
        ++k;
    }
    g_prof.used = 0;
    return k;
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
