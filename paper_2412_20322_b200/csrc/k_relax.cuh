// k_relax.cuh -- the decode stage (S5 + S7) of a heavily loaded chain as an exact
// parallel-in-time fixed point (DESIGN.md §4 "k_relax").
//
// k_decode walks a chain's decode stage serially and parallelises it only at idle
// points.  A chain loaded to ~0.75 of its decode capacity runs one busy period of
// ~10^5 requests without an idle point, so its serial walk is the step's critical
// path.  Here the same stage is solved for all requests at once (R57).
//
// Iteration domain.  Boundary I (= 0, 1, ...) of a chain's decode stage has a time
// tau(I); iteration I runs from tau(I) to tau(I + 1) with b(I) members.  Decode
// request q (FCFS order, ready at r_q, demand K_q iterations) joins at boundary J_q
// and leaves at F_q = J_q + K_q (R15, R16).  The serial simulation is equivalent to
//   b(I)     = #{q : J_q <= I < F_q}
//   tau(0)   = r_0
//   tau(I+1) = tau(I) + step[b(I)]                 if b(I) > 0
//            = max(tau(I), r_{q*}), q* = #{q : J_q <= I}   if b(I) = 0   (idle, R17)
//   J_q      = max(A_q, J_{q-1}, S_q)
//     A_q = min{I : tau(I) >= r_q}                        (ready, R16)
//     S_q = min{I : #{i : F_i <= I} >= q - cap + 1}       (a slot is free, R18)
// (an idle stage costs one empty iteration; S_q uses every request's F, which is
// exact wherever S_q <= J_q -- in particular at the fixed point).  Every rule is
// causal, so the system has exactly one solution, the serial simulation's.
//
// Relaxation.  Start from a guess of J and apply the rules as a map
//   J -> b, tau (scans over the boundaries) -> A, S (scattered / merged while the
//   boundaries are walked) -> J' (prefix max)
// until J' = J; the fixed point is the unique solution (bit-exact, integer).  The
// prefix before the first wrong J_q is exact after every sweep, so it converges;
// from a good guess it takes ~30 sweeps on config 4's chains 33 and 51, 88 on 63
// and 133 on 46, whose long saturated stretches fix joins by earlier leaves only
// (DESIGN.md §10).  The guess: k_relax_guess simulates every 1,024-request segment
// serially (one warp each, all segments at once) from an empty batch 128 requests
// earlier; the segments' local iteration numbers are stitched by a prefix sum.
// For convergence only, b > cap (possible in an iterate, never in the solution)
// extrapolates the step table linearly.
//
// k_relax is one cooperative kernel (grid barriers between phases) over all
// selected chains (slots); every block owns a contiguous chunk of each slot's
// boundaries and requests, every lane a contiguous run, and block carries come from
// the predecessors' aggregates after a grid barrier.  It races k_decode, which walks the same chains:
// whichever finishes a chain first owns its statistics (DChainX::pad bits); both
// write identical finish times, and the loser stops early (k_decode's leader polls
// the flag every 128 requests, k_relax every sweep).  A chain that outgrows its
// buffers or does not converge within RX_MAX_SWEEPS is simply left to k_decode.
#pragma once

#include <cooperative_groups.h>
#include <cstdio>

#include "common.cuh"

namespace gl {

constexpr int RX_SEG = 1024;      // decode requests per guess segment
constexpr int RX_WU = 128;        // warm-up requests simulated before a segment
constexpr int RX_GWARPS = 4;      // guess warps per block
constexpr int RX_THREADS = 256;   // k_relax block
constexpr int RX_BPS = 2;         // k_relax blocks per SM
constexpr int RX_EPT = 8;         // iterations per lane per warp step
constexpr int RX_WARPS = RX_THREADS / 32;
constexpr int RX_MAX_SLOTS = 16;
constexpr int RX_MAX_SWEEPS = 160;
constexpr int RX_LFACTOR = 40;    // iteration capacity per request
constexpr int RX_MAXCAP = 31;     // one member per lane in the guess
constexpr int32_t RX_MIN_M = 8192;
constexpr int64_t RX_MAX_N = 262144;
constexpr int32_t RX_MAX_NSEG = 4;
constexpr double RX_MAX_IPR = 10.0;  // iterations per request (estimated): a sweep costs O(iterations)   // k_segments' idle-point candidates: more = k_decode's helpers parallelise it  // default eligibility: traces up to this many requests
constexpr double RX_RHO_LO = 0.73, RX_RHO_HI = 0.82;
constexpr int RX_DEF_SLOTS = 8;   // slots per call (GL_RELAX=force: up to 16)

// one block's share of a slot's scans in the current sweep (zeroed per call; flags =
// sweep + 1 once the value is published)
struct RxBlk {
    int32_t f1, f2, fc, pad;
    unsigned long long s1;   // packed (joins << 32 | leaves) count of the block's iterations
    int64_t a2, b2;          // max-plus map x -> max(x + a2, b2) of the block's iterations
    int32_t mc, pad2;        // max of the block's requests' max(A_q, S_q)
    int32_t qa[256];         // per thread: its first request in the A merge (warm start)
    int64_t pad3;
};

// one relaxation slot: buffers (host), chain and state (device)
struct DRelax {
    int32_t *J;                 // [ncap] join boundary per decode request (the iterate)
    int32_t *A;                 // [ncap] A_q of the sweep, then the prefix max of max(A_q, S_q) per block
    int32_t *Sq;                // [ncap] S_q of the sweep
    int32_t *seg;               // [2 nsegcap] guess: local J of a segment's first request / of the next one
    uint32_t *h;                // [lcap] histogram per boundary: joins << 16 | leaves
    int64_t *tau;               // [lcap + 1]
    RxBlk *blk;                 // [grid blocks]
    int64_t lcap;
    int32_t ncap, nsegcap;
    // device-written
    int32_t chain;              // -1: unused
    int32_t M;
    int32_t Lc[2];              // max F of the iterate (by sweep parity)
    int32_t changed[2];
    int32_t state;              // 1 converged, 2 given up, 3 converged and owns the chain
    int32_t sweeps;
    int32_t Lf;                 // Lc of the converged iterate
    int32_t quit;               // k_decode's leader finished the chain first
    int64_t tend;               // tau(Lc + 1) of the sweep
    unsigned long long cnt[2][RX_MAXCAP + 1];  // iterations per batch size (by sweep parity)
};

// ---- selection: load factor of every eligible chain, slots to the heaviest ones
// rho = sum_q K_q * step[cap] / cap / (r_last - r_first): offered member-iterations
// per us over the stage's capacity at a full batch.
__global__ void __launch_bounds__(256)
    k_relax_rho(const DChain *__restrict__ chains, const gl_chain_stats *__restrict__ stats,
                double *__restrict__ rho, int32_t min_m, double ipr_max)
{
    __shared__ unsigned long long s_sum[8];
    const int c = blockIdx.x;
    const DChain &ch = chains[c];
    const int32_t M = ch.x->M;
    const bool ok = (ch.mode == GL_MODE_DPD || ch.mode == GL_MODE_DSD) && ch.cap >= 1 &&
                    ch.cap <= RX_MAXCAP && stats[c].status == 0 && M >= max(min_m, 1);
    if (!ok) {
        if (threadIdx.x == 0) rho[c] = -1.0;
        return;
    }
    unsigned long long s = 0;
    for (int32_t q = threadIdx.x; q < M; q += 256) s += __ldg(&ch.dec_dj[q].x);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) s += s_sum[w];
        const int64_t span = max((int64_t)1, ch.dec_r[M - 1] - ch.dec_r[0]);
        const double r_ = (double)s * (double)__ldg(ch.step + ch.cap) / (double)ch.cap / (double)span;
        // a sweep costs O(boundaries) ~ sum K / mean batch ~ sum K / (rho cap), the serial
        // walk O(requests): chains with many iterations per request (DPD chat chains,
        // ~20) are cheaper to walk than to relax (ipr_max: GL_RELAX=force passes 1e300)
        const double ipr = (double)s / (max(r_, 1e-9) * (double)ch.cap) / (double)M;
        rho[c] = ipr <= ipr_max ? r_ : -1.0;
    }
}

// one warp: slots to the chains with the largest rho in [rho_lo, rho_hi) (RX_RHO_LO, RX_RHO_HI)
__global__ void k_relax_pick(const DChain *__restrict__ chains, int32_t n_chains,
                             double *__restrict__ rho, DRelax *__restrict__ slots, int32_t nslots,
                             double rho_lo, double rho_hi)
{
    const int lane = threadIdx.x;
    for (int s = 0; s < nslots; ++s) {
        double best = -1.0;
        int32_t bc = -1;
        for (int32_t c = lane; c < n_chains; c += 32) {
            const double v = rho[c];
            // long busy periods only: a chain with many idle-point candidates is walked in
            // parallel by k_decode's helpers already (config 4's chain 21: 3 ms)
            if (v >= rho_lo && v < rho_hi && chains[c].x->M <= slots[s].ncap && v > best &&
                (rho_hi > 1e200 || chains[c].x->nseg <= RX_MAX_NSEG)) {
                best = v;
                bc = c;
            }
        }
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(FULL, best, o);
            const int32_t oc = __shfl_xor_sync(FULL, bc, o);
            if (ov > best || (ov == best && oc >= 0 && (bc < 0 || oc < bc))) {
                best = ov;
                bc = oc;
            }
        }
        if (bc < 0) break;
        if (lane == 0) {
            slots[s].chain = bc;
            slots[s].M = chains[bc].x->M;
            chains[bc].x->pad = s + 1;  // k_decode's first pass skips it
            rho[bc] = -1.0;
        }
        __syncwarp();
    }
}

// ---- the guess: one warp per (slot, segment) simulates requests [s - WU, e] from an
// empty batch, one member per lane, and writes the local join boundary of q in [s, e)
// (and of s and e to seg).  Same rules as k_decode's general event, plain code.
__global__ void __launch_bounds__(32 * RX_GWARPS)
    k_relax_guess(DRelax *__restrict__ slots, int32_t nslots, int32_t segs_per_slot,
                  const DChain *__restrict__ chains)
{
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * RX_GWARPS + (threadIdx.x >> 5);
    const int si = (int)(wid / segs_per_slot), k = (int)(wid % segs_per_slot);
    if (si >= nslots) return;
    DRelax &S = slots[si];
    const int32_t c = S.chain;
    if (c < 0) return;
    const int32_t M = S.M;
    const int32_t s = k * RX_SEG;
    if (s >= M) return;
    const int32_t e = min(s + RX_SEG, M);
    const DChain &ch = chains[c];
    const int cap = ch.cap;
    const int64_t *r = ch.dec_r;
    const uint2 *dj = ch.dec_dj;
    const int32_t st_l = lane <= cap ? __ldg(ch.step + lane) : 1;
    const uint64_t mg_l = st_l > 1 ? 0xFFFFFFFFFFFFFFFFull / (uint64_t)st_l + 1ull : 0ull;
    int32_t q = max(0, s - RX_WU);
    int64_t T = r[q];
    uint32_t I = 0, F = F_EMPTY;
    unsigned fr = (1u << cap) - 1u;
    int b = 0;
    int64_t hr = __ldg(r + q);
    uint32_t hk = __ldg(&dj[q].x);
    const int32_t qlast = e < M ? e : M - 1;  // run until this request has joined
    for (;;) {
        bool fin = false;
        while (b < cap && hr <= T) {  // FCFS joins at boundary I (R16, R18)
            const unsigned bit = fr & (0u - fr);
            fr ^= bit;
            if ((1u << lane) == bit) F = I + hk;
            ++b;
            if (lane == 0 && q >= s) {
                if (q < e) S.J[q] = (int32_t)I;
                if (q == s) S.seg[2 * k] = (int32_t)I;
                if (q == e) S.seg[2 * k + 1] = (int32_t)I;
            }
            if (q == qlast) {
                fin = true;
                break;
            }
            ++q;
            hr = __ldg(r + q);
            hk = __ldg(&dj[q].x);
        }
        if (fin) break;
        if (b == 0) {  // idle: one empty iteration, then the head is ready (R17)
            ++I;
            T = hr;
            continue;
        }
        const uint32_t kL = __reduce_min_sync(FULL, F) - I;
        const int32_t st = __shfl_sync(FULL, st_l, b);
        uint32_t kk = kL;
        if (b < cap) {
            const int64_t gap = hr - T;  // > 0: not admitted at T
            uint32_t kJ;
            if (gap < 0x80000000ll) {
                const uint64_t mg = __shfl_sync(FULL, mg_l, b);
                kJ = ceil_div_magic((uint32_t)gap, (uint32_t)st, mg);
            } else {
                kJ = (uint32_t)min((gap + st - 1) / st, (int64_t)0xFFFFFFFF);
            }
            kk = min(kL, kJ);
        }
        T += (int64_t)kk * st;
        I += kk;
        if (kk == kL) {  // leaves at I (before any join at I, R16)
            const bool lv = F == I;
            const unsigned lm = __ballot_sync(FULL, lv);
            if (lv) F = F_EMPTY;
            fr |= lm;
            b -= __popc(lm);
        }
    }
}

// ---- max-plus maps x -> max(x + a, b)
struct RxMap {
    int64_t a, b;
};
__device__ __forceinline__ RxMap rx_then(RxMap f, RxMap g)  // f first, then g
{
    return RxMap{f.a + g.a, max(f.b + g.a, g.b)};
}
__device__ __forceinline__ int64_t rx_apply(RxMap f, int64_t x) { return max(x + f.a, f.b); }

__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// first I in [lo, hi] with v(I) >= x (v nondecreasing), hi + 1 if none; galloping from s
__device__ unsigned long long g_rx_probes[4];  // GL_RX_TRACE builds: searches, probes
template <typename V>
__device__ __forceinline__ int32_t rx_search(V v, int64_t x, int32_t s, int32_t lo, int32_t hi)
{
    s = min(max(s, lo), hi);
    int32_t a, bnd;  // answer in (a, bnd]: v(a) < x (or a = lo - 1), v(bnd) >= x (or bnd = hi + 1)
    if (v(s) >= x) {
        bnd = s;
        int32_t d = 1;
        a = s - 1;
        while (a >= lo && v(a) >= x) {
            bnd = a;
            d *= 2;
            a = max(lo - 1, s - d);
        }
    } else {
        a = s;
        int32_t d = 1;
        bnd = s + 1;
        while (bnd <= hi && v(bnd) < x) {
            a = bnd;
            d *= 2;
            bnd = min(hi + 1, s + d);
        }
    }
    int np = 0;
    while (bnd - a > 1) {
        ++np;  // (GL_RX_TRACE)
        const int32_t m = a + (bnd - a) / 2;
        if (v(m) >= x) bnd = m;
        else a = m;
    }
#ifdef GL_RX_TRACE
    atomicAdd(&g_rx_probes[0], 1ull);
    atomicAdd(&g_rx_probes[1], (unsigned long long)(np + 2 * (32 - __clz(max(1, abs(bnd - s))))));
#endif
    return bnd;
}

// block-wide exclusive scan helpers (RX_THREADS threads)
__device__ __forceinline__ unsigned long long rx_block_excl_sum(unsigned long long v,
                                                                unsigned long long *sh,
                                                                unsigned long long &total)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    unsigned long long pre = 0, tot = 0;
    for (int i = 0; i < RX_THREADS / 32; ++i) {
        const unsigned long long t = sh[i];
        if (i < w) pre += t;
        tot += t;
    }
    __syncthreads();
    total = tot;
    return pre + x - v;
}

__device__ __forceinline__ int32_t rx_block_excl_max(int32_t v, int32_t *sh, int32_t &total)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x = max(x, y);
    }
    int32_t ex = __shfl_up_sync(FULL, x, 1);
    if (lane == 0) ex = INT32_MIN;
    if (lane == 31) sh[w] = x;
    __syncthreads();
    int32_t pre = INT32_MIN, tot = INT32_MIN;
    for (int i = 0; i < RX_THREADS / 32; ++i) {
        const int32_t t = sh[i];
        if (i < w) pre = max(pre, t);
        tot = max(tot, t);
    }
    __syncthreads();
    total = tot;
    return max(pre, ex);
}

__device__ __forceinline__ int64_t rx_step_ext(const int32_t *stp, int cap, int64_t b)
{
    if (b <= cap) return stp[b];
    const int64_t d = cap >= 2 ? (int64_t)stp[cap] - stp[cap - 1] : (int64_t)stp[cap];
    return (int64_t)stp[cap] + (b - cap) * max(d, (int64_t)0);
}

__device__ __forceinline__ void rx_spin() { __nanosleep(256); }  // spare k_decode's issue slots
__device__ __forceinline__ uint64_t rx_now()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}


// the map of boundary I's iteration from its packed prefix P = (GJ << 32 | G)
__device__ __forceinline__ RxMap rx_iter_map(unsigned long long P, const int32_t *stp, int cap,
                                             int32_t M, const int64_t *dec_r)
{
    const int64_t gj = (int64_t)(P >> 32), gl_ = (int64_t)(P & 0xFFFFFFFFull);
    const int64_t b = gj - gl_;
    if (b > 0) return RxMap{rx_step_ext(stp, cap, b), NEG_INF};
    return RxMap{0, gj < M ? __ldg(dec_r + gj) : NEG_INF};  // idle: the next request (R17)
}

__device__ __forceinline__ RxMap rx_shfl_up(RxMap m, int o)
{
    return RxMap{__shfl_up_sync(FULL, m.a, o), __shfl_up_sync(FULL, m.b, o)};
}
__device__ __forceinline__ RxMap rx_shfl(RxMap m, int l)
{
    return RxMap{__shfl_sync(FULL, m.a, l), __shfl_sync(FULL, m.b, l)};
}

// The relaxation of every slot, one cooperative grid of G blocks (one per SM).
// Per sweep: A scatter (J, F) -> grid barrier -> B1 block sums of the histogram;
// B2 the iterations' maps (block map) and S_q (one writer per request: the boundary
// where the leaves count G reaches q - cap + 1); B3 tau, and A_q by merging the
// sorted ready times into the tau of each 256-iteration tile -> grid barrier -> C1
// max(A_q, S_q) and its prefix max per block, C2 J' -> grid barrier -> convergence.
// Each block owns a contiguous chunk of every slot's iterations (and requests); its
// warps stream contiguous sub-chunks 256 iterations at a time with warp scans, and
// a block's carries come from its predecessors' published aggregates.
__global__ void __launch_bounds__(RX_THREADS, RX_BPS + 1)  // registers: room beside k_decode
    k_relax(DRelax *__restrict__ slots, int32_t nslots, const DChain *__restrict__ chains, int32_t dbg)
{
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ int32_t s_step[RX_MAX_SLOTS][RX_MAXCAP + 1];
    __shared__ int32_t s_cap[RX_MAX_SLOTS], s_M[RX_MAX_SLOTS], s_Lc[RX_MAX_SLOTS];
    __shared__ unsigned long long s_u64[RX_WARPS];
    __shared__ int32_t s_i32[RX_WARPS];
    __shared__ unsigned long long s_wsum[RX_MAX_SLOTS][RX_WARPS];
    __shared__ int64_t s_wa[RX_MAX_SLOTS][RX_WARPS], s_wb[RX_MAX_SLOTS][RX_WARPS];
    __shared__ unsigned long long s_c1[RX_MAX_SLOTS];
    __shared__ int64_t s_c2[RX_MAX_SLOTS], s_tend[RX_MAX_SLOTS];
    __shared__ int32_t s_cq[RX_MAX_SLOTS];
    __shared__ uint32_t s_hist[RX_MAXCAP + 2];
    // per slot and thread: lane carry (exclusive within the warp) and lane map prefix
    extern __shared__ __align__(16) unsigned char rx_dyn[];
    unsigned long long *s_lc = reinterpret_cast<unsigned long long *>(rx_dyn);          // [nslots][256]
    int64_t *s_la = reinterpret_cast<int64_t *>(rx_dyn) + (size_t)nslots * RX_THREADS;  // [nslots][256]
    int64_t *s_lb = s_la + (size_t)nslots * RX_THREADS;                                  // [nslots][256]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t G = (int32_t)gridDim.x, blk = (int32_t)blockIdx.x;
    const int64_t gthreads = (int64_t)G * RX_THREADS;
    const int64_t gtid = (int64_t)blk * RX_THREADS + tid;

    uint32_t active = 0;  // identical in every block: decided from the same flags
    for (int s = 0; s < nslots; ++s)
        if (slots[s].chain >= 0) active |= 1u << s;
    for (int i = tid; i < nslots * (RX_MAXCAP + 1); i += RX_THREADS) {
        const int s = i / (RX_MAXCAP + 1), bb = i % (RX_MAXCAP + 1);
        const int32_t c = slots[s].chain;
        s_step[s][bb] = (c >= 0 && bb <= chains[c].cap) ? __ldg(chains[c].step + bb) : 0;
    }
    if (tid < nslots) {
        const int32_t c = slots[tid].chain;
        s_cap[tid] = c >= 0 ? chains[c].cap : 0;
        s_M[tid] = c >= 0 ? slots[tid].M : 0;
    }
    if (tid < RX_MAXCAP + 2) s_hist[tid] = 0u;
    // phase 0: stitch the guess segments (block s: slot s) and zero the histograms
    if (blk < nslots && ((active >> blk) & 1)) {
        DRelax &S = slots[blk];
        const int32_t nseg = (S.M + RX_SEG - 1) / RX_SEG;
        // off_0 = -seg[0]; off_k = off_{k-1} + seg[2(k-1)+1] - seg[2k]
        int64_t carry = 0;
        for (int32_t k0 = 0; k0 < nseg; k0 += RX_THREADS) {
            const int32_t k = k0 + tid;
            int64_t dv = 0;
            if (k < nseg) dv = k == 0 ? -(int64_t)S.seg[0] : (int64_t)S.seg[2 * k - 1] - S.seg[2 * k];
            unsigned long long tot;
            const unsigned long long ex = rx_block_excl_sum((unsigned long long)dv, s_u64, tot);
            if (k < nseg) S.seg[2 * k] = (int32_t)(carry + (int64_t)(ex + (unsigned long long)dv));
            carry += (int64_t)tot;
        }
    }
    for (int s = 0; s < nslots; ++s) {
        if (!((active >> s) & 1)) continue;
        uint4 *h4 = reinterpret_cast<uint4 *>(slots[s].h);
        const int64_t L4 = slots[s].lcap / 4;
        for (int64_t i = gtid; i < L4; i += gthreads) h4[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
    grid.sync();

    uint64_t tph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pv[4] = {0, 0, 0, 0}, t_last = rx_now();
    auto lap = [&](int k) {
        const uint64_t t = rx_now();
        tph[k] += t - t_last;
        t_last = t;
    };
    // a warp's super-tiles (256 iterations) of n iterations: [w0, w1)
    auto warp_tiles = [&](int64_t n, int w, int64_t &w0, int64_t &w1) {
        const int64_t nst = (n + 255) / 256;
        const int64_t b0 = nst * blk / G, b1 = nst * (blk + 1) / G;
        w0 = b0 + (b1 - b0) * w / RX_WARPS;
        w1 = b0 + (b1 - b0) * (w + 1) / RX_WARPS;
    };
    // this lane's boundaries [a_l, b_l) of n: the warp's sub-chunk of the block's chunk,
    // split into lane-contiguous runs of whole 8-boundary units
    auto lane_range = [&](int64_t n, int64_t &a_l, int64_t &b_l) {
        int64_t w0, w1;
        warp_tiles(n, warp, w0, w1);
        const int64_t E0 = w0 * 256, E1 = min(w1 * 256, n);
        const int64_t nu = (E1 - E0 + RX_EPT - 1) / RX_EPT;
        a_l = min(E0 + RX_EPT * (nu * lane / 32), E1);
        b_l = min(E0 + RX_EPT * (nu * (lane + 1) / 32), E1);
    };
    // one lane's 8 boundaries of a super-tile: packed (joins << 32 | leaves) counts
    auto load8 = [&](const uint32_t *h, int64_t e0, int64_t n, unsigned long long (&v)[RX_EPT]) {
        if (e0 + RX_EPT <= n) {
            const uint4 *src = reinterpret_cast<const uint4 *>(h + e0);
            const uint4 x0 = __ldcg(src), x1 = __ldcg(src + 1);
            const uint32_t w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
            for (int k = 0; k < RX_EPT; ++k)
                v[k] = ((unsigned long long)(w[k] >> 16) << 32) | (w[k] & 0xFFFFu);
        } else {
#pragma unroll
            for (int k = 0; k < RX_EPT; ++k) {
                const uint32_t w = e0 + k < n ? __ldcg(h + e0 + k) : 0u;
                v[k] = ((unsigned long long)(w >> 16) << 32) | (w & 0xFFFFu);
            }
        }
    };
    int sw = 0;
    for (; active; ++sw) {
        const int32_t ep = sw + 1;
        const int par = sw & 1;
        // ---- A: histogram of (J, F) of the iterate; Lc = max F
        if (blk == 0 && tid < nslots && ((active >> tid) & 1)) {
            slots[tid].Lc[par ^ 1] = 0;
            slots[tid].changed[par] = 0;
            // the race: drop the chain once k_decode's leader has finished it
            if (ld_relaxed_gpu(&chains[slots[tid].chain].x->pad) & RX_SERIAL) slots[tid].quit = 1;
        }
        if (blk == 1 % G) {
            for (int i = tid; i < nslots * (RX_MAXCAP + 1); i += RX_THREADS) {
                const int s = i / (RX_MAXCAP + 1);
                if ((active >> s) & 1) slots[s].cnt[par][i % (RX_MAXCAP + 1)] = 0ull;
            }
        }
        for (int s = 0; s < nslots; ++s) {
            if (!((active >> s) & 1)) continue;
            DRelax &S = slots[s];
            const DChain &ch = chains[S.chain];
            const int32_t M = s_M[s];
            int32_t fv = INT32_MIN;
            for (int64_t q = gtid; q < M; q += gthreads) {
                int64_t j = __ldcg(S.J + q);
                if (sw == 0) {  // first sweep: the stitched guess
                    j += __ldcg(S.seg + 2 * (q / RX_SEG));
                    j = min(max(j, (int64_t)0), S.lcap - 8);
                    S.J[q] = (int32_t)j;
                }
                const int64_t F = j + __ldg(&ch.dec_dj[q].x);
                if (F + 4 < S.lcap) {
                    atomicAdd(S.h + j, 1u << 16);
                    atomicAdd(S.h + F, 1u);
                }
                fv = max(fv, (int32_t)min(F, (int64_t)INT32_MAX));
            }
            for (int o = 16; o; o >>= 1) fv = max(fv, __shfl_xor_sync(FULL, fv, o));
            if (lane == 0 && fv != INT32_MIN) atomicMax(&S.Lc[par], fv);
        }
        grid.sync();
        lap(0);
        // buffers outgrown, or k_decode was first: give the chain up
        if (tid < nslots) {
            const bool a = (active >> tid) & 1;
            s_Lc[tid] = a ? ld_relaxed_gpu(&slots[tid].Lc[par]) : 0;
            s_cq[tid] = a ? ld_relaxed_gpu(&slots[tid].quit) : 0;
        }
        __syncthreads();
        for (int s = 0; s < nslots; ++s) {
            if (!((active >> s) & 1)) continue;
            if ((int64_t)s_Lc[s] + 4 >= slots[s].lcap || s_cq[s]) {
                active &= ~(1u << s);
                if (blk == 0 && tid == 0) {
                    slots[s].state = 2;
                    slots[s].sweeps = sw;
                }
            }
        }
        if (!active) break;
        // ---- B1: lane sums over lane-contiguous ranges (8-boundary units) of the
        // warp's sub-chunk; lane carries (exclusive in the warp) and the block's sum
        for (int s = 0; s < nslots; ++s) {
            if (!((active >> s) & 1)) continue;
            const uint32_t *h = slots[s].h;
            const int64_t n = (int64_t)s_Lc[s] + 1;
            int64_t a_l, b_l;
            lane_range(n, a_l, b_l);
            unsigned long long sum = 0;
            for (int64_t e0 = a_l; e0 < b_l; e0 += 2 * RX_EPT) {  // two units in flight
                unsigned long long v[RX_EPT], w[RX_EPT];
                load8(h, e0, b_l, v);
                load8(h, e0 + RX_EPT, b_l, w);
#pragma unroll
                for (int k = 0; k < RX_EPT; ++k) sum += v[k] + w[k];
            }
            unsigned long long inc = sum;
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(FULL, inc, o);
                if (lane >= o) inc += y;
            }
            s_lc[s * RX_THREADS + tid] = inc - sum;
            if (lane == 31) s_wsum[s][warp] = inc;
        }
        __syncthreads();
        if (tid < nslots && ((active >> tid) & 1)) {
            unsigned long long t = 0;
            for (int w = 0; w < RX_WARPS; ++w) t += s_wsum[tid][w];
            RxBlk &B = slots[tid].blk[blk];
            B.s1 = t;
            __threadfence();
            st_release_gpu(&B.f1, ep);
        }
        grid.sync();  // every block's aggregate is published
        for (int s = warp; s < nslots; s += RX_WARPS) {  // carry: predecessors' sums
            if (!((active >> s) & 1)) continue;
            const RxBlk *bl = slots[s].blk;
            unsigned long long c = 0;
            for (int32_t j0 = 0; j0 < blk; j0 += 32) {
                const int32_t j = j0 + lane;
                if (j < blk) c += __ldcg(&bl[j].s1);
            }
            for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
            if (lane == 0) s_c1[s] = c;
        }
        __syncthreads();
        lap(4);
        // ---- B2: each lane walks its range: prefix P, the iterations' maps (lane map),
        // S_q at the boundary where the leave count G reaches q - cap + 1
        for (int s = 0; s < nslots; ++s) {
            if (!((active >> s) & 1)) continue;
            DRelax &S = slots[s];
            const int64_t *dec_r = chains[S.chain].dec_r;
            const int32_t M = s_M[s], cap = s_cap[s];
            const int64_t n = (int64_t)s_Lc[s] + 1;
            int64_t a_l, b_l;
            lane_range(n, a_l, b_l);
            unsigned long long P = s_c1[s] + s_lc[s * RX_THREADS + tid];
            for (int w = 0; w < warp; ++w) P += s_wsum[s][w];
            int64_t gprev = (int64_t)(P & 0xFFFFFFFFull);
            RxMap lm{0, NEG_INF};
            unsigned long long vn[RX_EPT];  // the next unit, loaded ahead
            if (a_l < b_l) load8(S.h, a_l, b_l, vn);
            for (int64_t e0 = a_l; e0 < b_l; e0 += RX_EPT) {
                unsigned long long v[RX_EPT];
#pragma unroll
                for (int k = 0; k < RX_EPT; ++k) v[k] = vn[k];
                if (e0 + RX_EPT < b_l) load8(S.h, e0 + RX_EPT, b_l, vn);
#pragma unroll
                for (int k = 0; k < RX_EPT; ++k) {
                    if (e0 + k < b_l) {
                        P += v[k];
                        lm = rx_then(lm, rx_iter_map(P, s_step[s], cap, M, dec_r));
                        const int64_t gk = (int64_t)(P & 0xFFFFFFFFull);
                        for (int64_t need = gprev + 1; need <= gk; ++need) {
                            const int64_t q = need + cap - 1;
                            if (q < M) S.Sq[q] = (int32_t)(e0 + k);
                        }
                        gprev = gk;
                    }
                }
            }
            RxMap in = lm;
            for (int o = 1; o < 32; o <<= 1) {
                const RxMap y = rx_shfl_up(in, o);
                if (lane >= o) in = rx_then(y, in);
            }
            RxMap ex = rx_shfl_up(in, 1);
            if (lane == 0) ex = RxMap{0, NEG_INF};
            s_la[s * RX_THREADS + tid] = ex.a;
            s_lb[s * RX_THREADS + tid] = ex.b;
            if (lane == 31) {
                s_wa[s][warp] = in.a;
                s_wb[s][warp] = in.b;
            }
        }
        __syncthreads();
        if (tid < nslots && ((active >> tid) & 1)) {
            RxMap m{0, NEG_INF};
            for (int w = 0; w < RX_WARPS; ++w) m = rx_then(m, RxMap{s_wa[tid][w], s_wb[tid][w]});
            RxBlk &B = slots[tid].blk[blk];
            B.a2 = m.a;
            B.b2 = m.b;
            __threadfence();
            st_release_gpu(&B.f2, ep);
        }
        grid.sync();  // every block's aggregate is published
        for (int s = warp; s < nslots; s += RX_WARPS) {  // carry: tau at the block's start
            if (!((active >> s) & 1)) continue;
            const RxBlk *bl = slots[s].blk;
            RxMap acc{0, NEG_INF};
            for (int32_t j0 = 0; j0 < blk; j0 += 32) {
                const int32_t j = j0 + lane;
                RxMap m{0, NEG_INF};
                if (j < blk) m = RxMap{__ldcg(&bl[j].a2), __ldcg(&bl[j].b2)};
                for (int o = 1; o < 32; o <<= 1) {  // in lane order: lane 0's map first
                    const RxMap y = RxMap{__shfl_down_sync(FULL, m.a, o), __shfl_down_sync(FULL, m.b, o)};
                    if ((lane & (2 * o - 1)) == 0 && lane + o < 32) m = rx_then(m, y);
                }
                acc = rx_then(acc, rx_shfl(m, 0));
            }
            if (lane == 0) s_c2[s] = rx_apply(acc, __ldg(chains[slots[s].chain].dec_r));
        }
        __syncthreads();
        lap(5);
        // ---- B3: each lane walks its range again: tau (written), h zeroed, iterations
        // per batch size, and A_q for the requests with tau(a_l) < r_q <= tau(b_l)
        // (the first range also r_q <= tau(0)), merged in ready order
        for (int s = 0; s < nslots; ++s) {
            if (!((active >> s) & 1)) continue;
            DRelax &S = slots[s];
            const int64_t *dec_r = chains[S.chain].dec_r;
            const int32_t M = s_M[s], cap = s_cap[s], Lc = s_Lc[s];
            const int64_t n = (int64_t)Lc + 1;
            int64_t a_l, b_l;
            lane_range(n, a_l, b_l);
            unsigned long long P = s_c1[s] + s_lc[s * RX_THREADS + tid];
            int64_t x = s_c2[s];
            for (int w = 0; w < warp; ++w) {
                P += s_wsum[s][w];
                x = rx_apply(RxMap{s_wa[s][w], s_wb[s][w]}, x);
            }
            x = rx_apply(RxMap{s_la[s * RX_THREADS + tid], s_lb[s * RX_THREADS + tid]}, x);  // tau(a_l)
            int32_t qp = 0;
            if (a_l < b_l && a_l > 0) {  // first request with r > tau(a_l) (warm start: last sweep's)
                qp = rx_search([&](int32_t i) { return __ldg(dec_r + i); }, x + 1,
                               min(max(__ldcg(&S.blk[blk].qa[tid]), 0), max(M - 1, 0)), 0, M - 1);
                S.blk[blk].qa[tid] = qp;
            }
            int64_t rq = (a_l < b_l && qp < M) ? __ldg(dec_r + qp) : INT64_MAX;
            int64_t rq2 = (a_l < b_l && qp + 1 < M) ? __ldg(dec_r + qp + 1) : INT64_MAX;
            auto consume = [&](int64_t tau_at, int64_t I) {
                while (rq <= tau_at) {
                    S.A[qp] = (int32_t)I;
                    ++qp;
                    rq = rq2;
                    rq2 = qp + 1 < M ? __ldg(dec_r + qp + 1) : INT64_MAX;
                }
            };
            if (a_l == 0 && a_l < b_l) consume(x, 0);  // ready by tau(0): boundary 0
            int64_t pb = -1;  // run-length histogram of b
            uint32_t run = 0;
            unsigned long long vn[RX_EPT];  // the next unit, loaded ahead
            if (a_l < b_l) load8(S.h, a_l, b_l, vn);
            for (int64_t e0 = a_l; e0 < b_l; e0 += RX_EPT) {
                unsigned long long v[RX_EPT];
#pragma unroll
                for (int k = 0; k < RX_EPT; ++k) v[k] = vn[k];
                if (e0 + RX_EPT < b_l) load8(S.h, e0 + RX_EPT, b_l, vn);
                int64_t tv[RX_EPT];
#pragma unroll
                for (int k = 0; k < RX_EPT; ++k) {
                    tv[k] = x;
                    if (e0 + k < b_l) {
                        P += v[k];
                        const int64_t b = (int64_t)(P >> 32) - (int64_t)(P & 0xFFFFFFFFull);
                        if (b != pb) {
                            if (run && pb >= 0 && pb <= RX_MAXCAP) atomicAdd(&s_hist[pb], run);
                            pb = b;
                            run = 0;
                        }
                        ++run;
                        x = rx_apply(rx_iter_map(P, s_step[s], cap, M, dec_r), x);  // tau(e + 1)
                        consume(x, e0 + k + 1);
                    }
                }
                if (e0 + RX_EPT <= b_l) {
                    longlong2 *dt = reinterpret_cast<longlong2 *>(S.tau + e0);
#pragma unroll
                    for (int k = 0; k < RX_EPT / 2; ++k) dt[k] = make_longlong2(tv[2 * k], tv[2 * k + 1]);
                    uint4 *dh = reinterpret_cast<uint4 *>(S.h + e0);
                    dh[0] = make_uint4(0u, 0u, 0u, 0u);
                    dh[1] = make_uint4(0u, 0u, 0u, 0u);
                } else {
#pragma unroll
                    for (int k = 0; k < RX_EPT; ++k)
                        if (e0 + k < b_l) {
                            S.tau[e0 + k] = tv[k];
                            S.h[e0 + k] = 0u;
                        }
                }
            }
            if (a_l < b_l && b_l == n) {  // the slot's last boundary: tau(Lc + 1)
                S.tau[n] = x;
                S.tend = x;
            }
            if (run && pb >= 0 && pb <= RX_MAXCAP) atomicAdd(&s_hist[pb], run);
            __syncthreads();
            if (tid <= RX_MAXCAP && s_hist[tid]) {
                atomicAdd(&S.cnt[par][tid], (unsigned long long)s_hist[tid]);
                s_hist[tid] = 0u;
            }
            if (tid == RX_MAXCAP + 1) s_hist[tid] = 0u;
            __syncthreads();
        }
        grid.sync();
        lap(1);
        if (tid < nslots) s_tend[tid] = ((active >> tid) & 1) ? __ldcg(&slots[tid].tend) : 0;
        __syncthreads();
        // ---- C1: m_q = max(A_q, S_q); prefix max within the block's chunk
        for (int s = 0; s < nslots; ++s) {
            if (!((active >> s) & 1)) continue;
            DRelax &S = slots[s];
            const int64_t *dec_r = chains[S.chain].dec_r;
            const int32_t M = s_M[s], cap = s_cap[s], Lc = s_Lc[s];
            const int64_t tend = s_tend[s];
            const int32_t c0 = (int32_t)((int64_t)M * blk / G), c1 = (int32_t)((int64_t)M * (blk + 1) / G);
            const int32_t t0 = c0 + (int32_t)((int64_t)(c1 - c0) * tid / RX_THREADS);
            const int32_t t1 = c0 + (int32_t)((int64_t)(c1 - c0) * (tid + 1) / RX_THREADS);
            int32_t run = INT32_MIN;
            for (int32_t q = t0; q < t1; ++q) {
                // unwritten A: ready after tau(Lc + 1), so not before boundary Lc + 2
                const int32_t a = __ldg(dec_r + q) > tend ? Lc + 2 : __ldcg(S.A + q);
                const int32_t sq = (int64_t)q - cap + 1 > 0 ? __ldcg(S.Sq + q) : 0;
                run = max(run, max(a, sq));
                S.A[q] = run;
            }
            int32_t tot;
            const int32_t exq = rx_block_excl_max(run, s_i32, tot);
            if (exq != INT32_MIN)
                for (int32_t q = t0; q < t1; ++q) S.A[q] = max(S.A[q], exq);
            if (tid == 0) {
                RxBlk &B = S.blk[blk];
                B.mc = tot;
                __threadfence();
                st_release_gpu(&B.fc, ep);
            }
        }
        grid.sync();  // every block's aggregate is published
        for (int s = warp; s < nslots; s += RX_WARPS) {  // carry: predecessors' maxima
            if (!((active >> s) & 1)) continue;
            const RxBlk *bl = slots[s].blk;
            int32_t c = INT32_MIN;
            for (int32_t j0 = 0; j0 < blk; j0 += 32) {
                const int32_t j = j0 + lane;
                if (j < blk) c = max(c, __ldcg(&bl[j].mc));
            }
            for (int o = 16; o; o >>= 1) c = max(c, __shfl_xor_sync(FULL, c, o));
            if (lane == 0) s_cq[s] = c;
        }
        __syncthreads();
        lap(2);
        // ---- C2: J' = max(carry, block prefix); changed?
        for (int s = 0; s < nslots; ++s) {
            if (!((active >> s) & 1)) continue;
            DRelax &S = slots[s];
            const int32_t M = s_M[s];
            const int32_t c0 = (int32_t)((int64_t)M * blk / G), c1 = (int32_t)((int64_t)M * (blk + 1) / G);
            const int32_t cq = s_cq[s];
            bool chg = false;
            for (int32_t q = c0 + tid; q < c1; q += RX_THREADS) {
                const int32_t jn = max(cq, S.A[q]);
                if (jn != __ldcg(S.J + q)) {
                    S.J[q] = jn;
                    chg = true;
                }
            }
            if (__syncthreads_or(chg) && tid == 0) st_relaxed_gpu(&S.changed[par], 1);
        }
        grid.sync();
        lap(3);
        if (dbg == 2 && blk == 0 && tid == 0)
            printf("sweep %d active %x: A %.1f B %.1f C1 %.1f C2 %.1f us (total %.3f ms)\n", sw, active,
                   (tph[0] - pv[0]) * 1e-3, (tph[1] - pv[1]) * 1e-3, (tph[2] - pv[2]) * 1e-3,
                   (tph[3] - pv[3]) * 1e-3, (tph[0] + tph[1] + tph[2] + tph[3]) * 1e-6);
        for (int k = 0; k < 4; ++k) pv[k] = tph[k];
        // ---- convergence: a slot whose iterate did not change is solved
        for (int s = 0; s < nslots; ++s) {
            if (!((active >> s) & 1)) continue;
            const bool chg = ld_relaxed_gpu(&slots[s].changed[par]) != 0;
            if (!chg || sw + 1 >= RX_MAX_SWEEPS) {
                active &= ~(1u << s);
                if (blk == 0 && tid == 0) {
                    // solved: claim the chain now, so that k_decode's leader stops; it is
                    // ours unless the leader finished it first (k_relax_out writes it)
                    int32_t st = 2;
                    if (!chg) st = (atomicOr(&chains[slots[s].chain].x->pad, RX_RELAXED) & RX_SERIAL) ? 1 : 3;
                    slots[s].state = st;
                    slots[s].sweeps = sw + 1;
                    slots[s].Lf = s_Lc[s];
                }
            }
        }
        __syncthreads();
    }
    if (dbg) {
        grid.sync();
        if (blk == 0 && tid == 0) {
            printf("k_relax %d sweeps: scatter %.3f ms, iterations %.3f ms (B1 %.3f, B2 %.3f, B3 %.3f), requests %.3f + %.3f ms\n", sw,
                   tph[0] * 1e-6, (tph[4] + tph[5] + tph[1]) * 1e-6, tph[4] * 1e-6, tph[5] * 1e-6, tph[1] * 1e-6,
                   tph[2] * 1e-6, tph[3] * 1e-6);
            for (int s = 0; s < nslots; ++s)
                if (slots[s].chain >= 0)
                    printf("k_relax slot %d chain %d M %d state %d sweeps %d Lf %d pad %x\n", s,
                           slots[s].chain, slots[s].M, ld_relaxed_gpu(&slots[s].state), slots[s].sweeps,
                           slots[s].Lf, ld_relaxed_gpu(&chains[slots[s].chain].x->pad));
        }
    }
}

// The owned slots' results, after k_decode (whose aborted leader may have written
// a few finish times of its unfinished batch): finish time of every decode request
// tau(J_q + K_q) into the rows; block 0 adds the sums and the makespan.
__global__ void __launch_bounds__(256)
    k_relax_out(const DRelax *__restrict__ slots, const DChain *__restrict__ chains,
                gl_chain_stats *__restrict__ stats, int64_t *__restrict__ perreq)
{
    const DRelax &S = slots[blockIdx.y];
    const int32_t c = S.chain;
    if (c < 0 || S.state != 3) return;
    const DChain &ch = chains[c];
    int64_t *rows_fin = perreq + 2 * ch.out_off + 1;
    for (int64_t q = (int64_t)blockIdx.x * 256 + threadIdx.x; q < S.M; q += (int64_t)gridDim.x * 256) {
        const uint2 dj = __ldg(ch.dec_dj + q);
        rows_fin[2 * (int64_t)dj.y] = S.tau[(int64_t)S.J[q] + dj.x];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        for (int bb = 1; bb <= ch.cap; ++bb) {
            const int64_t it = (int64_t)S.cnt[(S.sweeps - 1) & 1][bb];
            if (!it) continue;
            a0 += it * __ldg(ch.sbn + bb);
            a1 += it * __ldg(ch.sbo + bb);
            a2 += it * __ldg(ch.sen + bb);
            a3 += it * __ldg(ch.seo + bb);
        }
        gl_chain_stats &st = stats[c];
        st.busy_new_us += a0;
        st.busy_old_us += a1;
        st.e_new_uj += a2;
        st.e_old_uj += a3;
        st.makespan_us = max(st.makespan_us, S.tau[S.Lf]);
    }
}

}  // namespace gl
