// k_link.cuh -- link bandwidth demand of every disaggregated chain (SURVEY §8(f)
// NEXT #2; Fig. 4, "bandwidth requirement").
//
// Readings R45-R47: every payload is an impulse of bytes at its
// issue time -- a request's stage-2 payload bpt*(p+1) at its prefill completion
// c_i = a_i + TTFT_i (o_i > 1), and a decode iteration's payload b*pm at the
// iteration's start.  demand(t) = bytes issued in [t, t + W); the peak is its
// maximum over t, attained at an impulse time; peak_t is the earliest such time.
//
// The decode iterations come from the batch-size log k_decode<.., LOG> writes
// (runs write from position 2 q0, sentinels b = -1 elsewhere; k_link_scan compacts
// it, in order, into DLink::ev):
// between entries e and e+1 the batch size b_e is constant and iterations start
// at T_e, T_e + s_e, ..., k_e = (T_{e+1} - T_e) / s_e of them (s_e = step[b_e]).
// With C(x) = bytes issued before x (prefix sums over requests and over log
// entries), demand(t) = C(t + W) - C(t).
//   k_link_scan    exclusive prefix sums: per request (bytes) and per log entry
//                  (k_e * b_e * pm, after compacting the log), one 1024-thread block
//                  per (chain, side)
//   k_link_window  every candidate start: a request impulse (binary searches), or
//                  the k_e iteration starts of one log entry (binary search once,
//                  then two pointers that only move forward); per-block best
//   k_link_reduce  per chain: best over blocks -> gl_link_stats
// All integer, so the result is exact and independent of the launch geometry.
#pragma once

#include "common.cuh"

namespace gl {

struct DLink {
    int64_t bpt, pm;     // bytes per prompt token (+1), bytes per member-step
    int64_t *req_pre;    // [n + 1] exclusive prefix of request payload bytes
    int64_t *it_pre;     // [ev_cap + 1] exclusive prefix of iteration payload bytes
    longlong2 *part;     // [LINK_BLOCKS + 1] per-block (peak, t); [LINK_BLOCKS].x = iteration impulses
    longlong2 *ev;       // [ev_cap] the compacted batch-size log (k_link_scan)
    int64_t ev_cap;
};

constexpr int LINK_BLOCKS = 64;    // k_link_window blocks per chain
constexpr int LINK_THREADS = 256;

__device__ __forceinline__ int64_t link_req_bytes(const DChain &ch, const DLink &lk, int64_t i)
{
    return __ldg(ch.o + i) > 1u ? lk.bpt * ((int64_t)__ldg(ch.p + i) + 1) : 0;
}

// iterations of log entry e (0 for b = 0, for the last entry and for zero-length ones)
__device__ __forceinline__ int64_t link_iters(const DChain &ch, const longlong2 *ev, int32_t ne, int32_t e)
{
    if (e + 1 >= ne) return 0;
    const longlong2 a = ev[e], b = ev[e + 1];
    if (a.y <= 0) return 0;
    return (b.x - a.x) / (int64_t)__ldg(ch.step + a.y);
}

// exclusive block scan of int64 over 1024 threads
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t &total, int64_t *sw)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = shfl_up_i64(x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sw[w] = x;
    __syncthreads();
    if (w == 0) {
        int64_t s = sw[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = shfl_up_i64(s, o);
            if (lane >= o) s += y;
        }
        sw[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    total = sw[31];
    const int64_t r = x - v + (w ? sw[w - 1] : 0);
    __syncthreads();
    return r;
}

// blockIdx.x = chain, blockIdx.y = 0 (requests) / 1 (log entries); 1024 threads
__global__ void __launch_bounds__(1024)
    k_link_scan(const DChain *__restrict__ chains, const DLink *__restrict__ links)
{
    __shared__ int64_t sw[32];
    const DChain &ch = chains[blockIdx.x];
    if (ch.mode != GL_MODE_DPD && ch.mode != GL_MODE_DSD) return;
    const DLink &lk = links[blockIdx.x];
    const bool req = blockIdx.y == 0;
    if (!req) {  // compact the log (drop the b = -1 sentinels), keeping the order
        int64_t kept = 0;
        for (int64_t base = 0; base < lk.ev_cap; base += 1024) {
            const int64_t i = base + threadIdx.x;
            longlong2 v = make_longlong2(0, -1);
            if (i < lk.ev_cap) v = ch.ev[i];
            const int64_t f = v.y >= 0 ? 1 : 0;
            int64_t tot;
            const int64_t ex = block_excl_scan(f, tot, sw);
            if (f) lk.ev[kept + ex] = v;
            kept += tot;
        }
        if (threadIdx.x == 0) ch.x->n_ev = (int32_t)kept;
        __syncthreads();
    }
    const int32_t ne = ch.x->n_ev;
    const int64_t n = req ? ch.n : (int64_t)ne;
    int64_t *out = req ? lk.req_pre : lk.it_pre;
    int64_t carry = 0, cnt = 0;
    for (int64_t base = 0; base < n; base += 1024) {
        const int64_t i = base + threadIdx.x;
        int64_t v = 0;
        if (i < n) {
            if (req) {
                v = link_req_bytes(ch, lk, i);
            } else {
                const int64_t k = link_iters(ch, lk.ev, ne, (int32_t)i);
                v = k * lk.ev[i].y * lk.pm;
                cnt += v > 0 ? k : 0;  // iteration impulses with a payload
            }
        }
        int64_t tot;
        const int64_t ex = block_excl_scan(v, tot, sw);
        if (i < n) out[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) out[n] = carry;
    if (!req) {
        int64_t tot;
        block_excl_scan(cnt, tot, sw);
        if (threadIdx.x == 0) lk.part[LINK_BLOCKS] = make_longlong2(tot, 0);
    }
}

// first index in [lo, hi) whose key >= x (keys non-decreasing)
template <typename F>
__device__ __forceinline__ int64_t lower_bound_by(int64_t lo, int64_t hi, int64_t x, F key)
{
    while (lo < hi) {
        const int64_t m = (lo + hi) >> 1;
        if (key(m) < x) lo = m + 1;
        else hi = m;
    }
    return lo;
}

__device__ __forceinline__ void link_better(int64_t &bv, int64_t &bt, int64_t v, int64_t t)
{
    if (v > bv || (v == bv && t < bt)) {
        bv = v;
        bt = t;
    }
}

// grid (LINK_BLOCKS, n_chains) x LINK_THREADS
__global__ void __launch_bounds__(LINK_THREADS)
    k_link_window(const DChain *__restrict__ chains, const DLink *__restrict__ links,
                  const int64_t *__restrict__ perreq, int64_t window)
{
    __shared__ int64_t s_v[LINK_THREADS / 32], s_t[LINK_THREADS / 32];
    const DChain &ch = chains[blockIdx.y];
    const DLink &lk = links[blockIdx.y];
    int64_t bv = 0, bt = INT64_MAX;
    if (ch.mode == GL_MODE_DPD || ch.mode == GL_MODE_DSD) {
        const int64_t n = ch.n;
        const int32_t ne = ch.x->n_ev;
        const longlong2 *ev = lk.ev;
        const int64_t *ttft = perreq + 2 * ch.out_off;  // (ttft, finish) rows
        auto c_of = [&](int64_t i) { return __ldg(ch.a + i) + ttft[2 * i]; };
        // bytes issued before x: requests with c < x, and iteration starts < x
        auto c_req = [&](int64_t x) { return lk.req_pre[lower_bound_by(0, n, x, c_of)]; };
        auto c_it_at = [&](int32_t e, int64_t x) -> int64_t {  // e = last entry with T_e < x
            if (e < 0) return 0;
            const longlong2 en = ev[e];
            const int64_t k = link_iters(ch, ev, ne, e);
            int64_t m = 0;
            if (k > 0) {
                const int64_t s = __ldg(ch.step + en.y);
                m = min(k, (int64_t)((x - en.x + s - 1) / s));
            }
            return lk.it_pre[e] + m * en.y * lk.pm;
        };
        auto last_before = [&](int64_t x) -> int32_t {
            return (int32_t)lower_bound_by(0, ne, x, [&](int64_t e) { return ev[e].x; }) - 1;
        };
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        const int64_t total = n + ne;
        for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += stride) {
            if (g < n) {  // a request impulse at c_g
                if (link_req_bytes(ch, lk, g) == 0) continue;
                const int64_t t = c_of(g);
                const int64_t x = t + window;
                const int64_t v = c_req(x) + c_it_at(last_before(x), x) -
                                  (c_req(t) + c_it_at(last_before(t), t));
                link_better(bv, bt, v, t);
                continue;
            }
            // the iteration starts of log entry e
            const int32_t e = (int32_t)(g - n);
            const int64_t k = link_iters(ch, ev, ne, e);
            const int64_t w = ev[e].y * lk.pm;
            if (k == 0 || w == 0) continue;
            const int64_t T0 = ev[e].x, s = __ldg(ch.step + ev[e].y);
            // start side: C(t_m) = C_req(t_m) + it_pre[e] + m w
            int64_t is = lower_bound_by(0, n, T0, c_of);
            // end side: x_m = t_m + W; request pointer and log-entry pointer
            int64_t x = T0 + window;
            int64_t ie = lower_bound_by(0, n, x, c_of);
            int32_t ee = last_before(x);
            for (int64_t m = 0; m < k; ++m, x += s) {
                const int64_t t = T0 + m * s;
                while (is < n && c_of(is) < t) ++is;
                while (ie < n && c_of(ie) < x) ++ie;
                while (ee + 1 < ne && ev[ee + 1].x < x) ++ee;
                const int64_t v = lk.req_pre[ie] + c_it_at(ee, x) -
                                  (lk.req_pre[is] + lk.it_pre[e] + m * w);
                link_better(bv, bt, v, t);
            }
        }
    }
    // block reduce of (peak desc, t asc)
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const int64_t v = __shfl_xor_sync(FULL, bv, o), t = __shfl_xor_sync(FULL, bt, o);
        link_better(bv, bt, v, t);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_v[w] = bv;
        s_t[w] = bt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < LINK_THREADS / 32; ++i) link_better(bv, bt, s_v[i], s_t[i]);
        lk.part[blockIdx.x] = make_longlong2(bv, bt);
    }
}

// one warp per chain
__global__ void k_link_reduce(const DChain *__restrict__ chains, const DLink *__restrict__ links,
                              gl_link_stats *__restrict__ out, int32_t n_chains)
{
    const int c = blockIdx.x;
    const int lane = threadIdx.x;
    const DChain &ch = chains[c];
    const DLink &lk = links[c];
    gl_link_stats r{0, 0, -1, 0};
    if (ch.mode == GL_MODE_DPD || ch.mode == GL_MODE_DSD) {
        int64_t bv = 0, bt = INT64_MAX;
        for (int i = lane; i < LINK_BLOCKS; i += 32) link_better(bv, bt, lk.part[i].x, lk.part[i].y);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const int64_t v = __shfl_xor_sync(FULL, bv, o), t = __shfl_xor_sync(FULL, bt, o);
            link_better(bv, bt, v, t);
        }
        // impulse count: requests with a payload, iteration starts with one (k_link_scan)
        const int32_t ne = ch.x->n_ev;
        const int64_t cnt = lk.part[LINK_BLOCKS].x;
        const int64_t nreq = lk.bpt > 0 ? (int64_t)ch.x->M : 0;
        r.total_bytes = lk.req_pre[ch.n] + lk.it_pre[ne];
        r.n_impulses = nreq + cnt;
        if (bv > 0) {
            r.peak_bytes = bv;
            r.peak_t_us = bt;
        }
    }
    if (lane == 0) out[c] = r;
}

}  // namespace gl
