// k_chain.cuh -- one warp per timing chain: stages 1-2 as max-plus scans and the
// continuous-batching decode stage as a warp-uniform event loop (S1-S7).
//
//   stage 1  prefill FCFS on the new GPU   c_i = max(c_{i-1}, a_i) + t1[p_i]
//            (TTFT_i = c_i - a_i; R8-R10)
//   stage 2  DPD KV link (R11) / DSD handoff + draft prefill (R12):
//                                           r_i = max(r_{i-1}, c_i) + t2[p_i]  (o_i > 1)
//   decode   continuous batching (R15-R23): iterations run back to back while the
//            batch is non-empty; at each boundary members whose demand is met
//            leave (finish = boundary time), then ready requests (r <= T) join
//            FCFS while b < cap; an empty batch idles until the next r.
//
// Layout: the prompt-indexed t1/t2 tables and the batch-indexed step table are
// staged in shared memory by TMA bulk copies (cp.async.bulk + mbarrier).  Each
// 128-request chunk is read with 128-bit loads (4 requests per lane), both stages
// are warp scans on (A, B) max-plus pairs, and requests with o > 1 are compacted
// into a shared-memory ring.  The decode loop never steps single iterations: a
// member admitted at iteration I with demand d (DPD: o-1 tokens; DSD: K_j steps)
// finishes at iteration F = I + d, so the next event is min(REDUX-min F, the
// boundary at which the ring head becomes ready) and whole runs of iterations
// are jumped with T += k * step[b].  Active members live one per lane (SPL rows
// of 32 lanes); the loop only records finish times -- SLO counts and the hash are
// computed afterwards by k_finalize with the whole GPU.
#pragma once

#include "common.cuh"

namespace gl {

struct SmemLayout {
    int p1pad, cappad;
    size_t off_t1, off_t2, off_step, off_magic, off_r, off_dj, off_bar, total;
    __host__ __device__ SmemLayout(int max_prompt, int cap)
    {
        p1pad = round_up4(max_prompt + 1);
        cappad = round_up4(cap + 1);
        off_t1 = 0;
        off_t2 = off_t1 + 4 * (size_t)p1pad;
        off_step = off_t2 + 4 * (size_t)p1pad;
        off_magic = (off_step + 4 * (size_t)cappad + 15) & ~(size_t)15;
        off_r = off_magic + 8 * (size_t)cappad;
        off_dj = off_r + 8 * RING;
        off_bar = off_dj + 8 * RING;
        total = off_bar + 16;
    }
};

// ceil(gap / st) for 0 < gap < 2^31, 1 <= st < 2^31 without a division:
// Lemire, Kaser & Kurz (2019): with M = floor((2^64 - 1) / d) + 1, floor(x / d) =
// mulhi64(M, x) for every 32-bit x.  (d = 1 is stored as M = 0 and handled apart.)
__device__ __forceinline__ uint32_t ceil_div_magic(uint32_t gap, uint32_t st, uint64_t M)
{
    const uint32_t x = gap + st - 1u;
    const uint64_t hi = (uint64_t)(uint32_t)(M >> 32) * x + __umulhi((uint32_t)M, x);
    return st == 1u ? gap : (uint32_t)(hi >> 32);
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
    uint2 *ring_dj = reinterpret_cast<uint2 *>(smem + L.off_dj);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L.off_bar);
    int64_t *out = perreq + 2 * ch.out_off;  // this chain's (ttft, finish) rows

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
    uint64_t *magic = reinterpret_cast<uint64_t *>(smem + L.off_magic);
    {
        bool bad = false;
        for (int i = 1 + lane; i <= P; i += 32) bad |= (t1s[i] < 0) | (t2s[i] < 0);
        for (int b = 1 + lane; b <= cap; b += 32) {
            const int32_t s = steps[b];
            bad |= s < 1;
            magic[b] = s > 1 ? 0xFFFFFFFFFFFFFFFFull / (uint64_t)s + 1ull : 0ull;
        }
        if (lane == 0) magic[0] = 0;
        if (__any_sync(FULL, bad)) status |= GL_ST_TABLE;
        __syncwarp();
    }

    // lane-local accumulators
    int64_t acc_busy_new = 0, acc_busy_old = 0, acc_e_new = 0, acc_e_old = 0, acc_tokens = 0;
    int64_t acc_mk = 0;
    // iterations run at batch size b, held by lane b & 31 in row b >> 5: 32-bit
    // counters (flushed into 64-bit totals whenever the iteration counter rebases)
    uint64_t iters[SPL + 1];
    uint32_t cnt[SPL + 1];
#pragma unroll
    for (int s = 0; s <= SPL; ++s) {
        iters[s] = 0;
        cnt[s] = 0;
    }

    const int32_t n = (int32_t)ch.n;
    const bool dsd = ch.mode == GL_MODE_DSD;
    int32_t chunk_next = 0, produced = 0;
    int64_t carry_c = NEG_INF, carry_r = NEG_INF, carry_a = INT64_MIN;

    // ---- S1-S4: one 128-request chunk -> scans -> compacted decode ring -----
    auto produce = [&]() {
        const int32_t i0 = chunk_next + 4 * lane;
        int64_t av[4];
        uint32_t pv[4], ov[4], kv[4];
        if (i0 + 3 < n) {  // 128-bit loads: 2 x (2 x int64) + (4 x u32) per stream
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
        {  // sortedness across the lane boundary and the chunk boundary
            int64_t prev = shfl_up_i64(av[3], 1);
            if (lane == 0) prev = carry_a;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (valid[q] && av[q] < prev) status |= GL_ST_UNSORTED;
                if (valid[q]) prev = av[q];
            }
            carry_a = shfl_i64(prev, 31);
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
        // per request: TTFT row; o = 1 finishes at c (R13); others -> decode ring
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
            const int32_t j = i0 + q;
            if (!dec[q]) {
                *reinterpret_cast<longlong2 *>(out + 2 * (int64_t)j) =
                    make_longlong2(c[q] - av[q], c[q]);
                acc_mk = max(acc_mk, c[q]);
            } else {
                out[2 * (int64_t)j] = c[q] - av[q];
                const int e = (produced + pos) & RING_MASK;
                ring_r[e] = r[q];
                ring_dj[e] = make_uint2(dsd ? kv[q] : ov[q] - 1, (uint32_t)j);
                ++pos;
            }
        }
        produced += total;
        chunk_next += CHUNK;
        // after the last chunk, the two slots past the end read as "no request"
        if (chunk_next >= n && lane < 2) ring_r[(produced + lane) & RING_MASK] = INT64_MAX;
        __syncwarp();
    };

    if (status & GL_ST_TABLE) chunk_next = n;  // nothing to simulate

    // ---- S5: continuous-batching decode event loop ---------------------------
    // Warp-uniform state (every lane holds the same value): boundary time T,
    // iteration counter I, batch size b, ring head nxt with its fields (hr, hd,
    // hj) and one free-slot mask per slot row.  Lane-private: the members'
    // finish iterations F and request indices.
    uint32_t F[SPL], jl[SPL];
#pragma unroll
    for (int s = 0; s < SPL; ++s) {
        F[s] = F_EMPTY;
        jl[s] = 0;
    }
    int64_t T = 0, mk_dec = 0;
    uint32_t I = 0;
    int b = 0;
    int32_t nxt = 0;
    unsigned free_m[SPL];
#pragma unroll
    for (int s = 0; s < SPL; ++s) {
        const int lo = s * 32;
        free_m[s] = cap >= lo + 32 ? FULL : (cap > lo ? ((1u << (cap - lo)) - 1u) : 0u);
    }
    // Ring head (hr, hd, hj) and the request after it (nr, nd, nj), prefetched so
    // that a join never waits on shared memory.  hr = INT64_MAX: no head.
    int64_t hr = INT64_MAX, nr = INT64_MAX;
    uint32_t hd = 0, hj = 0, nd = 0, nj = 0;
    auto load_pair = [&]() {  // broadcast shared-memory loads
        hr = nxt < produced ? ring_r[nxt & RING_MASK] : INT64_MAX;
        const uint2 dh = ring_dj[nxt & RING_MASK];
        hd = dh.x;
        hj = dh.y;
        nr = nxt + 1 < produced ? ring_r[(nxt + 1) & RING_MASK] : INT64_MAX;
        const uint2 dn = ring_dj[(nxt + 1) & RING_MASK];
        nd = dn.x;
        nj = dn.y;
    };
    auto advance_head = [&]() {
        ++nxt;
        hr = nr;
        hd = nd;
        hj = nj;
        if (chunk_next < n && produced - nxt < LOOKAHEAD) {
            do produce();
            while (chunk_next < n && produced - nxt < LOOKAHEAD);
            load_pair();
        } else {
            const int e = (nxt + 1) & RING_MASK;
            nr = nxt + 1 < produced ? ring_r[e] : INT64_MAX;
            const uint2 dn = ring_dj[e];
            nd = dn.x;
            nj = dn.y;
        }
    };
    while (chunk_next < n && produced - nxt < LOOKAHEAD) produce();
    load_pair();
    const unsigned lane_bit = 1u << lane;
    if constexpr (SPL == 1) {
        // cap <= 31: one member per lane, b < 32.  fmin (the smallest finish
        // iteration) is kept warp-uniform: a join only lowers it (scalar min), so
        // the REDUX runs only after leaves.  The ring head and the request after
        // it are held in registers (h_*, n_*) so a join never waits on shared memory.
        uint32_t Fm = F_EMPTY, fmin = F_EMPTY;
        unsigned fr = free_m[0];
        uint32_t c_b = 0;  // iterations run at batch size b == lane
        int64_t *const fin_col = out + 1;
        int64_t *fa = fin_col;  // this lane's member's finish-time address
        int64_t h_r = hr, n_r = nr;
        uint2 h_dj = make_uint2(hd, hj), n_dj = make_uint2(nd, nj);
        // step[b] and its reciprocal for b-1, b, b+1 in registers, shifted when b
        // moves by one, so no shared-memory load sits on the event's critical path
        int32_t st_d = 0, st_c = 0, st_u = 0;
        uint64_t M_d = 0, M_c = 0, M_u = 0;
        auto load_nbr = [&](int nb) {
            st_c = steps[nb];
            M_c = magic[nb];
            st_u = steps[min(nb + 1, cap)];
            M_u = magic[min(nb + 1, cap)];
            st_d = steps[max(nb - 1, 0)];
            M_d = magic[max(nb - 1, 0)];
        };
        load_nbr(0);
        for (;;) {
            // ---- FCFS joins at boundary T (r <= T) while the batch has room (R16, R18)
            while (b < cap && h_r <= T) {
                if (I >= 0x80000000u) {  // rebase the 32-bit iteration counter
                    if (Fm != F_EMPTY) Fm -= I;
                    if (fmin != F_EMPTY) fmin -= I;
                    iters[0] += c_b;
                    c_b = 0;
                    I = 0;
                }
                const unsigned bit = fr & (0u - fr);
                fr ^= bit;
                const uint32_t fnew = I + h_dj.x;
                if (lane_bit == bit) {
                    Fm = fnew;
                    fa = fin_col + 2 * (int64_t)h_dj.y;
                }
                fmin = min(fmin, fnew);
                ++b;
                st_d = st_c;
                M_d = M_c;
                st_c = st_u;
                M_c = M_u;
                st_u = steps[min(b + 1, cap)];
                M_u = magic[min(b + 1, cap)];
                ++nxt;
                h_r = n_r;
                h_dj = n_dj;
                if (chunk_next < n && produced - nxt < LOOKAHEAD) {
                    do produce();
                    while (chunk_next < n && produced - nxt < LOOKAHEAD);
                    const int e = nxt & RING_MASK;
                    h_r = ring_r[e];
                    h_dj = ring_dj[e];
                }
                const int e1 = (nxt + 1) & RING_MASK;
                n_r = ring_r[e1];
                n_dj = ring_dj[e1];
            }
            if (b == 0) {  // idle until the next decode request is ready (R17)
                if (h_r == INT64_MAX) break;
                T = h_r;
                continue;
            }
            if (b == cap) {
                // Saturated fast path: with a full batch the next event is a leave;
                // while exactly one member leaves and the head is already ready, the
                // freed lane takes the head at the same boundary (R16).  Step time is
                // the constant step[cap]; any other case exits to the general loop.
                const int64_t stc = st_c;
                uint32_t it = 0;
                for (;;) {
                    const uint32_t kL = fmin - I;
                    I = fmin;
                    T += (int64_t)kL * stc;
                    it += kL;
                    const bool lv = Fm == I;
                    const unsigned lm = __ballot_sync(FULL, lv);
                    if (lv) *fa = T;
                    mk_dec = T;
                    const bool one = (lm & (lm - 1u)) == 0u;
                    if (!(one && h_r <= T && I < 0x80000000u)) {
                        if (lv) Fm = F_EMPTY;
                        fr |= lm;
                        b -= __popc(lm);
                        fmin = __reduce_min_sync(FULL, Fm);
                        break;
                    }
                    if (lv) {
                        Fm = I + h_dj.x;
                        fa = fin_col + 2 * (int64_t)h_dj.y;
                    }
                    fmin = __reduce_min_sync(FULL, Fm);
                    ++nxt;
                    h_r = n_r;
                    h_dj = n_dj;
                    if (chunk_next < n && produced - nxt < LOOKAHEAD) {
                        do produce();
                        while (chunk_next < n && produced - nxt < LOOKAHEAD);
                        const int e = nxt & RING_MASK;
                        h_r = ring_r[e];
                        h_dj = ring_dj[e];
                    }
                    const int e1 = (nxt + 1) & RING_MASK;
                    n_r = ring_r[e1];
                    n_dj = ring_dj[e1];
                }
                c_b += (lane == cap) ? it : 0u;
                if (b == cap - 1) {
                    st_u = st_c;
                    M_u = M_c;
                    st_c = st_d;
                    M_c = M_d;
                    st_d = steps[max(b - 1, 0)];
                    M_d = magic[max(b - 1, 0)];
                } else {
                    load_nbr(b);
                }
                continue;
            }
            {
                // Light-load fast path (0 < b < cap, head not ready at T): each
                // step is either the head's join at kJ = ceil(gap / step[b]) or the
                // next leave at kL; it exits to the general loop when a join finds
                // the batch full or another ready head, when the batch empties, or
                // (to the general event code below) on a very long gap or a rebase.
                bool slow = false;
                for (;;) {
                    const int64_t st = st_c;
                    const uint32_t kL = fmin - I;
                    const int64_t gap = h_r - T;
                    const uint32_t kJ = ceil_div_magic((uint32_t)gap, (uint32_t)st, M_c);
                    if (gap >= 0x80000000ll || I >= 0x80000000u) {
                        slow = true;
                        break;
                    }
                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;
                        I += kJ;
                        c_b += (lane == b) ? kJ : 0u;
                        const unsigned bit = fr & (0u - fr);
                        fr ^= bit;
                        const uint32_t fnew = I + h_dj.x;
                        if (lane_bit == bit) {
                            Fm = fnew;
                            fa = fin_col + 2 * (int64_t)h_dj.y;
                        }
                        fmin = min(fmin, fnew);
                        ++b;
                        st_d = st_c;
                        M_d = M_c;
                        st_c = st_u;
                        M_c = M_u;
                        st_u = steps[min(b + 1, cap)];
                        M_u = magic[min(b + 1, cap)];
                        ++nxt;
                        h_r = n_r;
                        h_dj = n_dj;
                        if (chunk_next < n && produced - nxt < LOOKAHEAD) {
                            do produce();
                            while (chunk_next < n && produced - nxt < LOOKAHEAD);
                            const int e = nxt & RING_MASK;
                            h_r = ring_r[e];
                            h_dj = ring_dj[e];
                        }
                        const int e1 = (nxt + 1) & RING_MASK;
                        n_r = ring_r[e1];
                        n_dj = ring_dj[e1];
                        if (b == cap || h_r <= T) break;
                    } else {  // leave at iteration fmin (R16)
                        T += (int64_t)kL * st;
                        I = fmin;
                        c_b += (lane == b) ? kL : 0u;
                        const bool lv = Fm == I;
                        const unsigned lm = __ballot_sync(FULL, lv);
                        if (lv) {
                            *fa = T;
                            Fm = F_EMPTY;
                        }
                        fr |= lm;
                        const int nl = __popc(lm);
                        b -= nl;
                        mk_dec = T;
                        fmin = __reduce_min_sync(FULL, Fm);
                        if (nl == 1) {
                            st_u = st_c;
                            M_u = M_c;
                            st_c = st_d;
                            M_c = M_d;
                            st_d = steps[max(b - 1, 0)];
                            M_d = magic[max(b - 1, 0)];
                        } else {
                            load_nbr(b);
                        }
                        if (b == 0 || h_r <= T) break;
                    }
                }
                if (!slow) continue;
            }
            // ---- next event: a join at kJ < kL, else the leave at kL (R16)
            const int64_t st = st_c;
            const uint32_t kL = fmin - I;
            if (b < cap) {  // the head may join before the next leave
                const int64_t gap = h_r - T;  // > 0: the head was not admitted at T
                uint32_t kJ = ceil_div_magic((uint32_t)gap, (uint32_t)st, M_c);
                const bool far = gap >= 0x80000000ll;  // rare: very long gap, or no head
                if (kJ < kL || far) {
                    if (far)  // exact 64-bit path; no head (INT64_MAX) never joins
                        kJ = (h_r != INT64_MAX && gap <= (int64_t)(kL - 1) * st)
                                 ? (uint32_t)((gap + st - 1) / st) : 0xFFFFFFFFu;
                    if (kJ < kL) {  // join event: nobody leaves before the head joins
                        T += (int64_t)kJ * st;
                        I += kJ;
                        c_b += (lane == b) ? kJ : 0u;
                        continue;
                    }
                }
            }
            T += (int64_t)kL * st;
            I = fmin;
            c_b += (lane == b) ? kL : 0u;
            const bool lv = Fm == I;
            const unsigned lm = __ballot_sync(FULL, lv);
            if (lv) {
                *fa = T;
                Fm = F_EMPTY;
            }
            fr |= lm;
            const int nl = __popc(lm);
            b -= nl;
            mk_dec = T;
            fmin = __reduce_min_sync(FULL, Fm);
            if (nl == 1) {
                st_u = st_c;
                M_u = M_c;
                st_c = st_d;
                M_c = M_d;
                st_d = steps[max(b - 1, 0)];
                M_d = magic[max(b - 1, 0)];
            } else {  // several members left at once
                load_nbr(b);
            }
        }
        iters[0] += c_b;
    } else for (;;) {
        // FCFS joins at boundary T (r <= T) while the batch has room (R16, R18)
        while (b < cap && hr <= T) {
            if (I >= 0x80000000u) {  // rebase the 32-bit iteration counter (F = I + d fits)
#pragma unroll
                for (int s = 0; s < SPL; ++s)
                    if (F[s] != F_EMPTY) F[s] -= I;
#pragma unroll
                for (int s = 0; s <= SPL; ++s) {
                    iters[s] += cnt[s];
                    cnt[s] = 0;
                }
                I = 0;
            }
            if (SPL == 1) {  // lowest free lane takes the head
                const unsigned bit = free_m[0] & (0u - free_m[0]);
                free_m[0] ^= bit;
                if (lane_bit == bit) {
                    F[0] = I + hd;
                    jl[0] = hj;
                }
            } else {
                int s_sel = SPL;
                unsigned bit = 0;
#pragma unroll
                for (int s = SPL - 1; s >= 0; --s)
                    if (free_m[s]) {
                        s_sel = s;
                        bit = free_m[s] & (0u - free_m[s]);
                    }
#pragma unroll
                for (int s = 0; s < SPL; ++s) {
                    if (s == s_sel) {
                        free_m[s] ^= bit;
                        if (lane_bit == bit) {
                            F[s] = I + hd;
                            jl[s] = hj;
                        }
                    }
                }
            }
            ++b;
            advance_head();
        }
        if (b == 0) {  // idle until the next decode request is ready (R17)
            if (hr == INT64_MAX) break;
            T = hr;
            continue;
        }
        // Next event: the first member leave (kL iterations away, REDUX min) or the
        // boundary at which the head joins (kJ = ceil(gap / step)); kJ does not
        // depend on kL, so the reciprocal multiply overlaps the REDUX latency.
        const int64_t st = steps[b];
        const int64_t gap = hr - T;  // > 0 whenever b < cap: the head was not admitted at T
        uint32_t kJ = ceil_div_magic((uint32_t)gap, (uint32_t)st, magic[b]);
        if (b >= cap) kJ = 0xFFFFFFFFu;
        if (gap >= 0x80000000ll && b < cap)  // rare: very long gaps, or no head (INT64_MAX)
            kJ = hr == INT64_MAX ? 0xFFFFFFFFu
                                 : (uint32_t)min((gap + st - 1) / st, (int64_t)0xFFFFFFFF);
        uint32_t fmin = F[0];
#pragma unroll
        for (int s = 1; s < SPL; ++s) fmin = min(fmin, F[s]);
        fmin = __reduce_min_sync(FULL, fmin);
        const uint32_t kL = fmin - I;
        const uint32_t k = min(kL, kJ);
        T += (int64_t)k * st;
        I += k;
        {
            const uint32_t kk = (lane == (b & 31)) ? k : 0u;
            const int row = b >> 5;
#pragma unroll
            for (int s = 0; s <= SPL; ++s) cnt[s] += (s == row) ? kk : 0u;
        }
        // leaves at boundary T (R16): finish = T.  No branch: when k < kL no
        // member has F == I.
        int nl = 0;
#pragma unroll
        for (int s = 0; s < SPL; ++s) {
            const bool lv = F[s] == I;
            free_m[s] |= __ballot_sync(FULL, lv);
            nl += (int)__reduce_add_sync(FULL, lv ? 1u : 0u);
            if (lv) out[2 * (int64_t)jl[s] + 1] = T;
            F[s] = lv ? F_EMPTY : F[s];
        }
        b -= nl;
        mk_dec = nl ? T : mk_dec;
    }
#pragma unroll
    for (int s = 0; s <= SPL; ++s) iters[s] += cnt[s];

    // ---- S7: chain reductions (SLO counts and the hash: k_finalize) ------------
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
    const int64_t tokens = warp_sum_i64(acc_tokens);
    const int64_t mk = max(warp_max_i64(acc_mk), mk_dec);
    status = __reduce_or_sync(FULL, status);
    if (lane == 0) {
        gl_chain_stats o;
        o.n = ch.n;
        o.slo_ok = 0;
        o.tokens = tokens;
        o.busy_new_us = busy_new;
        o.busy_old_us = busy_old;
        o.e_new_uj = e_new;
        o.e_old_uj = e_old;
        o.makespan_us = mk;
        o.req_hash = 0;
        o.status = status;
        o.capacity_ok = (uint32_t)ch.capacity_ok;
        stats[blockIdx.x] = o;
    }
}

// ---- S6 + S7: per-request SLO test and hash, the whole GPU over (chain, request)
//   ok_j = TTFT_j <= SLO_ttft and (o_j = 1 or finish_j - c_j <= SLO_tpot (o_j - 1))
//   (Table 2; R25-R27), hash += mix64(j, ttft_j, finish_j).
// Integer atomics commute, so the result is deterministic.
__global__ void __launch_bounds__(256)
    k_finalize(const DChain *__restrict__ chains, gl_chain_stats *__restrict__ stats,
               const int64_t *__restrict__ perreq, int per_thread)
{
    __shared__ unsigned long long s_ok[8], s_hash[8];
    const DChain &ch = chains[blockIdx.y];
    const int64_t n = ch.n;
    const int64_t *rows = perreq + 2 * ch.out_off;
    const int64_t ttft_slo = ch.ttft_slo, tpot_slo = ch.tpot_slo;
    unsigned long long ok = 0, hash = 0;
    const int64_t base = (int64_t)blockIdx.x * blockDim.x * per_thread;
    for (int q = 0; q < per_thread; ++q) {
        const int64_t j = base + (int64_t)q * blockDim.x + threadIdx.x;
        if (j < n) {
            const longlong2 tf = __ldg(reinterpret_cast<const longlong2 *>(rows) + j);
            const int64_t a = __ldg(ch.a + j);
            uint32_t o = __ldg(ch.o + j);
            o = min(max(o, 1u), O_LIMIT - 1);
            const int64_t c = a + tf.x;
            const bool good = tf.x <= ttft_slo &&
                              (o == 1 || tf.y - c <= tpot_slo * (int64_t)(o - 1));
            ok += good ? 1 : 0;
            hash += splitmix_fin((uint64_t)j ^ rotl64((uint64_t)tf.x, 21) ^
                                 rotl64((uint64_t)tf.y, 42));
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        ok += __shfl_xor_sync(FULL, ok, off);
        hash += __shfl_xor_sync(FULL, hash, off);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_ok[w] = ok;
        s_hash[w] = hash;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            ok += s_ok[i];
            hash += s_hash[i];
        }
        if (ok) atomicAdd(reinterpret_cast<unsigned long long *>(&stats[blockIdx.y].slo_ok), ok);
        atomicAdd(reinterpret_cast<unsigned long long *>(&stats[blockIdx.y].req_hash), hash);
    }
}

}  // namespace gl
