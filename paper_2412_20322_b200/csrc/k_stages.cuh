// k_stages.cuh -- S0-S4 for every timing chain and the segment starts the decode
// speculation uses.
//
//   stage 1  prefill FCFS on the new GPU   c_i = max(c_{i-1}, a_i) + t1[p_i]
//            (TTFT_i = c_i - a_i; R8-R10)
//   stage 2  DPD KV link (R11) / DSD handoff + draft prefill (R12):
//                                           r_i = max(r_{i-1}, c_i) + t2[p_i]  (o_i > 1)
//
// Both stages are max-plus recurrences: element i is the map x -> max(x + A_i, B_i)
// (A = s_i, B = a_i + s_i, resp. c_i + s_i) and a prefix is the composition
// (A, B) o (A', B') = (A + A', max(B + A', B')).  S blocks of ST_WARPS warps per
// chain (S from the host: as many as fit co-resident, S = 1 for many chains); warp w
// of block s owns the contiguous run s * ST_WARPS + w of 128-request chunks, and a
// block waits (acquire) for the aggregates its predecessors publish (release):
//   pass 1  aggregate of stage 1 over the run, decode count, stage sums, status
//   pass 2  carry-in = composition of the previous runs' aggregates -> c_i, and
//           the stage-2 aggregate of the run
//   pass 3  both carries -> c_i, r_i: TTFT rows (and the finish of o = 1 requests,
//           R13), and the compacted decode stream (r, demand, request index) in
//           HBM for k_decode, at the run's offset from the decode-count prefix.
// Within a chunk each lane holds 4 consecutive requests (128-bit loads) and the
// warp scans (A, B) pairs with shuffles.  The prompt-indexed t1/t2 tables are
// staged in shared memory by TMA bulk copies (cp.async.bulk + mbarrier).
#pragma once

#include "common.cuh"

namespace gl {

constexpr int ST_WARPS = 16;
constexpr int ST_MAX_SPLIT = 4;  // blocks per chain
constexpr int DEC_TAIL = 416;    // decode-stream entries written past M (< the 512 allocated)

struct MP {  // max-plus map x -> max(x + A, B)
    int64_t A, B;
};
__device__ __forceinline__ MP mp_then(const MP &f, const MP &g)  // g o f (f first)
{
    return MP{f.A + g.A, max(f.B + g.A, g.B)};
}

struct ChunkIn {
    int64_t av[4];
    uint32_t pc[4], oc[4], kv[4];
    bool valid[4], dec[4];
    int64_t s1[4], s2[4], xa[4];
};

__device__ __forceinline__ void load_chunk(const DChain &ch, const int32_t *t1s, const int32_t *t2s,
                                           int32_t i0, int32_t n, int P, bool dsd, ChunkIn &c,
                                           uint32_t &status)
{
    uint32_t pv[4], ov[4];
    if (i0 + 3 < n) {  // 128-bit loads: 2 x (2 x int64) + (4 x u32) per stream
        const longlong2 x0 = __ldg(reinterpret_cast<const longlong2 *>(ch.a + i0));
        const longlong2 x1 = __ldg(reinterpret_cast<const longlong2 *>(ch.a + i0) + 1);
        const uint4 pp = __ldg(reinterpret_cast<const uint4 *>(ch.p + i0));
        const uint4 oo = __ldg(reinterpret_cast<const uint4 *>(ch.o + i0));
        c.av[0] = x0.x; c.av[1] = x0.y; c.av[2] = x1.x; c.av[3] = x1.y;
        pv[0] = pp.x; pv[1] = pp.y; pv[2] = pp.z; pv[3] = pp.w;
        ov[0] = oo.x; ov[1] = oo.y; ov[2] = oo.z; ov[3] = oo.w;
        if (dsd) {
            const uint4 kk = __ldg(reinterpret_cast<const uint4 *>(ch.K + i0));
            c.kv[0] = kk.x; c.kv[1] = kk.y; c.kv[2] = kk.z; c.kv[3] = kk.w;
        } else {
            c.kv[0] = c.kv[1] = c.kv[2] = c.kv[3] = 0;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const bool v = i0 + q < n;
            c.av[q] = v ? __ldg(ch.a + i0 + q) : 0;
            pv[q] = v ? __ldg(ch.p + i0 + q) : 1;
            ov[q] = v ? __ldg(ch.o + i0 + q) : 1;
            c.kv[q] = (v && dsd) ? __ldg(ch.K + i0 + q) : 0;
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        c.valid[q] = i0 + q < n;
        uint32_t p = pv[q], o = ov[q];
        if (c.valid[q]) {
            if (c.av[q] < 0) status |= GL_ST_NEG_ARRIVAL;
            if (p < 1 || p > (uint32_t)P) status |= GL_ST_PROMPT_RANGE;
            if (o == 0) status |= GL_ST_OUTPUT_ZERO;
            if (o >= O_LIMIT) status |= GL_ST_OVERFLOW;
        }
        p = min(max(p, 1u), (uint32_t)P);
        o = min(max(o, 1u), O_LIMIT - 1);
        c.pc[q] = p;
        c.oc[q] = o;
        c.dec[q] = c.valid[q] && o > 1;
        c.s1[q] = c.valid[q] ? t1s[p] : 0;
        c.s2[q] = c.dec[q] ? t2s[p] : 0;
        c.xa[q] = c.valid[q] ? c.av[q] : NEG_INF;
    }
}

// inclusive warp scan of per-lane maps (lane order = request order)
__device__ __forceinline__ MP warp_scan_mp(MP f, int lane)
{
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int64_t Ap = shfl_up_i64(f.A, off), Bp = shfl_up_i64(f.B, off);
        if (lane >= off) f = mp_then(MP{Ap, Bp}, f);
    }
    return f;
}

// stage-1 values of a chunk given the carry c_prev; returns the new carry
__device__ __forceinline__ int64_t chunk_stage1(const ChunkIn &c, int64_t carry, int lane,
                                                int64_t (&cv)[4])
{
    MP f{0, NEG_INF};
#pragma unroll
    for (int q = 0; q < 4; ++q) f = mp_then(f, MP{c.s1[q], c.xa[q] + c.s1[q]});
    const MP inc = warp_scan_mp(f, lane);
    int64_t Ax = shfl_up_i64(inc.A, 1), Bx = shfl_up_i64(inc.B, 1);
    if (lane == 0) {
        Ax = 0;
        Bx = NEG_INF;
    }
    int64_t x = max(carry + Ax, Bx);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        x = max(x, c.xa[q]) + c.s1[q];
        cv[q] = c.valid[q] ? x : NEG_INF;
    }
    return shfl_i64(x, 31);
}

// stage-2 values of a chunk given c and the carry r_prev; returns the new carry
__device__ __forceinline__ int64_t chunk_stage2(const ChunkIn &c, const int64_t (&cv)[4],
                                                int64_t carry, int lane, int64_t (&rv)[4])
{
    MP f{0, NEG_INF};
#pragma unroll
    for (int q = 0; q < 4; ++q) f = mp_then(f, MP{c.s2[q], cv[q] + c.s2[q]});
    const MP inc = warp_scan_mp(f, lane);
    int64_t Ax = shfl_up_i64(inc.A, 1), Bx = shfl_up_i64(inc.B, 1);
    if (lane == 0) {
        Ax = 0;
        Bx = NEG_INF;
    }
    int64_t y = max(carry + Ax, Bx);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        y = max(y, cv[q]) + c.s2[q];
        rv[q] = y;
    }
    return shfl_i64(y, 31);
}

// aggregate map of a chunk's elements (lane 31's inclusive scan, broadcast)
__device__ __forceinline__ MP chunk_aggregate(const int64_t (&s)[4], const int64_t (&b)[4], int lane)
{
    MP f{0, NEG_INF};
#pragma unroll
    for (int q = 0; q < 4; ++q) f = mp_then(f, MP{s[q], b[q] + s[q]});
    const MP inc = warp_scan_mp(f, lane);
    return MP{shfl_i64(inc.A, 31), shfl_i64(inc.B, 31)};
}

// the composition of the predecessors' aggregates, as the B-value applied to -inf,
// and the sum of their decode counts (thread 0 of a block; spins on release flags)
__device__ __forceinline__ void stage_lookback(const DChain &ch, int s, bool second,
                                              int64_t &carry, int32_t &dbase)
{
    carry = NEG_INF;
    dbase = 0;
    for (int p = 0; p < s; ++p) {
        DStagePart &q = ch.stp[p];
        int32_t *flag = second ? &q.flag2 : &q.flag1;
        while (ld_acquire_gpu(flag) == 0) {
        }
        const int64_t A = __ldcg(second ? &q.agg2_A : &q.agg1_A);
        const int64_t B = __ldcg(second ? &q.agg2_B : &q.agg1_B);
        carry = max(carry + A, B);
        dbase += __ldcg(&q.dcount);
    }
}

__global__ void __launch_bounds__(32 * ST_WARPS, 1)
    k_stages(const DChain *__restrict__ chains, gl_chain_stats *__restrict__ stats,
             int64_t *__restrict__ perreq, int32_t S, int32_t *__restrict__ ticket,
             const int32_t *__restrict__ ids,  // chains to run (primaries), NULL = all
             int32_t defer_dsd)  // DSD chains: demand 0 in the stream, filled in later
{
    __shared__ int32_t s_vid;
    __shared__ int64_t s_carry;
    __shared__ int32_t s_dbase;
    __shared__ int32_t s_last;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int64_t agg_A[ST_WARPS], agg_B[ST_WARPS];
    __shared__ int32_t dcount[ST_WARPS];
    __shared__ int64_t red[6][ST_WARPS];
    __shared__ uint32_t red_status[ST_WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // virtual block ids in the order blocks start: a block only ever waits on blocks
    // with smaller ids, which are already running (no assumption on dispatch order)
    if (threadIdx.x == 0) s_vid = S > 1 ? atomicAdd(ticket, 1) : (int32_t)blockIdx.x;
    __syncthreads();
    const int32_t chain = ids ? ids[s_vid / S] : s_vid / S, sblk = s_vid % S;
    const DChain ch = chains[chain];
    const int P = ch.max_prompt, cap = ch.cap;
    const int p1pad = round_up4(P + 1);
    int32_t *t1s = reinterpret_cast<int32_t *>(smem);
    int32_t *t2s = t1s + p1pad;
    uint64_t *bar = reinterpret_cast<uint64_t *>(t2s + p1pad);
    int64_t *out = perreq + 2 * ch.out_off;

    // ---- S0: stage the prompt-indexed tables (TMA bulk copies + mbarrier) -----
    if (warp == 0) {
        if (lane == 0) mbar_init(bar, 1);
        __syncwarp();
        uint32_t tx = stage_table(t1s, ch.t1, P + 1, bar, lane);
        tx += stage_table(t2s, ch.t2, P + 1, bar, lane);
        if (lane == 0) mbar_arrive_expect_tx(bar, tx);
        mbar_wait(bar, 0);
    }
    __syncthreads();

    // invalid tables (GL_ST_TABLE): prompt-indexed ones skip the passes; a step table
    // does not (the passes never read it), so chains cloning this one's stage results
    // (k_stage_clone) get valid partials whatever this chain's own step table holds
    uint32_t status = 0;
    bool step_bad;
    {
        bool bad = false, sbad = false;
        for (int i = 1 + threadIdx.x; i <= P; i += blockDim.x) bad |= (t1s[i] < 0) | (t2s[i] < 0);
        for (int b = 1 + threadIdx.x; b <= cap; b += blockDim.x) sbad |= __ldg(ch.step + b) < 1;
        if (__syncthreads_or(bad)) status |= GL_ST_TABLE;
        step_bad = __syncthreads_or(sbad);
    }
    const bool skip = status & GL_ST_TABLE;

    const int32_t n = (int32_t)ch.n;
    const bool colo = ch.mode == GL_MODE_STANDALONE || ch.mode == GL_MODE_SPEC_COLO;
    // demand K_j -- or, deferred (disaggregated DSD while k_dsd_family / k_dsd_demand
    // still run on another stream), 0 now and k_stage_clone's fill pass writes K_j
    const bool dsd = (ch.mode == GL_MODE_DSD && !defer_dsd) || ch.mode == GL_MODE_SPEC_COLO;
    const int32_t nchunks = (n + CHUNK - 1) / CHUNK;
    const int32_t runs = ST_WARPS * S, run = sblk * ST_WARPS + warp;
    const int32_t per = (nchunks + runs - 1) / runs;
    const int32_t c_lo = min(run * per, nchunks), c_hi = min(c_lo + per, nchunks);

    // ---- pass 1: stage-1 aggregate, decode count, stage sums, status -----------
    int64_t acc_busy_new = 0, acc_busy_old = 0, acc_e_new = 0, acc_e_old = 0, acc_tokens = 0;
    MP agg1{0, NEG_INF};
    int32_t ndec = 0;
    int64_t carry_a = (c_lo > 0 && c_lo < nchunks) ? __ldg(ch.a + (int64_t)c_lo * CHUNK - 1) : INT64_MIN;
    for (int32_t ck = c_lo; ck < c_hi && !skip; ++ck) {
        ChunkIn c;
        load_chunk(ch, t1s, t2s, ck * CHUNK + 4 * lane, n, P, dsd, c, status);
        int cnt = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (c.valid[q]) {
                acc_busy_new += c.s1[q];
                acc_e_new += __ldg(ch.e1 + c.pc[q]);
                acc_tokens += c.oc[q];
            }
            if (c.dec[q] && !colo) {
                acc_busy_old += __ldg(ch.b2 + c.pc[q]);
                acc_e_old += __ldg(ch.e2 + c.pc[q]);
                ++cnt;
            }
        }
        if (colo) {
            // Co-located modes: no stage scans; every request enters the decode
            // stream at its arrival with its demand and prefill time (k_decode
            // runs prefills and iterations on the one GPU, R41-R42).
            const int32_t i0 = ck * CHUNK + 4 * lane;
            if (i0 + 3 < n) {
                int64_t *dr = ch.dec_r + i0;
                *reinterpret_cast<longlong2 *>(dr) = make_longlong2(c.av[0], c.av[1]);
                *reinterpret_cast<longlong2 *>(dr + 2) = make_longlong2(c.av[2], c.av[3]);
                uint4 *dd = reinterpret_cast<uint4 *>(ch.dec_dj + i0);
                const uint32_t d0 = dsd ? c.kv[0] : c.oc[0] - 1, d1 = dsd ? c.kv[1] : c.oc[1] - 1;
                const uint32_t d2 = dsd ? c.kv[2] : c.oc[2] - 1, d3 = dsd ? c.kv[3] : c.oc[3] - 1;
                dd[0] = make_uint4(d0, (uint32_t)i0, d1, (uint32_t)i0 + 1);
                dd[1] = make_uint4(d2, (uint32_t)i0 + 2, d3, (uint32_t)i0 + 3);
                *reinterpret_cast<int4 *>(ch.dec_pf + i0) =
                    make_int4((int)c.s1[0], (int)c.s1[1], (int)c.s1[2], (int)c.s1[3]);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (!c.valid[q]) continue;
                    ch.dec_r[i0 + q] = c.av[q];
                    ch.dec_dj[i0 + q] = make_uint2(dsd ? c.kv[q] : c.oc[q] - 1, (uint32_t)(i0 + q));
                    ch.dec_pf[i0 + q] = (int32_t)c.s1[q];
                }
            }
            cnt = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) cnt += c.valid[q] ? 1 : 0;
        }
        {  // sortedness across the lane boundary and the chunk / run boundary
            int64_t prev = shfl_up_i64(c.av[3], 1);
            if (lane == 0) prev = carry_a;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (c.valid[q] && c.av[q] < prev) status |= GL_ST_UNSORTED;
                if (c.valid[q]) prev = c.av[q];
            }
            carry_a = shfl_i64(prev, 31);
        }
        agg1 = mp_then(agg1, chunk_aggregate(c.s1, c.xa, lane));
        ndec += __reduce_add_sync(FULL, (unsigned)cnt);
    }
    if (lane == 0) {
        agg_A[warp] = agg1.A;
        agg_B[warp] = agg1.B;
        dcount[warp] = ndec;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // publish this block's aggregate, then look back
        DStagePart &me = ch.stp[sblk];
        MP a{0, NEG_INF};
        int32_t dc = 0;
        for (int w = 0; w < ST_WARPS; ++w) {
            a = mp_then(a, MP{agg_A[w], agg_B[w]});
            dc += dcount[w];
        }
        me.agg1_A = a.A;
        me.agg1_B = a.B;
        me.dcount = dc;
        __threadfence();
        st_release_gpu(&me.flag1, 1);
        int64_t cin;
        int32_t db;
        stage_lookback(ch, sblk, false, cin, db);
        s_carry = cin;
        s_dbase = db;
    }
    __syncthreads();
    int64_t carry_c = s_carry;  // = B of the composition of the previous runs
    int32_t dbase = s_dbase;
    for (int w = 0; w < warp; ++w) {
        carry_c = max(carry_c + agg_A[w], agg_B[w]);
        dbase += dcount[w];
    }
    int32_t M = 0;
    for (int w = 0; w < ST_WARPS; ++w) M += dcount[w];  // this block's share
    __syncthreads();

    // ---- pass 2: c with the true carry, stage-2 aggregate ---------------------
    MP agg2{0, NEG_INF};
    if (!colo) {
        int64_t cc = carry_c;
        for (int32_t ck = c_lo; ck < c_hi && !skip; ++ck) {
            ChunkIn c;
            uint32_t dummy = 0;
            load_chunk(ch, t1s, t2s, ck * CHUNK + 4 * lane, n, P, dsd, c, dummy);
            int64_t cv[4];
            cc = chunk_stage1(c, cc, lane, cv);
            agg2 = mp_then(agg2, chunk_aggregate(c.s2, cv, lane));
        }
    }
    if (lane == 0) {
        agg_A[warp] = agg2.A;
        agg_B[warp] = agg2.B;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        DStagePart &me = ch.stp[sblk];
        MP a{0, NEG_INF};
        for (int w = 0; w < ST_WARPS; ++w) a = mp_then(a, MP{agg_A[w], agg_B[w]});
        me.agg2_A = a.A;
        me.agg2_B = a.B;
        __threadfence();
        st_release_gpu(&me.flag2, 1);
        int64_t cin;
        int32_t db;
        stage_lookback(ch, sblk, true, cin, db);
        s_carry = cin;
    }
    __syncthreads();
    int64_t carry_r = s_carry;
    for (int w = 0; w < warp; ++w) carry_r = max(carry_r + agg_A[w], agg_B[w]);

    // ---- pass 3: c, r -> rows and the compacted decode stream -----------------
    int64_t acc_mk = 0;
    if (!colo) {
        int64_t cc = carry_c, rr = carry_r;
        int32_t produced = dbase;
        for (int32_t ck = c_lo; ck < c_hi && !skip; ++ck) {
            ChunkIn c;
            uint32_t dummy = 0;
            const int32_t i0 = ck * CHUNK + 4 * lane;
            load_chunk(ch, t1s, t2s, i0, n, P, dsd, c, dummy);
            int64_t cv[4], rv[4];
            cc = chunk_stage1(c, cc, lane, cv);
            rr = chunk_stage2(c, cv, rr, lane, rv);
            int cnt = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) cnt += c.dec[q] ? 1 : 0;
            const unsigned b0 = __ballot_sync(FULL, cnt & 1), b1 = __ballot_sync(FULL, cnt & 2),
                           b2 = __ballot_sync(FULL, cnt & 4);
            const unsigned lt = (1u << lane) - 1u;
            int pos = __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
            const int total = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (!c.valid[q]) continue;
                const int32_t j = i0 + q;
                if (!c.dec[q]) {
                    *reinterpret_cast<longlong2 *>(out + 2 * (int64_t)j) =
                        make_longlong2(cv[q] - c.av[q], cv[q]);
                    acc_mk = max(acc_mk, cv[q]);
                } else {  // finish 0 until k_decode writes it (rows always initialised)
                    *reinterpret_cast<longlong2 *>(out + 2 * (int64_t)j) =
                        make_longlong2(cv[q] - c.av[q], 0);
                    const int64_t e = (int64_t)produced + pos;
                    ch.dec_r[e] = rv[q];
                    ch.dec_dj[e] = make_uint2(dsd ? c.kv[q] : c.oc[q] - 1, (uint32_t)j);
                    ++pos;
                }
            }
            produced += total;
        }
    }

    // ---- block reductions and the chain's partial statistics ---------------------
    const int64_t v[6] = {warp_sum_i64(acc_busy_new), warp_sum_i64(acc_busy_old),
                          warp_sum_i64(acc_e_new), warp_sum_i64(acc_e_old),
                          warp_sum_i64(acc_tokens), warp_max_i64(acc_mk)};
    status = __reduce_or_sync(FULL, status);
    if (lane == 0) {
        for (int i = 0; i < 6; ++i) red[i][warp] = v[i];
        red_status[warp] = status;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // this block's partials; the chain's last block combines
        DStagePart &me = ch.stp[sblk];
        int64_t s[6] = {0, 0, 0, 0, 0, 0};
        uint32_t st = 0;
        for (int w = 0; w < ST_WARPS; ++w) {
            for (int i = 0; i < 5; ++i) s[i] += red[i][w];
            s[5] = max(s[5], red[5][w]);
            st |= red_status[w];
        }
        for (int i = 0; i < 6; ++i) me.sums[i] = s[i];
        me.status = st;
        __threadfence();
        s_last = atomicAdd(&ch.x->stage_done, 1) == S - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    M = 0;
    for (int p = 0; p < S; ++p) M += __ldcg(&ch.stp[p].dcount);
    // two sentinels after the last decode request, and the rest of the tail the
    // decode ring prefetches (up to 2 x 128 + 2 entries past M; the host allocates
    // n + 512) set to "no request", so no copy reads uninitialised memory
    for (int t = threadIdx.x; t < DEC_TAIL; t += blockDim.x) {
        ch.dec_r[(int64_t)M + t] = INT64_MAX;
        ch.dec_dj[(int64_t)M + t] = make_uint2(0u, 0u);
        ch.dec_pf[(int64_t)M + t] = 0;
    }
    if (threadIdx.x == 0) {
        int64_t s[6] = {0, 0, 0, 0, 0, 0};
        uint32_t st = 0;
        for (int p = 0; p < S; ++p) {
            const DStagePart &q = ch.stp[p];
            for (int i = 0; i < 5; ++i) s[i] += __ldcg(&q.sums[i]);
            s[5] = max(s[5], __ldcg(&q.sums[5]));
            st |= __ldcg(&q.status);
        }
        if (step_bad) st |= GL_ST_TABLE;
        // a chain with invalid input (any status bit) keeps only n and its status;
        // its decode stage is empty (M = 0) and k_finalize skips it, so every other
        // field is 0, as in the oracle, and Alg. 1 treats it as infeasible (R55)
        const bool valid = st == 0;
        gl_chain_stats o;
        o.n = ch.n;
        o.slo_ok = 0;
        o.tokens = valid ? s[4] : 0;
        o.busy_new_us = valid ? s[0] : 0;
        o.busy_old_us = valid ? s[1] : 0;
        o.e_new_uj = valid ? s[2] : 0;
        o.e_old_uj = valid ? s[3] : 0;
        o.makespan_us = valid ? s[5] : 0;
        o.req_hash = 0;
        o.status = st;
        o.capacity_ok = (uint32_t)ch.capacity_ok;
        stats[chain] = o;
        ch.x->M = valid ? M : 0;
    }
}

// Idle-point candidates for the decode speculation.  Request q can only find the
// decode stage empty if every earlier request has finished by r_q, and request q'
// cannot finish before r_q' + pf_q' + d_q' * step_min (it joins at or after r_q',
// after its prefill pf (co-located modes; 0 otherwise), and runs d_q' iterations of
// at least step_min = min_b step[b]).  So
//     slack_q = r_q - max_{q' < q} (r_q' + pf_q' + d_q' step_min) < 0
// proves q busy; the candidates are request 0 and, per window of SEG_LEN decode
// requests, the request with the largest slack if it is >= 0 (ties: the first).
// Any choice is exact -- k_decode verifies every candidate it uses -- this one
// makes almost all candidates true idle points (SEG_LEN bounds how many there are).
// S 1024-thread blocks per chain, each over a contiguous range of windows (its
// carry-in: a plain max over the earlier windows); windows in rounds of SEG_ROUND:
//   pass 1  warp per window: max of the lower bounds          -> smem
//   scan    exclusive prefix max over windows (carry across rounds)
//   pass 2  warp per window: in-window prefix max (8 warp scans), best slack
//   per-window candidates -> seg_wc[]; the chain's last block compacts them into
//   seg_start[] (in window order)
constexpr int SEG_ROUND = 128;  // windows per round: a round (512 KB per chain) stays in L2 for pass 2

__global__ void __launch_bounds__(1024)
    k_segments(const DChain *__restrict__ chains, int32_t S, int64_t wc_delta)
{
    __shared__ int64_t wpre[SEG_ROUND];
    __shared__ int32_t s_min_step;
    __shared__ int32_t s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int32_t chain = (int32_t)(blockIdx.x / S), sb = (int32_t)(blockIdx.x % S);
    const DChain &ch = chains[chain];
    // each window's candidate (q) or -1: a scratch array laid out like seg_start,
    // wc_delta entries after it (kept out of DChain, whose layout k_decode sees)
    int32_t *const seg_wc = ch.seg_start + wc_delta;
    const int32_t M = ch.x->M;
    const bool colo = ch.mode == GL_MODE_STANDALONE || ch.mode == GL_MODE_SPEC_COLO;
    if (threadIdx.x == 0) s_min_step = INT32_MAX;
    __syncthreads();
    {
        int32_t m = INT32_MAX;
        for (int b = 1 + threadIdx.x; b <= ch.cap; b += blockDim.x) m = min(m, __ldg(ch.step + b));
        m = __reduce_min_sync(FULL, (unsigned)m);
        if (lane == 0) atomicMin(&s_min_step, m);
    }
    __syncthreads();
    const int64_t smin = s_min_step;
    auto lb_of = [&](int32_t q) -> int64_t {  // finish-time lower bound of request q
        return __ldg(ch.dec_r + q) + (int64_t)__ldg(&ch.dec_dj[q].x) * smin +
               (colo ? __ldg(ch.dec_pf + q) : 0);
    };
    const int32_t nwin = (M + SEG_LEN - 1) / SEG_LEN;
    // block sb of the chain's S blocks takes a contiguous range of windows; its
    // carry-in is the max lower bound over all earlier windows (a plain reduction)
    const int32_t per = (nwin + S - 1) / S;
    const int32_t wlo = min(sb * per, nwin), whi = min(wlo + per, nwin);
    int64_t carry = NEG_INF;  // max lower bound over all earlier windows (warp 0)
    if (wlo > 0 && wlo < whi) {  // (earlier windows are full: wlo * SEG_LEN <= M)
        int64_t m = NEG_INF;
        const int32_t qe = wlo * SEG_LEN;
        for (int32_t q = threadIdx.x; q < qe; q += blockDim.x) m = max(m, lb_of(q));
        m = warp_max_i64(m);
        if (lane == 0) wpre[warp] = m;
        __syncthreads();
        if (warp == 0) carry = warp_max_i64(lane < nw ? wpre[lane] : NEG_INF);
        __syncthreads();
    }
    for (int32_t w0 = wlo; w0 < whi; w0 += SEG_ROUND) {
        const int32_t nwr = min(SEG_ROUND, whi - w0);
        for (int32_t w = warp; w < nwr; w += nw) {  // pass 1
            const int32_t lo = (w0 + w) * SEG_LEN, hi = min(lo + SEG_LEN, M);
            int64_t m = NEG_INF;
#pragma unroll
            for (int u = 0; u < SEG_LEN / 32; ++u) {  // all loads of the window in flight
                const int32_t q = lo + 32 * u + lane;
                if (q < hi) m = max(m, lb_of(q));
            }
            m = warp_max_i64(m);
            if (lane == 0) wpre[w] = m;
        }
        __syncthreads();
        if (warp == 0) {  // exclusive prefix max over the round's windows
            int64_t run = carry;
            for (int32_t base = 0; base < nwr; base += 32) {
                const int32_t w = base + lane;
                int64_t v = w < nwr ? wpre[w] : NEG_INF;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int64_t u = shfl_up_i64(v, off);
                    if (lane >= off) v = max(v, u);
                }
                int64_t ex = shfl_up_i64(v, 1);
                ex = lane == 0 ? run : max(run, ex);
                if (w < nwr) wpre[w] = ex;
                run = max(run, shfl_i64(v, 31));
            }
            carry = run;  // lane-uniform
        }
        __syncthreads();
        for (int32_t w = warp; w < nwr; w += nw) {  // pass 2
            const int32_t lo = (w0 + w) * SEG_LEN, hi = min(lo + SEG_LEN, M);
            int64_t pre = wpre[w];
            int64_t best = -1;
            int32_t best_q = INT32_MAX;
            int64_t rqs[SEG_LEN / 32], lbs[SEG_LEN / 32];
#pragma unroll
            for (int u = 0; u < SEG_LEN / 32; ++u) {  // all loads of the window in flight
                const int32_t q = lo + 32 * u + lane;
                const bool v = q < hi;
                rqs[u] = v ? __ldg(ch.dec_r + q) : 0;
                lbs[u] = v ? rqs[u] + (int64_t)__ldg(&ch.dec_dj[q].x) * smin +
                                 (colo ? __ldg(ch.dec_pf + q) : 0)
                           : NEG_INF;
            }
#pragma unroll
            for (int u = 0; u < SEG_LEN / 32; ++u) {
                const int32_t q = lo + 32 * u + lane;
                const bool v = q < hi;
                const int64_t rq = rqs[u];
                int64_t inc = lbs[u];
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int64_t t = shfl_up_i64(inc, off);
                    if (lane >= off) inc = max(inc, t);
                }
                int64_t ex = shfl_up_i64(inc, 1);
                ex = lane == 0 ? pre : max(pre, ex);
                const int64_t slack = rq - ex;
                if (v && slack >= 0 && (slack > best || (slack == best && q < best_q))) {
                    best = slack;
                    best_q = q;
                }
                pre = max(pre, shfl_i64(inc, 31));
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                const int64_t ob = __shfl_xor_sync(FULL, best, off);
                const int32_t oq = __shfl_xor_sync(FULL, best_q, off);
                if (ob > best || (ob == best && oq < best_q)) {
                    best = ob;
                    best_q = oq;
                }
            }
            if (lane == 0) seg_wc[w0 + w] = (w0 + w == 0) ? 0 : (best >= 0 ? best_q : -1);
        }
        __syncthreads();
    }
    // the chain's last block compacts every window's candidate into seg_start[]
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&ch.x->seg_done, 1) == S - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    int32_t ncand = 0;
    if (warp == 0) {
        for (int32_t base = 0; base < nwin; base += 32) {
            const int32_t w = base + lane;
            const int32_t cq = w < nwin ? __ldcg(seg_wc + w) : -1;
            const unsigned bal = __ballot_sync(FULL, cq >= 0);
            if (cq >= 0) ch.seg_start[ncand + __popc(bal & ((1u << lane) - 1u))] = cq;
            ncand += __popc(bal);
        }
        if (lane == 0) {
            ch.seg_start[ncand] = M;
            ch.x->nseg = ncand;
            ch.x->leader_pos = 0;
            ch.x->next_seg = 1;
        }
    }
}

// Stage results of a SECONDARY chain -- same trace and prompt-indexed tables as its
// primary (so identical stage-1/2 scans, TTFT rows and stage sums), its own mode,
// step table and demand -- taken from the primary's k_stages partials instead of
// re-running the scans (configuration 5: 320 chains, 8 primaries).  Per secondary:
// the statistics (its own step-table check and capacity flag, R55 if any status
// bit), the decode count, its decode stream's (demand, request) half over the
// primary's ready times (shared: DChain.dec_r points at the primary's), and, when the
// per-request rows are an output, the primary's (ttft, finish-of-o = 1) rows.
// Grid: (blocks per chain, secondaries) x 256.
__global__ void __launch_bounds__(256)
    k_stage_clone(const DChain *__restrict__ chains, gl_chain_stats *__restrict__ stats,
                  int64_t *__restrict__ perreq, const int32_t *__restrict__ sec,
                  const int32_t *__restrict__ prim_of, int32_t S, int32_t copy_rows,
                  int32_t fill_only)  // DSD primaries after a deferred k_stages: demands only
{
    const int32_t c = sec[blockIdx.y], pi = fill_only ? c : prim_of[c];
    const DChain &ch = chains[c];
    const DChain &pc = chains[pi];
    bool sbad = false;
    for (int b = 1 + threadIdx.x; b <= ch.cap; b += blockDim.x) sbad |= __ldg(ch.step + b) < 1;
    const bool step_bad = __syncthreads_or(sbad);
    int64_t sm[6] = {0, 0, 0, 0, 0, 0};
    uint32_t st = step_bad ? GL_ST_TABLE : 0u;
    int32_t M = 0;
    for (int p = 0; p < S; ++p) {
        const DStagePart &q = pc.stp[p];
        for (int i = 0; i < 5; ++i) sm[i] += __ldcg(&q.sums[i]);
        sm[5] = max(sm[5], __ldcg(&q.sums[5]));
        st |= __ldcg(&q.status);
        M += __ldcg(&q.dcount);
    }
    const bool valid = st == 0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && !fill_only) {  // R55 as in k_stages
        gl_chain_stats o;
        o.n = ch.n;
        o.slo_ok = 0;
        o.tokens = valid ? sm[4] : 0;
        o.busy_new_us = valid ? sm[0] : 0;
        o.busy_old_us = valid ? sm[1] : 0;
        o.e_new_uj = valid ? sm[2] : 0;
        o.e_old_uj = valid ? sm[3] : 0;
        o.makespan_us = valid ? sm[5] : 0;
        o.req_hash = 0;
        o.status = st;
        o.capacity_ok = (uint32_t)ch.capacity_ok;
        stats[c] = o;
        ch.x->M = valid ? M : 0;
    }
    const bool dsd = ch.mode == GL_MODE_DSD;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    auto demand = [&](uint32_t j) -> uint32_t {
        if (dsd) return __ldg(ch.K + j);
        return min(max(__ldg(ch.o + j), 1u), O_LIMIT - 1) - 1u;
    };
    // four entries per thread and trip (two 16-B loads of the primary's (d, j), four
    // independent demand loads, two 16-B stores): the stream is 16-B aligned (entry
    // offsets are multiples of 32), so only the sentinel tail is written one by one
    // (fill_only: in place over the primary's own stream; its tail is already written)
    const int64_t Q = (int64_t)M + (fill_only ? 0 : DEC_TAIL), Q4 = (int64_t)M / 4;
    const uint4 *src4 = reinterpret_cast<const uint4 *>(pc.dec_dj);
    uint4 *dst4 = reinterpret_cast<uint4 *>(ch.dec_dj);
    for (int64_t q4 = t0; q4 < Q4; q4 += stride) {
        const uint4 a = __ldcg(src4 + 2 * q4), b = __ldcg(src4 + 2 * q4 + 1);
        const uint32_t d0 = demand(a.y), d1 = demand(a.w), d2 = demand(b.y), d3 = demand(b.w);
        dst4[2 * q4] = make_uint4(d0, a.y, d1, a.w);
        dst4[2 * q4 + 1] = make_uint4(d2, b.y, d3, b.w);
    }
    for (int64_t q = 4 * Q4 + t0; q < Q; q += stride) {
        uint2 v = make_uint2(0u, 0u);  // tail: "no request" (dec_r's sentinels are shared)
        if (q < M) {
            const uint32_t j = __ldcg(&pc.dec_dj[q].y);
            v = make_uint2(demand(j), j);
        }
        ch.dec_dj[q] = v;
    }
    if (copy_rows && !fill_only) {  // the primary's (ttft, finish of o = 1 requests) rows
        const longlong2 *src = reinterpret_cast<const longlong2 *>(perreq + 2 * pc.out_off);
        longlong2 *dst = reinterpret_cast<longlong2 *>(perreq + 2 * ch.out_off);
        for (int64_t j = t0; j < ch.n; j += stride) dst[j] = __ldcg(src + j);
    }
}

// Launches without helper warps (many chains: every chain's leader walks it alone)
// need no idle-point candidates: one segment [0, M) per chain.  One thread per chain.
__global__ void __launch_bounds__(128) k_segments_single(const DChain *__restrict__ chains, int32_t n_chains)
{
    const int32_t c = (int32_t)(blockIdx.x * blockDim.x + threadIdx.x);
    if (c >= n_chains) return;
    const DChain &ch = chains[c];
    const int32_t M = ch.x->M;
    ch.seg_start[0] = 0;
    ch.seg_start[M > 0 ? 1 : 0] = M;
    ch.x->nseg = M > 0 ? 1 : 0;
    ch.x->leader_pos = 0;
    ch.x->next_seg = 1;
}

}  // namespace gl
