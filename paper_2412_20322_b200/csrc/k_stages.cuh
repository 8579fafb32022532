// k_stages.cuh -- S0-S4 for every timing chain (one warp per chain) and the
// segment starts the decode speculation uses.
//
//   stage 1  prefill FCFS on the new GPU   c_i = max(c_{i-1}, a_i) + t1[p_i]
//            (TTFT_i = c_i - a_i; R8-R10)
//   stage 2  DPD KV link (R11) / DSD handoff + draft prefill (R12):
//                                           r_i = max(r_{i-1}, c_i) + t2[p_i]  (o_i > 1)
//
// t1/t2 are staged in shared memory by TMA bulk copies (cp.async.bulk + mbarrier).
// Each 128-request chunk is read with 128-bit loads (4 requests per lane), both
// stages are warp scans on (A, B) max-plus pairs with carries across chunks, TTFT
// rows (and the finish of o = 1 requests, R13) are written, and requests with
// o > 1 are compacted into the decode stream (r, demand, request index) in HBM for
// k_decode.  The stage busy/energy sums, token count and status bits go to the
// chain's gl_chain_stats; k_decode and k_finalize add the rest.
#pragma once

#include "common.cuh"

namespace gl {

__global__ void __launch_bounds__(32, 1)
    k_stages(const DChain *__restrict__ chains, gl_chain_stats *__restrict__ stats,
             int64_t *__restrict__ perreq)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x;
    const DChain ch = chains[blockIdx.x];
    const int P = ch.max_prompt, cap = ch.cap;
    const int p1pad = round_up4(P + 1);
    int32_t *t1s = reinterpret_cast<int32_t *>(smem);
    int32_t *t2s = t1s + p1pad;
    uint64_t *bar = reinterpret_cast<uint64_t *>(t2s + p1pad + ((p1pad & 1) ? 1 : 0));
    int64_t *out = perreq + 2 * ch.out_off;

    // ---- S0: stage the prompt-indexed tables (TMA bulk copies + mbarrier) -----
    if (lane == 0) mbar_init(bar, 1);
    __syncwarp();
    uint32_t tx = stage_table(t1s, ch.t1, P + 1, bar, lane);
    tx += stage_table(t2s, ch.t2, P + 1, bar, lane);
    if (lane == 0) mbar_arrive_expect_tx(bar, tx);
    mbar_wait(bar, 0);
    __syncwarp();

    uint32_t status = 0;
    {
        bool bad = false;
        for (int i = 1 + lane; i <= P; i += 32) bad |= (t1s[i] < 0) | (t2s[i] < 0);
        for (int b = 1 + lane; b <= cap; b += 32) bad |= __ldg(ch.step + b) < 1;
        if (__any_sync(FULL, bad)) status |= GL_ST_TABLE;
    }

    int64_t acc_busy_new = 0, acc_busy_old = 0, acc_e_new = 0, acc_e_old = 0, acc_tokens = 0;
    int64_t acc_mk = 0;
    const int32_t n = (int32_t)ch.n;
    const bool dsd = ch.mode == GL_MODE_DSD;
    int32_t produced = 0;
    int64_t carry_c = NEG_INF, carry_r = NEG_INF, carry_a = INT64_MIN;

    for (int32_t chunk = 0; chunk < n && !(status & GL_ST_TABLE); chunk += CHUNK) {
        const int32_t i0 = chunk + 4 * lane;
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
        // per request: TTFT row; o = 1 finishes at c (R13); others -> decode stream
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
                const int64_t e = (int64_t)produced + pos;
                ch.dec_r[e] = r[q];
                ch.dec_dj[e] = make_uint2(dsd ? kv[q] : ov[q] - 1, (uint32_t)j);
                ++pos;
            }
        }
        produced += total;
    }
    // two sentinels after the last decode request read as "no request"
    if (lane < 2) {
        ch.dec_r[(int64_t)produced + lane] = INT64_MAX;
        ch.dec_dj[(int64_t)produced + lane] = make_uint2(0u, 0u);
    }
    const int64_t busy_new = warp_sum_i64(acc_busy_new), busy_old = warp_sum_i64(acc_busy_old);
    const int64_t e_new = warp_sum_i64(acc_e_new), e_old = warp_sum_i64(acc_e_old);
    const int64_t tokens = warp_sum_i64(acc_tokens);
    const int64_t mk = warp_max_i64(acc_mk);
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
        ch.x->M = produced;
    }
}

// Segment starts for the decode speculation: window w >= 1 of SEG_LEN decode
// requests contributes the request with the largest gap r_q - r_{q-1} in it (ties:
// the first), the request most likely to find the decode stage idle.  Any choice is
// exact -- k_decode verifies every boundary -- this one just makes most of them
// true idle points on lightly loaded chains.  One warp per chain.
__global__ void __launch_bounds__(32)
    k_segments(const DChain *__restrict__ chains)
{
    const int lane = threadIdx.x;
    const DChain &ch = chains[blockIdx.x];
    const int32_t M = ch.x->M;
    const int32_t nseg = M > 0 ? (M + SEG_LEN - 1) / SEG_LEN : 0;
    for (int32_t w = 1; w < nseg; ++w) {
        const int32_t lo = w * SEG_LEN, hi = min(lo + SEG_LEN, M);
        int64_t best_gap = -1;
        int32_t best_q = hi;
        for (int32_t q = lo + lane; q < hi; q += 32) {
            const int64_t g = __ldg(ch.dec_r + q) - __ldg(ch.dec_r + q - 1);
            if (g > best_gap) {
                best_gap = g;
                best_q = q;
            }
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            const int64_t og = __shfl_xor_sync(FULL, best_gap, off);
            const int32_t oq = __shfl_xor_sync(FULL, best_q, off);
            if (og > best_gap || (og == best_gap && oq < best_q)) {
                best_gap = og;
                best_q = oq;
            }
        }
        if (lane == 0) ch.seg_start[w] = best_q;
    }
    if (lane == 0) {
        ch.seg_start[0] = 0;
        ch.seg_start[nseg] = M;
        ch.x->nseg = nseg;
        ch.x->leader_pos = 0;
        ch.x->next_seg = 1;
    }
}

}  // namespace gl
