// k_decode.cuh -- S5 + S7: the continuous-batching decode stage (R15-R23) of every
// timing chain, with exact intra-chain speculation; and k_finalize (S6 + hash).
//
// The decode stage of one chain is a serial event chain.  It becomes parallel at
// idle points: if every decode request before q has finished by r_q, the decode
// stage is empty when q becomes ready, and the run from q onward depends only on
// requests >= q (R17: an empty batch restarts exactly at r_q).  k_segments picks
// candidates that are almost always idle points; in k_decode every run starts from
// an empty batch at a candidate and stops at the first later candidate where its
// batch is empty.
//   * Helper warps claim candidates in order and run them speculatively, keeping
//     the finish times in a buffer of their own; they publish (next candidate,
//     sums, last finish) and abort once the leader has moved past their start.
//   * One leader warp per chain hops from idle point to idle point.  Candidate 0
//     is one.  A run from an idle point is the true run, so the candidate where it
//     stopped (empty batch) is the next idle point: the leader copies the run's
//     finish times into the rows, adds its sums and moves there.  A candidate
//     nobody has claimed it runs itself, straight into the rows; one a helper is
//     running it waits for.
// Results are bit-identical to a single sequential run; speculation only changes
// how much of the chain one warp has to walk serially.
//
// Each run reads the decode stream (r, demand, request) from HBM through a
// 256-entry shared-memory window refilled in 128-entry halves by asynchronous
// 16-byte copies (cp.async, one commit group per half).  The loop never steps single
// iterations: a member admitted at iteration I with demand d finishes at
// F = I + d; the next event is min(REDUX-min F - I, the boundary where the head
// becomes ready) and T += k * step[b].  For cap <= 31 (one member per lane) a
// saturated fast path (full batch: one leaves, the freed lane takes the ready
// head) and a light-load fast path (alternate join / leave) carry almost all
// events; larger caps use the general multi-row loop (SPL members per lane).
#pragma once

#include "common.cuh"

namespace gl {

constexpr int DEC_WARPS = 1;  // one warp per k_decode block (leader or helper)
// dynamic shared memory layout of k_decode (bytes)
constexpr int SM_R = 0;                                   // [DEC_WARPS][RING] int64 ready times
constexpr int SM_DJ = DEC_WARPS * RING * 8;               // [DEC_WARPS][RING] (demand, j)
constexpr int SM_PF = DEC_WARPS * RING * 16;              // [DEC_WARPS][RING] prefill (co-located)
constexpr int SM_BARS = DEC_WARPS * RING * 20;            // mbarriers
constexpr int SM_MAGIC = SM_BARS + (2 * DEC_WARPS + 2) * 8;  // [cap+1] reciprocals, then steps

__device__ __forceinline__ void cp_async16(void *dst, const void *src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// One warp's shared-memory window on the decode stream of its chain, refilled
// in 128-entry halves by asynchronous 16-byte copies (cp.async / LDGSTS, one
// commit group per half).  The wait is a single dependency barrier (no retry
// loop), which keeps the decode loops free of forward-progress YIELDs.
struct RingW {
    int64_t *r;      // smem [RING]
    uint2 *dj;       // smem [RING]
    int32_t *pf;     // smem [RING] (co-located modes)
    const int64_t *gr;
    const uint2 *gdj;
    const int32_t *gpf;  // null unless co-located
    int32_t q_end;      // entries >= q_end read as "no request" (INT64_MAX)
    int32_t base;       // first chunk fetched by start()
    int32_t fill_next;  // next chunk to fetch
    int32_t ready_to;   // chunks below this are waited for

    __device__ __forceinline__ void issue(int32_t q, int lane)
    {
        const int h = (q >> 7) & 1;
        // 128 x 8 B of r and of (d, j): 64 x 16 B each, two copies per lane each
        const char *sr = reinterpret_cast<const char *>(gr + q);
        const char *sd = reinterpret_cast<const char *>(gdj + q);
        char *dr = reinterpret_cast<char *>(r + h * 128);
        char *dd = reinterpret_cast<char *>(dj + h * 128);
        cp_async16(dr + 16 * lane, sr + 16 * lane);
        cp_async16(dr + 16 * (lane + 32), sr + 16 * (lane + 32));
        cp_async16(dd + 16 * lane, sd + 16 * lane);
        cp_async16(dd + 16 * (lane + 32), sd + 16 * (lane + 32));
        if (gpf)  // 128 x 4 B of prefill times: one copy per lane
            cp_async16(reinterpret_cast<char *>(pf + h * 128) + 16 * lane,
                       reinterpret_cast<const char *>(gpf + q) + 16 * lane);
        cp_async_commit();
    }
    // all issued halves have landed (the newest one was issued long before)
    __device__ __forceinline__ void wait(int32_t q, int lane)
    {
        cp_async_wait_all();
        // the end of this run's input reads as "no request" (lanes 0 and 1)
        const int32_t qs = q_end + lane;
        if (lane < 2 && qs >= q && qs < q + 128) r[qs & RING_MASK] = INT64_MAX;
        __syncwarp();
    }
    __device__ __forceinline__ void start(int32_t q0, int lane)
    {
        cp_async_wait_all();  // fills the previous run left in flight
        __syncwarp();         // everyone is done with the previous run's window
        base = q0 & ~127;
        issue(base, lane);
        issue(base + 128, lane);
        cp_async_wait_all();
        const int32_t qs = q_end + lane;
        if (lane < 2 && qs >= base && qs < base + 256) r[qs & RING_MASK] = INT64_MAX;
        __syncwarp();
        fill_next = base + 256;
        ready_to = base + 256;
    }
    // called after the head index moved to nxt: recycle the consumed half, and
    // make sure the half holding nxt + 1 has landed
    __device__ __forceinline__ void advanced(int32_t nxt, int lane)
    {
        if ((nxt & 127) == 0 && nxt >= base + 128) {
            issue(fill_next, lane);
            fill_next += 128;
        }
        if (nxt + 1 >= ready_to) {
            wait(ready_to, lane);
            ready_to += 128;
        }
    }
};

struct RunOut {
    int64_t mk;       // last finish time of the run (0 if nothing finished)
    int32_t ne;       // LOG: batch-size log entries written so far (chain total)
    int64_t sums[4];  // decode busy_new, busy_old, e_new, e_old
    int32_t stop_seg; // candidate the run stopped at (idle there; nseg = end), -1 aborted
};

struct RunCtx {
    const DChain *ch;
    const int32_t *steps;   // smem [cap+1]
    const uint64_t *magic;  // smem [cap+1] Lemire reciprocals of steps
    int64_t *rows_fin;      // &perreq[2*out_off + 1]: finish column of this chain
    int64_t *spec;          // helpers: this helper's finish-time buffer, indexed by q
    int cap, lane;
    int32_t nseg;
    int32_t hid;  // helper index (buffer), -1 for the leader
    longlong2 *ev;  // LOG: the chain's batch-size log (T, b after the change)
    int32_t rx;     // the leader races k_relax on this chain (polls x->pad for RX_RELAXED)
};

// kept out of line so the decode loops stay free of memory-ordering operations
__device__ __noinline__ void publish_pos(bool p, int32_t *ptr, int32_t v) { st_relaxed_gpu_if(p, ptr, v); }
__device__ __noinline__ int32_t poll_pos(const int32_t *ptr) { return ld_relaxed_gpu(ptr); }

// sums of iterations x batch-indexed tables, reduced over the warp
template <int SPL>
__device__ __forceinline__ void run_sums(const RunCtx &cx, const uint64_t (&iters)[SPL + 1],
                                         int64_t (&s)[4])
{
    int64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
    for (int r = 0; r <= SPL; ++r) {
        const int bb = r * 32 + cx.lane;
        if (bb >= 1 && bb <= cx.cap && iters[r]) {
            const int64_t it = (int64_t)iters[r];
            a0 += it * __ldg(cx.ch->sbn + bb);
            a1 += it * __ldg(cx.ch->sbo + bb);
            a2 += it * __ldg(cx.ch->sen + bb);
            a3 += it * __ldg(cx.ch->seo + bb);
        }
    }
    s[0] = warp_sum_i64(a0);
    s[1] = warp_sum_i64(a1);
    s[2] = warp_sum_i64(a2);
    s[3] = warp_sum_i64(a3);
}

// One decode run from an empty batch at r_{q0} = r at candidate k0.  It continues
// across later candidates until it reaches one with an empty batch (an idle point:
// every earlier request finished by its ready time) and stops there.
//   ROWS   finish times go to the chain's (ttft, finish) rows (the leader's own
//          runs, whose start is a known idle point); the leader (pub) publishes
//          the candidate it has passed.
//   !ROWS  a helper's speculative run: finish times go to the helper's own buffer
//          (indexed by q); the run aborts once the leader has moved past k0 (the
//          result is then moot).
//   COLO   co-located modes (R41-R44): a join first runs the request's prefill alone
//          on the GPU (T += pf, its first token at T: the TTFT is written here), and a
//          request with no decode demand (o = 1) finishes there without joining.
//          Uses the general loop (the one-row fast paths assume free joins).
//   LOG    (link bandwidth demand) every change of the batch size b appends (T, b)
//          to cx.ev at index ne (ne0 = 2 q0 on entry: a run over decode requests
//          [q0, q1) has at most 2 (q1 - q0) changes); between two entries b is
//          constant and iterations run back to back from the first.
template <int SPL, bool ROWS, bool COLO, bool LOG = false>
__device__ RunOut decode_run(const RunCtx &cx, RingW &ring, int32_t q0, int32_t k0, bool pub,
                             int32_t ne0 = 0)
{
    constexpr bool to_rows = ROWS;
    const DChain &ch = *cx.ch;
    const int lane = cx.lane, cap = cx.cap;
    // shared-memory tables re-derived from the symbol (keeps plain LDS addressing;
    // layout as set up by k_decode: windows, mbarriers, reciprocals, steps)
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    // Table bases as opaque 32-bit shared addresses: kept in registers (ptxas would
    // otherwise rematerialise them from SR_CgaCtaId inside the loops) and read
    // with ld.shared (LDS).
    uint32_t magic_s = smem_u32(dyn_smem + SM_MAGIC);
    asm volatile("" : "+r"(magic_s));
    const uint32_t steps_s = magic_s + 8u * (uint32_t)round_up4(cap + 1);
    auto ld_step = [&](int bb) -> int32_t {
        int32_t v;
        asm("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(steps_s + 4u * (uint32_t)bb));
        return v;
    };
    auto ld_magic = [&](int bb) -> uint64_t {
        uint64_t v;
        asm("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(magic_s + 8u * (uint32_t)bb));
        return v;
    };
    int64_t *const fin_rows = cx.rows_fin;
    int64_t *const fin_spec = cx.spec;
    DChainX *const xx = ch.x;
    const unsigned lane_bit = 1u << lane;

    RunOut res;
    res.stop_seg = -1;
    ring.start(q0, lane);
    // the window again, straight from the shared-memory symbol (keeps LDS addressing)
    const int wid = threadIdx.x >> 5;
    const int64_t *const rr = reinterpret_cast<const int64_t *>(dyn_smem) + wid * RING;
    const uint2 *const rdj = reinterpret_cast<const uint2 *>(dyn_smem + SM_DJ) + wid * RING;
    const int32_t *const rpf = reinterpret_cast<const int32_t *>(dyn_smem + SM_PF) + wid * RING;
    // co-located: helper buffers hold finish times, then TTFTs (second half)
    int64_t *const ttft_spec = fin_spec + (COLO ? ch.spec_stride / 2 : 0);
    int32_t nxt = q0;
    int64_t h_r = rr[nxt & RING_MASK], n_r = rr[(nxt + 1) & RING_MASK];
    uint2 h_dj = rdj[nxt & RING_MASK], n_dj = rdj[(nxt + 1) & RING_MASK];
    // co-located: the head's prefill time, kept in a register like h_r (off the
    // event chain's shared-memory latency)
    int32_t h_pf = COLO ? rpf[nxt & RING_MASK] : 0, n_pf = COLO ? rpf[(nxt + 1) & RING_MASK] : 0;
    // next candidate after k0, for stop checks and leader_pos
    const int32_t nseg_r = cx.nseg;
    int32_t kb = k0 + 1;
    int32_t nb = ch.seg_start[kb];
    bool aborted = false;

    auto advance = [&]() {
        ++nxt;
        h_r = n_r;
        h_dj = n_dj;
        // all ring maintenance happens where nxt + 1 crosses a 128-entry half
        if (__builtin_expect((uint32_t)((nxt + 1) & 127) <= 1u, 0)) {
            ring.advanced(nxt, lane);
            if ((nxt & 127) == 0) {
                while (kb < nseg_r && nb < nxt) nb = ch.seg_start[++kb];
                if (ROWS) {  // publish the leader's progress
                    publish_pos(pub && lane == 0, &xx->leader_pos, kb - 1);
                    // k_relax solved the chain: end the input at the next half
                    if (cx.rx && !aborted && (__shfl_sync(FULL, poll_pos(&xx->pad), 0) & RX_RELAXED)) {
                        aborted = true;
                        ring.q_end = min(ring.q_end, ring.ready_to);
                    }
                } else if (!aborted && __shfl_sync(FULL, poll_pos(&xx->leader_pos), 0) > k0) {
                    // the leader is past this run's start: end the input at the next
                    // half (its sentinels are written when that half is waited for)
                    aborted = true;
                    ring.q_end = min(ring.q_end, ring.ready_to);
                }
            }
        }
        const int e1 = (nxt + 1) & RING_MASK;
        n_r = rr[e1];
        n_dj = rdj[e1];
        if constexpr (COLO) {
            h_pf = n_pf;
            n_pf = rpf[e1];
        }
    };
    // advance() when no ring maintenance is due ((nxt + 2) & 127 > 1): no
    // convergent operations, so no reconvergence region in the loops using it
    auto advance_fast = [&]() {
        ++nxt;
        h_r = n_r;
        h_dj = n_dj;
        const int e1 = (nxt + 1) & RING_MASK;
        n_r = rr[e1];
        n_dj = rdj[e1];
        if constexpr (COLO) {
            h_pf = n_pf;
            n_pf = rpf[e1];
        }
    };
    auto fin_addr = [&](uint32_t j, int32_t q) -> int64_t * {
        return to_rows ? fin_rows + 2 * (int64_t)j : fin_spec + q;
    };

    int64_t T = 0, mk = 0;
    uint32_t I = 0;
    int b = 0;
    int32_t ne = ne0;
    longlong2 *const evp = cx.ev;
    auto log_b = [&]() {
        if constexpr (LOG) {
            if (lane == 0) evp[ne] = make_longlong2(T, (int64_t)b);
            ++ne;
        }
    };
    uint64_t iters[SPL + 1];
#pragma unroll
    for (int s = 0; s <= SPL; ++s) iters[s] = 0;

    if constexpr (SPL == 1) {
        // caps <= 31, one member per lane.  Co-located modes (COLO, R41-R44) add, at
        // every admission, the request's prefill run alone on the GPU (T += t1[p],
        // its first token at T: the TTFT is written there); a request with no decode
        // demand (o = 1) finishes at its first token without taking a slot -- the
        // fast paths hand such heads to the admission loop.
        auto prefill = [&]() {
            if constexpr (COLO) {
                T += (int64_t)h_pf;
                if (lane == 0) {
                    if (to_rows) fin_rows[2 * (int64_t)h_dj.y - 1] = T - h_r;
                    else ttft_spec[nxt] = T - h_r;
                }
            }
        };
        uint32_t Fm = F_EMPTY, fmin = F_EMPTY;
        int64_t *fa = fin_rows;
        unsigned fr = cap >= 32 ? FULL : ((1u << cap) - 1u);
        uint32_t c_b = 0;  // iterations at batch size b == lane
        int32_t st_d = 0, st_c = 0, st_u = 0;
        uint64_t M_d = 0, M_c = 0, M_u = 0;
        auto load_nbr = [&](int nbb) {
            st_c = ld_step(nbb);
            M_c = ld_magic(nbb);
            st_u = ld_step(min(nbb + 1, cap));
            M_u = ld_magic(min(nbb + 1, cap));
            st_d = ld_step(max(nbb - 1, 0));
            M_d = ld_magic(max(nbb - 1, 0));
        };
        auto shift_up = [&]() {
            st_d = st_c;
            M_d = M_c;
            st_c = st_u;
            M_c = M_u;
            st_u = ld_step(min(b + 1, cap));
            M_u = ld_magic(min(b + 1, cap));
        };
        auto shift_down = [&]() {
            st_u = st_c;
            M_u = M_c;
            st_c = st_d;
            M_c = M_d;
            st_d = ld_step(max(b - 1, 0));
            M_d = ld_magic(max(b - 1, 0));
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
                if constexpr (COLO) {
                    prefill();
                    if (h_dj.x == 0) {  // o = 1: done at its first token (R13)
                        if (lane == 0) *fin_addr(h_dj.y, nxt) = T;
                        mk = T;
                        advance();
                        continue;
                    }
                }
                const unsigned bit = fr & (0u - fr);
                fr ^= bit;
                const uint32_t fnew = I + h_dj.x;
                if (lane_bit == bit) {
                    Fm = fnew;
                    fa = fin_addr(h_dj.y, nxt);
                }
                fmin = min(fmin, fnew);
                ++b;
                log_b();
                shift_up();
                advance();
            }
            if (b == 0) {  // idle until the next decode request is ready (R17)
                if (h_r == INT64_MAX) {
                    res.stop_seg = aborted ? -1 : nseg_r;
                    break;
                }
                if (nxt >= nb) {  // reached (or passed) the next candidate
                    while (kb < nseg_r && nb < nxt) nb = ch.seg_start[++kb];
                    if (nb == nxt) {  // an idle point: stop here
                        res.stop_seg = kb;
                        break;
                    }
                }
                T = h_r;
                continue;
            }
            if (b == cap) {
                // Saturated fast path: with a full batch the next event is a leave;
                // while exactly one member leaves and the head is already ready, the
                // freed lane takes the head at the same boundary (R16).
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
                    mk = T;
                    const bool one = (lm & (lm - 1u)) == 0u;
                    if (!(one && h_r <= T && I < 0x80000000u && ((nxt + 2) & 127) > 1 &&
                          (!COLO || h_dj.x != 0))) {
                        if (lv) Fm = F_EMPTY;
                        fr |= lm;
                        b -= __popc(lm);
                        log_b();
                        fmin = __reduce_min_sync(FULL, Fm);
                        break;
                    }
                    if (lv) {
                        Fm = I + h_dj.x;
                        fa = fin_addr(h_dj.y, nxt);
                    }
                    prefill();  // co-located: the freed slot's newcomer prefills first
                    fmin = __reduce_min_sync(FULL, Fm);
                    advance_fast();
                }
                c_b += (lane == cap) ? it : 0u;
                if (b == cap - 1) shift_down();
                else load_nbr(b);
                continue;
            }
            {
                // Light-load fast path (0 < b < cap, head not ready at T): each step
                // is the head's join at kJ = ceil(gap / step[b]) or the next leave at
                // kL.  Exits when a join fills the batch or finds another ready head,
                // when the batch empties, or (to the general code below) on a gap of
                // 2^31 us or more / a pending counter rebase.
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
                        if (((nxt + 2) & 127) <= 1) break;  // ring refill due: joins at the top
                        if constexpr (COLO) {
                            if (h_dj.x == 0) break;  // o = 1 head: admitted at the top
                            prefill();
                        }
                        const unsigned bit = fr & (0u - fr);
                        fr ^= bit;
                        const uint32_t fnew = I + h_dj.x;
                        if (lane_bit == bit) {
                            Fm = fnew;
                            fa = fin_addr(h_dj.y, nxt);
                        }
                        fmin = min(fmin, fnew);
                        ++b;
                        log_b();
                        shift_up();
                        advance_fast();
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
                        log_b();
                        mk = T;
                        fmin = __reduce_min_sync(FULL, Fm);
                        shift_down();
                        if (nl != 1) {  // several members left at once: leave the loop
                            load_nbr(b);
                            break;
                        }
                        if (b == 0 || h_r <= T) break;
                    }
                }
                if (!slow) continue;
            }
            // ---- general event: a join at kJ < kL, else the leave at kL (R16)
            const int64_t st = st_c;
            const uint32_t kL = fmin - I;
            if (b < cap) {
                const int64_t gap = h_r - T;  // > 0: the head was not admitted at T
                uint32_t kJ = ceil_div_magic((uint32_t)gap, (uint32_t)st, M_c);
                const bool far = gap >= 0x80000000ll;  // very long gap, or no head
                if (kJ < kL || far) {
                    if (far)  // exact 64-bit path; no head (INT64_MAX) never joins
                        kJ = (h_r != INT64_MAX && gap <= (int64_t)(kL - 1) * st)
                                 ? (uint32_t)((gap + st - 1) / st) : 0xFFFFFFFFu;
                    if (kJ < kL) {
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
            log_b();
            mk = T;
            fmin = __reduce_min_sync(FULL, Fm);
            if (nl == 1) shift_down();
            else load_nbr(b);
        }
        iters[0] += c_b;
    } else {
        // general loop, caps 32..256: SPL rows of 32 member slots per lane
        uint32_t F[SPL];
        int64_t *fa[SPL];
        unsigned free_m[SPL];
        uint32_t cnt[SPL + 1];
#pragma unroll
        for (int s = 0; s < SPL; ++s) {
            F[s] = F_EMPTY;
            fa[s] = fin_rows;
            const int lo = s * 32;
            free_m[s] = cap >= lo + 32 ? FULL : (cap > lo ? ((1u << (cap - lo)) - 1u) : 0u);
        }
#pragma unroll
        for (int s = 0; s <= SPL; ++s) cnt[s] = 0;
        for (;;) {
            while (b < cap && h_r <= T) {  // FCFS joins (R16, R18)
                if (I >= 0x80000000u) {     // rebase the 32-bit iteration counter
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
                if constexpr (COLO) {  // the prefill runs alone on the GPU (R42)
                    T += (int64_t)h_pf;
                    const uint32_t j = h_dj.y;
                    if (lane == 0) {
                        if (to_rows) fin_rows[2 * (int64_t)j - 1] = T - h_r;
                        else ttft_spec[nxt] = T - h_r;
                    }
                    if (h_dj.x == 0) {  // o = 1: done at its first token (R13)
                        if (lane == 0) *fin_addr(j, nxt) = T;
                        mk = T;
                        advance();
                        continue;
                    }
                }
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
                            F[s] = I + h_dj.x;
                            fa[s] = fin_addr(h_dj.y, nxt);
                        }
                    }
                }
                ++b;
                if constexpr (!COLO) log_b();
                advance();
            }
            if (b == 0) {  // idle (R17)
                if (h_r == INT64_MAX) {
                    res.stop_seg = aborted ? -1 : nseg_r;
                    break;
                }
                if (nxt >= nb) {  // reached (or passed) the next candidate
                    while (kb < nseg_r && nb < nxt) nb = ch.seg_start[++kb];
                    if (nb == nxt) {  // an idle point: stop here
                        res.stop_seg = kb;
                        break;
                    }
                }
                T = h_r;
                continue;
            }
            const int64_t st = ld_step(b);
            uint32_t kJ = 0xFFFFFFFFu;
            if (b < cap) {
                const int64_t gap = h_r - T;
                if (gap < 0x80000000ll) kJ = ceil_div_magic((uint32_t)gap, (uint32_t)st, ld_magic(b));
                else if (h_r != INT64_MAX)
                    kJ = (uint32_t)min((gap + st - 1) / st, (int64_t)0xFFFFFFFF);
            }
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
            int nl = 0;
#pragma unroll
            for (int s = 0; s < SPL; ++s) {  // leaves at T (none when k < kL)
                const bool lv = F[s] == I;
                const unsigned lm = __ballot_sync(FULL, lv);
                if (lv) {
                    *fa[s] = T;
                    F[s] = F_EMPTY;
                }
                free_m[s] |= lm;
                nl += __popc(lm);
            }
            b -= nl;
            if (nl) {
                mk = T;
                if constexpr (!COLO) log_b();
            }
        }
#pragma unroll
        for (int s = 0; s <= SPL; ++s) iters[s] += cnt[s];
    }
    res.mk = mk;
    res.ne = ne;
    run_sums<SPL>(cx, iters, res.sums);
    return res;
}

__device__ __forceinline__ void backoff() { __nanosleep(64); }

// Helpers: speculative runs from the candidates ahead of the leader.  Out of line
// so the kernel body holds a single (the leader's) copy of the decode loops.
// A helper's runs write disjoint stretches of its buffer: it skips candidates
// inside its previous run (if that run was the true one they are not idle points;
// if not, the leader runs them itself).
template <int SPL, bool COLO, bool LOG>
__device__ __noinline__ void helper_loop(const RunCtx cx, RingW ring)
{
    const DChain &ch = *cx.ch;
    const int lane = cx.lane;
    const int32_t nseg = cx.nseg;
    int32_t k_end = 0;  // candidate where this helper's previous run stopped
    for (;;) {
        int32_t k = 0;
        if (lane == 0) {
            k = atomicAdd(&ch.x->next_seg, 1);
            if (k < nseg && (k < k_end || k <= ld_relaxed_gpu(&ch.x->leader_pos) ||
                             atomicCAS(&ch.seg_out[k].state, SEG_FREE, SEG_CLAIMED) != SEG_FREE))
                k = -1;  // inside our last run, or the leader is there (or took it)
        }
        k = __shfl_sync(FULL, k, 0);
        if (k >= nseg) break;
        if (k < 0) continue;
        ring.q_end = ch.x->M;
        const int32_t q0 = ch.seg_start[k];
        const RunOut ro = decode_run<SPL, false, COLO, LOG>(cx, ring, q0, k, false, 2 * q0);
        if (ro.stop_seg < 0) continue;  // aborted: the leader passed k (moot values)
        k_end = ro.stop_seg;
        if (lane == 0) {
            DSegOut &so = ch.seg_out[k];
            so.maxfin = ro.mk;
            for (int i = 0; i < 4; ++i) so.sums[i] = ro.sums[i];
            so.next = ro.stop_seg;
            so.helper = cx.hid;
            so.nev = ro.ne - 2 * q0;
            __threadfence();
            st_release_gpu(&so.state, SEG_DONE);
        }
    }
}

// Leader + helpers (see the file comment).  One warp per block: blocks
// [0, n_chains) are the leaders of chain blockIdx.x, blocks >= n_chains are
// helpers of chain blockIdx.x % n_chains.
//   LOG: also writes the batch-size log of every disaggregated chain (link bandwidth
//   demand, k_link.cuh): the leader's runs into the chain's log, helper runs into
//   their own logs, copied by the leader with the finish times when accepted.
template <int SPL, bool COLO, bool LOG = false>
__global__ void __launch_bounds__(32 * DEC_WARPS, 1)
    k_decode(const DChain *__restrict__ chains, gl_chain_stats *__restrict__ stats,
             int64_t *__restrict__ perreq, int32_t n_chains, int32_t rxpass)
{
    static_assert(!(LOG && COLO), "the co-located modes have no link");
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x % n_chains;
    const bool leader = blockIdx.x < n_chains && warp == 0;
    const DChain &ch = chains[c];
    // one launch per family: the other launch handles this chain
    if ((ch.mode == GL_MODE_STANDALONE || ch.mode == GL_MODE_SPEC_COLO) != COLO) return;
    const int cap = ch.cap;
    const int cappad = round_up4(cap + 1);
    // smem: per-warp windows first (16-B aligned), then mbarriers, then tables
    int64_t *ring_r = reinterpret_cast<int64_t *>(smem + SM_R) + warp * RING;
    uint2 *ring_dj = reinterpret_cast<uint2 *>(smem + SM_DJ) + warp * RING;
    int32_t *ring_pf = reinterpret_cast<int32_t *>(smem + SM_PF) + warp * RING;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + SM_BARS);
    uint64_t *magic = reinterpret_cast<uint64_t *>(smem + SM_MAGIC);
    int32_t *steps = reinterpret_cast<int32_t *>(magic + cappad);

    // S0: batch-indexed step table by TMA (warp 0), reciprocals
    if (threadIdx.x == 0) mbar_init(bars + 2 * DEC_WARPS, 1);
    __syncthreads();
    if (warp == 0) {
        const uint32_t tx = stage_table(steps, ch.step, cap + 1, bars + 2 * DEC_WARPS, lane);
        if (lane == 0) mbar_arrive_expect_tx(bars + 2 * DEC_WARPS, tx);
        mbar_wait(bars + 2 * DEC_WARPS, 0);
    }
    __syncthreads();
    for (int bb = threadIdx.x; bb <= cap; bb += blockDim.x) {
        const int32_t s = steps[bb];
        magic[bb] = s > 1 ? 0xFFFFFFFFFFFFFFFFull / (uint64_t)s + 1ull : 0ull;
    }
    __syncthreads();

    const int32_t nseg = ch.x->nseg;
    const int32_t hid = leader ? -1 : (int32_t)(blockIdx.x / n_chains) - 1;
    // racing k_relax (rxpass 1): a chain with a relaxation slot is walked too; the
    // first to finish owns the statistics (x->pad bits), both write identical rows
    const int32_t rx = (rxpass > 0 && leader) ? (ld_relaxed_gpu(&ch.x->pad) & RX_SLOT_MASK) : 0;
    RunCtx cx{&ch, steps, magic, perreq + 2 * ch.out_off + 1,
              ch.spec_fin + (int64_t)max(hid, 0) * ch.spec_stride, cap, lane, nseg, hid,
              leader ? ch.ev : ch.ev_spec + (int64_t)max(hid, 0) * ch.ev_stride, rx};
    RingW ring;
    ring.r = ring_r;
    ring.dj = ring_dj;
    ring.pf = ring_pf;
    ring.gr = ch.dec_r;
    ring.gdj = ch.dec_dj;
    ring.gpf = COLO ? ch.dec_pf : nullptr;
    ring.fill_next = ring.ready_to = 0;

    if (!leader) {
        helper_loop<SPL, COLO, LOG>(cx, ring);
        return;
    }
    // The leader hops from idle point to idle point: candidate 0 is one, and a run
    // from an idle point is the true run, so where it stops is the next one.
    int64_t acc[4] = {0, 0, 0, 0};
    int64_t mk = 0;
    int32_t k = 0;
    const int32_t M = ch.x->M;
    bool lost = false;  // k_relax solved the chain first
    while (k < nseg) {
        if (rx && (__shfl_sync(FULL, ld_relaxed_gpu(&ch.x->pad), 0) & RX_RELAXED)) {
            lost = true;
            break;
        }
        if (lane == 0) st_relaxed_gpu(&ch.x->leader_pos, k);
        int32_t st = 0;
        if (lane == 0) {
            st = ld_acquire_gpu(&ch.seg_out[k].state);
            if (st == SEG_FREE) {
                st = atomicCAS(&ch.seg_out[k].state, SEG_FREE, SEG_CLAIMED);
                if (st == SEG_FREE) st = -1;  // ours now
            }
        }
        st = __shfl_sync(FULL, st, 0);
        if (st < 0) {  // nobody has run k: simulate it here, into the rows
            ring.q_end = M;
            const RunOut ro = decode_run<SPL, true, COLO, LOG>(cx, ring, ch.seg_start[k], k, true,
                                                              2 * ch.seg_start[k]);
            if (ro.stop_seg < 0) {  // aborted: k_relax solved the chain
                lost = true;
                break;
            }
            for (int i = 0; i < 4; ++i) acc[i] += ro.sums[i];
            mk = max(mk, ro.mk);
            k = ro.stop_seg;
            continue;
        }
        if (st != SEG_DONE) {  // a helper is running k: wait for it
            int32_t d = 0;
            do {
                if (lane == 0) d = ld_acquire_gpu(&ch.seg_out[k].state) == SEG_DONE;
                d = __shfl_sync(FULL, d, 0);
            } while (!d);
        }
        const DSegOut &so = ch.seg_out[k];
        const int32_t m = __ldcg(&so.next);
        for (int i = 0; i < 4; ++i) acc[i] += __ldcg(&so.sums[i]);
        mk = max(mk, __ldcg(&so.maxfin));
        {  // copy the run's finish times from the helper's buffer into the rows
            const int64_t *src = ch.spec_fin + (int64_t)__ldcg(&so.helper) * ch.spec_stride;
            const int32_t s_lo = ch.seg_start[k], s_hi = ch.seg_start[m];
            for (int32_t q0 = s_lo; q0 < s_hi; q0 += 128) {
                int64_t f[4];
                uint32_t j[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int32_t q = q0 + 32 * u + lane;
                    if (q < s_hi) {
                        f[u] = __ldcg(src + q);
                        j[u] = __ldcg(&ch.dec_dj[q].y);
                    }
                }
                if constexpr (COLO) {  // (ttft, finish) pairs: TTFTs in the second half
                    const int64_t *src_t = src + ch.spec_stride / 2;
                    int64_t t[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int32_t q = q0 + 32 * u + lane;
                        if (q < s_hi) t[u] = __ldcg(src_t + q);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (q0 + 32 * u + lane < s_hi)
                            *reinterpret_cast<longlong2 *>(cx.rows_fin - 1 + 2 * (int64_t)j[u]) =
                                make_longlong2(t[u], f[u]);
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (q0 + 32 * u + lane < s_hi) cx.rows_fin[2 * (int64_t)j[u]] = f[u];
                }
            }
        }
        if constexpr (LOG) {  // the run's batch-size log, at the same positions
            const int64_t p0 = 2 * (int64_t)ch.seg_start[k];
            const int32_t nev = __ldcg(&so.nev);
            const longlong2 *src = ch.ev_spec + (int64_t)__ldcg(&so.helper) * ch.ev_stride;
            for (int32_t e = lane; e < nev; e += 32) ch.ev[p0 + e] = __ldcg(src + p0 + e);
        }
        k = m;
    }
    if (lane == 0) {
        st_release_gpu(&ch.x->leader_pos, nseg);
        if (rx && !lost) lost = (atomicOr(&ch.x->pad, RX_SERIAL) & RX_RELAXED) != 0;
#ifdef GL_RX_TRACE
        if (rx) {
            uint64_t t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            printf("leader chain %d done lost %d k %d nseg %d t %llu\n", c, (int)lost, k, nseg, t);
        }
#endif
    }
    if (lane == 0 && !lost) {
        gl_chain_stats &s = stats[c];
        s.busy_new_us += acc[0];
        s.busy_old_us += acc[1];
        s.e_new_uj += acc[2];
        s.e_old_uj += acc[3];
        s.makespan_us = max(s.makespan_us, mk);
    }
}

__host__ __device__ inline size_t decode_smem_bytes(int cap)
{
    return (size_t)SM_MAGIC + (size_t)round_up4(cap + 1) * 12 + 16;
}

// ---- S6 + S7: per-request SLO test and hash, the whole GPU over (chain, request)
//   ok_j = TTFT_j <= SLO_ttft and (o_j = 1 or finish_j - c_j <= SLO_tpot (o_j - 1))
//   (Table 2; R25-R27), hash += mix64(j, ttft_j, finish_j).
// Integer atomics commute, so the result is deterministic.
__global__ void __launch_bounds__(256)
    k_finalize(const DChain *__restrict__ chains, gl_chain_stats *__restrict__ stats,
               const int64_t *__restrict__ perreq, int per_thread,
               const int32_t *__restrict__ prim_of)  // NULL: every chain has its own rows
{
    __shared__ unsigned long long s_ok[8], s_hash[8];
    const DChain &ch = chains[blockIdx.y];
    if (stats[blockIdx.y].status != 0) return;  // invalid input: only n and status (R55)
    const int64_t n = ch.n;
    const int64_t *rows = perreq + 2 * ch.out_off;
    // a secondary chain (k_stage_clone without row copies) reads its TTFTs and the
    // finish times of o = 1 requests from its primary's rows
    const int32_t pr = prim_of ? prim_of[blockIdx.y] : (int32_t)blockIdx.y;
    const int64_t *prow = perreq + 2 * chains[pr].out_off;
    const bool own = pr == (int32_t)blockIdx.y;
    const int64_t ttft_slo = ch.ttft_slo, tpot_slo = ch.tpot_slo;
    unsigned long long ok = 0, hash = 0;
    const int64_t base = (int64_t)blockIdx.x * blockDim.x * per_thread;
    for (int q = 0; q < per_thread; ++q) {
        const int64_t j = base + (int64_t)q * blockDim.x + threadIdx.x;
        if (j < n) {
            const int64_t a = __ldg(ch.a + j);
            uint32_t o = __ldg(ch.o + j);
            o = min(max(o, 1u), O_LIMIT - 1);
            longlong2 tf;
            if (own) {
                tf = __ldg(reinterpret_cast<const longlong2 *>(rows) + j);
            } else {  // the own row holds only the finish of a decode request
                tf.x = __ldg(prow + 2 * j);
                tf.y = __ldg((o == 1 ? prow : rows) + 2 * j + 1);
            }
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
