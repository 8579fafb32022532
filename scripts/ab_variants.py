"""Source edits for scripts/ab_build.py: name -> [(file, old, new), ...].

The record of the round's same-box A/B experiments (results in DESIGN.md §10).
Variants in MERGED were adopted and are part of the current source, so their
edits no longer apply; the others were measured against the source of their time
and may need the old text to build."""

MERGED = {"fastadv", "nl"}

LIGHT_HEAD_OLD = '''                    const int64_t gap = h_r - T;
                    const uint32_t kJ = ceil_div_magic((uint32_t)gap, (uint32_t)st, M_c);
                    if (gap >= 0x80000000ll || I >= 0x80000000u) {
                        slow = true;
                        break;
                    }
                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;'''

VARIANTS = {
    "base": [],
    # the rare far-gap / rebase check only on the join branch (clamped kJ)
    "clamp": [("k_decode.cuh", LIGHT_HEAD_OLD, '''                    const int64_t gap = h_r - T;
                    const uint32_t kJ = ceil_div_magic(
                        (uint32_t)min(gap, (int64_t)0x7FFFFFFF), (uint32_t)st, M_c);
                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        if (gap >= 0x80000000ll || I >= 0x80000000u) {
                            slow = true;
                            break;
                        }
                        T += (int64_t)kJ * st;''')],
    # join/leave decided by a warp vote: a uniform predicate needs no reconvergence
    "vote": [("k_decode.cuh", '''                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;''', '''                    if (__all_sync(FULL, kJ < kL)) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;''')],
    # multi-leave test from the ballot directly (no popc on the branch)
    "lm": [("k_decode.cuh", '''                        const int nl = __popc(lm);
                        b -= nl;
                        log_b();
                        mk = T;
                        fmin = __reduce_min_sync(FULL, Fm);
                        if (nl == 1) shift_down();
                        else load_nbr(b);
                        if (b == 0 || h_r <= T) break;''', '''                        const int nl = __popc(lm);
                        b -= nl;
                        log_b();
                        mk = T;
                        fmin = __reduce_min_sync(FULL, Fm);
                        if ((lm & (lm - 1u)) == 0u) shift_down();
                        else load_nbr(b);
                        if (b == 0 || h_r <= T) break;''')],
}

_ADV_OLD = '''    auto fin_addr = [&](uint32_t j, int32_t q) -> int64_t * {'''
_ADV_NEW = '''    // advance() when no ring maintenance is due ((nxt + 2) & 127 > 1): no
    // convergent operations, so no reconvergence region in the loops using it
    auto advance_fast = [&]() {
        ++nxt;
        h_r = n_r;
        h_dj = n_dj;
        const int e1 = (nxt + 1) & RING_MASK;
        n_r = rr[e1];
        n_dj = rdj[e1];
    };
    auto fin_addr = [&](uint32_t j, int32_t q) -> int64_t * {'''
_SAT_OLD = '''                    const bool one = (lm & (lm - 1u)) == 0u;
                    if (!(one && h_r <= T && I < 0x80000000u)) {'''
_SAT_NEW = '''                    const bool one = (lm & (lm - 1u)) == 0u;
                    if (!(one && h_r <= T && I < 0x80000000u && ((nxt + 2) & 127) > 1)) {'''
_SAT_ADV_OLD = '''                    fmin = __reduce_min_sync(FULL, Fm);
                    advance();
                }
                c_b += (lane == cap) ? it : 0u;'''
_SAT_ADV_NEW = '''                    fmin = __reduce_min_sync(FULL, Fm);
                    advance_fast();
                }
                c_b += (lane == cap) ? it : 0u;'''
_LIGHT_OLD = '''                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;
                        I += kJ;
                        c_b += (lane == b) ? kJ : 0u;
                        const unsigned bit = fr & (0u - fr);'''
_LIGHT_NEW = '''                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;
                        I += kJ;
                        c_b += (lane == b) ? kJ : 0u;
                        if (((nxt + 2) & 127) <= 1) break;  // ring refill due: joins at the top
                        const unsigned bit = fr & (0u - fr);'''
_LIGHT_ADV_OLD = '''                        ++b;
                        log_b();
                        shift_up();
                        advance();
                        if (b == cap || h_r <= T) break;'''
_LIGHT_ADV_NEW = '''                        ++b;
                        log_b();
                        shift_up();
                        advance_fast();
                        if (b == cap || h_r <= T) break;'''
VARIANTS["fastadv"] = [("k_decode.cuh", _ADV_OLD, _ADV_NEW), ("k_decode.cuh", _SAT_OLD, _SAT_NEW),
                       ("k_decode.cuh", _SAT_ADV_OLD, _SAT_ADV_NEW),
                       ("k_decode.cuh", _LIGHT_OLD, _LIGHT_NEW),
                       ("k_decode.cuh", _LIGHT_ADV_OLD, _LIGHT_ADV_NEW)]
VARIANTS["fastadv_sat"] = VARIANTS["fastadv"][:3]
VARIANTS["fastadv_light"] = [VARIANTS["fastadv"][0]] + VARIANTS["fastadv"][3:]

# one branch decides leave vs (join or slow path); the slow test moves inside
_MERGE_OLD = '''                    if (gap >= 0x80000000ll || I >= 0x80000000u) {
                        slow = true;
                        break;
                    }
                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;'''
_MERGE_NEW = '''                    const bool far = gap >= 0x80000000ll || I >= 0x80000000u;
                    if (far || kJ < kL) {  // the head joins at T + kJ * step[b]
                        if (far) {
                            slow = true;
                            break;
                        }
                        T += (int64_t)kJ * st;'''
VARIANTS["merge"] = [("k_decode.cuh", _MERGE_OLD, _MERGE_NEW)]
# the leave branch's multi-leave test on the ballot (no popc) and predicated refill
_NL_OLD = '''                        if (nl == 1) shift_down();
                        else load_nbr(b);
                        if (b == 0 || h_r <= T) break;'''
_NL_NEW = '''                        shift_down();
                        if (nl != 1) {  // several members left at once: leave the loop
                            load_nbr(b);
                            break;
                        }
                        if (b == 0 || h_r <= T) break;'''
VARIANTS["nl"] = [("k_decode.cuh", _NL_OLD, _NL_NEW)]
VARIANTS["merge_nl"] = VARIANTS["merge"] + VARIANTS["nl"]

# join/leave decided in the time domain: kJ < kL  <=>  gap <= (kL - 1) st; the
# division is computed only on the join path
_TDEC_OLD = '''                    const uint32_t kJ = ceil_div_magic((uint32_t)gap, (uint32_t)st, M_c);
                    if (gap >= 0x80000000ll || I >= 0x80000000u) {
                        slow = true;
                        break;
                    }
                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;'''
_TDEC_NEW = '''                    if (gap >= 0x80000000ll || I >= 0x80000000u) {
                        slow = true;
                        break;
                    }
                    if (gap <= ((int64_t)kL - 1) * st) {  // the head joins at T + kJ * step[b]
                        const uint32_t kJ = ceil_div_magic((uint32_t)gap, (uint32_t)st, M_c);
                        T += (int64_t)kJ * st;'''
VARIANTS["tdec"] = [("k_decode.cuh", _TDEC_OLD, _TDEC_NEW)]
# saturated loop: exit test without the popc / multi-leave combination on the chain
_SATX_OLD = '''                    const bool one = (lm & (lm - 1u)) == 0u;
                    if (!(one && h_r <= T && I < 0x80000000u && ((nxt + 2) & 127) > 1)) {'''
_SATX_NEW = '''                    const bool one = lm == lane_bit_of_min;
                    if (!(one && h_r <= T && I < 0x80000000u && ((nxt + 2) & 127) > 1)) {'''

# a join that fills the batch stays in the light-load loop (the next event is then
# a forced leave): near-saturated chains stop bouncing into the saturated loop
VARIANTS["capjoin"] = [
    ("k_decode.cuh", '''                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;''', '''                    if (kJ < kL && b < cap) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;'''),
    ("k_decode.cuh", '''                        if (b == cap || h_r <= T) break;''',
     '''                        if (h_r <= T && b < cap) break;'''),
]

# decision in the time domain while kJ is still computed before the branch
VARIANTS["tdec2"] = [("k_decode.cuh", '''                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;''', '''                    if (gap <= ((int64_t)kL - 1) * st) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;''')]

# the light loop keeps fmin2 = the next distinct finish iteration above fmin, so a
# leave sets fmin = fmin2 at once and the REDUX (for the new fmin2) leaves the chain
VARIANTS["fmin2"] = [
    ("k_decode.cuh", '''                bool slow = false;
                for (;;) {
                    const int64_t st = st_c;
                    const uint32_t kL = fmin - I;''', '''                bool slow = false;
                uint32_t fmin2 = __reduce_min_sync(FULL, Fm > fmin ? Fm : F_EMPTY);
                for (;;) {
                    const int64_t st = st_c;
                    const uint32_t kL = fmin - I;'''),
    ("k_decode.cuh", '''                        fmin = min(fmin, fnew);
                        ++b;
                        log_b();
                        shift_up();
                        advance_fast();''', '''                        fmin2 = fnew < fmin ? fmin : (fnew > fmin ? min(fmin2, fnew) : fmin2);
                        fmin = min(fmin, fnew);
                        ++b;
                        log_b();
                        shift_up();
                        advance_fast();'''),
    ("k_decode.cuh", '''                        mk = T;
                        fmin = __reduce_min_sync(FULL, Fm);
                        shift_down();
                        if (nl != 1) {  // several members left at once: leave the loop''', '''                        mk = T;
                        fmin = fmin2;  // every member at the old minimum has left
                        fmin2 = __reduce_min_sync(FULL, Fm > fmin ? Fm : F_EMPTY);
                        shift_down();
                        if (nl != 1) {  // several members left at once: leave the loop'''),
]

# general loop (caps >= 32, co-located modes): fmin kept across join events (REDUX
# only after leaves) and step[b +- 1] / reciprocals cached in registers
VARIANTS["gen1"] = [
    ("k_decode.cuh", '''#pragma unroll
        for (int s = 0; s <= SPL; ++s) cnt[s] = 0;
        for (;;) {
            while (b < cap && h_r <= T) {  // FCFS joins (R16, R18)''', '''#pragma unroll
        for (int s = 0; s <= SPL; ++s) cnt[s] = 0;
        uint32_t fmin = F_EMPTY;  // min over members, kept across joins
        int32_t g_st_d = 0, g_st_c = ld_step(0), g_st_u = ld_step(min(1, cap));
        uint64_t g_M_d = 0, g_M_c = ld_magic(0), g_M_u = ld_magic(min(1, cap));
        auto g_load = [&](int nbb) {
            g_st_c = ld_step(nbb);
            g_M_c = ld_magic(nbb);
            g_st_u = ld_step(min(nbb + 1, cap));
            g_M_u = ld_magic(min(nbb + 1, cap));
            g_st_d = ld_step(max(nbb - 1, 0));
            g_M_d = ld_magic(max(nbb - 1, 0));
        };
        for (;;) {
            while (b < cap && h_r <= T) {  // FCFS joins (R16, R18)'''),
    ("k_decode.cuh", '''                    for (int s = 0; s < SPL; ++s)
                        if (F[s] != F_EMPTY) F[s] -= I;
#pragma unroll
                    for (int s = 0; s <= SPL; ++s) {''', '''                    for (int s = 0; s < SPL; ++s)
                        if (F[s] != F_EMPTY) F[s] -= I;
                    if (fmin != F_EMPTY) fmin -= I;
#pragma unroll
                    for (int s = 0; s <= SPL; ++s) {'''),
    ("k_decode.cuh", '''                        if (lane_bit == bit) {
                            F[s] = I + h_dj.x;
                            fa[s] = fin_addr(h_dj.y, nxt);
                        }
                    }
                }
                ++b;
                if constexpr (!COLO) log_b();
                advance();''', '''                        if (lane_bit == bit) {
                            F[s] = I + h_dj.x;
                            fa[s] = fin_addr(h_dj.y, nxt);
                        }
                    }
                }
                fmin = min(fmin, I + h_dj.x);
                ++b;
                g_st_d = g_st_c;
                g_M_d = g_M_c;
                g_st_c = g_st_u;
                g_M_c = g_M_u;
                g_st_u = ld_step(min(b + 1, cap));
                g_M_u = ld_magic(min(b + 1, cap));
                if constexpr (!COLO) log_b();
                advance();'''),
    ("k_decode.cuh", '''            const int64_t st = ld_step(b);
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
            const uint32_t kL = fmin - I;''', '''            const int64_t st = g_st_c;
            uint32_t kJ = 0xFFFFFFFFu;
            if (b < cap) {
                const int64_t gap = h_r - T;
                if (gap < 0x80000000ll) kJ = ceil_div_magic((uint32_t)gap, (uint32_t)st, g_M_c);
                else if (h_r != INT64_MAX)
                    kJ = (uint32_t)min((gap + st - 1) / st, (int64_t)0xFFFFFFFF);
            }
            const uint32_t kL = fmin - I;'''),
    ("k_decode.cuh", '''            b -= nl;
            if (nl) {
                mk = T;
                if constexpr (!COLO) log_b();
            }''', '''            b -= nl;
            if (nl) {
                mk = T;
                if constexpr (!COLO) log_b();
                uint32_t f = F[0];
#pragma unroll
                for (int s = 1; s < SPL; ++s) f = min(f, F[s]);
                fmin = __reduce_min_sync(FULL, f);
                if (nl == 1) {
                    g_st_u = g_st_c;
                    g_M_u = g_M_c;
                    g_st_c = g_st_d;
                    g_M_c = g_M_d;
                    g_st_d = ld_step(max(b - 1, 0));
                    g_M_d = ld_magic(max(b - 1, 0));
                } else {
                    g_load(b);
                }
            }'''),
]

# the one-leave path decrements b without waiting for popc(ballot)
VARIANTS["nl2"] = [("k_decode.cuh", '''                        fr |= lm;
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
                        if (b == 0 || h_r <= T) break;''', '''                        fr |= lm;
                        mk = T;
                        fmin = __reduce_min_sync(FULL, Fm);
                        if ((lm & (lm - 1u)) != 0u) {  // several left at once: leave the loop
                            b -= __popc(lm);
                            log_b();
                            load_nbr(b);
                            break;
                        }
                        --b;
                        log_b();
                        shift_down();
                        if (b == 0 || h_r <= T) break;''')]

# packed keys (F << 5 | lane) for DPD/DSD caps <= 31: one REDUX gives the leaver
# (no ballot / popc), joins update kmin uniformly; ring refills hoisted
_PK_BLOCK = open(__import__("os").path.join(__import__("os").path.dirname(__file__), "ab_blocks",
                                            "packed_spl1.txt")).read()
VARIANTS["packed"] = [
    ("k_decode.cuh", '''constexpr int DEC_WARPS = 1;  // one warp per k_decode block (leader or helper)''',
     '''constexpr int DEC_WARPS = 1;  // one warp per k_decode block (leader or helper)
constexpr uint32_t KEY_INF = 0xFFFFFFFFu;  // packed-key decode loop (caps <= 31)
constexpr uint32_t PK_REBASE = 1u << 25;   // keys hold F < 2^27: rebase I at 2^25
constexpr uint32_t PK_MAXD = 1u << 25;     // ... which needs every demand < 2^25'''),
    ("k_decode.cuh", '''        };
        uint32_t Fm = F_EMPTY, fmin = F_EMPTY;
        int64_t *fa = fin_rows;''', '''        };
''' + _PK_BLOCK + '''        uint32_t Fm = F_EMPTY, fmin = F_EMPTY;
        int64_t *fa = fin_rows;'''),
    ("k_decode.cuh", '''        iters[0] += c_b;
    } else {
        // general loop, caps 32..256: SPL rows of 32 member slots per lane''', '''        iters[0] += c_b;
        }
    } else {
        // general loop, caps 32..256: SPL rows of 32 member slots per lane'''),
    ("common.cuh", '''    int32_t n_ev;        // LOG launches: batch-size log entries written
    int32_t pad[3];''', '''    int32_t n_ev;        // LOG launches: batch-size log entries written
    uint32_t maxd;       // largest decode demand of the chain (k_segments)
    int32_t pad[2];'''),
    ("k_stages.cuh", '''    __shared__ int32_t s_min_step;''', '''    __shared__ int32_t s_min_step;
    __shared__ uint32_t s_maxd;'''),
    ("k_stages.cuh", '''    if (threadIdx.x == 0) s_min_step = INT32_MAX;
    __syncthreads();''', '''    if (threadIdx.x == 0) {
        s_min_step = INT32_MAX;
        s_maxd = 0;
    }
    __syncthreads();
    uint32_t maxd = 0;'''),
    ("k_stages.cuh", '''            for (int32_t q = lo + lane; q < hi; q += 32)
                m = max(m, __ldg(ch.dec_r + q) + (int64_t)__ldg(&ch.dec_dj[q].x) * smin +
                               (colo ? __ldg(ch.dec_pf + q) : 0));''', '''            for (int32_t q = lo + lane; q < hi; q += 32) {
                const uint32_t dq = __ldg(&ch.dec_dj[q].x);
                maxd = max(maxd, dq);
                m = max(m, __ldg(ch.dec_r + q) + (int64_t)dq * smin +
                               (colo ? __ldg(ch.dec_pf + q) : 0));
            }'''),
    ("k_stages.cuh", '''    if (threadIdx.x == 0) {
        ch.seg_start[ncand] = M;''', '''    maxd = __reduce_max_sync(FULL, maxd);
    if (lane == 0) atomicMax(&s_maxd, maxd);
    __syncthreads();
    if (threadIdx.x == 0) {
        ch.x->maxd = s_maxd;
        ch.seg_start[ncand] = M;'''),
]

# each 4-lane unit walks a contiguous run of C requests: per-warp work is a sum over
# 8 x C requests, so the long-tailed lengths average out
VARIANTS["dsdC"] = [
    ("k_dsd_demand.cuh", '''    const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / DSD_QL;
    const bool valid = j < g->n;''', '''  const int64_t unit = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / DSD_QL;
  for (int64_t jj = 0; jj < DSD_C; ++jj) {
    const int64_t j = unit * DSD_C + jj;
    if (__all_sync(gmask, j >= g->n)) break;
    const bool valid = j < g->n;'''),
    ("k_dsd_demand.cuh", '''    if (valid && sub == 0) g->K[j] = K;
}''', '''    if (valid && sub == 0) g->K[j] = K;
  }
}'''),
    ("k_dsd_demand.cuh", '''constexpr int DSD_QL = 4;  // lanes per request''', '''constexpr int DSD_QL = 4;  // lanes per request
constexpr int DSD_C = 16;  // requests per 4-lane unit'''),
    ("greenllm.cu", '''        dim3 grid((unsigned)((gmax * gl::DSD_QL + 255) / 256), (unsigned)groups.size());''',
     '''        dim3 grid((unsigned)(((gmax + gl::DSD_C - 1) / gl::DSD_C * gl::DSD_QL + 255) / 256),
                  (unsigned)groups.size());'''),
]

VARIANTS["st32"] = [("k_stages.cuh", "constexpr int ST_WARPS = 16;", "constexpr int ST_WARPS = 32;")]

# 32-bit threshold compares: u < thr with thr <= 2^32 is u < min(thr, 2^32 - 1) except
# u = 2^32 - 1 against thr = 2^32 (alpha = 1), counted separately
VARIANTS["thr32"] = [("k_dsd_demand.cuh", '''template <int G>
__device__ __forceinline__ uint32_t accepted_tokens(uint32_t u, const uint64_t (&thr)[G])
{
    uint32_t acc = 1;
#pragma unroll
    for (int c = 0; c < G; ++c) acc += ((uint64_t)u < thr[c]) ? 1u : 0u;
    return acc;
}''', '''template <int G>
__device__ __forceinline__ uint32_t accepted_tokens(uint32_t u, const uint32_t (&thr)[G],
                                                    uint32_t nfull)
{
    uint32_t acc = 1 + (u == 0xFFFFFFFFu ? nfull : 0u);
#pragma unroll
    for (int c = 0; c < G; ++c) acc += (u < thr[c]) ? 1u : 0u;
    return acc;
}'''), ("k_dsd_demand.cuh", '''    uint64_t thr[G];
#pragma unroll
    for (int c = 0; c < G; ++c) thr[c] = g->thr[c];''', '''    uint32_t thr[G];
    uint32_t nfull = 0;  // thresholds equal to 2^32 (always accepted)
#pragma unroll
    for (int c = 0; c < G; ++c) {
        const uint64_t t = g->thr[c];
        thr[c] = t >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)t;
        nfull += t > 0xFFFFFFFFull ? 1u : 0u;
    }'''), ("k_dsd_demand.cuh", '''        const uint32_t a0 = accepted_tokens<G>(w.x, thr), a1 = accepted_tokens<G>(w.y, thr);
        const uint32_t a2 = accepted_tokens<G>(w.z, thr), a3 = accepted_tokens<G>(w.w, thr);''', '''        const uint32_t a0 = accepted_tokens<G>(w.x, thr, nfull), a1 = accepted_tokens<G>(w.y, thr, nfull);
        const uint32_t a2 = accepted_tokens<G>(w.z, thr, nfull), a3 = accepted_tokens<G>(w.w, thr, nfull);''')]

# a head that is already ready joins inside the light loop (kJ = 0) instead of
# leaving to the admission loop
VARIANTS["nohr"] = [
    ("k_decode.cuh", '''                    const int64_t gap = h_r - T;
                    const uint32_t kJ = ceil_div_magic((uint32_t)gap, (uint32_t)st, M_c);
                    if (gap >= 0x80000000ll || I >= 0x80000000u) {''', '''                    const int64_t gap = h_r - T;
                    const uint32_t kJ = ceil_div_magic((uint32_t)max(gap, (int64_t)0), (uint32_t)st, M_c);
                    if (gap >= 0x80000000ll || I >= 0x80000000u) {'''),
    ("k_decode.cuh", '''                        advance_fast();
                        if (b == cap || h_r <= T) break;''', '''                        advance_fast();
                        if (b == cap) break;'''),
    ("k_decode.cuh", '''                        shift_down();
                        if (nl != 1) {  // several members left at once: leave the loop
                            load_nbr(b);
                            break;
                        }
                        if (b == 0 || h_r <= T) break;''', '''                        shift_down();
                        if (nl != 1) {  // several members left at once: leave the loop
                            load_nbr(b);
                            break;
                        }
                        if (b == 0) break;'''),
]

# packed keys only for chains k_segments flags as overloaded (rho >= 1.2): the
# saturated loop wins there, the near-saturated / light chains keep the base loops
def _pksel():
    v = []
    for f, old, new in VARIANTS["packed"]:
        if f == "k_decode.cuh" and "pk_done = true" in new:
            new = new.replace("if (xx->maxd < PK_MAXD) {", "if (xx->maxd < PK_MAXD && xx->pk) {", 1)
        if f == "common.cuh":
            new = new.replace('''    uint32_t maxd;       // largest decode demand of the chain (k_segments)
    int32_t pad[2];''', '''    uint32_t maxd;       // largest decode demand of the chain (k_segments)
    int32_t pk;          // 1: overloaded chain, packed-key loops (k_segments)
    int32_t pad;''')
        if f == "k_stages.cuh" and "s_maxd = 0;" in new:
            new = new.replace("    uint32_t maxd = 0;", "    uint32_t maxd = 0;\n    unsigned long long sumd = 0;")
            new = new.replace("        s_maxd = 0;", "        s_maxd = 0;\n        s_sumd = 0;")
        if f == "k_stages.cuh" and "__shared__ uint32_t s_maxd;" in new:
            new = new + "\n    __shared__ unsigned long long s_sumd;"
        if f == "k_stages.cuh" and "maxd = max(maxd, dq);" in new:
            new = new.replace("maxd = max(maxd, dq);", "maxd = max(maxd, dq);\n                sumd += dq;")
        if f == "k_stages.cuh" and "ch.x->maxd = s_maxd;" in new:
            new = new.replace('''    maxd = __reduce_max_sync(FULL, maxd);
    if (lane == 0) atomicMax(&s_maxd, maxd);''', '''    maxd = __reduce_max_sync(FULL, maxd);
    for (int o = 16; o; o >>= 1) sumd += __shfl_xor_sync(FULL, sumd, o);
    if (lane == 0) {
        atomicMax(&s_maxd, maxd);
        atomicAdd(&s_sumd, sumd);
    }''')
            new = new.replace('''        ch.x->maxd = s_maxd;''', '''        ch.x->maxd = s_maxd;
        // offered decode load at a full batch: rho = sum(d) step[cap] / (cap span)
        const int64_t span = M > 1 ? __ldg(ch.dec_r + M - 1) - __ldg(ch.dec_r) : 0;
        const double work = (double)s_sumd * (double)__ldg(ch.step + ch.cap);
        ch.x->pk = (!colo && M > 1 && work >= 1.2 * (double)ch.cap * (double)span) ? 1 : 0;''')
        v.append((f, old, new))
    return v


VARIANTS["pksel"] = _pksel()

# the time / counter advance k = min(kJ, kL) happens before the join/leave branch
VARIANTS["kfirst"] = [
    ("k_decode.cuh", '''                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;
                        I += kJ;
                        c_b += (lane == b) ? kJ : 0u;
                        if (((nxt + 2) & 127) <= 1) break;  // ring refill due: joins at the top''',
     '''                    const bool jn = kJ < kL;
                    const uint32_t k = jn ? kJ : kL;
                    T += (int64_t)k * st;
                    I += k;
                    c_b += (lane == b) ? k : 0u;
                    if (jn) {  // the head joins at T + kJ * step[b]
                        if (((nxt + 2) & 127) <= 1) break;  // ring refill due: joins at the top'''),
    ("k_decode.cuh", '''                    } else {  // leave at iteration fmin (R16)
                        T += (int64_t)kL * st;
                        I = fmin;
                        c_b += (lane == b) ? kL : 0u;
                        const bool lv = Fm == I;''', '''                    } else {  // leave at iteration fmin (R16)
                        const bool lv = Fm == I;'''),
]
# branch layout hint: the leave is the more frequent event
VARIANTS["expect"] = [("k_decode.cuh", '''                    if (kJ < kL) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;''', '''                    if (__builtin_expect(kJ < kL, 0)) {  // the head joins at T + kJ * step[b]
                        T += (int64_t)kJ * st;''')]

# 32-bit relative time inside the light-load loop (DPD/DSD)
_T32 = open(__import__("os").path.join(__import__("os").path.dirname(__file__), "ab_blocks",
                                       "t32_light.txt")).read()
VARIANTS["t32"] = [
    ("k_decode.cuh", '''                bool slow = false;
                for (;;) {
                    const int64_t st = st_c;
                    const uint32_t kL = fmin - I;
                    const int64_t gap = h_r - T;''', _T32 + '''                for (;;) {
                    const int64_t st = st_c;
                    const uint32_t kL = fmin - I;
                    const int64_t gap = h_r - T;'''),
    ("k_decode.cuh", '''                        if (b == 0 || h_r <= T) break;
                    }
                }
                if (!slow) continue;''', '''                        if (b == 0 || h_r <= T) break;
                    }
                }
              }
                if (!slow) continue;'''),
]

# branch layout hints on the light loop's exits (the common one-leave / one-join
# path falls through to the back edge)
_EXP_NL = ("k_decode.cuh", '''                        if (nl != 1) {  // several members left at once: leave the loop''',
           '''                        if (__builtin_expect(nl != 1, 0)) {  // several members left at once''')
_EXP_LV = ("k_decode.cuh", '''                        if (b == 0 || h_r <= T) break;
                    }''', '''                        if (__builtin_expect(b == 0 || h_r <= T, 0)) break;
                    }''')
_EXP_JN = ("k_decode.cuh", '''                        if (((nxt + 2) & 127) <= 1) break;  // ring refill due: joins at the top''',
           '''                        if (__builtin_expect(((nxt + 2) & 127) <= 1, 0)) break;  // refill due''')
_EXP_JN2 = ("k_decode.cuh", '''                        if (b == cap || h_r <= T) break;
                    } else {''', '''                        if (__builtin_expect(b == cap || h_r <= T, 0)) break;
                    } else {''')
VARIANTS["expnl"] = [_EXP_NL]
VARIANTS["explv"] = [_EXP_NL, _EXP_LV]
VARIANTS["expjn"] = [_EXP_JN, _EXP_JN2]
VARIANTS["expall"] = [_EXP_NL, _EXP_LV, _EXP_JN, _EXP_JN2]

# the run's makespan from T where the batch empties (idle branch) instead of a
# 64-bit move at every leave of the SPL = 1 fast loops
VARIANTS["nomk"] = [
    ("k_decode.cuh", '''                    if (lv) *fa = T;
                    mk = T;
                    const bool one = (lm & (lm - 1u)) == 0u;''', '''                    if (lv) *fa = T;
                    const bool one = (lm & (lm - 1u)) == 0u;'''),
    ("k_decode.cuh", '''                        b -= nl;
                        log_b();
                        mk = T;
                        fmin = __reduce_min_sync(FULL, Fm);
                        shift_down();''', '''                        b -= nl;
                        log_b();
                        fmin = __reduce_min_sync(FULL, Fm);
                        shift_down();'''),
    ("k_decode.cuh", '''            if (b == 0) {  // idle until the next decode request is ready (R17)
                if (h_r == INT64_MAX) {''', '''            if (b == 0) {  // idle until the next decode request is ready (R17)
                mk = T;  // the batch emptied at its last finish
                if (h_r == INT64_MAX) {'''),
]

# co-located light loop: heads already ready after a join's prefill join at once
# inside the loop (each after its own prefill) instead of via the admission loop
VARIANTS["colojoin"] = [("k_decode.cuh", '''                        ++b;
                        log_b();
                        shift_up();
                        advance_fast();
                        if (b == cap || h_r <= T) break;
                    } else {  // leave at iteration fmin (R16)''', '''                        ++b;
                        log_b();
                        shift_up();
                        advance_fast();
                        if constexpr (COLO) {
                            while (b < cap && h_r <= T && h_dj.x != 0 && ((nxt + 2) & 127) > 1) {
                                prefill();
                                const unsigned bit2 = fr & (0u - fr);
                                fr ^= bit2;
                                const uint32_t fnew2 = I + h_dj.x;
                                if (lane_bit == bit2) {
                                    Fm = fnew2;
                                    fa = fin_addr(h_dj.y, nxt);
                                }
                                fmin = min(fmin, fnew2);
                                ++b;
                                log_b();
                                shift_up();
                                advance_fast();
                            }
                        }
                        if (b == cap || h_r <= T) break;
                    } else {  // leave at iteration fmin (R16)''')]

# DChain layout variants (ptxas schedules k_decode differently per layout; adding a
# pointer field after seg_start cost 2.6%)
_DC_END = '''    int32_t mode, cap, max_prompt, capacity_ok;
};'''
VARIANTS["lay_pad8"] = [("common.cuh", _DC_END, '''    int32_t mode, cap, max_prompt, capacity_ok;
    int64_t pad0;
};''')]
VARIANTS["lay_pad16"] = [("common.cuh", _DC_END, '''    int32_t mode, cap, max_prompt, capacity_ok;
    int64_t pad0, pad1;
};''')]
VARIANTS["lay_stp_end"] = [
    ("common.cuh", '''    DStagePart *stp;    // [stage_split] k_stages partials of this chain
''', ''),
    ("common.cuh", _DC_END, '''    int32_t mode, cap, max_prompt, capacity_ok;
    DStagePart *stp;
};''')]
VARIANTS["lay_pad_front"] = [("common.cuh", '''    int64_t *dec_r;
    uint2 *dec_dj;''', '''    void *pad_front;
    int64_t *dec_r;
    uint2 *dec_dj;''')]
VARIANTS["lay_x_first"] = [
    ("common.cuh", '''    DChainX *x;
    DStagePart *stp;''', '''    DStagePart *stp;'''),
    ("common.cuh", '''struct DChain {
    const int64_t *a;''', '''struct DChain {
    DChainX *x;
    const int64_t *a;''')]

# k_stages: 8-warp blocks (two per SM by registers), split width up to 8
VARIANTS["st8"] = [("k_stages.cuh", '''constexpr int ST_WARPS = 16;
constexpr int ST_MAX_SPLIT = 4;  // blocks per chain''', '''constexpr int ST_WARPS = 8;
constexpr int ST_MAX_SPLIT = 8;  // blocks per chain''')]
