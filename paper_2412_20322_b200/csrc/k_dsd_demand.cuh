// k_dsd_demand.cuh -- DSD demand K_j: speculative steps request j needs (R22, R23).
//
// Speculative decoding (§2.2): the verifier accepts draft token
// x with probability min(1, q/p); collapsed to a marginal per-token rate alpha
// (SPEC S:297), one step yields acc = 1 + #{c in 1..gamma : u < thr_c} tokens with
// thr_c = floor(alpha^c 2^32) and u = Philox word (s mod 4) of counter
// (s/4, j, ACCEPT_STREAM, 0) for request j's own step s.  Because the draw is keyed
// by (request, its own step), K_j = min{k : sum_{s<k} acc_s >= o_j - 1} does not
// depend on batching, so chains with equal (output lengths, gamma, alpha, seed)
// share it.
//
// Work split: QL = 4 lanes per request.  In round t lane l evaluates Philox call
// 4t + l (steps 16t + 4l .. +3); the four calls' token counts are prefix-summed with
// two shuffles and the crossing step is found without a serial walk.  The quads are
// persistent (a grid of a few waves per group): a finished quad starts its next
// request in the same loop trip, so lanes idle only at the end of the group.
// The gamma thresholds sit in registers (the kernel is instantiated per gamma;
// the block's group picks the instance), compared as 64-bit (thr = 2^32 at alpha = 1).
#pragma once

#include "common.cuh"

namespace gl {

constexpr int DSD_QL = 4;  // lanes per request

template <int G>
__device__ __forceinline__ uint32_t accepted_tokens(uint32_t u, const uint64_t (&thr)[G])
{
    uint32_t acc = 1;
#pragma unroll
    for (int c = 0; c < G; ++c) acc += ((uint64_t)u < thr[c]) ? 1u : 0u;
    return acc;
}

template <int G>
__device__ __forceinline__ void dsd_demand_body(const DGroup *g)
{
    uint64_t thr[G];
#pragma unroll
    for (int c = 0; c < G; ++c) thr[c] = g->thr[c];
    const int lane = threadIdx.x & 31, sub = lane & (DSD_QL - 1);
    const int qbase = lane & ~(DSD_QL - 1);
    // persistent quads: quad q of the group's blocks takes requests q, q + Q, ...; a
    // quad whose request is done takes its next one at the top of the same loop, so
    // the warp's lanes stay busy until the group's requests run out (not until the
    // longest of the warp's 8 current requests finishes)
    const int64_t Q = (int64_t)gridDim.x * (blockDim.x / DSD_QL);
    int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / DSD_QL;
    const int64_t n = g->n;
    const uint32_t k0 = (uint32_t)g->seed, k1 = (uint32_t)(g->seed >> 32);
    auto need_of = [&](int64_t jj) -> int64_t {
        uint32_t o = jj < n ? __ldg(g->o + jj) : 1u;
        if (o >= O_LIMIT) o = O_LIMIT - 1;
        return (int64_t)o - 1;
    };
    int64_t need = need_of(j);
    int64_t tok = 0;  // tokens accepted before this round
    uint32_t t = 0;
    while (__any_sync(FULL, j < n)) {
        // this lane's call: steps s0 .. s0+3 of request j
        const uint32_t call = DSD_QL * t + sub;
        const uint4 w = philox4x32_10(make_uint4(call, (uint32_t)j, ACCEPT_STREAM, 0u), k0, k1);
        const uint32_t a0 = accepted_tokens<G>(w.x, thr), a1 = accepted_tokens<G>(w.y, thr);
        const uint32_t a2 = accepted_tokens<G>(w.z, thr), a3 = accepted_tokens<G>(w.w, thr);
        const uint32_t mine = a0 + a1 + a2 + a3;
        // inclusive prefix over the 4 lanes of this request
        uint32_t inc = mine;
        uint32_t y = __shfl_up_sync(FULL, inc, 1, DSD_QL);
        if (sub >= 1) inc += y;
        y = __shfl_up_sync(FULL, inc, 2, DSD_QL);
        if (sub >= 2) inc += y;
        const uint32_t round_tot = __shfl_sync(FULL, inc, DSD_QL - 1, DSD_QL);
        const int64_t before = tok + (inc - mine);  // tokens before this lane's call
        // the crossing lies in this lane's call iff before < need <= before + mine
        int64_t cum = before;
        uint32_t ks = 0;
        if (before < need && need <= before + mine) {
            cum += a0;
            ks = 1;
            if (cum < need) { cum += a1; ks = 2; }
            if (cum < need) { cum += a2; ks = 3; }
            if (cum < need) { ks = 4; }
        }
        const unsigned hit = (__ballot_sync(FULL, ks != 0) >> qbase) & 0xFu;
        const int src = __ffs(hit | 0x10u) - 1;  // 4: no crossing this round
        const uint32_t kk = __shfl_sync(FULL, ks, (qbase + (src & 3)) & 31);
        if (hit != 0u || need <= 0) {  // request j done: K_j, then its next request
            const uint32_t K = need <= 0 ? 0u : 4 * (DSD_QL * t + (uint32_t)src) + kk;
            if (j < n && sub == 0) g->K[j] = K;
            j += Q;
            need = need_of(j);
            tok = 0;
            t = 0;
        } else {
            tok += round_tot;
            ++t;
        }
    }
}

__global__ void __launch_bounds__(256) k_dsd_demand(const DGroup *__restrict__ groups)
{
    const DGroup *g = groups + blockIdx.y;
    switch (g->gamma) {
        case 1: dsd_demand_body<1>(g); break;
        case 2: dsd_demand_body<2>(g); break;
        case 3: dsd_demand_body<3>(g); break;
        case 4: dsd_demand_body<4>(g); break;
        case 5: dsd_demand_body<5>(g); break;
        case 6: dsd_demand_body<6>(g); break;
        case 7: dsd_demand_body<7>(g); break;
        case 8: dsd_demand_body<8>(g); break;
        case 9: dsd_demand_body<9>(g); break;
        case 10: dsd_demand_body<10>(g); break;
        case 11: dsd_demand_body<11>(g); break;
        case 12: dsd_demand_body<12>(g); break;
        case 13: dsd_demand_body<13>(g); break;
        case 14: dsd_demand_body<14>(g); break;
        case 15: dsd_demand_body<15>(g); break;
        default: dsd_demand_body<16>(g); break;
    }
}

// Families (several (alpha, gamma) groups on one set of draws; configs 2 and 5 have one
// family of 5 alphas x 8 gammas): one thread per request evaluates each Philox word
// ONCE for every group.  Per draft step s and alpha-set a, m_a = #{c : u_s < thr_a[c]}
// (thresholds decrease in c, so the accepted drafts are a prefix); group (a, gamma)
// accepts 1 + min(gamma, m_a) tokens, and its K is the number of steps taken while
// its running total is still below o - 1.  Running totals grow with alpha and gamma
// (thresholds grow with alpha), so the group (smallest alpha, gamma = 1) is the last
// to finish: the loop for a request ends when it has.  Threads are persistent: a lane
// whose request is done takes its next one (stride = all threads of the family) in
// the same loop trip.
//
// m_a for all alpha-sets comes from one shared-memory table indexed by the top
// FAM_LUT_BITS bits of u: entry .x packs m_a (4 bits per set) at the bucket's top
// value; a bucket holding exactly one threshold thr_a[c] stores it in .y and its set
// a in bits 28-30 of .x, so m_a(u) = m_a(top) + (u < .y) (.y = 0 elsewhere: never
// true); a bucket holding more thresholds sets bit 31 and the lane counts by compares.
// Per group and step: r -= 1 + min(gamma, m) and K += (r > 0) before it (r = tokens
// still needed).
constexpr int FAM_LUT_BITS = 11;
constexpr int FAM_LUT = 1 << FAM_LUT_BITS;

__global__ void __launch_bounds__(128) k_dsd_family(const DFamily *__restrict__ fams)
{
    const DFamily *f = fams + blockIdx.y;
    __shared__ uint32_t *s_K[FAM_NA * FAM_GM];
    __shared__ uint2 s_lut[FAM_LUT];
    if (threadIdx.x < FAM_NA * FAM_GM) s_K[threadIdx.x] = f->K[threadIdx.x / FAM_GM][threadIdx.x % FAM_GM];
    uint32_t thr[FAM_NA][FAM_GM];
    bool all[FAM_NA];
#pragma unroll
    for (int a = 0; a < FAM_NA; ++a) {
        all[a] = __ldg(&f->all[a]) != 0u;
#pragma unroll
        for (int c = 0; c < FAM_GM; ++c) thr[a][c] = __ldg(&f->thr[a][c]);
    }
    auto count = [&](int a, uint32_t u) -> uint32_t {
        uint32_t m = 0;
#pragma unroll
        for (int c = 0; c < FAM_GM; ++c) m += u < thr[a][c] ? 1u : 0u;
        return all[a] ? (uint32_t)FAM_GM : m;
    };
    for (int bkt = threadIdx.x; bkt < FAM_LUT; bkt += blockDim.x) {
        const uint32_t lo = (uint32_t)bkt << (32 - FAM_LUT_BITS);
        const uint32_t hi = lo + ((1u << (32 - FAM_LUT_BITS)) - 1u);
        uint32_t x = 0, y = 0, nbreak = 0;
#pragma unroll
        for (int a = 0; a < FAM_NA; ++a) {
            const uint32_t mh = count(a, hi), ml = count(a, lo);
            x |= mh << (4 * a);
            nbreak += ml - mh;
            if (ml != mh) {
                x |= (uint32_t)a << 28;
#pragma unroll
                for (int c = 0; c < FAM_GM; ++c)
                    if (thr[a][c] > lo && thr[a][c] <= hi) y = thr[a][c];
            }
        }
        if (nbreak > 1) x |= 0x80000000u;  // several thresholds in the bucket: compares
        s_lut[bkt] = make_uint2(x, nbreak == 1 ? y : 0u);
    }
    __syncthreads();
    const int na = __ldg(&f->na);
    const int64_t n = __ldg(&f->n);
    const uint64_t seed = __ldg(&f->seed);
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    const uint32_t *const o = f->o;
    const int64_t Q = (int64_t)gridDim.x * blockDim.x;
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int32_t r[FAM_NA][FAM_GM];   // tokens still needed (the request's o - 1 at first)
    uint32_t kk[FAM_NA][FAM_GM];  // steps taken while r > 0
    uint32_t call = 0;
    // next request with demand > 0 (requests with o = 1 get K = 0 right away)
    auto take = [&]() {
        uint32_t need = 0;
        for (; j < n; j += Q) {
            uint32_t ov = __ldg(o + j);
            if (ov >= O_LIMIT) ov = O_LIMIT - 1;
            need = ov > 0 ? ov - 1 : 0;
            if (need > 0) break;
            for (int i = 0; i < na * FAM_GM; ++i)
                if (s_K[i]) s_K[i][j] = 0u;
        }
#pragma unroll
        for (int a = 0; a < FAM_NA; ++a)
#pragma unroll
            for (int g = 0; g < FAM_GM; ++g) {
                r[a][g] = (int32_t)need;
                kk[a][g] = 0u;
            }
        call = 0;
    };
    take();
    while (__any_sync(FULL, j < n)) {
        if (j < n) {
            const uint4 w = philox4x32_10(make_uint4(call, (uint32_t)j, ACCEPT_STREAM, 0u), k0, k1);
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t u = ws[q];
                const uint2 e = s_lut[u >> (32 - FAM_LUT_BITS)];
                uint32_t pk = (e.x & 0x0FFFFFFFu) + ((u < e.y) ? (1u << (4 * ((e.x >> 28) & 7u))) : 0u);
                if (e.x & 0x80000000u) {  // several thresholds in this bucket
                    pk = 0;
#pragma unroll
                    for (int a = 0; a < FAM_NA; ++a) pk |= count(a, u) << (4 * a);
                }
#pragma unroll
                for (int a = 0; a < FAM_NA; ++a) {
                    const int32_t m1 = (int32_t)((pk >> (4 * a)) & 15u) + 1;
#pragma unroll
                    for (int g = 0; g < FAM_GM; ++g) {
                        kk[a][g] += r[a][g] > 0 ? 1u : 0u;
                        r[a][g] -= min(g + 2, m1);
                    }
                }
            }
            ++call;
            if (r[0][0] <= 0) {  // the last group has crossed: write K, next request
#pragma unroll
                for (int a = 0; a < FAM_NA; ++a)
#pragma unroll
                    for (int g = 0; g < FAM_GM; ++g) {
                        uint32_t *K = s_K[a * FAM_GM + g];
                        if (a < na && K) K[j] = kk[a][g];
                    }
                j += Q;
                take();
            }
        }
    }
}

}  // namespace gl
