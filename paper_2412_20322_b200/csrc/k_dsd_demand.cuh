// k_dsd_demand.cuh -- DSD demand K_j: speculative steps request j needs (R22, R23).
//
// Speculative decoding (§2.2): the verifier accepts draft token
// x with probability min(1, q/p); collapsed to a marginal per-token rate alpha
// (SPEC S:297), one step yields acc = 1 + #{c in 1..gamma : u < thr_c} tokens with
// thr_c = floor(alpha^c 2^32) and u = Philox word (s mod 4) of counter
// (s/4, j, ACCEPT_STREAM, 0) for request j's own step s.  Because the draw is keyed
// by (request, its own step), K_j = min{k : sum_{s<k} acc_s >= o_j - 1} does not
// depend on batching, so one thread per (group, request) computes it up front and
// chains with equal (output lengths, gamma, alpha, seed) share it.
#pragma once

#include "common.cuh"

namespace gl {

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

}  // namespace gl
