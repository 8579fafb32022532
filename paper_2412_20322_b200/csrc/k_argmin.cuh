// k_argmin.cuh -- Alg. 1 on the carbon matrix of Eqs. 1-3.
//
// One warp per row (workload x scenario); lanes stride over the columns
// (candidate configurations, Fig. 8).  Per cell: fp64 total carbon in
// the fixed R34 order with explicit round-to-nearest intrinsics (never contracted
// to FMA, so it is bit-identical to the CPU oracle), feasibility
// slo_den*ok >= slo_num*n by integer cross-products, then a lexicographic
// warp-shuffle argmin: lower total, higher attainment, lower column (R36); the
// fallback (R37) ranks higher attainment, lower total, lower column.
#pragma once

#include "common.cuh"

namespace gl {

// Eqs. 1-3: op = (kWh_new + kWh_old) * CI;  emb = t_new/LT_new*Ce_new + t_old/LT_old*Ce_old
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
    int32_t col;  // -1 = none
};

__device__ __forceinline__ int cmp_att(int64_t ok1, int64_t n1, int64_t ok2, int64_t n2)
{
    const int64_t l = ok1 * n2, r = ok2 * n1;  // n < 2^31 => no overflow
    return (l > r) - (l < r);
}

__device__ __forceinline__ bool better_feasible(const Cand &x, const Cand &y)
{
    if (x.col < 0) return false;
    if (y.col < 0) return true;
    if (x.total != y.total) return x.total < y.total;
    const int c = cmp_att(x.ok, x.n, y.ok, y.n);
    if (c) return c > 0;
    return x.col < y.col;
}

__device__ __forceinline__ bool better_fallback(const Cand &x, const Cand &y)
{
    if (x.col < 0) return false;
    if (y.col < 0) return true;
    const int c = cmp_att(x.ok, x.n, y.ok, y.n);
    if (c) return c > 0;
    if (x.total != y.total) return x.total < y.total;
    return x.col < y.col;
}

__device__ __forceinline__ Cand shfl_xor_cand(const Cand &c, int mask)
{
    Cand o;
    o.total = __shfl_xor_sync(FULL, c.total, mask);
    o.ok = __shfl_xor_sync(FULL, c.ok, mask);
    o.n = __shfl_xor_sync(FULL, c.n, mask);
    o.col = __shfl_xor_sync(FULL, c.col, mask);
    return o;
}

__global__ void __launch_bounds__(256)
    k_argmin(const gl_chain_stats *__restrict__ stats, const DCarbon *__restrict__ cpar,
             const gl_scenario *__restrict__ scen, const int32_t *__restrict__ row_scen,
             const int32_t *__restrict__ cells, int32_t rows, int32_t cols, int32_t slo_num,
             int32_t slo_den, int32_t priority, int32_t default_col, double *__restrict__ carbon_out,
             double *__restrict__ per_token_out, int32_t *__restrict__ choice_out,
             uint8_t *__restrict__ fb_out)
{
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (row >= rows) return;  // warp-uniform
    const gl_scenario sc = scen[row_scen[row]];
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    Cand bf{0.0, 0, 1, -1}, bb{0.0, 0, 1, -1};
    for (int col = lane; col < cols; col += 32) {
        const int32_t k = cells[row * cols + col];
        if (k < 0) {
            const double nan = __longlong_as_double(0x7ff8000000000000ll);
            if (carbon_out) carbon_out[row * cols + col] = nan;
            if (per_token_out) per_token_out[row * cols + col] = nan;
            continue;
        }
        const gl_chain_stats s = stats[k];
        const DCarbon cp = cpar[k];
        const double total = carbon_total(s, cp, sc);
        if (carbon_out) carbon_out[row * cols + col] = total;
        // carbon per token (R33): one IEEE division after the total
        if (per_token_out) per_token_out[row * cols + col] = __ddiv_rn(total, (double)s.tokens);
        // capacity-infeasible (R38) or invalid input (status bits, R55): never
        // feasible, and ok = 0 / total = +inf in the fallback (R37)
        const bool cap_ok = cp.cap_ok != 0 && s.status == 0;
        const bool feas = cap_ok && (int64_t)slo_den * s.slo_ok >= (int64_t)slo_num * s.n;
        const Cand cf{total, s.slo_ok, s.n, col};
        if (feas && better_feasible(cf, bf)) bf = cf;
        const Cand cb{cap_ok ? total : inf, cap_ok ? s.slo_ok : 0, s.n, col};
        if (better_fallback(cb, bb)) bb = cb;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        const Cand of = shfl_xor_cand(bf, off), ob = shfl_xor_cand(bb, off);
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

// Alg. 1 lines 2-9 on explicit matrices (e.g. completed by gl_complete_matrices,
// line 1): fractional attainments, feasible iff present and att >= target (R54).
// One warp per row, same lexicographic shuffle argmin as k_argmin.
struct CandF {
    double c, a;
    int32_t col;
};

__device__ __forceinline__ bool better_feasible_f(const CandF &x, const CandF &y)
{
    if (x.col < 0) return false;
    if (y.col < 0) return true;
    if (x.c != y.c) return x.c < y.c;
    if (x.a != y.a) return x.a > y.a;
    return x.col < y.col;
}

__device__ __forceinline__ bool better_fallback_f(const CandF &x, const CandF &y)
{
    if (x.col < 0) return false;
    if (y.col < 0) return true;
    if (x.a != y.a) return x.a > y.a;
    if (x.c != y.c) return x.c < y.c;
    return x.col < y.col;
}

__global__ void __launch_bounds__(256)
    k_argmin_matrices(const double *__restrict__ carbon, const double *__restrict__ att,
                      const uint8_t *__restrict__ present, int32_t rows, int32_t cols,
                      double target, int32_t priority, int32_t default_col,
                      int32_t *__restrict__ choice_out, uint8_t *__restrict__ fb_out)
{
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (row >= rows) return;  // warp-uniform
    CandF bf{0.0, 0.0, -1}, bb{0.0, 0.0, -1};
    for (int col = lane; col < cols; col += 32) {
        const int64_t k = row * cols + col;
        if (present && !present[k]) continue;
        const CandF c{carbon[k], att[k], col};
        if (c.a >= target && better_feasible_f(c, bf)) bf = c;
        if (better_fallback_f(c, bb)) bb = c;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        CandF of, ob;
        of.c = __shfl_xor_sync(FULL, bf.c, off);
        of.a = __shfl_xor_sync(FULL, bf.a, off);
        of.col = __shfl_xor_sync(FULL, bf.col, off);
        ob.c = __shfl_xor_sync(FULL, bb.c, off);
        ob.a = __shfl_xor_sync(FULL, bb.a, off);
        ob.col = __shfl_xor_sync(FULL, bb.col, off);
        if (better_feasible_f(of, bf)) bf = of;
        if (better_fallback_f(ob, bb)) bb = ob;
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

}  // namespace gl
