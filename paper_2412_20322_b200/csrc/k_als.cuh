// k_als.cuh -- collaborative filtering of partially observed Alg. 1 matrices
// (Alg. 1 line 1) by alternating least
// squares (readings R50-R53).
//
// One 512-thread CTA per matrix of the batch; V [cols x K] lives in shared
// memory, U [rows x K] in global memory (L2-resident).  Per iteration:
//   U-step  one thread per row: Gram = lambda I + sum_{j observed} V_j V_j^T and
//           rhs = sum_j x_ij V_j over the row's columns IN ORDER, then a k x k
//           Cholesky solve -- the same operations in the same order as the oracle,
//           with explicit round-to-nearest intrinsics (no FMA contraction).
//   V-step  per column, the rows split over one or more warps (lanes stride the
//           rows), shuffle-tree and fixed-order partial combination, then the same
//           Cholesky solve by one thread.  The summation order differs from the
//           oracle's sequential one, so results agree to rounding, not bit for bit
//           (tolerance derived in DESIGN.md §2, R50).
// Finally out = x where observed (verbatim), else clamp(U_i . V_j, lo, hi).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace gl {

constexpr int ALS_THREADS = 512;
constexpr int ALS_WARPS = ALS_THREADS / 32;

__device__ __forceinline__ double dfma_free(double acc, double a, double b)
{
    return __dadd_rn(acc, __dmul_rn(a, b));  // acc + a*b, never contracted
}

// A: K x K row-major lower part used (SPD), b: rhs -> solution (oracle's order)
template <int K>
__device__ __forceinline__ void chol_solve(double (&A)[K * K], double (&b)[K])
{
#pragma unroll
    for (int c = 0; c < K; ++c) {
        double d = A[c * K + c];
#pragma unroll
        for (int m = 0; m < c; ++m) d = __dsub_rn(d, __dmul_rn(A[c * K + m], A[c * K + m]));
        d = __dsqrt_rn(d);
        A[c * K + c] = d;
#pragma unroll
        for (int r = c + 1; r < K; ++r) {
            double v = A[r * K + c];
#pragma unroll
            for (int m = 0; m < c; ++m) v = __dsub_rn(v, __dmul_rn(A[r * K + m], A[c * K + m]));
            A[r * K + c] = __ddiv_rn(v, d);
        }
    }
#pragma unroll
    for (int r = 0; r < K; ++r) {
        double v = b[r];
#pragma unroll
        for (int m = 0; m < r; ++m) v = __dsub_rn(v, __dmul_rn(A[r * K + m], b[m]));
        b[r] = __ddiv_rn(v, A[r * K + r]);
    }
#pragma unroll
    for (int r = K - 1; r >= 0; --r) {
        double v = b[r];
#pragma unroll
        for (int m = r + 1; m < K; ++m) v = __dsub_rn(v, __dmul_rn(A[m * K + r], b[m]));
        b[r] = __ddiv_rn(v, A[r * K + r]);
    }
}

struct DAls {
    const double *x;       // [batch][rows][cols]
    const uint8_t *obs;    // [batch][rows][cols]
    const double *v0;      // [batch][cols][K]
    double *u;             // [batch][rows][K]
    double *v_out;         // [batch][cols][K] or null
    double *out;           // [batch][rows][cols]
    int32_t *status;       // [batch]
    int64_t rows;
    int32_t cols, iters;
    double lambda, lo, hi;
};

template <int K>
__global__ void __launch_bounds__(ALS_THREADS, 1) k_als(const DAls p)
{
    constexpr int NS = K * (K + 1) / 2 + K;  // Gram lower triangle + rhs
    extern __shared__ __align__(16) double als_smem[];
    double *V = als_smem;                                  // [cols][K]
    double *part = als_smem + (size_t)p.cols * K;           // [32][NS] (cols <= 32)
    __shared__ int s_flags;
    const int64_t rows = p.rows;
    const int32_t cols = p.cols;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t mo = (size_t)blockIdx.x * (size_t)rows * cols;
    const double *x = p.x + mo;
    const uint8_t *obs = p.obs + mo;
    double *u = p.u + (size_t)blockIdx.x * rows * K;
    for (int i = tid; i < cols * K; i += ALS_THREADS) V[i] = p.v0[(size_t)blockIdx.x * cols * K + i];
    for (int64_t i = tid; i < rows * K; i += ALS_THREADS) u[i] = 0.0;  // U = 0 before iteration 1
    if (tid == 0) s_flags = 0;
    __syncthreads();

    // R53: a row or a column without an observed entry (status bits 1, 2)
    for (int64_t i = tid; i < rows; i += ALS_THREADS) {
        int any = 0;
        for (int32_t j = 0; j < cols; ++j) any |= obs[i * cols + j];
        if (!any) atomicOr(&s_flags, 1);
    }
    for (int32_t j = warp; j < cols; j += ALS_WARPS) {
        int any = 0;
        for (int64_t i = lane; i < rows; i += 32) any |= obs[i * cols + j];
        if (!__any_sync(FULL, any) && lane == 0) atomicOr(&s_flags, 2);
    }

    // V-step work split: cols <= 32 -> g warps per column, partials in smem
    const int g = cols <= ALS_WARPS ? ALS_WARPS / cols : 1;
    for (int it = 0; it < p.iters; ++it) {
        // ---- U-step: one thread per row, columns in order
        for (int64_t i = tid; i < rows; i += ALS_THREADS) {
            double A[K * K], b[K];
#pragma unroll
            for (int a = 0; a < K * K; ++a) A[a] = 0.0;
#pragma unroll
            for (int a = 0; a < K; ++a) b[a] = 0.0;
            for (int32_t j = 0; j < cols; ++j) {
                if (!obs[i * cols + j]) continue;
                const double xv = x[i * cols + j];
                double vj[K];
#pragma unroll
                for (int r = 0; r < K; ++r) vj[r] = V[j * K + r];
#pragma unroll
                for (int r = 0; r < K; ++r) {
#pragma unroll
                    for (int c = 0; c <= r; ++c) A[r * K + c] = dfma_free(A[r * K + c], vj[r], vj[c]);
                    b[r] = dfma_free(b[r], xv, vj[r]);
                }
            }
#pragma unroll
            for (int r = 0; r < K; ++r) A[r * K + r] = __dadd_rn(A[r * K + r], p.lambda);
            chol_solve<K>(A, b);
#pragma unroll
            for (int r = 0; r < K; ++r) u[i * K + r] = b[r];
        }
        __syncthreads();
        // ---- V-step: (column, part) per warp
        for (int w = warp; w < (cols <= ALS_WARPS ? cols * g : cols); w += ALS_WARPS) {
            const int32_t j = cols <= ALS_WARPS ? w / g : w;
            const int part_i = cols <= ALS_WARPS ? w % g : 0;
            const int nparts = cols <= ALS_WARPS ? g : 1;
            double s[NS];
#pragma unroll
            for (int a = 0; a < NS; ++a) s[a] = 0.0;
            for (int64_t i = (int64_t)part_i * 32 + lane; i < rows; i += 32 * nparts) {
                if (!obs[i * cols + j]) continue;
                const double xv = x[i * cols + j];
                double ui[K];
#pragma unroll
                for (int r = 0; r < K; ++r) ui[r] = u[i * K + r];
                int a = 0;
#pragma unroll
                for (int r = 0; r < K; ++r)
#pragma unroll
                    for (int c = 0; c <= r; ++c) {
                        s[a] = dfma_free(s[a], ui[r], ui[c]);
                        ++a;
                    }
#pragma unroll
                for (int r = 0; r < K; ++r) s[a + r] = dfma_free(s[a + r], xv, ui[r]);
            }
#pragma unroll
            for (int a = 0; a < NS; ++a)
#pragma unroll
                for (int o = 16; o; o >>= 1) s[a] = __dadd_rn(s[a], __shfl_xor_sync(FULL, s[a], o));
            if (cols <= ALS_WARPS) {
                if (lane == 0)
#pragma unroll
                    for (int a = 0; a < NS; ++a) part[w * NS + a] = s[a];
            } else if (lane == 0) {
                double A[K * K], b[K];
                int a = 0;
#pragma unroll
                for (int r = 0; r < K; ++r)
#pragma unroll
                    for (int c = 0; c <= r; ++c) A[r * K + c] = s[a++];
#pragma unroll
                for (int r = 0; r < K; ++r) {
                    b[r] = s[a + r];
                    A[r * K + r] = __dadd_rn(A[r * K + r], p.lambda);
                }
                chol_solve<K>(A, b);
#pragma unroll
                for (int r = 0; r < K; ++r) V[j * K + r] = b[r];
            }
        }
        if (cols <= ALS_WARPS) {
            __syncthreads();
            if (tid < cols) {  // combine the column's g partials in order, solve
                const int32_t j = tid;
                double s[NS];
#pragma unroll
                for (int a = 0; a < NS; ++a) s[a] = part[(j * g) * NS + a];
                for (int q = 1; q < g; ++q)
#pragma unroll
                    for (int a = 0; a < NS; ++a) s[a] = __dadd_rn(s[a], part[(j * g + q) * NS + a]);
                double A[K * K], b[K];
                int a = 0;
#pragma unroll
                for (int r = 0; r < K; ++r)
#pragma unroll
                    for (int c = 0; c <= r; ++c) A[r * K + c] = s[a++];
#pragma unroll
                for (int r = 0; r < K; ++r) {
                    b[r] = s[a + r];
                    A[r * K + r] = __dadd_rn(A[r * K + r], p.lambda);
                }
                chol_solve<K>(A, b);
#pragma unroll
                for (int r = 0; r < K; ++r) V[j * K + r] = b[r];
            }
        }
        __syncthreads();
    }

    // ---- completion: observed entries verbatim, the rest clamp(U_i . V_j)
    double *out = p.out + mo;
    const int64_t cells = rows * cols;
    for (int64_t q = tid; q < cells; q += ALS_THREADS) {
        if (obs[q]) {
            out[q] = x[q];
            continue;
        }
        const int64_t i = q / cols;
        const int32_t j = (int32_t)(q - i * cols);
        double v = 0.0;
#pragma unroll
        for (int r = 0; r < K; ++r) v = dfma_free(v, u[i * K + r], V[j * K + r]);
        out[q] = v < p.lo ? p.lo : (v > p.hi ? p.hi : v);
    }
    if (p.v_out)
        for (int i = tid; i < cols * K; i += ALS_THREADS) p.v_out[(size_t)blockIdx.x * cols * K + i] = V[i];
    __syncthreads();
    if (tid == 0) p.status[blockIdx.x] = s_flags;
}

__host__ __device__ inline size_t als_smem_bytes(int cols, int k)
{
    const int ns = k * (k + 1) / 2 + k;
    return sizeof(double) * ((size_t)cols * k + (cols <= ALS_WARPS ? (size_t)ALS_WARPS * ns : 0));
}

// ---- multi-CTA ALS for small batches: P CTAs per matrix, one grid-wide barrier
// per iteration (cooperative launch).  CTA p owns a contiguous block of rows: its
// U-step, its partial V-step sums (warp per column, lanes striding its rows) into
// a double-buffered global array; after the barrier EVERY CTA combines the P
// partials of each column in order p = 0..P-1 and solves V itself (no second
// barrier).  Fixed assignment and order => deterministic.

constexpr int ALSC_THREADS = 256;
constexpr int ALSC_WARPS = ALSC_THREADS / 32;

template <int K>
__global__ void __launch_bounds__(ALSC_THREADS)
    k_als_coop(const DAls p, double *__restrict__ part, uint32_t *__restrict__ colmask,
               int32_t *__restrict__ rowflag, int P)
{
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    constexpr int NS = K * (K + 1) / 2 + K;
    extern __shared__ __align__(16) double alsc_smem[];
    double *V = alsc_smem;  // [cols][K]
    const int mat = blockIdx.x / P, pi = blockIdx.x % P;
    const int64_t rows = p.rows;
    const int32_t cols = p.cols;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = rows * pi / P, r1 = rows * (pi + 1) / P;
    const size_t mo = (size_t)mat * (size_t)rows * cols;
    const double *x = p.x + mo;
    const uint8_t *obs = p.obs + mo;
    double *u = p.u + (size_t)mat * rows * K;
    const int cw = (cols + 31) / 32;
    for (int i = tid; i < cols * K; i += ALSC_THREADS) V[i] = p.v0[(size_t)mat * cols * K + i];
    for (int64_t i = r0 * K + tid; i < r1 * K; i += ALSC_THREADS) u[i] = 0.0;  // U = 0 before iteration 1

    // R53 status: rows without an observed entry; columns observed somewhere
    for (int64_t i = r0 + tid; i < r1; i += ALSC_THREADS) {
        int any = 0;
        for (int32_t j = 0; j < cols; ++j) any |= obs[i * cols + j];
        if (!any) atomicOr(rowflag + mat, 1);
    }
    for (int32_t j = warp; j < cols; j += ALSC_WARPS) {
        int any = 0;
        for (int64_t i = r0 + lane; i < r1; i += 32) any |= obs[i * cols + j];
        if (__any_sync(FULL, any) && lane == 0) atomicOr(colmask + (size_t)mat * cw + j / 32, 1u << (j & 31));
    }
    __syncthreads();

    for (int it = 0; it < p.iters; ++it) {
        // U-step over this CTA's rows (the oracle's order within a row)
        for (int64_t i = r0 + tid; i < r1; i += ALSC_THREADS) {
            double A[K * K], b[K];
#pragma unroll
            for (int a = 0; a < K * K; ++a) A[a] = 0.0;
#pragma unroll
            for (int a = 0; a < K; ++a) b[a] = 0.0;
            for (int32_t j = 0; j < cols; ++j) {
                if (!obs[i * cols + j]) continue;
                const double xv = x[i * cols + j];
                double vj[K];
#pragma unroll
                for (int r = 0; r < K; ++r) vj[r] = V[j * K + r];
#pragma unroll
                for (int r = 0; r < K; ++r) {
#pragma unroll
                    for (int c = 0; c <= r; ++c) A[r * K + c] = dfma_free(A[r * K + c], vj[r], vj[c]);
                    b[r] = dfma_free(b[r], xv, vj[r]);
                }
            }
#pragma unroll
            for (int r = 0; r < K; ++r) A[r * K + r] = __dadd_rn(A[r * K + r], p.lambda);
            chol_solve<K>(A, b);
#pragma unroll
            for (int r = 0; r < K; ++r) u[i * K + r] = b[r];
        }
        __syncthreads();
        // partial V-step sums of this CTA's rows: warp per column
        double *pb = part + (((size_t)(it & 1) * gridDim.x + blockIdx.x) * cols) * NS;
        for (int32_t j = warp; j < cols; j += ALSC_WARPS) {
            double s[NS];
#pragma unroll
            for (int a = 0; a < NS; ++a) s[a] = 0.0;
            for (int64_t i = r0 + lane; i < r1; i += 32) {
                if (!obs[i * cols + j]) continue;
                const double xv = x[i * cols + j];
                double ui[K];
#pragma unroll
                for (int r = 0; r < K; ++r) ui[r] = u[i * K + r];
                int a = 0;
#pragma unroll
                for (int r = 0; r < K; ++r)
#pragma unroll
                    for (int c = 0; c <= r; ++c) {
                        s[a] = dfma_free(s[a], ui[r], ui[c]);
                        ++a;
                    }
#pragma unroll
                for (int r = 0; r < K; ++r) s[a + r] = dfma_free(s[a + r], xv, ui[r]);
            }
#pragma unroll
            for (int a = 0; a < NS; ++a)
#pragma unroll
                for (int o = 16; o; o >>= 1) s[a] = __dadd_rn(s[a], __shfl_xor_sync(FULL, s[a], o));
            if (lane == 0)
#pragma unroll
                for (int a = 0; a < NS; ++a) pb[(size_t)j * NS + a] = s[a];
        }
        grid.sync();
        // every CTA combines its matrix's P partials per column (warp per column: lane
        // l sums partials l, l+32, ... in order, then a fixed shuffle tree) and solves V
        const double *pa = part + ((size_t)(it & 1) * gridDim.x + (size_t)mat * P) * cols * NS;
        for (int32_t j = warp; j < cols; j += ALSC_WARPS) {
            double s[NS];
#pragma unroll
            for (int a = 0; a < NS; ++a) s[a] = 0.0;
            for (int q = lane; q < P; q += 32)
#pragma unroll
                for (int a = 0; a < NS; ++a)
                    s[a] = __dadd_rn(s[a], __ldcg(pa + ((size_t)q * cols + j) * NS + a));
#pragma unroll
            for (int a = 0; a < NS; ++a)
#pragma unroll
                for (int o = 16; o; o >>= 1) s[a] = __dadd_rn(s[a], __shfl_xor_sync(FULL, s[a], o));
            if (lane != 0) continue;
            double A[K * K], b[K];
            int a = 0;
#pragma unroll
            for (int r = 0; r < K; ++r)
#pragma unroll
                for (int c = 0; c <= r; ++c) A[r * K + c] = s[a++];
#pragma unroll
            for (int r = 0; r < K; ++r) {
                b[r] = s[a + r];
                A[r * K + r] = __dadd_rn(A[r * K + r], p.lambda);
            }
            chol_solve<K>(A, b);
#pragma unroll
            for (int r = 0; r < K; ++r) V[j * K + r] = b[r];
        }
        __syncthreads();
    }
    if (p.iters == 0) grid.sync();  // the status flags below need every CTA's pre-pass

    // completion of this CTA's rows
    double *out = p.out + mo;
    for (int64_t q = r0 * cols + tid; q < r1 * cols; q += ALSC_THREADS) {
        if (obs[q]) {
            out[q] = x[q];
            continue;
        }
        const int64_t i = q / cols;
        const int32_t j = (int32_t)(q - i * cols);
        double v = 0.0;
#pragma unroll
        for (int r = 0; r < K; ++r) v = dfma_free(v, u[i * K + r], V[j * K + r]);
        out[q] = v < p.lo ? p.lo : (v > p.hi ? p.hi : v);
    }
    if (pi == 0) {
        if (p.v_out)
            for (int i = tid; i < cols * K; i += ALSC_THREADS) p.v_out[(size_t)mat * cols * K + i] = V[i];
        if (tid == 0) {
            int32_t f = __ldcg(rowflag + mat) ? 1 : 0;
            for (int32_t j = 0; j < cols; ++j)
                if (!((__ldcg(colmask + (size_t)mat * cw + j / 32) >> (j & 31)) & 1u)) f |= 2;
            p.status[mat] = f;
        }
    }
}

}  // namespace gl
