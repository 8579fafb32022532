// k_savings.cuh -- §5 carbon-efficiency analysis surfaces (
// PAPER.md:355-414, Eqs. 4-6) as an epilogue over the chain statistics.
//
// One thread per (pair, scenario): Case 2 = a disaggregated (or co-located
// SpecDecode) chain d, Case 1 = the Standalone chain s on the same trace
// (P:358-362); the scenario gives the carbon intensity alpha and the lifetimes
// T_A (new GPU), T_B (old GPU).  Case totals are Eqs. 1-3 in the fixed R34 order
// with round-to-nearest intrinsics (no FMA), so every output is bit-identical
// to the oracle:
//   ratio     = (O_A' + E_A' + O_B + E_B) / (O_A + E_A)        Eq. 5, first line
//   op_saved  = O_A - (O_A' + O_B),  emb_saved = E_A - (E_A' + E_B)   (grams)
//   eq6_term  = (t_B/T_B B) / (N_A alpha + t_A'/T_A A)         Eq. 6 as printed (R49)
//   eq4       = N_A > N_A' + N_B on integer energies           Eq. 4 (energy, G1)
// Pair-major output: out[p * n_scen + s]; consecutive threads write consecutive
// 40-B records (coalesced), the pair's two 80-B stats records stay in L1/L2.
#pragma once

#include "common.cuh"

namespace gl {

struct DPairC {
    int32_t d, s;
    double ce_new_d, ce_old_d, ce_new_s, ce_old_s;
};

__device__ __forceinline__ void carbon_parts(const gl_chain_stats &st, double ce_new, double ce_old,
                                             const gl_scenario &sc, double &op, double &emb)
{
    const double kwh_new = __ddiv_rn((double)st.e_new_uj, 3.6e12);
    const double kwh_old = __ddiv_rn((double)st.e_old_uj, 3.6e12);
    op = __dmul_rn(__dadd_rn(kwh_new, kwh_old), sc.ci_g_per_kwh);
    const double emb_new = __dmul_rn(__ddiv_rn(__ddiv_rn((double)st.busy_new_us, 1e6), sc.lt_new_s), ce_new);
    const double emb_old = __dmul_rn(__ddiv_rn(__ddiv_rn((double)st.busy_old_us, 1e6), sc.lt_old_s), ce_old);
    emb = __dadd_rn(emb_new, emb_old);
}

__global__ void __launch_bounds__(256)
    k_savings(const gl_chain_stats *__restrict__ stats, const DPairC *__restrict__ pairs,
              const gl_scenario *__restrict__ scen, int32_t n_pairs, int32_t n_scen,
              gl_savings *__restrict__ out)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (int64_t)n_pairs * n_scen) return;
    const int32_t p = (int32_t)(g / n_scen), si = (int32_t)(g % n_scen);
    const DPairC pc = pairs[p];
    const gl_chain_stats &d = stats[pc.d];
    const gl_chain_stats &s = stats[pc.s];
    const gl_scenario sc = scen[si];
    double op_d, emb_d, op_s, emb_s;
    carbon_parts(d, pc.ce_new_d, pc.ce_old_d, sc, op_d, emb_d);
    carbon_parts(s, pc.ce_new_s, pc.ce_old_s, sc, op_s, emb_s);
    gl_savings r;
    r.ratio = __ddiv_rn(__dadd_rn(op_d, emb_d), __dadd_rn(op_s, emb_s));
    r.op_saved_g = __dsub_rn(op_s, op_d);
    r.emb_saved_g = __dsub_rn(emb_s, emb_d);
    const double n_a = __dadd_rn(__ddiv_rn((double)s.e_new_uj, 3.6e12), __ddiv_rn((double)s.e_old_uj, 3.6e12));
    const double e_b = __dmul_rn(__ddiv_rn(__ddiv_rn((double)d.busy_old_us, 1e6), sc.lt_old_s), pc.ce_old_d);
    const double e_a2 = __dmul_rn(__ddiv_rn(__ddiv_rn((double)d.busy_new_us, 1e6), sc.lt_new_s), pc.ce_new_d);
    r.eq6_term = __ddiv_rn(e_b, __dadd_rn(__dmul_rn(n_a, sc.ci_g_per_kwh), e_a2));
    r.eq4_energy_less = (s.e_new_uj + s.e_old_uj) > (d.e_new_uj + d.e_old_uj) ? 1 : 0;
    r.pad = 0;
    out[g] = r;
}

}  // namespace gl
