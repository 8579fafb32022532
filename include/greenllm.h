/*
 * greenllm.h -- C ABI of libgreenllm.so, the B200-native (sm_100a) batched
 * SLO / carbon grid evaluator for GreenLLM (arXiv 2412.20322).
 *
 * The problem statement this ABI follows is Alg. 1 (§4.3):
 *   input  a profiling database D, workloads W = {(req_size, qps)},
 *          SLO_target and a fallback priority;
 *   output the Optimal configuration per workload.
 * gl_eval_grid replaces D by exact simulation of every candidate configuration
 * on a request trace; gl_argmin_feasible IS Alg. 1 with
 * the carbon matrix C computed from Eqs. 1-3.  gl_evaluate_host runs
 * both end to end from host buffers.
 *
 * Conventions
 *  - Times are integer microseconds (int64 absolute, int32 table entries),
 *    energies integer microjoules, carbon grams (fp64), lifetimes seconds
 *    (365-day years), carbon intensity gCO2/kWh.  DESIGN.md §2 lists every
 *    rule (R1-R40) the simulation implements; the CPU oracle under oracle/
 *    implements the same rules independently.
 *  - "device" = CUDA device memory of the current device; "host" = CPU memory.
 *  - The caller owns every buffer.  The library keeps no global state besides
 *    a cached device-capability check and, per host thread and device, up to five
 *    side streams with their events (created on first use, kept for the process);
 *    it allocates only stream-ordered scratch (cudaMallocAsync / cudaFreeAsync
 *    on `stream`) and never synchronises except in gl_evaluate_host.  When one
 *    gl_eval_grid call holds both disaggregated and co-located chains, it forks
 *    a side stream from `stream` (event record / wait) for the co-located decode
 *    launch and joins it back before returning, so the call remains ordered on
 *    `stream`; if the fork fails the two launches run one after the other.
 *  - Calls are asynchronous and stream-ordered (except gl_evaluate_host):
 *    device buffers must stay valid until `stream` has passed the call; host
 *    descriptor arrays are consumed before the call returns.
 *  - Outputs are deterministic: bit-identical for identical inputs, for any
 *    launch geometry, chain order or sharding.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Errors: invalid host-visible arguments return a gl_status synchronously
 *    and launch nothing.  Data-dependent violations found on the device are
 *    reported per chain in gl_chain_stats.status (GL_ST_* bits); the chain's
 *    other statistics are then 0 (n and status kept; R55) and Alg. 1 never
 *    selects it as feasible.
 */
#ifndef GREENLLM_H
#define GREENLLM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GL_VERSION 3  /* 2: carbon_per_token_out in gl_argmin_feasible; 3: gl_schedule hints */
#define GL_MAX_CAP 256        /* batch cap: 8 active-set slots per lane x 32 lanes */
#define GL_MAX_GAMMA 16       /* DSD draft length */
#define GL_MAX_PROMPT 16384   /* prompt-indexed tables live in shared memory */

typedef int32_t gl_status;
enum {
    GL_OK = 0,
    GL_E_INVALID = -1,     /* null pointer, n <= 0, cap/gamma/max_prompt out of range, misaligned */
    GL_E_DOMAIN = -2,      /* alpha not in [0,1], negative SLO, CI < 0, LT <= 0, Ce <= 0, non-finite */
    GL_E_LOOKUP = -3,      /* trace_idx, row_scenario, cell_chain or default_col out of range */
    GL_E_CUDA = -4,        /* a CUDA runtime call or launch failed */
    GL_E_UNSUPPORTED = -5  /* current device is not sm_100 (B200) */
};

/* Disg-Pref-Decode / Disg-Spec-Decode, and the two single-GPU
 * configurations the paper compares against: Standalone (target
 * only) and SpecDecode (draft + target) co-located on the new GPU. */
enum { GL_MODE_DPD = 0, GL_MODE_DSD = 1, GL_MODE_STANDALONE = 2, GL_MODE_SPEC_COLO = 3 };
enum { GL_PRIORITY_SLO = 0, GL_PRIORITY_DEFAULT = 1 }; /* Alg. 1 FallbackStrategy */

/* per-chain status bits, set on the device */
enum {
    GL_ST_UNSORTED = 1u,      /* arrival_us decreases somewhere */
    GL_ST_PROMPT_RANGE = 2u,  /* prompt_len outside [1, max_prompt] */
    GL_ST_OUTPUT_ZERO = 4u,   /* output_len == 0 */
    GL_ST_OVERFLOW = 8u,      /* output_len >= 2^30 */
    GL_ST_NEG_ARRIVAL = 16u,  /* arrival_us < 0 */
    GL_ST_TABLE = 32u         /* t1/t2 < 0, or step_us[b] < 1 for some b in [1, batch_cap] */
};

/* One request trace, structure of arrays, sorted by arrival (R6).
 * Device pointers for gl_eval_grid, host pointers for gl_evaluate_host
 * (pinned memory recommended).  Each array must be 16-byte aligned. */
typedef struct {
    const int64_t *arrival_us;   /* [n] non-decreasing, >= 0 */
    const uint32_t *prompt_len;  /* [n] in [1, max_prompt of every chain using the trace] */
    const uint32_t *output_len;  /* [n] >= 1; counts prefill's first token (R7) */
    int64_t n;                   /* 1 <= n < 2^31 */
} gl_trace;

/* One timing chain = one candidate configuration's timing: (trace, GPU pair,
 * mode, gamma, alpha, batch cap, link).  Table pointers are DEVICE memory and
 * stand in for the profiling database D.  Prompt-indexed tables have
 * max_prompt+1 entries, batch-indexed ones batch_cap+1 entries (index 0 unused).
 *   t1_us[p]      prefill latency of a p-token prompt on the new GPU (stage 1)
 *   e1_new_uj[p]  its energy
 *   t2_us[p]      stage-2 service: DPD KV transfer of p+1 tokens over the link
 *                 (P:50-52); DSD prompt handoff + draft prefill (R12)
 *   b2_old_us[p]  stage-2 busy time of the old GPU; e2_old_uj[p] its energy
 *   step_us[b]    decode iteration (DPD) / speculative step (DSD, Fig. 7) latency
 *                 at batch size b; step_busy_{new,old}_us[b], step_e_{new,old}_uj[b]
 *                 the per-GPU busy time and energy of that iteration
 * Co-located modes (STANDALONE, SPEC_COLO; R41-R44): one GPU runs prefills
 * (t1_us, e1_new_uj) and decode iterations / speculative steps (step_*) one at a
 * time, prefill first: at every iteration boundary each arrived request is
 * admitted FCFS while the batch has room, its prefill runs alone (first token at
 * its end), and it then joins the batch if o > 1.  t2_us, b2_old_us, e2_old_uj
 * are not used; old-GPU step tables are added as given (normally zero).
 * DSD / SPEC_COLO acceptance: thr_c = floor(alpha^c * 2^32) (alpha^c by repeated products),
 * accepted tokens per member-step = 1 + #{c in 1..gamma : u < thr_c}, u = word
 * (s mod 4) of Philox4x32-10(counter (s/4, j, 0x41434350, 0), key = seed) for
 * request j's own step s (R22; rejection rule P:111-114 as a marginal rate). */
typedef struct {
    int32_t mode;          /* GL_MODE_DPD, _DSD, _STANDALONE or _SPEC_COLO */
    int32_t trace_idx;     /* index into the traces array */
    int32_t batch_cap;     /* [1, GL_MAX_CAP] */
    int32_t gamma;         /* DSD, SPEC_COLO: [1, GL_MAX_GAMMA]; ignored otherwise */
    int32_t max_prompt;    /* [1, GL_MAX_PROMPT] */
    int32_t capacity_ok;   /* 0 => excluded from Alg. 1's feasible set (R38), still simulated */
    double alpha;          /* DSD, SPEC_COLO: marginal acceptance rate in [0, 1] */
    uint64_t seed;         /* DSD, SPEC_COLO: Philox key */
    const int32_t *t1_us;
    const int64_t *e1_new_uj;
    const int32_t *t2_us;
    const int32_t *b2_old_us;
    const int64_t *e2_old_uj;
    const int32_t *step_us;
    const int32_t *step_busy_new_us;
    const int32_t *step_busy_old_us;
    const int64_t *step_e_new_uj;
    const int64_t *step_e_old_uj;
    int64_t ttft_slo_us;   /* Table 2 TTFT SLO, >= 0 */
    int64_t tpot_slo_us;   /* Table 2 TPOT SLO, >= 0 */
    double ce_new_g;       /* Table 1 embodied carbon of the new GPU, grams (> 0) */
    double ce_old_g;       /* ... of the old GPU (>= 0; 0 for the co-located modes) */
} gl_chain;

/* Sufficient statistics of one simulated chain (integers => bit-exact). 80 B. */
typedef struct {
    int64_t n;             /* requests */
    int64_t slo_ok;        /* requests meeting TTFT and TPOT SLOs (R27) */
    int64_t tokens;        /* sum of output_len */
    int64_t busy_new_us;   /* new-GPU busy time (Eq. 1's t, R31) */
    int64_t busy_old_us;
    int64_t e_new_uj;      /* new-GPU energy (Eq. 2's E, R32) */
    int64_t e_old_uj;
    int64_t makespan_us;   /* max finish time */
    uint64_t req_hash;     /* sum_j mix64(j, ttft_j, finish_j) mod 2^64 */
    uint32_t status;       /* GL_ST_* bits */
    uint32_t capacity_ok;  /* copied from the chain */
} gl_chain_stats;

/* One carbon scenario (a row's CI and lifetimes; changes only carbon). */
typedef struct {
    double ci_g_per_kwh;   /* >= 0, finite */
    double lt_new_s;       /* > 0 */
    double lt_old_s;       /* > 0 */
} gl_scenario;

/* Alg. 1 matrices (Fig. 8): rows = workloads/scenarios, cols =
 * candidate configurations.  HOST arrays. */
typedef struct {
    int32_t rows, cols;           /* >= 1 */
    const int32_t *row_scenario;  /* [rows] index into the scenarios */
    const int32_t *cell_chain;    /* [rows*cols] chain scored in that cell, -1 = absent */
} gl_grid;

/*
 * Simulate every timing chain on its trace (stages 1-2 as max-plus scans,
 * continuous-batching decode as a per-warp event loop) and write one
 * gl_chain_stats per chain.
 *   traces, chains   HOST descriptor arrays; their data pointers are DEVICE
 *   stats_out        DEVICE [n_chains]
 *   per_request_out  DEVICE int64 [sum over chains of n(trace)][2] = (ttft_us,
 *                    finish_us), chain-major in chain order; NULL to skip
 */
gl_status gl_eval_grid(const gl_trace *traces, int32_t n_traces, const gl_chain *chains,
                       int32_t n_chains, gl_chain_stats *stats_out, int64_t *per_request_out,
                       void *stream);

/*
 * Launch-order hint.  The step lasts as long as its slowest chain's serial decode
 * walk, and that walk can only start once the chain's DSD demand and
 * stage scans exist.  With a hint, the chains [first_lo, first_hi) -- e.g. the
 * trace predicted to hold the slowest chain -- run first: their DSD demand, stage
 * scans (and those of the primaries they copy from) and segment starts, then their
 * decode on a side stream forked from `stream`, while the other chains' prologue
 * kernels and decodes follow on `stream` (and a second side stream); both are
 * joined back before the per-request SLO pass, so the call stays ordered on
 * `stream`.  Results never depend on the hint (outputs are bit-identical with or
 * without it).  Ignored when the call holds co-located chains, for gl_link_demand,
 * and for an empty or full range.
 *   first_lo, first_hi   0 <= first_lo <= first_hi <= n_chains, else GL_E_INVALID
 */
typedef struct {
    int32_t first_lo, first_hi;
} gl_schedule;

/* gl_eval_grid with an optional launch-order hint (NULL: as gl_eval_grid). */
gl_status gl_eval_grid_sched(const gl_trace *traces, int32_t n_traces, const gl_chain *chains,
                             int32_t n_chains, gl_chain_stats *stats_out,
                             int64_t *per_request_out, const gl_schedule *sched, void *stream);

/*
 * Alg. 1 on the carbon matrix of Eqs. 1-3:
 *   total = ((e_new/3.6e12) + (e_old/3.6e12)) * CI
 *         + ((busy_new/1e6)/LT_new)*Ce_new + ((busy_old/1e6)/LT_old)*Ce_old
 * (fixed order, no contraction: R34).  A cell is feasible iff capacity_ok and
 * slo_den*slo_ok >= slo_num*n (SLO_att >= SLO_target).  Per row: argmin
 * total over feasible cells, ties -> higher attainment -> lower column; if none
 * is feasible via_fallback = 1 and: priority SLO -> argmax attainment (capacity-
 * infeasible cells count as 0 and +inf), ties -> lower total -> lower column,
 * -1 if the row has no present cell; priority DEFAULT -> default_col.
 * A chain with status bits (invalid input) is never feasible and counts like a
 * capacity-infeasible one (R55).
 *   stats            DEVICE [n_chains] (all chains, e.g. after an allgather)
 *   chains           HOST [n_chains] (ce_new_g, ce_old_g, capacity_ok are read)
 *   scen             HOST [n_scen];  grid: HOST arrays
 *   carbon_out       DEVICE double [rows*cols] (absent cells: NaN) or NULL
 *   carbon_per_token_out  DEVICE double [rows*cols] or NULL: the paper's reported
 *                    metric, gCO2 per token (R33) = total / (double)tokens
 *                    (one IEEE division after the total; absent cells NaN).  A
 *                    row's cells share one trace, hence one token count, so the
 *                    argmin over totals is the argmin over per-token carbon.
 *   choice_out       DEVICE int32 [rows];  via_fallback_out DEVICE uint8 [rows]
 */
gl_status gl_argmin_feasible(const gl_chain_stats *stats, int32_t n_chains,
                             const gl_chain *chains, const gl_scenario *scen, int32_t n_scen,
                             const gl_grid *grid, int32_t slo_num, int32_t slo_den,
                             int32_t priority, int32_t default_col, double *carbon_out,
                             double *carbon_per_token_out, int32_t *choice_out,
                             uint8_t *via_fallback_out, void *stream);

/*
 * End to end from host buffers: copies the traces host->device (each distinct
 * host array once -- traces sharing an array share its device copy; the arrival
 * arrays on a side stream forked from `stream`, overlapping the DSD demand
 * kernel), runs gl_eval_grid and gl_argmin_feasible, copies the results
 * device->host and synchronises `stream` before returning.  Host arrays should
 * be pinned for the copies to be asynchronous.
 *   host_traces      HOST descriptors with HOST data pointers
 *   chains           as for gl_eval_grid (tables stay in DEVICE memory)
 *   stats_host       HOST [n_chains];  carbon_host HOST [rows*cols] or NULL
 *   carbon_per_token_host  HOST [rows*cols] or NULL (as gl_argmin_feasible's)
 *   choice_host      HOST [rows];      via_fallback_host HOST [rows]
 */
gl_status gl_evaluate_host(const gl_trace *host_traces, int32_t n_traces,
                           const gl_chain *chains, int32_t n_chains, const gl_scenario *scen,
                           int32_t n_scen, const gl_grid *grid, int32_t slo_num,
                           int32_t slo_den, int32_t priority, int32_t default_col,
                           gl_chain_stats *stats_host, double *carbon_host,
                           double *carbon_per_token_host, int32_t *choice_host,
                           uint8_t *via_fallback_host, void *stream);

/* gl_evaluate_host with an optional launch-order hint (as gl_eval_grid_sched). */
gl_status gl_evaluate_host_sched(const gl_trace *host_traces, int32_t n_traces,
                                 const gl_chain *chains, int32_t n_chains,
                                 const gl_scenario *scen, int32_t n_scen, const gl_grid *grid,
                                 int32_t slo_num, int32_t slo_den, int32_t priority,
                                 int32_t default_col, gl_chain_stats *stats_host,
                                 double *carbon_host, double *carbon_per_token_host,
                                 int32_t *choice_host, uint8_t *via_fallback_host,
                                 const gl_schedule *sched, void *stream);

/* ---- Link bandwidth demand (Fig. 4, "bandwidth
 * requirement"; "peak bandwidth demand over a 1 s sliding window").
 * Readings R45-R47: every payload the timing model puts on the
 * GPU-GPU link is an impulse of bytes at its ISSUE time --
 *   a request with o > 1: bytes_per_token * (p + 1) at its prefill completion
 *     c = a + TTFT (DPD: its KV cache, R11; DSD: its prompt IDs, R12);
 *   a decode iteration at batch b: b * bytes_per_member_step at its start (DSD:
 *     draft IDs, probabilities and accepted IDs of every member, R21; DPD: 0).
 * demand(t) = bytes issued in [t, t + window_us); peak = max over t (attained at
 * an impulse time); peak_t_us = the earliest impulse time attaining it.  The
 * co-located modes have no link: all zero, peak_t_us = -1. */
typedef struct {
    int64_t bytes_per_token;        /* >= 0 */
    int64_t bytes_per_member_step;  /* >= 0 */
} gl_link_params;

typedef struct {
    int64_t total_bytes;   /* all payload bytes (SPEC S:372's bandwidth accounting) */
    int64_t peak_bytes;    /* max bytes issued in one window (x 8 / window = peak bits/s) */
    int64_t peak_t_us;     /* earliest impulse time whose window attains the peak, -1 if none */
    int64_t n_impulses;    /* payloads with a positive size */
} gl_link_stats;           /* 32 B */

/*
 * Simulate every chain exactly as gl_eval_grid does (recording the decode
 * batch-size changes of every run) and compute its link demand.  Stream-ordered
 * like gl_eval_grid.
 *   traces, chains   as for gl_eval_grid (HOST descriptors, DEVICE data)
 *   params           HOST [n_chains] payload sizes
 *   window_us        >= 1 (1,000,000 = SPEC's 1 s window)
 *   stats_out        DEVICE [n_chains] or NULL (the same statistics gl_eval_grid writes)
 *   link_out         DEVICE [n_chains]
 * Errors: as gl_eval_grid; GL_E_INVALID for window_us < 1 or a NULL params /
 * link_out, GL_E_DOMAIN for a negative payload size.
 */
gl_status gl_link_demand(const gl_trace *traces, int32_t n_traces, const gl_chain *chains,
                         int32_t n_chains, const gl_link_params *params, int64_t window_us,
                         gl_chain_stats *stats_out, gl_link_stats *link_out, void *stream);

/* ---- §5 carbon-efficiency analysis surfaces.
 * Case 1 (Standalone): the service on the new GPU A alone; Case 2
 * (disaggregation): the same trace on A and an old GPU B (or any other
 * candidate chain).  Per (pair, scenario), with Case totals from Eqs. 1-3 in the
 * fixed R34 order (bit-identical to gl_argmin_feasible's carbon):
 *   ratio       Eq. 5 first line (O_A' + E_A' + O_B + E_B) / (O_A + E_A);
 *               carbon savings = 1 - ratio
 *   op_saved_g  O_A - (O_A' + O_B);  emb_saved_g  E_A - (E_A' + E_B)  (grams)
 *   eq6_term    (t_B/T_B * B) / (N_A * alpha + (t_A'/T_A) * A), Eq. 6's variable
 *               term exactly as printed (R49: an approximation; never decisive)
 *   eq4_energy_less  1 iff N_A > N_A' + N_B (Eq. 4, integer energies) */
typedef struct {
    int32_t disagg_chain;      /* Case 2 chain index */
    int32_t standalone_chain;  /* Case 1 chain index */
} gl_savings_pair;

typedef struct {
    double ratio, op_saved_g, emb_saved_g, eq6_term;
    int32_t eq4_energy_less, pad;
} gl_savings;              /* 40 B */

/*
 *   stats      DEVICE [n_chains] (e.g. from gl_eval_grid)
 *   chains     HOST [n_chains] (ce_new_g, ce_old_g are read)
 *   pairs      HOST [n_pairs];  scen HOST [n_scen]
 *   out        DEVICE [n_pairs * n_scen], pair-major (out[p * n_scen + s])
 * Errors: GL_E_INVALID for NULL / non-positive counts, GL_E_LOOKUP for a chain
 * index out of range, GL_E_DOMAIN as gl_argmin_feasible for scenarios and Ce.
 */
gl_status gl_savings_surface(const gl_chain_stats *stats, int32_t n_chains,
                             const gl_chain *chains, const gl_savings_pair *pairs,
                             int32_t n_pairs, const gl_scenario *scen, int32_t n_scen,
                             gl_savings *out, void *stream);

/* ---- Collaborative filtering (Alg. 1 line 1, P:309;
 * missing entries of C and SLO_att are filled "only once after
 * profiling").  The paper names no algorithm; this is alternating least squares
 * with ridge regularisation (readings R50-R53):
 *   each of `iters` iterations: for every row i,
 *     U_i = (sum_{j observed} V_j V_j^T + lambda I)^-1 sum_j x_ij V_j,
 *   then for every column j the same with U and V swapped; k x k Cholesky solves.
 *   out_ij = x_ij where observed (verbatim), else clamp(U_i . V_j, lo, hi).
 * The matrices of a batch are independent (SPEC completes C and SLO_att
 * separately); all arrays are row-major fp64 / uint8 in DEVICE memory:
 *   x, observed   [batch][rows][cols]     (observed != 0 marks a known entry)
 *   v0            [batch][cols][rank]     initial V (seeded input, R51)
 *   out           [batch][rows][cols]
 *   u_out, v_out  [batch][rows][rank], [batch][cols][rank] final factors, or NULL
 *   status_out    [batch] int32: bit 1 = a row without an observed entry, bit 2 =
 *                 a column without one (the completion is then undefined)
 * Limits: 1 <= rank <= GL_MAX_RANK, rank <= min(rows, cols), cols <= 1024,
 * lambda >= 0 finite, iters >= 0, lo <= hi.  Results match the CPU oracle to
 * rounding (the V-step sums rows in a parallel order; R50). */
#define GL_MAX_RANK 8
gl_status gl_complete_matrices(const double *x, const uint8_t *observed, int32_t batch,
                               int32_t rows, int32_t cols, int32_t rank, double lambda,
                               int32_t iters, const double *v0, double lo, double hi,
                               double *out, double *u_out, double *v_out, int32_t *status_out,
                               void *stream);

/*
 * Alg. 1 lines 2-9 on explicit matrices -- C and SLO_att as the paper
 * states them, e.g. after gl_complete_matrices filled the unmeasured cells
 * (line 1).  Attainments are fractions (R54): a cell is feasible iff present and
 * att >= slo_target; per row argmin carbon, ties -> higher att -> lower column;
 * nothing feasible -> via_fallback = 1 and priority SLO -> argmax att (ties ->
 * lower carbon -> lower column; -1 if no present cell), DEFAULT -> default_col.
 *   carbon, att   DEVICE double [rows*cols] row-major; present DEVICE uint8 or NULL
 *   choice_out    DEVICE int32 [rows];  via_fallback_out DEVICE uint8 [rows]
 * Errors: GL_E_INVALID (NULL, rows/cols <= 0, bad priority), GL_E_DOMAIN (target
 * not in [0, 1] or non-finite), GL_E_LOOKUP (default_col out of range).
 */
gl_status gl_argmin_matrices(const double *carbon, const double *att, const uint8_t *present,
                             int32_t rows, int32_t cols, double slo_target, int32_t priority,
                             int32_t default_col, int32_t *choice_out, uint8_t *via_fallback_out,
                             void *stream);

/* Number of CUDA kernels the last successful call on this thread enqueued. */
int32_t gl_last_launch_count(void);

/* Benchmark instrumentation (per calling thread).  When enabled (on != 0),
 * gl_eval_grid and gl_argmin_feasible record CUDA events on `stream` around
 * every kernel they enqueue.  After the stream is synchronised,
 * gl_kernel_times writes up to `max` (name, milliseconds) pairs of the
 * kernels enqueued since the previous gl_kernel_times call and returns how
 * many it wrote (names are static strings).  Disabled by default. */
gl_status gl_profile_enable(int32_t on);
int32_t gl_kernel_times(const char **names_out, float *ms_out, int32_t max);
/* As gl_kernel_times, plus each kernel's start in milliseconds after the first
 * recorded kernel's (the launches of one call may overlap on several streams). */
int32_t gl_kernel_timeline(const char **names_out, float *start_ms_out, float *ms_out,
                           int32_t max);
const char *gl_strerror(gl_status status);
int32_t gl_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GREENLLM_H */
