/*
 * greenllm_oracle.c -- plain, slow, single-threaded CPU oracle for the
 * batched SLO / carbon evaluation of GreenLLM (arXiv 2412.20322).
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant generator with the CUDA path
 * (paper_2412_20322_b200/csrc), and neither side includes the other.
 *
 * What it computes, literally and in the
 * paper's order:
 *   stage 1  prefill FCFS on the new GPU: c_i = max(c_{i-1}, a_i) + t1[p_i]
 *            (§2.1; TTFT_i = c_i - a_i)
 *   stage 2  FIFO KV link (DPD) or prompt handoff + draft
 *            prefill (DSD): r_i = max(r_{i-1}, c_i) + t2[p_i]
 *   decode   continuous batching stepped ONE ITERATION AT A TIME (no event
 *            jumping, no precomputed demand): every member advances each
 *            iteration; DPD by one token, DSD by 1 + #accepted draft tokens
 *            drawn per member-step from Philox4x32-10 against the acceptance
 *            thresholds floor(alpha^c * 2^32) (rejection rule P:111-114
 *            collapsed to a marginal rate alpha, R22)
 *   SLO      TTFT <= SLO_ttft and (o = 1 or finish - c <= SLO_tpot (o-1))
 *            (Table 2; per-request mean TPOT, R25)
 *   carbon   Eqs. 1-3 with the fixed expression of R34
 *   Alg. 1   feasible set, argmin, fallback
 * and the SURVEY §8(f) NEXT rows:
 *   co-located Standalone / SpecDecode serving (R41-R44)
 *   link bandwidth demand, 1 s sliding-window peak (R45-R47; Fig. 4)
 *   §5 savings analysis per (Case 2, Standalone) pair (R48-R49; Eqs. 4-6)
 *   collaborative filtering by ALS (R50-R53; Alg. 1 line 1)
 * Every rule R1-R53 it follows is listed in DESIGN.md §2.
 *
 * Pins (tests/test_oracle_pins.py): Philox known-answer vectors; the E[acc]
 * closed form (1-alpha^(g+1))/(1-alpha); hand-worked queueing examples
 * (SURVEY Appendix A.1-A.5); an independent 1-us tick brute force on <=10
 * requests and exhaustive tiny enumerations; the max-plus longest-path form of
 * stages 1-2; the cap=1 Lindley recursion; the isolated-request and D/D/1
 * closed forms; carbon closed forms S:55-74; Alg. 1 against brute force;
 * link demand against closed forms, S:372 accounting and the tick brute force
 * scanning every window start (tests/test_oracle_link.py); the savings analysis
 * against S:500 / S:499 and Eq. 5's three lines (tests/test_oracle_savings.py);
 * ALS against numpy's ridge solves and exact rank-1 recovery, Alg. 1 on explicit
 * matrices against SPEC's examples and the integer Alg. 1 (tests/test_oracle_cf.py).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -shared -fPIC (no threads, no SIMD
 * intrinsics).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_ST_UNSORTED 1u
#define OR_ST_PROMPT_RANGE 2u
#define OR_ST_OUTPUT_ZERO 4u
#define OR_ST_OVERFLOW 8u
#define OR_ST_NEG_ARRIVAL 16u

#define OR_ACCEPT_STREAM 0x41434350u /* "ACCP": third Philox counter word */

typedef struct {
    int32_t mode; /* 0 = DPD, 1 = DSD, 2 = Standalone, 3 = SpecDecode (co-located) */
    int32_t cap;
    int32_t gamma;
    int32_t max_prompt;
    double alpha;
    uint64_t seed;
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
    int64_t ttft_slo_us;
    int64_t tpot_slo_us;
} or_chain;

typedef struct {
    int64_t n, slo_ok, tokens, busy_new_us, busy_old_us, e_new_uj, e_old_uj, makespan_us;
    uint64_t req_hash;
    uint32_t status, capacity_ok;
} or_stats;

/* ---------------- Philox4x32-10 (Salmon et al.; own implementation) ------- */
static void or_philox(uint32_t ctr[4], uint32_t k0, uint32_t k1)
{
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * ctr[0];
        uint64_t p1 = (uint64_t)0xCD9E8D57u * ctr[2];
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ ctr[1] ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ ctr[3] ^ k1;
        uint32_t n3 = (uint32_t)p0;
        ctr[0] = n0;
        ctr[1] = n1;
        ctr[2] = n2;
        ctr[3] = n3;
    }
}

void oracle_philox4x32_10(const uint32_t in_ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4])
{
    uint32_t c[4] = {in_ctr[0], in_ctr[1], in_ctr[2], in_ctr[3]};
    or_philox(c, k0, k1);
    memcpy(out, c, sizeof c);
}

/* The acceptance draw of request j at its own step s (R22): word (s mod 4) of
 * Philox(counter = (s/4, j, ACCEPT_STREAM, 0), key = seed). */
static uint32_t or_accept_word(uint64_t seed, uint32_t j, uint32_t s)
{
    uint32_t c[4] = {s / 4u, j, OR_ACCEPT_STREAM, 0u};
    or_philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    return c[s % 4u];
}

/* thr_c = floor(alpha^c * 2^32), alpha^c by left-to-right repeated products */
void oracle_thresholds(double alpha, int32_t gamma, uint64_t *thr)
{
    double x = 1.0;
    for (int c = 1; c <= gamma; ++c) {
        x = x * alpha;
        thr[c - 1] = (uint64_t)floor(x * 4294967296.0);
    }
}

/* accepted tokens of one speculative step: 1 (target's own token) + the
 * number of thresholds the uniform word falls under (R22) */
int32_t oracle_accept_count(uint32_t u, const uint64_t *thr, int32_t gamma)
{
    int32_t acc = 1;
    for (int c = 1; c <= gamma; ++c)
        if ((uint64_t)u < thr[c - 1]) acc += 1;
    return acc;
}

static uint64_t or_rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

/* SplitMix64 finaliser of j ^ rotl(ttft,21) ^ rotl(finish,42) */
uint64_t oracle_mix64(uint64_t j, int64_t ttft, int64_t finish)
{
    uint64_t z = j ^ or_rotl((uint64_t)ttft, 21) ^ or_rotl((uint64_t)finish, 42);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static int64_t or_max(int64_t x, int64_t y) { return x > y ? x : y; }

typedef struct {
    int64_t j;
    int64_t rem;
    uint32_t s;
} or_member;

/* Link impulses of one chain (NEXT #2, R45-R47): payload bytes put on the
 * GPU-GPU link at their issue times.  Two streams, each in time order:
 * per-request stage-2 payloads and per-iteration decode payloads. */
typedef struct {
    int64_t bytes_per_token;       /* request payload = bytes_per_token * (p + 1) */
    int64_t bytes_per_member_step; /* iteration payload = b * bytes_per_member_step */
    int64_t *req_t, *req_w, n_req;
    int64_t *it_t, *it_w, n_it, cap_it;
} or_link;

static void or_link_iter(or_link *lk, int64_t t, int64_t w)
{
    if (!lk || w <= 0) return;
    if (lk->n_it == lk->cap_it) {
        lk->cap_it = lk->cap_it ? 2 * lk->cap_it : 1024;
        lk->it_t = realloc(lk->it_t, sizeof(int64_t) * lk->cap_it);
        lk->it_w = realloc(lk->it_w, sizeof(int64_t) * lk->cap_it);
    }
    lk->it_t[lk->n_it] = t;
    lk->it_w[lk->n_it] = w;
    lk->n_it += 1;
}

/*
 * Simulate one timing chain.  ttft_out / finish_out / ready_out (stage-2
 * completion r_i) may be NULL.  Returns the status bits (0 = valid input).
 * lk (may be NULL) collects the link impulses of the disaggregated modes.
 */
static uint32_t or_simulate(const int64_t *a, const uint32_t *p, const uint32_t *o, int64_t n,
                            const or_chain *ch, or_stats *st, int64_t *ttft_out,
                            int64_t *finish_out, int64_t *ready_out, or_link *lk)
{
    memset(st, 0, sizeof *st);
    st->n = n;
    uint32_t status = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (a[i] < 0) status |= OR_ST_NEG_ARRIVAL;
        if (i > 0 && a[i] < a[i - 1]) status |= OR_ST_UNSORTED;
        if (p[i] < 1 || (int64_t)p[i] > ch->max_prompt) status |= OR_ST_PROMPT_RANGE;
        if (o[i] < 1) status |= OR_ST_OUTPUT_ZERO;
    }
    st->status = status;
    if (status || n <= 0) return status;

    int64_t *c = malloc(sizeof(int64_t) * n);
    int64_t *r = malloc(sizeof(int64_t) * n);
    int64_t *fin = malloc(sizeof(int64_t) * n);
    or_member *A = malloc(sizeof(or_member) * (ch->cap > 0 ? ch->cap : 1));
    uint64_t thr[64];
    if (ch->mode == 1 || ch->mode == 3) oracle_thresholds(ch->alpha, ch->gamma, thr);
    const int colo = ch->mode >= 2;

    if (colo) {
        /* Co-located serving on one GPU: Standalone (target only) and SpecDecode
         * (draft + target).  At every iteration boundary T the
         * scheduler first admits, FCFS, every arrived request (a <= T) while the
         * running batch has room; each admitted prefill runs alone on the GPU
         * (T += t1[p], first token at T) and a request with o > 1 then joins the
         * batch.  Decode iterations run only when no admissible request waits
         * (prefill priority, R41-R44).  Stepped one iteration at a time. */
        int64_t T = 0;
        int32_t size = 0;
        int64_t nxt = 0;
        while (nxt < n || size > 0) {
            while (nxt < n && size < ch->cap && a[nxt] <= T) {
                T += ch->t1_us[p[nxt]];
                st->busy_new_us += ch->t1_us[p[nxt]];
                st->e_new_uj += ch->e1_new_uj[p[nxt]];
                c[nxt] = T;
                r[nxt] = a[nxt];
                fin[nxt] = T;
                if (o[nxt] > 1) {
                    A[size].j = nxt;
                    A[size].rem = (int64_t)o[nxt] - 1;
                    A[size].s = 0;
                    ++size;
                }
                ++nxt;
            }
            if (size == 0) { /* idle until the next arrival */
                if (nxt >= n) break; /* the last admissions were o = 1 requests */
                T = or_max(T, a[nxt]);
                continue;
            }
            int32_t b = size;
            T += ch->step_us[b];
            st->busy_new_us += ch->step_busy_new_us[b];
            st->busy_old_us += ch->step_busy_old_us[b];
            st->e_new_uj += ch->step_e_new_uj[b];
            st->e_old_uj += ch->step_e_old_uj[b];
            for (int32_t m = 0; m < size;) {
                if (ch->mode == 2) {
                    A[m].rem -= 1;
                } else {
                    uint32_t u = or_accept_word(ch->seed, (uint32_t)A[m].j, A[m].s);
                    A[m].rem -= oracle_accept_count(u, thr, ch->gamma);
                    A[m].s += 1;
                }
                if (A[m].rem <= 0) {
                    fin[A[m].j] = T;
                    A[m] = A[size - 1];
                    --size;
                } else {
                    ++m;
                }
            }
        }
        goto slo;
    }

    /* stage 1: prefill FCFS on the new GPU */
    for (int64_t i = 0; i < n; ++i) {
        int64_t start = (i == 0) ? a[i] : or_max(c[i - 1], a[i]);
        c[i] = start + ch->t1_us[p[i]];
        st->busy_new_us += ch->t1_us[p[i]];
        st->e_new_uj += ch->e1_new_uj[p[i]];
    }
    /* stage 2: KV link (DPD) / handoff + draft prefill (DSD); o = 1 skips it */
    for (int64_t i = 0; i < n; ++i) {
        int64_t s2 = (o[i] > 1) ? ch->t2_us[p[i]] : 0;
        int64_t start = (i == 0) ? c[i] : or_max(r[i - 1], c[i]);
        r[i] = start + s2;
        if (o[i] > 1) {
            st->busy_old_us += ch->b2_old_us[p[i]];
            st->e_old_uj += ch->e2_old_uj[p[i]];
            /* R46: the stage-2 payload (DPD: KV of p+1 tokens, R11; DSD: the
             * prompt-ID handoff, R12) is issued when the prefill completes */
            if (lk && lk->bytes_per_token > 0) {
                lk->req_t[lk->n_req] = c[i];
                lk->req_w[lk->n_req] = lk->bytes_per_token * ((int64_t)p[i] + 1);
                lk->n_req += 1;
            }
        }
    }
    /* requests with a single output token finish at prefill completion */
    for (int64_t i = 0; i < n; ++i) fin[i] = c[i];

    /* decode: continuous batching, one iteration per loop pass */
    int64_t T = 0;
    int32_t size = 0;
    int64_t nxt = 0;
    while (nxt < n && o[nxt] <= 1) ++nxt;
    while (nxt < n || size > 0) {
        /* admit FCFS ready requests (r <= T) while there is room */
        while (nxt < n && size < ch->cap && r[nxt] <= T) {
            A[size].j = nxt;
            A[size].rem = (int64_t)o[nxt] - 1;
            A[size].s = 0;
            ++size;
            ++nxt;
            while (nxt < n && o[nxt] <= 1) ++nxt;
        }
        if (size == 0) { /* idle until the next request is ready */
            T = r[nxt];
            continue;
        }
        /* one iteration at batch size b; R47: its link payload (DSD: draft IDs,
         * probabilities and accepted IDs of every member, R21) is issued at its start */
        int32_t b = size;
        if (lk) or_link_iter(lk, T, (int64_t)b * lk->bytes_per_member_step);
        T += ch->step_us[b];
        st->busy_new_us += ch->step_busy_new_us[b];
        st->busy_old_us += ch->step_busy_old_us[b];
        st->e_new_uj += ch->step_e_new_uj[b];
        st->e_old_uj += ch->step_e_old_uj[b];
        for (int32_t m = 0; m < size;) {
            if (ch->mode == 0) {
                A[m].rem -= 1;
            } else {
                uint32_t u = or_accept_word(ch->seed, (uint32_t)A[m].j, A[m].s);
                A[m].rem -= oracle_accept_count(u, thr, ch->gamma);
                A[m].s += 1;
            }
            if (A[m].rem <= 0) {
                fin[A[m].j] = T;
                A[m] = A[size - 1];
                --size;
            } else {
                ++m;
            }
        }
    }

slo:
    /* per-request SLO and chain statistics */
    for (int64_t i = 0; i < n; ++i) {
        int64_t ttft = c[i] - a[i];
        int ok = (ttft <= ch->ttft_slo_us) &&
                 (o[i] == 1 || fin[i] - c[i] <= ch->tpot_slo_us * (int64_t)(o[i] - 1));
        st->slo_ok += ok;
        st->tokens += o[i];
        if (fin[i] > st->makespan_us) st->makespan_us = fin[i];
        st->req_hash += oracle_mix64((uint64_t)i, ttft, fin[i]);
        if (ttft_out) ttft_out[i] = ttft;
        if (finish_out) finish_out[i] = fin[i];
        if (ready_out) ready_out[i] = r[i];
    }
    free(c);
    free(r);
    free(fin);
    free(A);
    return 0;
}

/* Eqs. 1-3 with the fixed expression of R34 (no contraction: -ffp-contract=off) */
void oracle_carbon(const or_stats *st, double ce_new_g, double ce_old_g, double ci,
                   double lt_new_s, double lt_old_s, double out[3])
{
    double kwh_new = (double)st->e_new_uj / 3.6e12;
    double kwh_old = (double)st->e_old_uj / 3.6e12;
    double op = (kwh_new + kwh_old) * ci;
    double emb = ((double)st->busy_new_us / 1e6) / lt_new_s * ce_new_g +
                 ((double)st->busy_old_us / 1e6) / lt_old_s * ce_old_g;
    out[0] = op;
    out[1] = emb;
    out[2] = op + emb;
}

/* Carbon per token (§6 "Carbon Per Token: gCO2 of carbon emission per
 * token"; R33): the chain's Eq. 3 total over the tokens it generated, sum of o_j
 * (every output token, prefill's first included, R7).  0 tokens (a chain whose
 * statistics are void, R55) gives total/0 by IEEE rules. */
double oracle_carbon_per_token(const or_stats *st, double total)
{
    return total / (double)st->tokens;
}

/*
 * §5 carbon-efficiency analysis for one
 * (Case 2 = disaggregated chain d, Case 1 = Standalone chain s) pair under one
 * scenario (carbon intensity alpha = ci, lifetimes T_A = lt_new, T_B = lt_old).
 * Case totals are Eqs. 1-3 with the fixed expression of R34 (oracle_carbon):
 *   out[0] ratio     = (O_A' + E_A' + O_B + E_B) / (O_A + E_A)   (Eq. 5, first line)
 *   out[1] op_saved  = O_A - (O_A' + O_B)      grams (Fig. 9 right / Fig. 14 split)
 *   out[2] emb_saved = E_A - (E_A' + E_B)      grams
 *   out[3] eq6_term  = (t_B/T_B * B) / (N_A * alpha + (t_A'/T_A) * A)   (Eq. 6 as printed,
 *                      R49: its index slip kept -- an approximation, never the decision)
 * and *eq4 = (N_A > N_A' + N_B) on integer energies (Eq. 4 with E read as energy N, G1).
 */
void oracle_savings(const or_stats *d, double ce_new_d, double ce_old_d, const or_stats *s,
                    double ce_new_s, double ce_old_s, double ci, double lt_new_s, double lt_old_s,
                    double out[4], int32_t *eq4)
{
    double cd[3], cs[3];
    oracle_carbon(d, ce_new_d, ce_old_d, ci, lt_new_s, lt_old_s, cd);
    oracle_carbon(s, ce_new_s, ce_old_s, ci, lt_new_s, lt_old_s, cs);
    out[0] = cd[2] / cs[2];
    out[1] = cs[0] - cd[0];
    out[2] = cs[1] - cd[1];
    double n_a = (double)s->e_new_uj / 3.6e12 + (double)s->e_old_uj / 3.6e12;
    double e_b = ((double)d->busy_old_us / 1e6) / lt_old_s * ce_old_d;
    double e_a2 = ((double)d->busy_new_us / 1e6) / lt_new_s * ce_new_d;
    out[3] = e_b / (n_a * ci + e_a2);
    *eq4 = (s->e_new_uj + s->e_old_uj) > (d->e_new_uj + d->e_old_uj);
}

/* attainment comparison by cross-multiplication: sign(ok1/n1 - ok2/n2) */
static int or_cmp_att(int64_t ok1, int64_t n1, int64_t ok2, int64_t n2)
{
    __int128 l = (__int128)ok1 * n2, rr = (__int128)ok2 * n1;
    return (l > rr) - (l < rr);
}

/*
 * Alg. 1 over a rows x cols grid.  present[i] = 0 marks an absent
 * cell.  cap_ok = 0 cells are infeasible and count as ok = 0, total = +inf in
 * the fallback (R37).
 */
void oracle_alg1(int32_t rows, int32_t cols, const uint8_t *present, const double *total,
                 const int64_t *ok, const int64_t *n, const uint8_t *cap_ok, int32_t slo_num,
                 int32_t slo_den, int32_t priority, int32_t default_col, int32_t *choice,
                 uint8_t *via_fallback)
{
    for (int32_t row = 0; row < rows; ++row) {
        int32_t best = -1;
        for (int32_t col = 0; col < cols; ++col) {
            int64_t k = (int64_t)row * cols + col;
            if (!present[k] || !cap_ok[k]) continue;
            if ((__int128)slo_den * ok[k] < (__int128)slo_num * n[k]) continue; /* SLO_att < target */
            if (best < 0) {
                best = col;
                continue;
            }
            int64_t kb = (int64_t)row * cols + best;
            if (total[k] < total[kb] ||
                (total[k] == total[kb] && or_cmp_att(ok[k], n[k], ok[kb], n[kb]) > 0))
                best = col;
        }
        if (best >= 0) {
            choice[row] = best;
            via_fallback[row] = 0;
            continue;
        }
        via_fallback[row] = 1;
        if (priority != 0) {
            choice[row] = default_col;
            continue;
        }
        /* FallbackStrategy, priority = SLO: argmax attainment, then lower total */
        for (int32_t col = 0; col < cols; ++col) {
            int64_t k = (int64_t)row * cols + col;
            if (!present[k]) continue;
            int64_t okk = cap_ok[k] ? ok[k] : 0;
            double tk = cap_ok[k] ? total[k] : INFINITY;
            if (best < 0) {
                best = col;
                continue;
            }
            int64_t kb = (int64_t)row * cols + best;
            int64_t okb = cap_ok[kb] ? ok[kb] : 0;
            double tb = cap_ok[kb] ? total[kb] : INFINITY;
            int cmp = or_cmp_att(okk, n[k], okb, n[kb]);
            if (cmp > 0 || (cmp == 0 && tk < tb)) best = col;
        }
        choice[row] = best;
    }
}

uint32_t oracle_simulate_chain(const int64_t *a, const uint32_t *p, const uint32_t *o, int64_t n,
                               const or_chain *ch, or_stats *st, int64_t *ttft_out,
                               int64_t *finish_out, int64_t *ready_out)
{
    return or_simulate(a, p, o, n, ch, st, ttft_out, finish_out, ready_out, NULL);
}

/*
 * Bandwidth demand of one chain's GPU-GPU link (Fig. 4,
 * P:230-247, "bandwidth requirement"; "peak bandwidth demand over a
 * 1 s sliding window", S:372 bandwidth accounting).  Readings R45-R47
 * (DESIGN.md §2): every payload is an impulse of bytes at its issue time; the
 * demand at t is the bytes issued in the half-open window [t, t + window_us);
 * the peak is its maximum over t, which is attained at an impulse time.
 *   out[0] total bytes, out[1] peak window bytes, out[2] the earliest impulse
 *   time whose window attains the peak (-1 if there is no impulse), out[3] the
 *   number of impulses.
 * Stepped the plain way: the chain is simulated one iteration at a time
 * recording every impulse, the two time-ordered streams are merged, and a
 * two-pointer sweep evaluates the window at every distinct impulse time.
 */
uint32_t oracle_link_demand(const int64_t *a, const uint32_t *p, const uint32_t *o, int64_t n,
                            const or_chain *ch, int64_t bytes_per_token,
                            int64_t bytes_per_member_step, int64_t window_us, or_stats *st,
                            int64_t out[4])
{
    or_link lk;
    memset(&lk, 0, sizeof lk);
    lk.bytes_per_token = bytes_per_token;
    lk.bytes_per_member_step = bytes_per_member_step;
    lk.req_t = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    lk.req_w = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    out[0] = 0;
    out[1] = 0;
    out[2] = -1;
    out[3] = 0;
    /* the co-located modes have no link (R45) */
    uint32_t status = or_simulate(a, p, o, n, ch, st, NULL, NULL, NULL, ch->mode >= 2 ? NULL : &lk);
    if (status == 0) {
        int64_t K = lk.n_req + lk.n_it;
        int64_t *t = malloc(sizeof(int64_t) * (K > 0 ? K : 1));
        int64_t *w = malloc(sizeof(int64_t) * (K > 0 ? K : 1));
        int64_t *pre = malloc(sizeof(int64_t) * (K + 1));
        int64_t x = 0, y = 0;
        for (int64_t k = 0; k < K; ++k) { /* merge of the two time-ordered streams */
            if (y >= lk.n_it || (x < lk.n_req && lk.req_t[x] <= lk.it_t[y])) {
                t[k] = lk.req_t[x];
                w[k] = lk.req_w[x];
                ++x;
            } else {
                t[k] = lk.it_t[y];
                w[k] = lk.it_w[y];
                ++y;
            }
        }
        pre[0] = 0;
        for (int64_t k = 0; k < K; ++k) pre[k + 1] = pre[k] + w[k];
        int64_t hi = 0;
        for (int64_t k = 0; k < K; ++k) {
            if (k > 0 && t[k] == t[k - 1]) continue; /* same window as the group's first */
            while (hi < K && t[hi] < t[k] + window_us) ++hi;
            int64_t v = pre[hi] - pre[k];
            if (v > out[1]) {
                out[1] = v;
                out[2] = t[k];
            }
        }
        out[0] = pre[K];
        out[3] = K;
        free(t);
        free(w);
        free(pre);
    }
    free(lk.req_t);
    free(lk.req_w);
    free(lk.it_t);
    free(lk.it_w);
    return status;
}

/*
 * Collaborative filtering (Alg. 1 line 1; P:343-345:
 * "GreenLLM employs collaborative filtering" to fill the missing entries of C and
 * SLO_att; the algorithm is unspecified -- SPEC S:415-423, S:451 choose alternating
 * least squares).  Readings R50-R53, step by step:
 *   X [rows x cols], observed mask M, rank k, ridge lambda, `iters` iterations,
 *   V [cols x k] initialised from the caller's v0 (seeded input, R51).
 *   each iteration (R50):
 *     U-step: for every row i, U_i = argmin_u sum_{j in M_i} (x_ij - u.V_j)^2 + lambda |u|^2
 *             i.e. (sum_j V_j V_j^T + lambda I) U_i = sum_j x_ij V_j   (columns in order)
 *     V-step: for every column j, the same with the roles swapped (rows in order)
 *   each k x k system is solved by a textbook Cholesky factorisation.
 *   out_ij = x_ij where observed (verbatim), else U_i.V_j clamped to [lo, hi] (R52).
 * Returns bit 1 if some row has no observed entry, bit 2 for a column (R53: the
 * completion is then undefined); out is still written.
 */
static void or_chol_solve(double *A, double *b, int k)
{
    /* A (k x k, SPD, row-major) = L L^T in place (lower), then L y = b, L^T x = y */
    for (int c = 0; c < k; ++c) {
        double d = A[c * k + c];
        for (int m = 0; m < c; ++m) d -= A[c * k + m] * A[c * k + m];
        d = sqrt(d);
        A[c * k + c] = d;
        for (int r = c + 1; r < k; ++r) {
            double v = A[r * k + c];
            for (int m = 0; m < c; ++m) v -= A[r * k + m] * A[c * k + m];
            A[r * k + c] = v / d;
        }
    }
    for (int r = 0; r < k; ++r) {
        double v = b[r];
        for (int m = 0; m < r; ++m) v -= A[r * k + m] * b[m];
        b[r] = v / A[r * k + r];
    }
    for (int r = k - 1; r >= 0; --r) {
        double v = b[r];
        for (int m = r + 1; m < k; ++m) v -= A[m * k + r] * b[m];
        b[r] = v / A[r * k + r];
    }
}

int32_t oracle_als_complete(const double *x, const uint8_t *obs, int32_t rows, int32_t cols,
                            int32_t k, double lambda, int32_t iters, const double *v0,
                            double lo, double hi, double *out, double *u_out, double *v_out)
{
    double *U = calloc((size_t)rows * k, sizeof(double));
    double *V = malloc(sizeof(double) * (size_t)cols * k);
    double A[64], b[8];
    int32_t status = 0;
    memcpy(V, v0, sizeof(double) * (size_t)cols * k);
    for (int32_t i = 0; i < rows; ++i) {
        int any = 0;
        for (int32_t j = 0; j < cols; ++j) any |= obs[(int64_t)i * cols + j] != 0;
        if (!any) status |= 1;
    }
    for (int32_t j = 0; j < cols; ++j) {
        int any = 0;
        for (int32_t i = 0; i < rows; ++i) any |= obs[(int64_t)i * cols + j] != 0;
        if (!any) status |= 2;
    }
    for (int32_t it = 0; it < iters; ++it) {
        for (int32_t i = 0; i < rows; ++i) { /* U-step */
            for (int a = 0; a < k * k; ++a) A[a] = 0.0;
            for (int a = 0; a < k; ++a) b[a] = 0.0;
            for (int32_t j = 0; j < cols; ++j) {
                if (!obs[(int64_t)i * cols + j]) continue;
                const double *vj = V + (int64_t)j * k;
                for (int r = 0; r < k; ++r) {
                    for (int c = 0; c <= r; ++c) A[r * k + c] += vj[r] * vj[c];
                    b[r] += x[(int64_t)i * cols + j] * vj[r];
                }
            }
            for (int r = 0; r < k; ++r) A[r * k + r] += lambda;
            or_chol_solve(A, b, k);
            for (int r = 0; r < k; ++r) U[(int64_t)i * k + r] = b[r];
        }
        for (int32_t j = 0; j < cols; ++j) { /* V-step */
            for (int a = 0; a < k * k; ++a) A[a] = 0.0;
            for (int a = 0; a < k; ++a) b[a] = 0.0;
            for (int32_t i = 0; i < rows; ++i) {
                if (!obs[(int64_t)i * cols + j]) continue;
                const double *ui = U + (int64_t)i * k;
                for (int r = 0; r < k; ++r) {
                    for (int c = 0; c <= r; ++c) A[r * k + c] += ui[r] * ui[c];
                    b[r] += x[(int64_t)i * cols + j] * ui[r];
                }
            }
            for (int r = 0; r < k; ++r) A[r * k + r] += lambda;
            or_chol_solve(A, b, k);
            for (int r = 0; r < k; ++r) V[(int64_t)j * k + r] = b[r];
        }
    }
    for (int32_t i = 0; i < rows; ++i) {
        for (int32_t j = 0; j < cols; ++j) {
            int64_t q = (int64_t)i * cols + j;
            if (obs[q]) {
                out[q] = x[q];
                continue;
            }
            double v = 0.0;
            for (int r = 0; r < k; ++r) v += U[(int64_t)i * k + r] * V[(int64_t)j * k + r];
            out[q] = v < lo ? lo : (v > hi ? hi : v);
        }
    }
    if (u_out) memcpy(u_out, U, sizeof(double) * (size_t)rows * k);
    if (v_out) memcpy(v_out, V, sizeof(double) * (size_t)cols * k);
    free(U);
    free(V);
    return status;
}

/*
 * Alg. 1 lines 2-9 on explicit matrices C and SLO_att -- e.g. the ones
 * collaborative filtering completed (line 1) -- with fractional attainments (R54):
 * feasible iff present and SLO_att >= target; argmin C, ties -> higher SLO_att ->
 * lower column; nothing feasible -> via_fallback = 1 and priority SLO -> argmax
 * SLO_att (ties -> lower C -> lower column), priority DEFAULT -> default_col; a row
 * without a present cell -> -1 (SLO) .  present may be NULL (all present).
 */
void oracle_alg1_matrices(int32_t rows, int32_t cols, const double *carbon, const double *att,
                          const uint8_t *present, double target, int32_t priority,
                          int32_t default_col, int32_t *choice, uint8_t *via_fallback)
{
    for (int32_t row = 0; row < rows; ++row) {
        int32_t best = -1;
        for (int32_t col = 0; col < cols; ++col) {
            int64_t k = (int64_t)row * cols + col;
            if (present && !present[k]) continue;
            if (!(att[k] >= target)) continue;
            if (best < 0) {
                best = col;
                continue;
            }
            int64_t kb = (int64_t)row * cols + best;
            if (carbon[k] < carbon[kb] || (carbon[k] == carbon[kb] && att[k] > att[kb])) best = col;
        }
        if (best >= 0) {
            choice[row] = best;
            via_fallback[row] = 0;
            continue;
        }
        via_fallback[row] = 1;
        if (priority != 0) {
            choice[row] = default_col;
            continue;
        }
        for (int32_t col = 0; col < cols; ++col) {
            int64_t k = (int64_t)row * cols + col;
            if (present && !present[k]) continue;
            if (best < 0) {
                best = col;
                continue;
            }
            int64_t kb = (int64_t)row * cols + best;
            if (att[k] > att[kb] || (att[k] == att[kb] && carbon[k] < carbon[kb])) best = col;
        }
        choice[row] = best;
    }
}

int32_t oracle_version(void) { return 1; }
