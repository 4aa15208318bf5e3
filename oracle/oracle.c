/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * implementation of EdgeServing's online scheduler (arxiv 2605.05527, §V,
 * Algorithm 1) and of the statistics the paper reports (Eq. 2, P95).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It shares NO code, header,
 * table generator or constant with the CUDA path in paper_2605_05527_b200/.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n,
 * "Qn" = reading n of DESIGN.md §3 (ambiguity register).
 *
 * Arithmetic (reading Q5): the real-valued urgency f(w) = min(exp(w/tau-1), C)
 * (Eq. 3) and the score S = sum f (Eq. 4) are evaluated
 * in fixed point with F = 28 fractional bits:
 *   x_c   = ceil(tau * (1 + ln C))                 clip boundary (Q6)
 *   r     = (1024 - tau mod 1024) mod 1024
 *   A[h]  = floor(2^F * exp((h*1024 - r - tau)/tau))  h = 0 .. (x_c-1+r)>>10
 *   Bt[l] = floor(2^F * exp(l/tau))                 l = 0 .. 1023
 *   G(w)  = (A[(w+r)>>10] * Bt[(w+r)&1023]) >> F    0 <= w < x_c
 *   H(L)  = floor(2^F * exp(L/tau))                 0 <= L < x_c
 *   S_q(m)= C*2^F * K_m + floor(H(L_m) * U_m / 2^F)
 * where, after the hypothetical batch of candidate m (prediction),
 * K_m counts remaining tasks whose predicted wait w+L_m >= x_c and U_m sums
 * G(w) over the others.  Every table entry is the exact floor of a real
 * number; it is computed here with long double expl/logl (64-bit mantissa) and
 * the distance of the real value to the nearest integer is returned so tests
 * can prove the floor is unambiguous (margin >> the expl error bound).
 *
 * Parity pins: see tests/test_oracle_*.py.  The float64 "shadow" score
 * (literal Eq. 3-4 in double) is returned beside the integer score so tests
 * can pin the encoding to the paper's real-valued definition.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_F 28
#define OR_SBITS 10
#define OR_S 1024u

/* status codes (numbers mirror nothing; the Python side maps them) */
enum { OR_OK = 0, OR_ERR_ARG = 1, OR_ERR_PROFILE = 2, OR_ERR_RANGE = 3, OR_ERR_UNSORTED = 4 };

/*
 * Selection policies (numbering = the C ABI's ES_POLICY_*).  EDGESERVING is
 * Algorithm 1.  The others are the paper's baselines (§VI-A) and
 * core-design ablations (§VI-H), with DESIGN.md reading Q26:
 *   ALL_FINAL    longest queue first (LQF), B from Eq. 5, deepest allowed exit
 *   ALL_EARLY    LQF, B from Eq. 5, shallowest allowed exit
 *   EE_LQF       LQF, then Eq. 5 / Eq. 6 for the chosen queue
 *   EE_EDF       least remaining slack tau - w_head (= largest head wait), Eq. 5 / 6
 *   ALLFINAL_DA  Eq. 7 stability-score selection, every candidate at its deepest exit
 *   OURS_BS1     Algorithm 1 with the batch fixed to 1 (bs[0])
 *   SYMPHONY     deferred batching (§VI-A; reading Q27): at the deepest
 *                exit with B of Eq. 5, queue m is triggered when w_head + L >= tau
 *                (one more idle microsecond would miss the SLO) or |Q_m| >= B_max;
 *                the triggered queue with the largest w_head + L is dispatched
 *                (ties lowest m); with none triggered the GPU idles until the
 *                earliest trigger instant or the next arrival, whichever first
 *   GRID         (north star's 1,280 candidates per decision; f2) every admissible
 *                (m, e, b): allowed e, profiled b <= min(|Q_m|, B_max), scored
 *                like Eq. 4 with L(m, e, b) and b served tasks; argmin of the
 *                key (S, m, e, b index); feasible iff w_head + L <= tau
 * LQF / EDF ties go to the lowest model index; those policies score nothing
 * (S = 0).  A fixed exit is feasible iff w_head + L <= tau.
 */
enum { OR_POL_EDGESERVING = 0, OR_POL_ALL_FINAL = 1, OR_POL_ALL_EARLY = 2, OR_POL_EE_LQF = 3,
       OR_POL_EE_EDF = 4, OR_POL_ALLFINAL_DA = 5, OR_POL_OURS_BS1 = 6, OR_POL_SYMPHONY = 7, OR_POL_GRID = 8,
       OR_POL_N = 9 };

/* ------------------------------------------------------------------ tables */

/* distance of a real value to the nearest integer */
static long double frac_dist(long double v) {
  long double f = v - floorl(v);
  return f < 0.5L ? f : 1.0L - f;
}

/* floor(2^F * exp(num/den)) for integers num, den>0, with margin tracking */
static uint64_t fx_exp(long long num, long long den, long double *min_margin) {
  long double q = (long double)num / (long double)den;
  long double v = ldexpl(expl(q), OR_F);
  long double d = frac_dist(v);
  if (num != 0 && d < *min_margin) *min_margin = d; /* num==0 -> exactly 2^F */
  return (uint64_t)floorl(v);
}

/*
 * Build the per-tau tables of reading Q5.  A must hold a_cap entries.
 * Returns OR_ERR_ARG if tau/C are outside the supported range
 * (1024 <= tau <= 2^20 us, 1 <= C <= 15: keeps A, Bt, G in u32).
 */
int or_build_tables(uint32_t tau, uint32_t C, uint64_t *x_c_out, uint32_t *r_out,
                    uint32_t *A, int a_cap, int *nA_out, uint32_t *Bt,
                    double *min_margin_out) {
  if (tau < 1024u || tau > (1u << 20) || C < 1u || C > 15u) return OR_ERR_ARG;
  long double margin = 1.0L;
  /* x_c = ceil(tau (1 + ln C)); C = 1 gives exactly tau (ln 1 = 0) */
  uint64_t x_c;
  if (C == 1u) {
    x_c = tau;
  } else {
    long double y = (long double)tau * (1.0L + logl((long double)C));
    long double d = frac_dist(y);
    if (d < margin) margin = d;
    x_c = (uint64_t)ceill(y);
  }
  uint32_t r = (OR_S - tau % OR_S) % OR_S;
  int nA = (int)(((x_c - 1u) + r) >> OR_SBITS) + 1;
  if (nA > a_cap) return OR_ERR_ARG;
  for (int h = 0; h < nA; ++h) {
    long long num = (long long)h * OR_S - (long long)r - (long long)tau;
    uint64_t v = fx_exp(num, tau, &margin);
    A[h] = (uint32_t)v;
  }
  for (uint32_t l = 0; l < OR_S; ++l) Bt[l] = (uint32_t)fx_exp((long long)l, tau, &margin);
  *x_c_out = x_c;
  *r_out = r;
  *nA_out = nA;
  *min_margin_out = (double)margin;
  return OR_OK;
}

/* H(L) = floor(2^F exp(L/tau)); only defined (and only used) for L < x_c */
uint64_t or_H(uint32_t tau, uint32_t L, double *min_margin_out) {
  long double margin = 1.0L;
  uint64_t v = fx_exp((long long)L, tau, &margin);
  if (min_margin_out) *min_margin_out = (double)margin;
  return v;
}

/* ---------------------------------------------------------- oracle context */

typedef struct {
  /* profile */
  int M, E, nb;
  const int32_t *bs;    /* [nb] strictly increasing, bs[0] == 1 (Q8) */
  const uint32_t *lat;  /* [M][E][nb] microseconds */
  const uint8_t *mask;  /* [M][E] allowed exits, nonzero = allowed */
  const uint16_t *acc;  /* [M][E] top-1 accuracy in basis points (Table I), or NULL */
  /* scheduler config */
  uint32_t tau, C, b_max, warmup;
  uint32_t policy; /* OR_POL_*: Algorithm 1 or one of the paper's baselines / ablations */
  /* derived tables (Q5) */
  uint64_t x_c, C_q;
  uint32_t r;
  int nA;
  uint32_t *A;
  uint32_t Bt[OR_S];
  uint64_t *H; /* [M][E][nb], UINT64_MAX where L >= x_c */
} or_ctx;

static uint32_t LAT(const or_ctx *c, int m, int e, int b) {
  return c->lat[((size_t)m * c->E + e) * c->nb + b];
}

/* G(w) for 0 <= w < x_c (Q5) */
static uint64_t G_of(const or_ctx *c, uint64_t w) {
  uint64_t v = w + c->r;
  uint64_t prod = (uint64_t)c->A[v >> OR_SBITS] * (uint64_t)c->Bt[v & (OR_S - 1u)];
  return prod >> OR_F;
}

/*
 * Profile validation: complete grid (implied by the dense
 * array), latencies > 0, non-decreasing in batch, strictly increasing in exit,
 * bs strictly increasing with bs[0] == 1, every model has an allowed exit.
 * On failure returns OR_ERR_PROFILE and names the offending cell.
 */
int or_validate_profile(int M, int E, int nb, const int32_t *bs, const uint32_t *lat,
                        const uint8_t *mask, int32_t *bad_cell /* [3] m,e,b */) {
  bad_cell[0] = bad_cell[1] = bad_cell[2] = -1;
  if (M < 1 || M > 8 || E < 1 || E > 8 || nb < 1 || nb > 64) return OR_ERR_ARG;
  if (bs[0] != 1) { bad_cell[2] = 0; return OR_ERR_PROFILE; }
  for (int b = 1; b < nb; ++b)
    if (bs[b] <= bs[b - 1] || bs[b] > 65535) { bad_cell[2] = b; return OR_ERR_PROFILE; }
  for (int m = 0; m < M; ++m) {
    int any = 0;
    for (int e = 0; e < E; ++e) any |= mask ? mask[m * E + e] != 0 : 1;
    if (!any) { bad_cell[0] = m; return OR_ERR_PROFILE; }
    for (int e = 0; e < E; ++e)
      for (int b = 0; b < nb; ++b) {
        uint32_t v = lat[((size_t)m * E + e) * nb + b];
        int bad = v == 0u;
        if (b > 0 && v < lat[((size_t)m * E + e) * nb + b - 1]) bad = 1;
        if (e > 0 && v <= lat[((size_t)m * E + e - 1) * nb + b]) bad = 1;
        if (bad) { bad_cell[0] = m; bad_cell[1] = e; bad_cell[2] = b; return OR_ERR_PROFILE; }
      }
  }
  return OR_OK;
}

static int ctx_init(or_ctx *c, int M, int E, int nb, const int32_t *bs, const uint32_t *lat,
                    const uint8_t *mask, uint32_t tau, uint32_t C, uint32_t b_max,
                    uint32_t warmup, uint32_t policy) {
  memset(c, 0, sizeof(*c));
  int32_t bad[3];
  int st = or_validate_profile(M, E, nb, bs, lat, mask, bad);
  if (st) return st;
  if (b_max < 1u || b_max > (uint32_t)bs[nb - 1]) return OR_ERR_ARG;
  if (policy >= OR_POL_N) return OR_ERR_ARG;
  c->M = M; c->E = E; c->nb = nb; c->bs = bs; c->lat = lat; c->mask = mask;
  c->tau = tau; c->C = C; c->b_max = b_max; c->warmup = warmup; c->policy = policy;
  int cap = (int)((((uint64_t)tau * 4u) >> OR_SBITS) + 4);
  c->A = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)cap);
  double mg;
  st = or_build_tables(tau, C, &c->x_c, &c->r, c->A, cap, &c->nA, c->Bt, &mg);
  if (st) { free(c->A); c->A = NULL; return st; }
  c->C_q = (uint64_t)C << OR_F;
  c->H = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)M * E * nb);
  for (int i = 0; i < M * E * nb; ++i)
    c->H[i] = (lat[i] < c->x_c) ? or_H(tau, lat[i], NULL) : UINT64_MAX;
  return OR_OK;
}

static void ctx_free(or_ctx *c) {
  free(c->A);
  free(c->H);
  c->A = NULL;
  c->H = NULL;
}

static int allowed(const or_ctx *c, int m, int e) { return c->mask ? c->mask[m * c->E + e] != 0 : 1; }

/* Eq. 5 with reading Q8: index of the largest profiled batch <= min(len, B_max) */
static int batch_index(const or_ctx *c, uint64_t len) {
  uint64_t cap = len < c->b_max ? len : c->b_max;
  int bi = 0;
  for (int i = 0; i < c->nb; ++i)
    if ((uint64_t)c->bs[i] <= cap) bi = i;
  return bi;
}

/* Eq. 6 by linear search, reading Q2 for the infeasible case */
static int exit_select(const or_ctx *c, int m, int bi, uint64_t w_max, int *feasible) {
  int e_sel = -1;
  for (int e = 0; e < c->E; ++e)
    if (allowed(c, m, e) && w_max + LAT(c, m, e, bi) <= c->tau) e_sel = e; /* deepest wins */
  *feasible = e_sel >= 0;
  if (e_sel < 0)
    for (int e = c->E - 1; e >= 0; --e)
      if (allowed(c, m, e)) e_sel = e; /* shallowest allowed */
  return e_sel;
}

static int n_allowed(const or_ctx *c, int m) {
  int k = 0;
  for (int e = 0; e < c->E; ++e) k += allowed(c, m, e);
  return k;
}

/*
 * The per-candidate score of Algorithm 1 lines 394-398 on a queue snapshot.
 * waits[m][i], i = 0 (head, oldest) .. len[m]-1.  Candidate m serves the B
 * oldest tasks of Q_m (removed); every other task's wait grows
 * by L; future arrivals are excluded.
 */
typedef struct {
  int e, B, bi, feasible;
  uint32_t L;
  uint64_t S_q;
  double S_dbl;
} or_cand;

static int deepest_allowed(const or_ctx *c, int m) {
  for (int e = c->E - 1; e >= 0; --e)
    if (allowed(c, m, e)) return e;
  return 0;
}

static int shallowest_allowed(const or_ctx *c, int m) {
  for (int e = 0; e < c->E; ++e)
    if (allowed(c, m, e)) return e;
  return 0;
}

static int uses_score(const or_ctx *c) {
  return c->policy == OR_POL_EDGESERVING || c->policy == OR_POL_ALLFINAL_DA || c->policy == OR_POL_OURS_BS1 ||
         c->policy == OR_POL_GRID;
}

/* a3 + a4 of candidate m under the cfg's policy: batch (Eq. 5, or 1 for
   OURS_BS1) and exit (Eq. 6, or the policy's fixed exit) */
static void cand_params(const or_ctx *c, int m, uint64_t len, uint64_t w_max, or_cand *out) {
  int bi = c->policy == OR_POL_OURS_BS1 ? 0 : batch_index(c, len);
  int e, feasible;
  if (c->policy == OR_POL_ALL_FINAL || c->policy == OR_POL_ALLFINAL_DA || c->policy == OR_POL_ALL_EARLY ||
      c->policy == OR_POL_SYMPHONY) {
    e = c->policy == OR_POL_ALL_EARLY ? shallowest_allowed(c, m) : deepest_allowed(c, m);
    feasible = w_max + LAT(c, m, e, bi) <= c->tau;
  } else {
    e = exit_select(c, m, bi, w_max, &feasible);
  }
  out->e = e; out->B = c->bs[bi]; out->bi = bi; out->feasible = feasible; out->L = LAT(c, m, e, bi);
  out->S_q = 0; out->S_dbl = 0.0;
}

/* Eq. 4 on the predicted state of serving b = bs[bi] tasks of Q_m at exit e */
static void score_at(const or_ctx *c, int m, int e, int bi, const uint64_t *len, const uint32_t *const *waits,
                     or_cand *out) {
  int B = c->bs[bi];
  uint32_t L = LAT(c, m, e, bi);
  out->e = e; out->bi = bi; out->B = B; out->L = L;
  out->feasible = (uint64_t)waits[m][0] + L <= c->tau;
  uint64_t K = 0;
  unsigned __int128 U = 0;
  double S_dbl = 0.0;
  for (int m2 = 0; m2 < c->M; ++m2) {
    uint64_t start = (m2 == m) ? (uint64_t)B : 0u;
    for (uint64_t i = start; i < len[m2]; ++i) {
      uint64_t w = waits[m2][i];
      if (w + L >= c->x_c) K++;
      else U += G_of(c, w);
      /* shadow: literal Eq. 3 on the predicted wait, float64 */
      double f = exp((double)(w + L) / (double)c->tau - 1.0);
      S_dbl += f < (double)c->C ? f : (double)c->C;
    }
  }
  uint64_t S = c->C_q * K;
  if (L < c->x_c) {
    unsigned __int128 HU = (unsigned __int128)c->H[((size_t)m * c->E + e) * c->nb + bi] * U;
    S += (uint64_t)(HU >> OR_F);
  }
  out->S_q = S; out->S_dbl = S_dbl;
}

static void score_candidate(const or_ctx *c, int m, const uint64_t *len,
                            const uint32_t *const *waits, or_cand *out) {
  cand_params(c, m, len[m], waits[m][0], out);
  int feasible = out->feasible;
  score_at(c, m, out->e, out->bi, len, waits, out);
  out->feasible = feasible; /* Eq. 6's flag (Q2) */
}

/*
 * decide() on one snapshot (Algorithm 1; Eq. 7 argmin with
 * tie-break lowest model index, Q3; or the cfg's baseline policy, Q26).
 * Returns the chosen model or -1 when every queue is empty (no-work signal,
 * S:233).  *n_cand = non-empty queues.
 */
static int decide(const or_ctx *c, const uint64_t *len, const uint32_t *const *waits,
                  or_cand *cands /* [M] */, int *n_cand) {
  int best = -1;
  *n_cand = 0;
  if (c->policy == OR_POL_GRID) {
    /* every admissible (m, e, b), in (m, e, b) order: strict < keeps the
       lowest (m, e, b index) on equal scores */
    or_cand x;
    for (int m = 0; m < c->M; ++m) {
      if (len[m] == 0) continue;
      int have = 0; /* cands[m] = model m's best cell */
      uint64_t cap = len[m] < c->b_max ? len[m] : c->b_max;
      for (int e = 0; e < c->E; ++e) {
        if (!allowed(c, m, e)) continue;
        for (int bi = 0; bi < c->nb && (uint64_t)c->bs[bi] <= cap; ++bi) {
          score_at(c, m, e, bi, len, waits, &x);
          (*n_cand)++;
          if (!have || x.S_q < cands[m].S_q) { cands[m] = x; have = 1; }
        }
      }
      if (best < 0 || cands[m].S_q < cands[best].S_q) best = m;
    }
    return best;
  }
  if (uses_score(c)) {
    for (int m = 0; m < c->M; ++m) {
      if (len[m] == 0) continue;
      score_candidate(c, m, len, waits, &cands[m]);
      (*n_cand)++;
      if (best < 0 || cands[m].S_q < cands[best].S_q) best = m;
    }
    return best;
  }
  /* LQF: most queued tasks; EDF: least slack tau - w_head, i.e. the largest
     head wait; strict > keeps the lowest model index on ties */
  for (int m = 0; m < c->M; ++m) {
    if (len[m] == 0) continue;
    (*n_cand)++;
    if (best < 0) { best = m; continue; }
    if (c->policy == OR_POL_EE_EDF ? waits[m][0] > waits[best][0] : len[m] > len[best]) best = m;
  }
  if (best >= 0) cand_params(c, best, len[best], waits[best][0], &cands[best]);
  return best;
}

/*
 * Snapshot decisions (the K1 contract): n snapshots, CSR q_off[n*M+1] into
 * waits (head first, non-increasing per queue, Q7).  Per snapshot outputs
 * m,e,B,L,S_q,flags (bit0 feasible, bit1 no_work, bit2 bad_input),
 * cand_S[n*M] (UINT64_MAX for empty queues), shadow cand_dbl[n*M] (NaN empty).
 */
int or_decide_batch(int M, int E, int nb, const int32_t *bs, const uint32_t *lat,
                    const uint8_t *mask, const uint32_t *tau, const uint32_t *C,
                    const uint32_t *b_max, const uint32_t *policy, int ncfg, int64_t n,
                    const uint16_t *cfg_idx,
                    const uint64_t *q_off, const uint32_t *waits, uint8_t *o_m, uint8_t *o_e,
                    uint16_t *o_B, uint32_t *o_L, uint64_t *o_S, uint8_t *o_flags,
                    uint64_t *o_cand, double *o_cand_dbl) {
  or_ctx *ctx = (or_ctx *)calloc((size_t)ncfg, sizeof(or_ctx));
  for (int k = 0; k < ncfg; ++k) {
    int st = ctx_init(&ctx[k], M, E, nb, bs, lat, mask, tau[k], C[k], b_max[k], 0, policy ? policy[k] : 0u);
    if (st) {
      for (int j = 0; j < k; ++j) ctx_free(&ctx[j]);
      free(ctx);
      return st;
    }
  }
  uint64_t len[8];
  const uint32_t *wp[8];
  or_cand cands[8];
  for (int64_t s = 0; s < n; ++s) {
    int k = cfg_idx ? cfg_idx[s] : 0;
    o_m[s] = 0; o_e[s] = 0; o_B[s] = 0; o_L[s] = 0; o_S[s] = 0; o_flags[s] = 0;
    for (int m = 0; m < M; ++m) {
      if (o_cand) o_cand[s * M + m] = UINT64_MAX;
      if (o_cand_dbl) o_cand_dbl[s * M + m] = NAN;
    }
    if (k >= ncfg) { o_flags[s] = 4; continue; }
    const or_ctx *c = &ctx[k];
    if (c->policy == OR_POL_SYMPHONY) { o_flags[s] = 4; continue; } /* replay-only policy (timer instants) */
    int bad = 0;
    for (int m = 0; m < M; ++m) {
      uint64_t lo = q_off[s * M + m], hi = q_off[s * M + m + 1];
      len[m] = hi - lo;
      wp[m] = waits + lo;
      for (uint64_t i = 1; i < len[m]; ++i)
        if (wp[m][i] > wp[m][i - 1]) bad = 1;
    }
    if (bad) { o_flags[s] = 4; continue; }
    int nc;
    int best = decide(c, len, wp, cands, &nc);
    if (best < 0) { o_flags[s] = 2; continue; }
    o_m[s] = (uint8_t)best;
    o_e[s] = (uint8_t)cands[best].e;
    o_B[s] = (uint16_t)cands[best].B;
    o_L[s] = cands[best].L;
    o_S[s] = cands[best].S_q;
    o_flags[s] = (uint8_t)(cands[best].feasible ? 1 : 0);
    for (int m = 0; m < M; ++m)
      if (len[m] && uses_score(c)) { /* LQF / EDF policies score nothing */
        if (o_cand) o_cand[s * M + m] = cands[m].S_q;
        if (o_cand_dbl) o_cand_dbl[s * M + m] = cands[m].S_dbl;
      }
  }
  for (int k = 0; k < ncfg; ++k) ctx_free(&ctx[k]);
  free(ctx);
  return OR_OK;
}

/* ---------------------------------------------------------------- replay */

/* per-scenario statistics columns (same meaning as the library's, own enum) */
enum {
  ST_DECISIONS = 0, ST_CANDIDATES, ST_CELLS, ST_COMPLETED, ST_VIOLATIONS,
  ST_INFEASIBLE, ST_MAX_DEPTH, ST_STATUS, ST_SUM_LAT, ST_LIVE, ST_TERMS,
  ST_ACC_BP, /* accuracy (basis points) of the served exit, summed over post-warmup tasks */
  ST_EXIT0,  /* ST_EXIT0 + e: post-warmup tasks served at exit e (Fig. exit_depth) */
  ST_NCOL = ST_EXIT0 + 8
};

static int cmp_u32(const void *a, const void *b) {
  uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
  return (x > y) - (x < y);
}

/* Nearest-rank P95 (Q15): the ceil(0.95 N)-th smallest. */
uint32_t or_p95(const uint32_t *v, int64_t n) {
  if (n <= 0) return 0;
  uint32_t *tmp = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n);
  memcpy(tmp, v, sizeof(uint32_t) * (size_t)n);
  qsort(tmp, (size_t)n, sizeof(uint32_t), cmp_u32);
  int64_t k = (95 * n + 99) / 100; /* ceil(0.95 n) */
  uint32_t out = tmp[k - 1];
  free(tmp);
  return out;
}

/*
 * Whole-trace replay of one scenario (P:161-167 online loop; Q10-Q14).
 * a[m] = arrivals of model m (sorted, u32 us).  Outputs (each optional):
 * completion[m][i], exit[m][i] aligned with a; lat[seq] = total latency T in
 * dispatch order (Eq. 1); dec_* = first dec_cap decisions.
 */
static int replay_one(const or_ctx *c, const uint64_t *n, const uint32_t *const *a,
                      uint32_t *const *completion, uint8_t *const *exit_used, uint32_t *lat,
                      uint64_t *stats, uint32_t *p95, int64_t dec_cap, uint32_t *dec_t,
                      uint8_t *dec_m, uint8_t *dec_e, uint16_t *dec_B, uint32_t *dec_L,
                      uint64_t *dec_S, uint8_t *dec_f) {
  const int M = c->M;
  uint64_t head[8] = {0}, tail[8] = {0}, total = 0, served = 0, seq = 0;
  for (int k = 0; k < ST_NCOL; ++k) stats[k] = 0;
  *p95 = 0;
  for (int m = 0; m < M; ++m) {
    total += n[m];
    for (uint64_t i = 1; i < n[m]; ++i)
      if (a[m][i] < a[m][i - 1]) { stats[ST_STATUS] = OR_ERR_UNSORTED; return OR_ERR_UNSORTED; }
  }
  if (total == 0) return OR_OK;
  uint32_t *lat_local = lat ? lat : (uint32_t *)malloc(sizeof(uint32_t) * (size_t)total);
  uint64_t t = UINT64_MAX;
  for (int m = 0; m < M; ++m)
    if (n[m] && a[m][0] < t) t = a[m][0];
  uint64_t len[8];
  uint32_t *wbuf[8];
  for (int m = 0; m < M; ++m) wbuf[m] = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n[m] + 1));
  or_cand cands[8];
  int status = OR_OK;
  while (served < total) {
    /* admission: a decision at t sees every arrival with a <= t (Q10) */
    for (int m = 0; m < M; ++m)
      while (tail[m] < n[m] && a[m][tail[m]] <= t) tail[m]++;
    int any = 0;
    for (int m = 0; m < M; ++m) any |= tail[m] > head[m];
    if (!any) { /* idle GPU: jump to the next arrival (Q12) */
      uint64_t nt = UINT64_MAX;
      for (int m = 0; m < M; ++m)
        if (tail[m] < n[m] && a[m][tail[m]] < nt) nt = a[m][tail[m]];
      t = nt;
      continue;
    }
    /* Algorithm 1: current queuing times */
    for (int m = 0; m < M; ++m) {
      len[m] = tail[m] - head[m];
      if (len[m] > stats[ST_MAX_DEPTH]) stats[ST_MAX_DEPTH] = len[m];
      for (uint64_t i = 0; i < len[m]; ++i) wbuf[m][i] = (uint32_t)(t - a[m][head[m] + i]);
    }
    int nc;
    int best;
    if (c->policy == OR_POL_SYMPHONY) {
      /* deferred batching (Q27): dispatch only a triggered queue, else idle */
      uint64_t wake = UINT64_MAX, best_need = 0;
      best = -1;
      nc = 0;
      for (int m = 0; m < M; ++m) {
        if (len[m] == 0) continue;
        nc++;
        cand_params(c, m, len[m], wbuf[m][0], &cands[m]);
        uint64_t need = (uint64_t)wbuf[m][0] + cands[m].L; /* head latency if started now */
        if (need >= c->tau || len[m] >= c->b_max) {
          if (best < 0 || need > best_need) { best = m; best_need = need; }
        } else if (t + (c->tau - need) < wake) {
          wake = t + (c->tau - need); /* latest start that still meets tau */
        }
      }
      if (best < 0) {
        for (int m = 0; m < M; ++m)
          if (tail[m] < n[m] && a[m][tail[m]] < wake) wake = a[m][tail[m]];
        t = wake; /* idle until the earliest trigger or the next arrival */
        continue;
      }
    } else {
      best = decide(c, len, (const uint32_t *const *)wbuf, cands, &nc);
    }
    const or_cand *d = &cands[best];
    if (t + d->L > 0xFFFFFFFFull) { status = OR_ERR_RANGE; break; }
    uint32_t done = (uint32_t)(t + d->L);
    int64_t k = (int64_t)stats[ST_DECISIONS];
    if (k < dec_cap) {
      if (dec_t) dec_t[k] = (uint32_t)t;
      if (dec_m) dec_m[k] = (uint8_t)best;
      if (dec_e) dec_e[k] = (uint8_t)d->e;
      if (dec_B) dec_B[k] = (uint16_t)d->B;
      if (dec_L) dec_L[k] = d->L;
      if (dec_S) dec_S[k] = d->S_q;
      if (dec_f) dec_f[k] = (uint8_t)d->feasible;
    }
    stats[ST_DECISIONS]++;
    stats[ST_CANDIDATES] += (uint64_t)nc;
    /* work counters: pending tasks not yet clipped at zero prediction (w < x_c)
       and the Eq. 4 terms they generate (one per candidate) */
    uint64_t live = 0;
    for (int m = 0; m < M; ++m)
      for (uint64_t i = 0; i < len[m]; ++i) live += (uint64_t)wbuf[m][i] < c->x_c;
    stats[ST_LIVE] += live;
    if (uses_score(c)) stats[ST_TERMS] += live * (uint64_t)nc; /* Eq. 4 terms: scoring policies only */
    for (int m = 0; m < M; ++m)
      if (len[m]) stats[ST_CELLS] += (uint64_t)n_allowed(c, m);
    if (!d->feasible) stats[ST_INFEASIBLE]++;
    /* commit: exclusive time-division execution of the batch */
    for (int j = 0; j < d->B; ++j) {
      uint64_t i = head[best] + (uint64_t)j;
      if (completion) completion[best][i] = done;
      if (exit_used) exit_used[best][i] = (uint8_t)d->e;
      uint32_t T = done - a[best][i]; /* Eq. 1: T = w + t */
      lat_local[seq] = T;
      if (seq >= c->warmup) { /* Q14: drop the first W completions */
        stats[ST_COMPLETED]++;
        stats[ST_SUM_LAT] += T;
        if (T > c->tau) stats[ST_VIOLATIONS]++; /* Eq. 2, strict (Q16) */
        /* "for each completed task we record the exit point used,
           look up the corresponding per-exit accuracy from Table I" */
        if (c->acc) stats[ST_ACC_BP] += c->acc[best * c->E + d->e];
        stats[ST_EXIT0 + d->e]++;
      }
      seq++;
    }
    head[best] += (uint64_t)d->B;
    served += (uint64_t)d->B;
    t = done; /* next round starts on completion */
  }
  stats[ST_STATUS] = (uint64_t)status;
  if (status == OR_OK && seq > c->warmup) *p95 = or_p95(lat_local + c->warmup, (int64_t)(seq - c->warmup));
  for (int m = 0; m < M; ++m) free(wbuf[m]);
  if (!lat) free(lat_local);
  return status;
}

typedef struct {
  const or_ctx *ctx;
  int ncfg, M, tid, nthreads;
  int64_t n_scen;
  const uint16_t *cfg_idx;
  const uint64_t *arr_off;
  const uint32_t *arrival;
  uint32_t *completion;
  uint8_t *exit_used;
  uint32_t *lat;
  uint64_t *stats;
  uint32_t *p95;
  int64_t dec_cap;
  uint32_t *dec_t;
  uint8_t *dec_m, *dec_e;
  uint16_t *dec_B;
  uint32_t *dec_L;
  uint64_t *dec_S;
  uint8_t *dec_f;
} replay_job;

static void *replay_worker(void *arg) {
  replay_job *j = (replay_job *)arg;
  const int M = j->M;
  for (int64_t s = j->tid; s < j->n_scen; s += j->nthreads) {
    int k = j->cfg_idx ? j->cfg_idx[s] : 0;
    uint64_t *st = j->stats + s * ST_NCOL;
    if (k >= j->ncfg) {
      for (int q = 0; q < ST_NCOL; ++q) st[q] = 0;
      st[ST_STATUS] = OR_ERR_ARG;
      j->p95[s] = 0;
      continue;
    }
    uint64_t n[8];
    const uint32_t *a[8];
    uint32_t *comp[8];
    uint8_t *ex[8];
    uint64_t base = j->arr_off[s * M];
    for (int m = 0; m < M; ++m) {
      uint64_t lo = j->arr_off[s * M + m], hi = j->arr_off[s * M + m + 1];
      n[m] = hi - lo;
      a[m] = j->arrival + lo;
      comp[m] = j->completion ? j->completion + lo : NULL;
      ex[m] = j->exit_used ? j->exit_used + lo : NULL;
    }
    int64_t dc = j->dec_cap;
    int64_t doff = s * dc;
    replay_one(&j->ctx[k], n, a, j->completion ? comp : NULL, j->exit_used ? ex : NULL,
               j->lat ? j->lat + base : NULL, st, &j->p95[s], dc,
               j->dec_t ? j->dec_t + doff : NULL, j->dec_m ? j->dec_m + doff : NULL,
               j->dec_e ? j->dec_e + doff : NULL, j->dec_B ? j->dec_B + doff : NULL,
               j->dec_L ? j->dec_L + doff : NULL, j->dec_S ? j->dec_S + doff : NULL,
               j->dec_f ? j->dec_f + doff : NULL);
  }
  return NULL;
}

/*
 * Replay n_scen scenarios.  arr_off[n_scen*M+1] is the CSR of
 * (scenario, model) segments into arrival.  completion / exit_used are
 * aligned with arrival; lat is in dispatch order within each scenario's
 * segment [arr_off[s*M], arr_off[s*M+M]).  stats[n_scen][ST_NCOL].
 * Scenarios are independent; nthreads > 1 only splits them over threads.
 */
int or_replay_batch(int M, int E, int nb, const int32_t *bs, const uint32_t *lat,
                    const uint8_t *mask, const uint16_t *acc, const uint32_t *tau, const uint32_t *C,
                    const uint32_t *b_max, const uint32_t *warmup, const uint32_t *policy, int ncfg,
                    int64_t n_scen,
                    const uint16_t *cfg_idx, const uint64_t *arr_off, const uint32_t *arrival,
                    uint32_t *completion, uint8_t *exit_used, uint32_t *lat_out,
                    uint64_t *stats, uint32_t *p95, int64_t dec_cap, uint32_t *dec_t,
                    uint8_t *dec_m, uint8_t *dec_e, uint16_t *dec_B, uint32_t *dec_L,
                    uint64_t *dec_S, uint8_t *dec_f, int nthreads) {
  or_ctx *ctx = (or_ctx *)calloc((size_t)ncfg, sizeof(or_ctx));
  for (int k = 0; k < ncfg; ++k) {
    int st = ctx_init(&ctx[k], M, E, nb, bs, lat, mask, tau[k], C[k], b_max[k], warmup[k], policy ? policy[k] : 0u);
    ctx[k].acc = acc;
    if (st) {
      for (int q = 0; q < k; ++q) ctx_free(&ctx[q]);
      free(ctx);
      return st;
    }
  }
  if (nthreads < 1) nthreads = 1;
  replay_job *jobs = (replay_job *)calloc((size_t)nthreads, sizeof(replay_job));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int i = 0; i < nthreads; ++i) {
    replay_job *j = &jobs[i];
    j->ctx = ctx; j->ncfg = ncfg; j->M = M; j->tid = i; j->nthreads = nthreads;
    j->n_scen = n_scen; j->cfg_idx = cfg_idx; j->arr_off = arr_off; j->arrival = arrival;
    j->completion = completion; j->exit_used = exit_used; j->lat = lat_out;
    j->stats = stats; j->p95 = p95; j->dec_cap = dec_cap; j->dec_t = dec_t;
    j->dec_m = dec_m; j->dec_e = dec_e; j->dec_B = dec_B; j->dec_L = dec_L;
    j->dec_S = dec_S; j->dec_f = dec_f;
    if (nthreads > 1) pthread_create(&th[i], NULL, replay_worker, j);
  }
  if (nthreads == 1) replay_worker(&jobs[0]);
  else
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
  free(jobs);
  for (int k = 0; k < ncfg; ++k) ctx_free(&ctx[k]);
  free(ctx);
  return OR_OK;
}
