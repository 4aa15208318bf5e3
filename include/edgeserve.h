/*
 * edgeserve.h -- C ABI of the B200-native EdgeServing stability-score engine.
 *
 * The engine evaluates the online scheduler of EdgeServing (arxiv 2605.05527,
 * PAPER.md §V) batched over many independent scheduling scenarios:
 *   - es_load_profile      the offline profile table L(m, e, B) (P:140-142,
 *                          P:187-196) plus the per-SLO fixed-point
 *                          urgency tables of Eq. 3 (Q5)
 *   - es_score_candidates  one scheduling decision per queue snapshot:
 *                          Algorithm 1 = Eq. 5 batch,
 *                          Eq. 6 exit, queue-status prediction
 *                          (P:347-353), stability score Eq. 3-4,
 *                          Eq. 7 argmin
 *   - es_replay_traces     whole request traces replayed decision by decision
 *                          (online serving loop P:161-167, exclusive
 *                          time-division execution P:152-153), per-scenario
 *                          violations (Eq. 2) and nearest-rank P95
 *   - es_group_*           per-group merge of counters and exact P95 via
 *                          three-level integer histograms (all-reducible)
 *
 * Conventions
 *   - Times are integer microseconds in uint32 relative to the trace start.
 *   - "device" pointers are CUDA global-memory pointers on the profile's
 *     device; "host" pointers are ordinary CPU memory.  All buffers are owned
 *     by the caller unless stated otherwise; the library owns the profile
 *     handle, its device tables and a small scratch pool inside the handle.
 *   - es_stream is a cudaStream_t passed as void* (0 = legacy default
 *     stream).  Device-pointer calls are asynchronous on that stream; host
 *     validation errors are returned synchronously before anything is launched.
 *   - No exception crosses the ABI.  es_last_error() returns a thread-local
 *     message for the last failing call (it names the offending cell / item).
 *   - A handle is immutable after es_load_profile and may be used from several
 *     host threads on different streams, except the es_*_host entry points,
 *     which use the handle's scratch pool and must not run concurrently on the
 *     same handle.
 */
#ifndef EDGESERVE_H
#define EDGESERVE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ES_OK = 0,
  ES_ERR_ARG = 1,              /* null pointer, bad dimension, cfg out of range  */
  ES_ERR_PROFILE_GRID = 2,     /* batch grid: bs[0]!=1, not strictly increasing */
  ES_ERR_PROFILE_MONOTONE = 3, /* L<=0, decreasing in B, not increasing in e     */
  ES_ERR_OUT_OF_GRID = 4,      /* b_max above the largest profiled batch        */
  ES_ERR_RANGE = 5,            /* completion time past 2^32-1 us (Q19)          */
  ES_ERR_CUDA = 6,             /* CUDA runtime error (message has the name)     */
  ES_ERR_OOM = 7,              /* device allocation failed                      */
  ES_ERR_UNSORTED = 8,         /* arrivals not sorted within a (scen, model)    */
  ES_ERR_NUMERIC = 9,          /* a table value too close to an integer to floor */
  ES_ERR_INTERNAL = 10         /* a kernel invariant failed (e.g. replay made no progress) */
} es_status;

#if defined(__GNUC__)
#define ES_API __attribute__((visibility("default")))
#else
#define ES_API
#endif

typedef void *es_stream; /* cudaStream_t */

ES_API const char *es_last_error(void);
ES_API const char *es_version(void);

/* ------------------------------------------------------------------ profile */

#define ES_MAX_MODELS 8  /* M */
#define ES_MAX_EXITS 8   /* E */
#define ES_MAX_BATCHES 64 /* nb */

typedef struct es_profile es_profile; /* opaque, library-owned */

/* The offline profile.  Host pointers, copied. */
typedef struct {
  int32_t M, E, nb;
  const int32_t *batch_sizes; /* host [nb], strictly increasing, [0] == 1, <= 65535 */
  const uint32_t *latency_us; /* host [M][E][nb] row-major, L(m, e, bs[b])         */
  const uint8_t *exit_mask;   /* host [M][E] nonzero = exit allowed, or NULL = all */
  const uint16_t *accuracy_bp; /* host [M][E] top-1 accuracy of (model, exit) in basis
                                  points (0.01 %; Table I), <= 10000, or NULL
                                  (= 0: the accuracy column then stays 0)            */
} es_profile_desc;

/* One scheduler configuration (SLO and knobs).  Bound to the handle at load. */
typedef struct {
  uint32_t tau_us;  /* SLO deadline tau, 1024 <= tau <= 2^20 us          */
  uint32_t clip_C;  /* clip constant C of Eq. 3, 1..15 (C = 10)           */
  uint32_t b_max;   /* B_max of Eq. 5, 1 <= b_max <= bs[nb-1]                    */
  uint32_t warmup;  /* completions dropped from the statistics (100)      */
  uint32_t policy;  /* selection rule, ES_POLICY_* below (Algorithm 1 = 0)          */
} es_sched_cfg;

/*
 * Selection policies.  EDGESERVING is Algorithm 1.  The others
 * are the paper's baselines (§VI-A) and core-design ablations
 * (§VI-H), read as DESIGN.md Q26; they reuse a1-a5 and a8-a10:
 *   ALL_FINAL    longest queue first (LQF; ties lowest m), B* of Eq. 5, deepest allowed exit
 *   ALL_EARLY    LQF, B* of Eq. 5, shallowest allowed exit
 *   EE_LQF       LQF, then Eq. 5 / Eq. 6 for the chosen queue
 *   EE_EDF       least slack tau - w_head (largest head wait; ties lowest m), Eq. 5 / Eq. 6
 *   ALLFINAL_DA  Eq. 7 stability-score selection with every candidate at its deepest exit
 *   OURS_BS1     Algorithm 1 with B* = 1
 *   SYMPHONY     deferred batching (Q27): deepest exit, B* of Eq. 5; a queue is
 *                triggered when w_head + L >= tau or |Q| >= B_max; the triggered queue with the
 *                largest w_head + L is served (ties lowest m); with none triggered the GPU idles
 *                until the earliest trigger instant or the next arrival (not work-conserving)
 *   GRID         every admissible (m, e, b) -- allowed exit, profiled b <= min(|Q_m|, B_max) --
 *                scored like Eq. 4 with L(m, e, b) and b served tasks; argmin of (S, m, e, b
 *                index) (the north star's "1,280 candidates per decision", f2; Q28)
 * A fixed exit is feasible iff w_head + L <= tau.  LQF / EDF policies score
 * nothing: the decision's S is 0 and their candidate scores are UINT64_MAX;
 * under GRID a model's candidate score is its best cell.  Replay
 * (es_replay_traces) accepts every policy; es_score_candidates (K1) every
 * policy but SYMPHONY (ES_ERR_ARG: its "wait until" needs a replay clock).
 */
#define ES_POLICY_EDGESERVING 0u
#define ES_POLICY_ALL_FINAL 1u
#define ES_POLICY_ALL_EARLY 2u
#define ES_POLICY_EE_LQF 3u
#define ES_POLICY_EE_EDF 4u
#define ES_POLICY_ALLFINAL_DA 5u
#define ES_POLICY_OURS_BS1 6u
#define ES_POLICY_SYMPHONY 7u
#define ES_POLICY_GRID 8u
#define ES_POLICY_COUNT 9u

/*
 * Validate the profile (complete grid; L > 0; non-decreasing in batch;
 * strictly increasing in exit; every model has an allowed exit -- S:26-34),
 * validate every cfg, upload it to `device` and build the per-cfg fixed-point
 * urgency tables on the GPU (reading Q5: x_c, r, A, Bt, H).  Synchronous.
 * Errors: ES_ERR_ARG, ES_ERR_PROFILE_GRID, ES_ERR_PROFILE_MONOTONE (the
 * message names (m, e, b)), ES_ERR_OUT_OF_GRID (b_max), ES_ERR_NUMERIC,
 * ES_ERR_CUDA, ES_ERR_OOM.  *out is NULL on failure.  Capacity: the kernels
 * stage the image core (latency tables + per-cfg A / Bt, ~5.4 KB per cfg for
 * tau = 100 ms) in shared memory and read the per-cfg H tables from global
 * memory, so a handle holds as many cfgs as fit ~220 KB of core (about 38 for
 * an 8 x 5 x 32 profile); beyond that ES_ERR_ARG asks to split the cfgs.
 */
ES_API es_status es_load_profile(const es_profile_desc *desc, const es_sched_cfg *cfgs, int32_t ncfg,
                          int32_t device, es_profile **out);
ES_API es_status es_free_profile(es_profile *prof);

/*
 * Copy the profile's device tables to host for inspection (tests compare them
 * bitwise with the oracle's independently built tables).  For cfg k:
 * x_c_out / r_out / nA_out scalars, A_out [>= nA], Bt_out [1024],
 * H_out [M*E*nb] (UINT64_MAX where L >= x_c).  Synchronous.  Any output may
 * be NULL.
 */
ES_API es_status es_get_tables(const es_profile *prof, int32_t k, uint64_t *x_c_out, uint32_t *r_out,
                        int32_t *nA_out, uint32_t *A_out, int32_t A_cap, uint32_t *Bt_out,
                        uint64_t *H_out);

/* ------------------------------------------------- K1: snapshot decisions */

/* n independent queue snapshots (the system state of S:112-115). Device. */
typedef struct {
  int64_t n;
  const uint16_t *cfg_idx;  /* [n] index into the handle's cfgs, or NULL = all 0   */
  const uint64_t *q_off;    /* [n*M+1] CSR: queue (s,m) = waits[q_off[s*M+m] ..
                               q_off[s*M+m+1])                                      */
  const uint32_t *waits_us; /* head (oldest) first, non-increasing per queue (Q7)  */
  int64_t n_waits;          /* q_off[n*M] if known (host value), else 0.  Selects the
                               mapping: >= 1024 waits per snapshot on average -> the
                               streamed three-phase mapping (deep queues), else one
                               thread per snapshot (Algorithm 1; warp segments for the
                               baseline policies and GRID).  Results never depend on it */
} es_snapshots;

#define ES_FLAG_FEASIBLE 1u  /* Eq. 6 satisfiable for the chosen model            */
#define ES_FLAG_NO_WORK 2u   /* every queue empty: no decision            */
#define ES_FLAG_BAD_INPUT 4u /* waits increase inside the read window or bad cfg  */

/* Per-snapshot outputs.  Device [n] each (cand_score_q [n*M] or NULL). */
typedef struct {
  uint8_t *m;              /* m*                                                 */
  uint8_t *e;              /* e* (exit ordinal, 0 = shallowest)                  */
  uint16_t *B;             /* B*                                                 */
  uint32_t *L_us;          /* L(m*, e*, B*)                                      */
  uint64_t *score_q;       /* S_q(m*) = stability score * 2^28 (Q5)              */
  uint8_t *flags;          /* ES_FLAG_*                                          */
  uint64_t *cand_score_q;  /* S_q(m) per model, UINT64_MAX for an empty queue    */
} es_decisions;

/*
 * Algorithm 1 on every snapshot.  Tasks whose wait is already >= x_c are
 * clipped for every candidate (Eq. 3 clip); they are counted from the
 * CSR by a search on the non-increasing waits and never read, so a wait
 * inversion inside that clipped prefix is not detected (ES_FLAG_BAD_INPUT
 * covers the read window).  All-empty snapshots get ES_FLAG_NO_WORK and zero
 * outputs.  Async on `stream`.
 */
ES_API es_status es_score_candidates(const es_profile *prof, const es_snapshots *snaps,
                              es_decisions *out, es_stream stream);

/* ---------------------------------------------- K2 + K3: trace replay */

/* n_scen independent scenarios. Device pointers. */
typedef struct {
  int64_t n_scen;
  const uint16_t *cfg_idx;    /* [n_scen] or NULL = all cfg 0                        */
  const uint32_t *group_id;   /* [n_scen] or NULL = all group 0 (es_group_* only)   */
  const uint64_t *arr_off;    /* [n_scen*M+1] CSR of (scenario, model) segments      */
  const uint32_t *arrival_us; /* sorted non-decreasing within each segment           */
} es_traces;

/* per-scenario statistics columns of es_replay_out.scen_stats */
enum {
  ES_ST_DECISIONS = 0, /* Algorithm 1 invocations                                  */
  ES_ST_CANDIDATES,    /* stability scores evaluated (non-empty queues)            */
  ES_ST_CELLS,         /* (m, e) profile cells examined by Eq. 6                   */
  ES_ST_COMPLETED,     /* completions after the warmup                             */
  ES_ST_VIOLATIONS,    /* post-warmup completions with T > tau (Eq. 2)            */
  ES_ST_INFEASIBLE,    /* decisions whose chosen exit failed Eq. 6 (Q2)            */
  ES_ST_MAX_DEPTH,     /* largest queue length seen at a decision                  */
  ES_ST_STATUS,        /* es_status of this scenario (other columns undefined if != 0) */
  ES_ST_SUM_LAT,       /* sum of post-warmup T, us                                  */
  ES_ST_LIVE,          /* sum over decisions of pending tasks with w < x_c (read)   */
  ES_ST_TERMS,         /* sum over decisions of live tasks x candidates (Eq. 4 terms) */
  ES_ST_ACC_BP,        /* sum over post-warmup completions of accuracy_bp(m, e) of the
                          exit that served them: effective accuracy = ACC_BP / COMPLETED
                          basis points                               */
  ES_ST_EXIT0,         /* post-warmup completions served at exit 0 (shallowest) ...   */
  ES_ST_EXIT7 = ES_ST_EXIT0 + 7, /* ... exit 7: the exit-depth histogram (Fig. exit_depth) */
  ES_NSTAT
};

typedef struct {
  uint32_t *completion_us; /* [total] aligned with arrival_us, or NULL (stats only)  */
  uint8_t *exit_used;      /* [total] aligned with arrival_us, or NULL               */
  uint32_t *latency_us;    /* [total] REQUIRED: T per request in dispatch order
                              within each scenario's segment [arr_off[s*M], ...)     */
  uint64_t *scen_stats;    /* [n_scen][ES_NSTAT] REQUIRED                            */
  uint32_t *scen_p95_us;   /* [n_scen] nearest-rank P95 of post-warmup T, or NULL    */
  /* optional decision log: first dec_cap decisions of every scenario */
  int64_t dec_cap;
  uint32_t *dec_t_us;
  uint8_t *dec_m;
  uint8_t *dec_e;
  uint16_t *dec_B;
  uint32_t *dec_L_us;
  uint64_t *dec_score_q;
  uint8_t *dec_flags;
} es_replay_out;

/*
 * Replay every scenario (K2) and compute per-scenario P95 (K3).  Semantics
 * (DESIGN.md §3): t starts at the first arrival; a decision at t sees every
 * arrival with a <= t (Q10); with all queues empty t jumps to the next arrival
 * (Q12); a decision (m*, e*, B*) serves the B* oldest requests of Q_m* which
 * complete at t + L (Eq. 1); the next decision happens at completion;
 * the run drains every request (Q13).  Async on `stream`.
 */
ES_API es_status es_replay_traces(const es_profile *prof, const es_traces *traces, es_replay_out *out,
                           es_stream stream);

/*
 * K3 alone: per-scenario nearest-rank P95 of the post-warmup latencies that a
 * previous es_replay_traces wrote to out->latency_us (requires scen_stats and
 * scen_p95_us).  es_replay_traces already runs it when scen_p95_us != NULL.
 */
ES_API es_status es_scen_p95(const es_profile *prof, const es_traces *traces, es_replay_out *out,
                             es_stream stream);

/*
 * End-to-end variant: the same call with HOST traces and HOST outputs.  The
 * library copies inputs to device scratch, runs K2/K3, copies the outputs back
 * and synchronises `stream` before returning.  Pinned host memory gives
 * asynchronous copies; pageable memory works but is slower.
 */
ES_API es_status es_replay_traces_host(es_profile *prof, const es_traces *host_traces,
                                es_replay_out *host_out, es_stream stream);

/*
 * Pipelined end-to-end replay of nbatch independent host batches (each with its
 * own host traces and outputs, as in es_replay_traces_host): batch k's inputs
 * are copied to one of two device buffers on a library-owned copy stream while
 * batch k-1 replays on `stream`, so the host->device transfer overlaps the
 * replay.  Every batch still moves its own inputs in and its outputs out.
 * Synchronises `stream` before returning.  Errors as es_replay_traces_host.
 */
ES_API es_status es_replay_traces_host_pipelined(es_profile *prof, const es_traces *host_traces,
                                          es_replay_out *host_outs, int32_t nbatch, es_stream stream);

/* ------------------------------------------------ group merge (multi-GPU) */

#define ES_NGSTAT 16 /* decisions, candidates, cells, completed, violations, infeasible, sum_lat,
                        acc_bp, exit0 .. exit7 */
#define ES_HIST_BINS 4096

/*
 * Accumulate (+=) per-group counters [n_groups][ES_NGSTAT] and the level-0
 * (coarse) latency histogram [n_groups][4096], bin = min(T >> 12, 4095)
 * (4.096 ms bins, 4095 = overflow T >= 16.77 s), over the post-warmup requests
 * of every scenario with status OK.  Buffers are device u64 and must be
 * zeroed by the caller before the first call.  Integer sums: an
 * all_reduce(sum) across ranks gives bit-identical results for any rank count.
 */
ES_API es_status es_group_accumulate(const es_profile *prof, const es_traces *traces,
                                     const es_replay_out *out, uint32_t n_groups, uint64_t *group_counts,
                                     uint64_t *hist0, es_stream stream);

/*
 * K3 fused with es_group_accumulate: per-scenario P95 into out->scen_p95_us
 * (if non-NULL) and, if group_counts != NULL, the group counters and level-0
 * histogram -- one pass over the latencies instead of two.
 */
ES_API es_status es_scen_stats(const es_profile *prof, const es_traces *traces, es_replay_out *out,
                               uint32_t n_groups, uint64_t *group_counts, uint64_t *hist0, es_stream stream);

/*
 * Exact group P95 by radix selection on digits that are identical on every
 * rank (so histograms can be summed across ranks before each selection):
 *   level 0: coarse bin min(T >> 12, 4095)        (es_group_accumulate / es_scen_stats)
 *   level 1: T & 0xFFF inside the coarse bin       -> the exact P95 (normal case)
 *            or, for a group whose P95 lies in the overflow bin, T >> 20
 *   level 2: (T >> 8) & 0xFFF (overflow groups only)
 *   level 3: T & 0xFF          (overflow groups only)
 * Call order: [all_reduce counts + hist0] -> es_group_p95_select(0); then for
 * level 1, 2, 3: es_group_hist(level) -> [all_reduce hist] ->
 * es_group_p95_select(level).  Levels 2 and 3 are no-ops unless some group is
 * in the overflow bin.  state is u64 [n_groups][2]; after level 3 (or level 1
 * when no group overflows) state[g][0] is the nearest-rank P95 of group g (0
 * for an empty group).  es_group_hist overwrites hist (no need to zero).
 */
ES_API es_status es_group_hist(const es_profile *prof, const es_traces *traces, const es_replay_out *out,
                               uint32_t n_groups, int32_t level, const uint64_t *state, uint64_t *hist,
                               es_stream stream);
ES_API es_status es_group_p95_select(uint32_t n_groups, int32_t level, const uint64_t *group_counts,
                                     const uint64_t *hist, uint64_t *state, es_stream stream);

/*
 * Synchronise `stream` and report the first device-side error recorded by any
 * kernel launched with this handle since the last call (code 0 = none) and
 * the item (snapshot / scenario index) that raised it.  Clears the record.
 */
ES_API es_status es_device_status(es_profile *prof, es_stream stream, uint32_t *code, int64_t *item);

/* number of kernel launches issued through this handle (for launch counting) */
ES_API int64_t es_launch_count(const es_profile *prof);

#ifdef __cplusplus
}
#endif
#endif /* EDGESERVE_H */
