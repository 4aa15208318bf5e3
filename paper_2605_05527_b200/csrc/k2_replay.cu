// k2_replay.cu -- K2: whole-trace replay (steps a2-a8), one warp segment per
// scenario.
//
// The online serving loop of EdgeServing with exclusive
// time-division GPU execution, replayed decision by
// decision on a request trace:
//   a2  admission: a decision at t sees every arrival with a <= t (reading
//       Q10); queue Q_m is the index range [head_m, tail_m) of model m's
//       sorted arrival segment (no ring buffer, any depth).  Each lane group
//       tests GL upcoming arrivals per step with one coalesced load + ballot.
//   a3-a7  one decision (decide.cuh).  Tasks with w >= x_c form a prefix of
//       each queue (FIFO, waits non-increasing); the boundary `live_m` only
//       moves forward, so deep backlogs cost O(advance), not O(depth).
//   a8  commit: the B* oldest requests of Q_m* complete at t + L (Eq. 1);
//       their latency T = completion - arrival is written in dispatch order;
//       the next decision happens at completion, or at the next
//       arrival if every queue is empty (work-conserving idle, reading Q12).
//   a9  per-scenario counters (Eq. 2 strict violations after the warmup of
//       reading Q14); the P95 is K3 (k3_stats.cu).
//
// Execution model: a warp holds 32/LPS segments; each segment replays one
// scenario at a time and pulls the next from a device-wide atomic counter as
// soon as its scenario drains (chain lengths differ ~4x across rho and tau).
// All segments step in lockstep -- one decision (or one idle jump) per
// iteration -- with per-segment predicates, so every warp-synchronous
// primitive is executed by the whole warp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "k2_common.cuh"

namespace es {
namespace {

__device__ __forceinline__ uint32_t ldg_u32(const uint32_t *p) { return __ldg(p); }

// L1 prefetch of an upcoming arrival line (admission reads it a few decisions later)
__device__ __forceinline__ void prefetch_l1(const uint32_t *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// some segment is running (go) with all its queues empty: per-segment test of two ballots
template <int LPS>
__device__ __forceinline__ bool segs_idle(unsigned b_go, unsigned b_has) {
  bool idle = false;
#pragma unroll
  for (int k = 0; k < 32 / LPS; ++k) {
    const unsigned m = (LPS == 32 ? 0xFFFFFFFFu : ((1u << LPS) - 1u)) << (k * LPS);
    idle |= (b_go & m) != 0u && (b_has & m) == 0u;
  }
  return idle;
}


#ifndef ES_PF_LINES
#define ES_PF_LINES 2
#endif
constexpr int PF_LINES = ES_PF_LINES;

template <int LPS, int MM, bool POL, bool OUT>
// OUT = false compiles the stats-only replay (no completion / exit / decision
// log outputs: the bench and sweep path) without their per-decision tests.
// register budget: ptxas's own (127 registers for 8-model segments: 2 CTAs
// per SM; an explicit minimum of 1 CTA gives 136 and one CTA).  Forcing 3 CTAs
// (80 registers, spills) helped a 16,384-scenario cfg3 slice (-24 %) but
// slowed full cfg3 and the latency-bound cfg5-A chains, so it is left to
// ES_K2_MINB builds
#ifdef ES_K2_MINB
#define ES_K2_BOUNDS __launch_bounds__(256, ES_K2_MINB)
#else
#define ES_K2_BOUNDS __launch_bounds__(512)
#endif
__global__ void ES_K2_BOUNDS k2_replay(const uint8_t *__restrict__ gimg, ImgLayout lay, ReplayArgs a) {
  constexpr int GL = Seg<LPS, MM>::GL;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  stage_image(smem, gimg, a.stage_bytes, &mbar);
  SmemProf P = smem_prof(smem, lay);
  if (a.stage_bytes < lay.bytes) P.hb = gimg;  // H tables stay in global memory (L1-cached)
  uint8_t *flat = smem + ((a.stage_bytes + 15u) & ~15u) + (threadIdx.x >> 5) * FLAT_BYTES;  // this warp's scratch
  const Seg<LPS, MM> sg;
  const int g = sg.grp;
  const int M = P.M;
  const uint32_t mbits = g < M ? P.mask[g] : 0u;
  const uint32_t nallow = __popc(mbits);

  // ---- per-segment scenario state (uniform within a segment, per group for queues)
  bool active = false, exhausted = false;
  int64_t s = 0;
  SmemCfg C{};
  uint64_t base0 = 0, qb = 0;
  const uint32_t *Aq = a.arrival;
  uint32_t n = 0, head = 0, tail = 0, live = 0, last = 0, next_arr = 0xFFFFFFFFu;
  // admission window: WA consecutive arrivals per lane, a GW-arrival window
  // per group per round (narrow groups take several per lane: bursts admit in
  // fewer rounds), loaded one decision ahead
#ifndef ES_K2_WIN
#define ES_K2_WIN 4
#endif
  constexpr int WA = GL >= ES_K2_WIN ? 1 : ES_K2_WIN / GL;
  constexpr int GW = GL * WA;
  uint32_t win[WA];
#pragma unroll
  for (int k = 0; k < WA; ++k) win[k] = 0xFFFFFFFFu;
  uint32_t t = 0, total = 0, served = 0, seq = 0, status = 0, iters = 0;
  uint64_t decisions = 0, candidates = 0, infeasible = 0;
  // lane-local counters (reduced once per scenario)
  uint32_t completed = 0, viol = 0, cells = 0, maxd = 0;
  uint64_t sum_lat = 0, live_sum = 0, terms = 0;
  // f1 statistics: the accuracy sum (lane 0 of the segment) and the exit-depth
  // histogram, bin e held by segment lane e (LPS >= MAXE)
  uint64_t acc_bp = 0;
  uint32_t exit_n = 0;

  for (;;) {
    // ---- refill: segments without a scenario fetch the next one
    const bool need = !active && !exhausted;
    if (__any_sync(FULL, need)) {
      unsigned long long got = 0;
      if (need && sg.sl == 0) got = atomicAdd(a.work, 1ull);
      got = sg.bcast(got, 0);
      bool fresh = false;
      if (need) {
        if ((int64_t)got >= a.n_scen) exhausted = true;
        else fresh = true;
      }
      int k = 0;
      uint32_t n_new = 0, a0 = 0xFFFFFFFFu;
      if (fresh) {
        s = a.order ? (int64_t)a.order[got] : (int64_t)got;
        k = a.cfg_idx ? (int)a.cfg_idx[s] : 0;
        qb = 0;
        if (k < P.ncfg) {
          C = smem_cfg(P, k);
          base0 = a.arr_off[s * M];
          if (g < M) {
            qb = a.arr_off[s * M + g];
            n_new = (uint32_t)(a.arr_off[s * M + g + 1] - qb);
          }
        }
        Aq = a.arrival + qb;
        if (n_new) a0 = ldg_u32(Aq);
#pragma unroll
        for (int k = 0; k < WA; ++k) {
          const uint32_t i = (uint32_t)(sg.gl * WA + k);
          win[k] = i < n_new ? ldg_u32(Aq + i) : 0xFFFFFFFFu;
        }
      }
      const uint32_t tot = sg.sum(sg.gl == 0 ? n_new : 0u);
      const uint32_t t0 = sg.vmin(a0);
      if (fresh) {
        active = true;
        n = n_new;
        next_arr = a0;
        total = tot;
        t = t0;
        head = tail = live = last = 0;
        served = seq = iters = 0;
        status = (k < P.ncfg) ? (uint32_t)ES_OK : (uint32_t)ES_ERR_ARG;
        decisions = candidates = infeasible = 0;
        completed = viol = cells = maxd = 0;
        sum_lat = live_sum = terms = 0;
        acc_bp = exit_n = 0;
      }
    }
    if (__all_sync(FULL, exhausted)) break;

    // ---- decisions until some segment of the warp drains its scenario
    for (;;) {
      // progress guard: each iteration serves >= 1 request or jumps to an arrival
      // (deferred batching adds at most one idle step per arrival or dispatch)
      if (active && status == ES_OK && ++iters > 4u * total + 8u) status = ES_ERR_INTERNAL;
      const bool run = active && status == ES_OK && served < total;
      // a2: admission (every arrival with a <= t)
      const bool pre_ok = run && head < tail;
      const uint32_t ahead_pre = pre_ok ? ldg_u32(Aq + head) : 0u;  // head arrival, issued early
      bool more = true, first = true;
      while (more) {
        // window positions tail + gl WA + k; the first round reads the
        // registers loaded at the end of the previous admission (off the chain)
        uint32_t v[WA];
        uint32_t c = 0u;
        bool bad = false;
#pragma unroll
        for (int k = 0; k < WA; ++k) {
          const uint32_t idx = tail + (uint32_t)(sg.gl * WA + k);
          const bool valid = run && idx < n;
          v[k] = !valid ? 0xFFFFFFFFu : first ? win[k] : ldg_u32(Aq + idx);
          c += valid && v[k] <= t ? 1u : 0u;
          if (k > 0) bad |= valid && v[k] < v[k - 1];
        }
        first = false;
        uint32_t prev = last;  // order check across lanes: the previous lane's last element
        if constexpr (GL > 1) {
          const uint32_t pl = __shfl_up_sync(FULL, v[WA - 1], 1, GL);
          if (sg.gl != 0) prev = pl;
        }
        bad |= run && tail + (uint32_t)(sg.gl * WA) < n && v[0] < prev;
        // admitted = a prefix of the group window (sorted): its length
        uint32_t cnt = c;
#pragma unroll
        for (int o = 1; o < GL; o <<= 1) cnt += __shfl_xor_sync(FULL, cnt, o, GL);
        const unsigned badb = __ballot_sync(FULL, bad);
        // last admitted (window position cnt - 1) and next pending (position cnt)
        const uint32_t jl = cnt ? cnt - 1u : 0u, jn = cnt < (uint32_t)GW ? cnt : (uint32_t)GW - 1u;
        uint32_t el = v[0], en = v[0];
#pragma unroll
        for (int k = 1; k < WA; ++k) {
          if (jl % WA == (uint32_t)k) el = v[k];
          if (jn % WA == (uint32_t)k) en = v[k];
        }
        const uint32_t lv = __shfl_sync(FULL, el, sg.grp * GL + (int)(jl / WA), LPS);
        const uint32_t nx = __shfl_sync(FULL, en, sg.grp * GL + (int)(jn / WA), LPS);
        if (run) {
          next_arr = nx;
          if (cnt) last = lv;
          tail += cnt;
          if (sg.sbits(badb)) status = ES_ERR_UNSORTED;
        }
        more = __any_sync(FULL, run && status == ES_OK && cnt == (uint32_t)GW);
      }
      // the next decision's first admission round reads this window
      if (run) {
#pragma unroll
        for (int k = 0; k < WA; ++k) {
          const uint32_t idx = tail + (uint32_t)(sg.gl * WA + k);
          if (idx < n) win[k] = ldg_u32(Aq + idx);
        }
      }
      // keep the next PF_LINES 128-byte lines of this model's arrivals in L1
      // (the admission loads above are the head of the per-decision chain)
      if (run && sg.gl < PF_LINES) {
        const uint32_t pf = (tail & ~31u) + 32u * (uint32_t)(sg.gl + 1);
        if (pf < n) prefetch_l1(Aq + pf);
      }
      const bool go = run && status == ES_OK;
      uint32_t len = go ? tail - head : 0u;
      // a3/a4 inputs: head wait (issued before admission), clipped-for-everyone prefix
      const uint32_t ahead = len == 0u ? t : (pre_ok ? ahead_pre : ldg_u32(Aq + head));
      uint32_t wmax = t - ahead;
      // every warp-uniform decision of this step from one round of independent
      // ballots (they pipeline; a chain of votes would not)
      const unsigned b_go = __ballot_sync(FULL, go);
      const unsigned b_has = __ballot_sync(FULL, len > 0u);
      const unsigned b_xc = __ballot_sync(FULL, len > 0u && wmax >= C.x_c);
      const unsigned b_slow = __ballot_sync(FULL, len > 0u && wmax >= C.fast_lim);
      const bool has = sg.sbits(b_has) != 0u;
      // idle GPU (Q12): a running segment with every queue empty jumps to the next arrival
      if (segs_idle<LPS>(b_go, b_has)) {
        const uint32_t tn = sg.vmin(go ? next_arr : 0xFFFFFFFFu);
        if (go && !has) t = tn;
      }
      const bool dec = go && has;
      if (!dec) len = 0u;
      maxd = max(maxd, len);
      if (live < head) live = head;
      if (b_xc != 0u) {
        bool adv = true;
        while (adv) {
          const uint32_t idx = live + sg.gl;
          const bool pr = len > 0u && idx < tail && (t - ldg_u32(Aq + idx)) >= C.x_c;
          const uint32_t cnt = __popc(sg.gbits(__ballot_sync(FULL, pr)));
          live += cnt;
          adv = __any_sync(FULL, cnt == (uint32_t)GL);
        }
      }
      const uint32_t c = len ? live - head : 0u;
      const Cand cand = cand_params<LPS, MM, POL>(sg, P, C, len, wmax);
      const uint32_t tt = t;
      const uint32_t *Ah = Aq + head;
      // a5-a7: Eq. 7 on the stability score, or the LQF / EDF rule of a
      // baseline policy (each runs warp-wide when some segment needs it)
      const bool sc = !POL || policy_scores(C.policy);
      Decision d{};
      if (!POL || (a.any_score && (!a.any_simple || __any_sync(FULL, dec && sc)))) {
        // fast path of 8-lane segments: the warp's queued positions flattened
        // (four scenarios per warp: the per-group walk would cost the warp's
        // longest queue; measured cfg3 K2 46.7 -> 43.4 ms).  Wider segments
        // keep the per-group walk (flattening measured slower there).
        if (LPS == 8 && b_slow == 0u)
          d = decide_fast_flat<LPS, MM>(sg, P, C, len, cand, Ah, tt, flat);
        else
          d = decide<LPS, MM>(sg, P, C, len, c, b_slow == 0u, cand, [&](uint32_t p) { return tt - ldg_u32(Ah + p); });
      }
      if (POL && a.any_simple && __any_sync(FULL, dec && !sc)) {
        const Decision ds = select_simple<LPS, MM>(sg, cand, len, wmax, C);
        if (!sc) d = ds;
      }
      const bool grid = POL && C.policy == ES_POLICY_GRID;
      uint32_t ngrid = 0u;
      if (POL && a.any_grid && __any_sync(FULL, dec && grid)) {
        uint32_t ng = 0u;
        uint64_t own = 0ull;
        const Decision dg = decide_grid<LPS, MM>(sg, P, C, len, c, wmax, [&](uint32_t p) { return tt - ldg_u32(Ah + p); },
                                                 ng, own);
        if (grid) {
          d = dg;
          ngrid = ng;
        }
      }
      // SYMPHONY with no triggered queue (Q27): no dispatch; the GPU idles
      // until the earliest trigger instant or the next arrival
      bool disp = dec;
      if (POL && a.any_simple) {
        const bool sym = C.policy == ES_POLICY_SYMPHONY;
        const bool wait = dec && sym && d.m == 0xFFu;
        if (__any_sync(FULL, wait)) {
          const uint64_t need = (uint64_t)wmax + cand.L;
          const uint32_t rel = sg.vmin(wait && len > 0u ? (uint32_t)(C.tau - need) : 0xFFFFFFFFu);
          const uint32_t na = sg.vmin(wait ? next_arr : 0xFFFFFFFFu);
          if (wait) {
            t = (uint32_t)min((uint64_t)t + rel, (uint64_t)na);
            disp = false;
          }
        }
      }
      const uint32_t nq = __popc(sg.sbits(b_has)) / (uint32_t)GL;  // non-empty queues (all GL lanes of a group agree)
      const uint32_t ncand = grid ? ngrid : nq;  // scored candidates: queues, or (m, e, b) cells
      // a8: commit
      const int src = (int)(d.m & (MM - 1)) * GL;
      const uint64_t qb_w = sg.bcast(qb, src);
      const uint32_t head_w = sg.bcast(head, src);
      if (disp) {
        const uint64_t done64 = (uint64_t)t + d.L;
        if (done64 > 0xFFFFFFFFull) {
          status = ES_ERR_RANGE;
        } else {
          const uint32_t done = (uint32_t)done64;
          decisions++;
          candidates += ncand;
          if (!d.feas) infeasible++;
          {  // f1: the batch's post-warmup tasks served at (m*, e*)
            const uint32_t pre_w = seq < C.warmup ? min(C.warmup - seq, d.B) : 0u;
            const uint32_t npost = d.B - pre_w;
            if (sg.sl == 0) acc_bp += (uint64_t)npost * P.acc[d.m * P.E + d.e];
            if ((uint32_t)sg.sl == d.e) exit_n += npost;
          }
          if (sg.gl == 0 && len > 0u) {
            cells += nallow;
            live_sum += len - c;
            if (sc || grid) terms += (uint64_t)(len - c) * ncand;  // Eq. 4 terms: scoring policies only
          }
          for (uint32_t j = sg.sl; j < d.B; j += LPS) {
            const uint64_t i = qb_w + head_w + j;
            const uint32_t T = done - ldg_u32(a.arrival + i);  // Eq. 1: T = w + t
            if (a.completion) a.completion[i] = done;
            if (a.exit_used) a.exit_used[i] = (uint8_t)d.e;
            const uint32_t q = seq + j;
            a.lat[base0 + q] = T;
            if (q >= C.warmup) {  // reading Q14
              completed++;
              sum_lat += T;
              viol += T > C.tau ? 1u : 0u;  // Eq. 2, strict
            }
          }
          if (OUT && a.dec_cap && sg.sl == 0 && (int64_t)decisions <= a.dec_cap) {
            const int64_t o = s * a.dec_cap + (int64_t)decisions - 1;
            if (a.dec_t) a.dec_t[o] = t;
            if (a.dec_m) a.dec_m[o] = (uint8_t)d.m;
            if (a.dec_e) a.dec_e[o] = (uint8_t)d.e;
            if (a.dec_B) a.dec_B[o] = (uint16_t)d.B;
            if (a.dec_L) a.dec_L[o] = d.L;
            if (a.dec_S) a.dec_S[o] = d.S;
            if (a.dec_f) a.dec_f[o] = d.feas ? 1 : 0;
          }
          if (g == (int)d.m) head += d.B;
          seq += d.B;
          served += d.B;
          t = done;  // next round on completion
        }
      }
      if (__any_sync(FULL, active && (served >= total || status != ES_OK))) break;
    }

    // ---- a9: drained (or failed) scenarios write their counters
    const bool fin = active && (served >= total || status != ES_OK);
    const uint32_t r_comp = sg.sum(completed), r_viol = sg.sum(viol), r_cells = sg.sum(cells);
    const uint32_t r_maxd = sg.vmax(maxd);
    const uint64_t r_sum = sg.sum64(sum_lat), r_live = sg.sum64(live_sum), r_terms = sg.sum64(terms);
    if (fin) {
      if (sg.sl == 0) {
        uint64_t *st = a.stats + s * ES_NSTAT;
        st[ES_ST_DECISIONS] = decisions;
        st[ES_ST_CANDIDATES] = candidates;
        st[ES_ST_CELLS] = r_cells;
        st[ES_ST_COMPLETED] = r_comp;
        st[ES_ST_VIOLATIONS] = r_viol;
        st[ES_ST_INFEASIBLE] = infeasible;
        st[ES_ST_MAX_DEPTH] = r_maxd;
        st[ES_ST_STATUS] = status;
        st[ES_ST_SUM_LAT] = r_sum;
        st[ES_ST_LIVE] = r_live;
        st[ES_ST_TERMS] = r_terms;
        st[ES_ST_ACC_BP] = acc_bp;
        if (status) report(a.dstat, status, s);
      }
      if (sg.sl < MAXE) a.stats[s * ES_NSTAT + ES_ST_EXIT0 + sg.sl] = exit_n;
      active = false;
    }
  }
}

// ---- hand-out order: K2's time is its longest chain, so the segments pick up
// the scenarios in decreasing order of trace span (last - first arrival; at a
// fixed request count a longer span means lighter load, smaller batches, more
// decisions) -- longest-processing-time-first.  64 span buckets (counting
// sort); the order inside a bucket is arbitrary.  Results do not depend on it
// (scenarios are independent and write fixed slots).
constexpr int NBK = 64;

__global__ void k2_order_span(int64_t n_scen, int M, const uint64_t *__restrict__ arr_off,
                              const uint32_t *__restrict__ arrival, uint32_t *span, unsigned *sc) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_scen; s += (int64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0xFFFFFFFFu, hi = 0u;
    for (int m = 0; m < M; ++m) {
      const uint64_t b = arr_off[s * M + m], e = arr_off[s * M + m + 1];
      if (e > b) {
        lo = min(lo, __ldg(arrival + b));
        hi = max(hi, __ldg(arrival + e - 1));
      }
    }
    const uint32_t v = hi >= lo ? hi - lo : 0u;
    span[s] = v;
    atomicMax(sc, v);
  }
}

__global__ void k2_order_hist(int64_t n_scen, const uint32_t *span, unsigned *sc) {
  const uint64_t mx = (uint64_t)sc[0] + 1u;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_scen; s += (int64_t)gridDim.x * blockDim.x) {
    const int b = NBK - 1 - (int)((uint64_t)span[s] * NBK / mx);  // longest spans -> bucket 0
    atomicAdd(sc + 1 + b, 1u);
  }
}

__global__ void k2_order_scatter(int64_t n_scen, const uint32_t *span, unsigned *sc, uint32_t *order) {
  __shared__ unsigned base[NBK];
  if (threadIdx.x == 0) {
    unsigned acc = 0;
    for (int b = 0; b < NBK; ++b) {
      base[b] = acc;
      acc += sc[1 + b];
    }
  }
  __syncthreads();
  const uint64_t mx = (uint64_t)sc[0] + 1u;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_scen; s += (int64_t)gridDim.x * blockDim.x) {
    const int b = NBK - 1 - (int)((uint64_t)span[s] * NBK / mx);
    order[base[b] + atomicAdd(sc + 1 + NBK + b, 1u)] = (uint32_t)s;
  }
}

template <int LPS, int MM>
cudaError_t launch_t(const uint8_t *img, const ImgLayout &lay, const ReplayArgs &a, cudaStream_t st, int sms) {
  // Algorithm 1 alone compiles without the policy code (no cost on the bench path)
  const bool alg1 = lay.pol_mask == (1u << ES_POLICY_EDGESERVING);
  const bool out = a.completion || a.exit_used || a.dec_cap;
  auto kern = alg1 ? (out ? k2_replay<LPS, MM, false, true> : k2_replay<LPS, MM, false, false>)
                   : (out ? k2_replay<LPS, MM, true, true> : k2_replay<LPS, MM, true, false>);
  // dynamic shared memory: the staged image + one flat-path scratch per warp
  auto dyn_of = [&](int threads) {
    return (((size_t)a.stage_bytes + 15u) & ~(size_t)15u) + (LPS == 8 ? (size_t)(threads / 32) * FLAT_BYTES : 0u);
  };
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_of(512));
  if (e != cudaSuccess) return e;
  // threads per block: the smallest of 64 / 128 / 256 that keeps the resident
  // thread count of 256-thread blocks (small blocks deal the longest-first
  // scenarios round-robin over the SMs in finer grains; a large profile image
  // -- one CTA per SM by shared memory -- keeps 256).  ES_K2_BLOCK overrides.
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, dyn_of(256));
  if (e != cudaSuccess) return e;
  int threads = 256;
  for (int t = 64; t < 256; t *= 2) {
    int o = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, t, dyn_of(t));
    if (e != cudaSuccess) return e;
    // (and only while the extra per-CTA image copies leave L1 room: the
    // pending waits are re-read from L1 every decision)
    if (o * t >= occ * 256 && (size_t)o * dyn_of(t) <= 96u * 1024u) {
      threads = t;
      occ = o;
      break;
    }
  }
  // a throughput batch (>= 256 scenarios per SM) takes 512-thread CTAs: one
  // staged image per 16 warps leaves L1 the most room for the re-read waits
  // (cfg3: 43.2 -> 41.8 ms vs 256-thread CTAs)
  if (a.n_scen >= (int64_t)256 * sms) {
    int o = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, 512, dyn_of(512));
    if (e != cudaSuccess) return e;
    if (o >= 1 && o * 512 >= occ * threads) {
      threads = 512;
      occ = o;
    }
  }
  if (const char *env = getenv("ES_K2_BLOCK")) {
    const int v = atoi(env);
    if (v == 32 || v == 64 || v == 128 || v == 256 || v == 512) {
      threads = v;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, dyn_of(threads));
      if (e != cudaSuccess) return e;
    }
  }
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const int seg_per_block = threads / LPS;
  int64_t blocks = (a.n_scen + seg_per_block - 1) / seg_per_block;
  if (const char *env = getenv("ES_K2_OCC")) occ = std::max(1, std::min(occ, atoi(env)));  // resident CTAs/SM cap
  const int64_t cap = (int64_t)sms * occ;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, threads, dyn_of(threads), st>>>(img, lay, a);
  return cudaGetLastError();
}

template <int LPS>
cudaError_t launch_lps(const uint8_t *img, const ImgLayout &lay, const ReplayArgs &a, cudaStream_t st, int sms) {
  if (lay.M <= 2) return launch_t<LPS, 2>(img, lay, a, st, sms);
  if (lay.M <= 4) return launch_t<LPS, 4>(img, lay, a, st, sms);
  return launch_t<LPS, 8>(img, lay, a, st, sms);
}

// lanes per scenario: a latency-bound batch (few chains per SM: the longest
// chain is the kernel's time) takes wide segments -- 16 lanes for M <= 4, a
// whole warp for M > 4 -- so one decision has more lanes on its chain; a
// throughput-bound batch (>= 256 scenarios per SM) takes 8-lane segments, so
// each warp instruction serves four decisions (and the flattened fast path
// balances the four).  Measured (1 x B200, K2 alone): cfg2 16 lanes 2.90 ms
// vs 8 lanes 3.77; cfg5-A 32: 105 vs 16: 175; cfg5-B 32: 281 vs 16: 323;
// cfg3 8 (flat): 43.4 vs 16: 48.1 vs 32: 59.1; cfg4 8: 52.5 vs 16: 64.9.
// ES_LPS overrides.
int choose_lps(const ImgLayout &lay, int64_t n_scen, int sms) {
  const char *env = getenv("ES_LPS");
  if (env) {
    int v = atoi(env);
    if (v == 8 || v == 16 || v == 32) return v;
  }
  const int wide = lay.M <= 4 ? 16 : 32;
  return n_scen >= (int64_t)256 * sms ? 8 : wide;
}

}  // namespace

cudaError_t launch_replay(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                          const es_replay_out &out, DevStatus *dstat, cudaStream_t st, int sms, int *n_launch) {
  ReplayArgs a;
  a.n_scen = tr.n_scen;
  a.cfg_idx = tr.cfg_idx;
  a.arr_off = tr.arr_off;
  a.arrival = tr.arrival_us;
  a.completion = out.completion_us;
  a.exit_used = out.exit_used;
  a.lat = out.latency_us;
  a.stats = out.scen_stats;
  a.dec_cap = out.dec_cap;
  a.dec_t = out.dec_t_us;
  a.dec_m = out.dec_m;
  a.dec_e = out.dec_e;
  a.dec_B = out.dec_B;
  a.dec_L = out.dec_L_us;
  a.dec_S = out.dec_score_q;
  a.dec_f = out.dec_flags;
  a.dstat = dstat;
  a.order = nullptr;
  // a large image (many SLOs: cfg3's nine, cfg4's sixteen) would leave one CTA
  // per SM: stage only the core and read H (one load per candidate) from global
  a.stage_bytes = lay.bytes > 64u * 1024u ? lay.core_bytes : lay.bytes;
  constexpr uint32_t SCORE_POLS =
      (1u << ES_POLICY_EDGESERVING) | (1u << ES_POLICY_ALLFINAL_DA) | (1u << ES_POLICY_OURS_BS1);
  constexpr uint32_t GRID_POLS = 1u << ES_POLICY_GRID;
  a.any_score = (lay.pol_mask & SCORE_POLS) != 0u;
  a.any_grid = (lay.pol_mask & GRID_POLS) != 0u;
  a.any_simple = (lay.pol_mask & ~(SCORE_POLS | GRID_POLS)) != 0u;
  // per-call scratch (stream-ordered, so concurrent calls on one handle never
  // share it): the scenario work counter, and the longest-span-first hand-out
  // order (ES_K2_ORDER=0: scenario index order)
  const char *oe = getenv("ES_K2_ORDER");
  const bool ordered = tr.n_scen > 1 && tr.n_scen < (int64_t)0xFFFFFFFF && !(oe && oe[0] == '0');
  const size_t ob = ordered ? 4u * (size_t)tr.n_scen : 0u, sb = ordered ? 4u * (1 + 2 * NBK) : 0u;
  void *buf = nullptr;
  cudaError_t e = cudaMallocAsync(&buf, 16 + 2 * ob + sb, st);
  if (e != cudaSuccess) return e;
  a.work = static_cast<unsigned long long *>(buf);
  e = cudaMemsetAsync(buf, 0, 16, st);
  if (e == cudaSuccess && ordered) {
    uint32_t *order = reinterpret_cast<uint32_t *>(static_cast<uint8_t *>(buf) + 16), *span = order + tr.n_scen;
    unsigned *sc = reinterpret_cast<unsigned *>(span + tr.n_scen);
    e = cudaMemsetAsync(sc, 0, sb, st);
    const int blocks = (int)std::min<int64_t>((tr.n_scen + 255) / 256, (int64_t)sms * 8);
    if (e == cudaSuccess) k2_order_span<<<blocks, 256, 0, st>>>(tr.n_scen, lay.M, tr.arr_off, tr.arrival_us, span, sc);
    if (e == cudaSuccess) k2_order_hist<<<blocks, 256, 0, st>>>(tr.n_scen, span, sc);
    if (e == cudaSuccess) k2_order_scatter<<<blocks, 256, 0, st>>>(tr.n_scen, span, sc, order);
    if (e == cudaSuccess) e = cudaGetLastError();
    a.order = order;
    *n_launch += 3;
  }
  if (e == cudaSuccess) {
    const int lps = choose_lps(lay, tr.n_scen, sms);
    e = lps == 8 && lay.M <= 8 ? launch_lps<8>(img, lay, a, st, sms)
        : lps == 16            ? launch_lps<16>(img, lay, a, st, sms)
                               : launch_lps<32>(img, lay, a, st, sms);
    *n_launch += 1;
  }
  const cudaError_t f = cudaFreeAsync(buf, st);
  return e != cudaSuccess ? e : f;
}

}  // namespace es
