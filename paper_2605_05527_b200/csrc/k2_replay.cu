// k2_replay.cu -- K2: whole-trace replay, one warp per scenario (steps a2-a8).
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
// Scenarios are handed out by a device-wide atomic counter (persistent warps)
// because chain lengths differ by ~4x across rho and tau.
#include <cuda_runtime.h>

#include "decide.cuh"

namespace es {
namespace {

struct ReplayArgs {
  int64_t n_scen;
  const uint16_t *cfg_idx;
  const uint64_t *arr_off;
  const uint32_t *arrival;
  uint32_t *completion;
  uint8_t *exit_used;
  uint32_t *lat;
  uint64_t *stats;
  int64_t dec_cap;
  uint32_t *dec_t;
  uint8_t *dec_m, *dec_e;
  uint16_t *dec_B;
  uint32_t *dec_L;
  uint64_t *dec_S;
  uint8_t *dec_f;
  DevStatus *dstat;
  unsigned long long *work;
};

__device__ __forceinline__ uint32_t ldg_u32(const uint32_t *p) { return __ldg(p); }

__device__ __forceinline__ void report(DevStatus *ds, uint32_t code, int64_t item) {
  if (atomicCAS(&ds->code, 0u, code) == 0u) ds->item = (unsigned long long)item;
}

template <int MM>
__device__ void replay_one(const Lanes<MM> &ln, const uint8_t *sm, const SmemProf &P, const ReplayArgs &a,
                           int64_t s) {
  constexpr int GL = Lanes<MM>::GL;
  const int g = ln.grp;
  const int M = P.M;
  uint64_t *st = a.stats + s * ES_NSTAT;
  const int k = a.cfg_idx ? (int)a.cfg_idx[s] : 0;
  if (k >= P.ncfg) {
    if (ln.lane < ES_NSTAT) st[ln.lane] = (ln.lane == ES_ST_STATUS) ? (uint64_t)ES_ERR_ARG : 0ull;
    if (ln.lane == 0) report(a.dstat, ES_ERR_ARG, s);
    return;
  }
  const SmemCfg C = smem_cfg(sm, P, k);
  const uint64_t base0 = a.arr_off[s * M];
  uint64_t qb = 0;
  uint32_t n = 0;
  if (g < M) {
    qb = a.arr_off[s * M + g];
    n = (uint32_t)(a.arr_off[s * M + g + 1] - qb);
  }
  const uint32_t *Aq = a.arrival + qb;
  const uint32_t total = red_u32(ln.gl == 0 ? n : 0u);
  uint32_t next_arr = n ? ldg_u32(Aq) : 0xFFFFFFFFu;
  uint32_t t = __reduce_min_sync(FULL, next_arr);
  uint32_t head = 0, tail = 0, live = 0, last = 0;
  uint32_t served = 0, seq = 0;
  uint32_t status = ES_OK;
  // uniform counters
  uint64_t decisions = 0, candidates = 0, infeasible = 0, live_sum = 0, terms = 0;
  // lane-local counters (reduced at the end)
  uint32_t completed = 0, viol = 0, cells = 0, maxd = 0;
  uint64_t sum_lat = 0;
  const uint32_t mbits = g < M ? P.mask[g] : 0u;
  const uint32_t nallow = __popc(mbits);
  while (served < total) {
    // ---- a2: admission (every arrival with a <= t)
    bool more = true;
    while (more) {
      const uint32_t idx = tail + ln.gl;
      const uint32_t v = idx < n ? ldg_u32(Aq + idx) : 0xFFFFFFFFu;
      uint32_t prev = __shfl_up_sync(FULL, v, 1, GL);
      if (ln.gl == 0) prev = last;
      const bool bad = idx < n && v < prev;
      const bool ok = idx < n && v <= t;
      const unsigned b = ln.gbits(__ballot_sync(FULL, ok));
      const uint32_t cnt = __popc(b);
      const uint32_t lv = __shfl_sync(FULL, v, g * GL + (cnt ? cnt - 1 : 0));
      next_arr = __shfl_sync(FULL, v, g * GL + (cnt < GL ? cnt : GL - 1));
      if (cnt) last = lv;
      tail += cnt;
      if (__any_sync(FULL, bad)) {
        status = ES_ERR_UNSORTED;
        break;
      }
      more = __any_sync(FULL, cnt == (uint32_t)GL);
    }
    if (status) break;
    uint32_t len = tail - head;
    if (!__any_sync(FULL, len > 0u)) {  // idle GPU: jump to the next arrival (Q12)
      t = __reduce_min_sync(FULL, next_arr);
      continue;
    }
    maxd = max(maxd, len);
    // ---- a3/a4 inputs: head wait, clipped-for-everyone prefix
    const uint32_t ahead = len ? ldg_u32(Aq + head) : t;
    const uint32_t wmax = t - ahead;
    if (live < head) live = head;
    if (__any_sync(FULL, len > 0u && wmax >= C.x_c)) {
      bool adv = true;
      while (adv) {
        const uint32_t idx = live + ln.gl;
        const bool pr = idx < tail && (t - ldg_u32(Aq + idx)) >= C.x_c;
        const uint32_t cnt = __popc(ln.gbits(__ballot_sync(FULL, pr)));
        live += cnt;
        adv = __any_sync(FULL, cnt == (uint32_t)GL);
      }
    }
    const uint32_t c = live - head;
    const Cand cand = cand_params<MM>(ln, P, C, g, len, wmax);
    const uint32_t hq = head;
    const uint32_t tt = t;
    const Decision d = decide<MM>(ln, C, len, c, cand, [&](uint32_t p) { return tt - ldg_u32(Aq + hq + p); });
    // ---- a8: commit
    const uint64_t done64 = (uint64_t)t + d.L;
    if (done64 > 0xFFFFFFFFull) {
      status = ES_ERR_RANGE;
      break;
    }
    const uint32_t done = (uint32_t)done64;
    decisions++;
    const uint32_t ncand = __popc(__ballot_sync(FULL, ln.gl == 0 && len > 0u));
    const uint32_t nlive = red_u32(ln.gl == 0 ? len - c : 0u);
    candidates += ncand;
    live_sum += nlive;
    terms += (uint64_t)nlive * ncand;
    if (ln.gl == 0 && len > 0u) cells += nallow;
    if (!d.feas) infeasible++;
    const int src = (int)d.m * GL;
    const uint64_t qb_w = __shfl_sync(FULL, qb, src);
    const uint32_t head_w = __shfl_sync(FULL, head, src);
    for (uint32_t j = ln.lane; j < d.B; j += 32) {
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
    if (a.dec_cap && ln.lane == 0 && (int64_t)decisions <= a.dec_cap) {
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
  // ---- a9: per-scenario counters
  completed = red_u32(completed);
  viol = red_u32(viol);
  cells = red_u32(cells);
  maxd = __reduce_max_sync(FULL, maxd);
  sum_lat = red_u64(sum_lat);
  if (ln.lane == 0) {
    st[ES_ST_DECISIONS] = decisions;
    st[ES_ST_CANDIDATES] = candidates;
    st[ES_ST_CELLS] = cells;
    st[ES_ST_COMPLETED] = completed;
    st[ES_ST_VIOLATIONS] = viol;
    st[ES_ST_INFEASIBLE] = infeasible;
    st[ES_ST_MAX_DEPTH] = maxd;
    st[ES_ST_STATUS] = status;
    st[ES_ST_SUM_LAT] = sum_lat;
    st[ES_ST_LIVE] = live_sum;
    st[ES_ST_TERMS] = terms;
    if (status) report(a.dstat, status, s);
  }
}

template <int MM>
__global__ void __launch_bounds__(256) k2_replay(const uint8_t *__restrict__ gimg, ImgLayout lay, ReplayArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  stage_image(smem, gimg, lay.bytes, &mbar);
  const SmemProf P = smem_prof(smem, lay);
  const Lanes<MM> ln;
  for (;;) {
    unsigned long long s = 0;
    if (ln.lane == 0) s = atomicAdd(a.work, 1ull);
    s = __shfl_sync(FULL, s, 0);
    if ((int64_t)s >= a.n_scen) break;
    replay_one<MM>(ln, smem, P, a, (int64_t)s);
  }
}

template <int MM>
cudaError_t launch_mm(const uint8_t *img, const ImgLayout &lay, const ReplayArgs &a, cudaStream_t st, int sms) {
  auto kern = k2_replay<MM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.bytes);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, lay.bytes);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const int64_t warps_needed = a.n_scen;
  int64_t blocks = (warps_needed + 7) / 8;
  const int64_t cap = (int64_t)sms * occ;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, 256, lay.bytes, st>>>(img, lay, a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_replay(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                          const es_replay_out &out, DevStatus *dstat, uint32_t *work_ctr,
                          cudaStream_t st, int sms, int *n_launch) {
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
  a.work = reinterpret_cast<unsigned long long *>(work_ctr);
  cudaError_t e = cudaMemsetAsync(work_ctr, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  *n_launch += 1;
  if (lay.M <= 2) return launch_mm<2>(img, lay, a, st, sms);
  if (lay.M <= 4) return launch_mm<4>(img, lay, a, st, sms);
  return launch_mm<8>(img, lay, a, st, sms);
}

}  // namespace es
