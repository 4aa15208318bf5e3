// k2_lane.cu -- K2, latency-optimised mapping: one LANE per model queue.
//
// Same method and same integers as k2_replay.cu (steps a2-a8, see there and
// decide.cuh); only the mapping differs.  K2 is a dependent chain per scenario
// (each decision needs the previous completion time), so its speed is the
// length of one decision's dependency chain.  Here a scenario is a segment of
// MM lanes (MM = M rounded up to 2/4/8), lane g owns model g's queue and does
// its queue's work serially with instruction-level parallelism (admission,
// Eq. 5-6 for its own candidate, G(w) of its own tasks); only the cross-queue
// steps (sum of U, Eq. 7 argmin, winner broadcast) cross lanes, as log2(MM)
// shuffle butterflies.  32/MM scenarios share a warp; every warp-synchronous
// primitive is executed by the whole warp (lane predicates, never branches).
//
// Measured on cfg2 (profiles/r01_*): this mapping issues ~40 % fewer
// instructions than k2_replay.cu but its per-lane serial loops make the
// per-decision chain longer (1.5 vs 1.0 us alone), so k2_replay.cu is the
// default and this kernel is selected with ES_K2=lane (tests cover both).
#include <cuda_runtime.h>

#include <cstdlib>

#include "decide.cuh"

namespace es {
namespace {

struct LaneArgs {
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

__device__ __forceinline__ uint32_t ldg(const uint32_t *p) { return __ldg(p); }

template <int MM>
struct LSeg {  // segment of MM lanes, lane g = model g
  int lane, seg, g, base;
  __device__ __forceinline__ LSeg() {
    lane = threadIdx.x & 31;
    seg = lane / MM;
    g = lane % MM;
    base = seg * MM;
  }
  __device__ __forceinline__ unsigned sbits(unsigned b) const { return (b >> base) & low_mask(MM); }
  __device__ __forceinline__ bool any(bool p) const { return sbits(__ballot_sync(FULL, p)) != 0u; }
  template <typename T>
  __device__ __forceinline__ T bcast(T v, int src) const {
    return __shfl_sync(FULL, v, src, MM);
  }
  __device__ __forceinline__ uint32_t sum(uint32_t v) const {
#pragma unroll
    for (int o = MM / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o, MM);
    return v;
  }
  __device__ __forceinline__ uint64_t sum64(uint64_t v) const {
#pragma unroll
    for (int o = MM / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o, MM);
    return v;
  }
  __device__ __forceinline__ uint32_t vmin(uint32_t v) const {
#pragma unroll
    for (int o = MM / 2; o >= 1; o >>= 1) v = min(v, __shfl_xor_sync(FULL, v, o, MM));
    return v;
  }
  __device__ __forceinline__ uint32_t vmax(uint32_t v) const {
#pragma unroll
    for (int o = MM / 2; o >= 1; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o, MM));
    return v;
  }
};

__device__ __forceinline__ void lreport(DevStatus *ds, uint32_t code, int64_t item) {
  if (atomicCAS(&ds->code, 0u, code) == 0u) ds->item = (unsigned long long)item;
}

template <int MM>
__global__ void __launch_bounds__(256) k2_lane(const uint8_t *__restrict__ gimg, ImgLayout lay, LaneArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  stage_image(smem, gimg, lay.bytes, &mbar);
  const SmemProf P = smem_prof(smem, lay);
  const LSeg<MM> sg;
  const int g = sg.g;
  const int M = P.M;
  const bool real = g < M;
  const uint32_t mbits = real ? P.mask[g] : 0u;
  const uint32_t nallow = __popc(mbits);
  const uint32_t e_shallow = mbits ? (uint32_t)(__ffs(mbits) - 1) : 0u;

  bool active = false, exhausted = false;
  int64_t s = 0;
  SmemCfg C{};
  uint64_t base0 = 0, qb = 0;
  const uint32_t *Aq = a.arrival;
  uint32_t n = 0, head = 0, tail = 0, live = 0, last = 0, nxt = 0xFFFFFFFFu, ahead = 0;
  uint32_t t = 0, total = 0, served = 0, seq = 0, status = 0, iters = 0;
  uint64_t decisions = 0, candidates = 0, infeasible = 0;
  uint32_t completed = 0, viol = 0, cells = 0, maxd = 0;
  uint64_t sum_lat = 0, live_sum = 0, terms = 0;

  for (;;) {
    // ---- refill
    const bool need = !active && !exhausted;
    if (__any_sync(FULL, need)) {
      unsigned long long got = 0;
      if (need && g == 0) got = atomicAdd(a.work, 1ull);
      got = sg.bcast(got, 0);
      bool fresh = false;
      if (need) {
        if ((int64_t)got >= a.n_scen) exhausted = true;
        else fresh = true;
      }
      int k = 0;
      uint32_t n_new = 0, a0 = 0xFFFFFFFFu;
      if (fresh) {
        s = (int64_t)got;
        k = a.cfg_idx ? (int)a.cfg_idx[s] : 0;
        qb = 0;
        if (k < P.ncfg) {
          C = smem_cfg(P, k);
          base0 = a.arr_off[s * M];
          if (real) {
            qb = a.arr_off[s * M + g];
            n_new = (uint32_t)(a.arr_off[s * M + g + 1] - qb);
          }
        }
        Aq = a.arrival + qb;
        if (n_new) a0 = ldg(Aq);
      }
      const uint32_t tot = sg.sum(n_new);
      const uint32_t t0 = sg.vmin(a0);
      if (fresh) {
        active = true;
        n = n_new;
        total = tot;
        t = t0;
        head = tail = live = last = 0;
        nxt = a0;
        served = seq = iters = 0;
        status = (k < P.ncfg) ? (uint32_t)ES_OK : (uint32_t)ES_ERR_ARG;
        decisions = candidates = infeasible = 0;
        completed = viol = cells = maxd = 0;
        sum_lat = live_sum = terms = 0;
      }
    }
    if (__all_sync(FULL, exhausted)) break;

    for (;;) {
      if (active && status == ES_OK && ++iters > 2u * total + 4u) status = ES_ERR_INTERNAL;
      const bool run = active && status == ES_OK && served < total;
      // ---- a2: admission of this lane's queue, serial, 4 arrivals per step
      if (run) {
        const bool was_empty = head == tail;
        while (nxt <= t && tail < n) {
          // nxt = a[tail] is already known; look ahead 3 more
          const uint32_t v0 = nxt;
          const uint32_t v1 = tail + 1 < n ? ldg(Aq + tail + 1) : 0xFFFFFFFFu;
          const uint32_t v2 = tail + 2 < n ? ldg(Aq + tail + 2) : 0xFFFFFFFFu;
          const uint32_t v3 = tail + 3 < n ? ldg(Aq + tail + 3) : 0xFFFFFFFFu;
          const uint32_t v4 = tail + 4 < n ? ldg(Aq + tail + 4) : 0xFFFFFFFFu;
          // sortedness of the admitted prefix and its successor (Q19 input contract)
          bool bad = v0 < last;
          uint32_t c = 1;
          bad |= (tail + 1 < n) && v1 < v0;
          if (tail + 1 < n && v1 <= t) {
            c = 2;
            bad |= (tail + 2 < n) && v2 < v1;
            if (tail + 2 < n && v2 <= t) {
              c = 3;
              bad |= (tail + 3 < n) && v3 < v2;
              if (tail + 3 < n && v3 <= t) {
                c = 4;
                bad |= (tail + 4 < n) && v4 < v3;
              }
            }
          }
          last = c == 1 ? v0 : (c == 2 ? v1 : (c == 3 ? v2 : v3));
          nxt = c == 1 ? v1 : (c == 2 ? v2 : (c == 3 ? v3 : v4));
          tail += c;
          if (bad) {
            status = ES_ERR_UNSORTED;
            break;
          }
        }
        if (was_empty && tail > head) ahead = ldg(Aq + head);
      }
      const bool bad_any = sg.any(run && status == ES_ERR_UNSORTED);
      if (run && bad_any) status = ES_ERR_UNSORTED;
      const bool go = run && status == ES_OK;
      uint32_t len = go ? tail - head : 0u;
      const bool has = sg.any(len > 0u);
      if (__any_sync(FULL, go && !has)) {  // idle GPU: jump to the next arrival (Q12)
        const uint32_t tn = sg.vmin(go ? nxt : 0xFFFFFFFFu);
        if (go && !has) t = tn;
      }
      const bool dec = go && has;
      if (!dec) len = 0u;
      maxd = max(maxd, len);
      const uint32_t wmax = len ? t - ahead : 0u;
      // ---- clipped-for-everyone prefix [head, live): waits >= x_c (rare)
      if (live < head) live = head;
      if (len && wmax >= C.x_c) {
        while (live < tail && t - ldg(Aq + live) >= C.x_c) ++live;
      }
      const uint32_t c = len ? live - head : 0u;
      // ---- a3/a4 for this lane's candidate (Eq. 5, Eq. 6)
      uint32_t B = 0, e = 0, L = 0, thr = 0;
      uint64_t H = 0;
      bool feas = false;
      if (len) {
        const uint32_t cap = len < C.b_max ? len : C.b_max;
        const uint32_t bi = P.sm[C.off_bidx + cap];
        B = P.bs[bi];
        const uint32_t *row = P.lat + (size_t)g * P.E * P.nb + bi;
        const uint64_t lim = (uint64_t)C.tau;
        int best = -1;
#pragma unroll
        for (int ee = 0; ee < MAXE; ++ee) {
          if (ee < P.E && ((mbits >> ee) & 1u) && (uint64_t)wmax + row[ee * P.nb] <= lim) best = ee;
        }
        feas = best >= 0;
        e = feas ? (uint32_t)best : e_shallow;
        L = row[e * P.nb];
        thr = L < C.x_c ? C.x_c - L : 0u;
        H = L < C.x_c ? reinterpret_cast<const uint64_t *>(P.hb + C.off_H)[((size_t)g * P.E + e) * P.nb + bi] : 0ull;
      }
      // ---- a5/a6: stability score of every candidate (Eq. 3-4, reading Q5)
      const uint32_t tt = t;
      const uint32_t *Ah = Aq + head;
      uint64_t Sq = ~0ull;
      const bool fast = !__any_sync(FULL, len > 0u && wmax >= C.fast_lim);
      if (fast) {
        // no task can clip under any candidate: U_m = sum_all G - sum_own_served G
        uint64_t tot = 0, srv = 0;
        uint32_t p = 0;
        for (; p + 4u <= len; p += 4u) {  // 4 independent loads in flight
          const uint32_t x0 = ldg(Ah + p), x1 = ldg(Ah + p + 1), x2 = ldg(Ah + p + 2), x3 = ldg(Ah + p + 3);
          const uint64_t g0 = G_of(P, C, tt - x0), g1 = G_of(P, C, tt - x1);
          const uint64_t g2 = G_of(P, C, tt - x2), g3 = G_of(P, C, tt - x3);
          tot += (g0 + g1) + (g2 + g3);
          srv += (p < B ? g0 : 0ull) + (p + 1 < B ? g1 : 0ull) + (p + 2 < B ? g2 : 0ull) + (p + 3 < B ? g3 : 0ull);
        }
        for (; p < len; ++p) {
          const uint64_t gw = G_of(P, C, tt - ldg(Ah + p));
          tot += gw;
          if (p < B) srv += gw;
        }
        tot = sg.sum64(tot);
        if (len) {
          const uint64_t u = tot - srv;
          const uint64_t lo = H * u, hi = __umul64hi(H, u);
          Sq = (hi << (64 - F)) | (lo >> F);
        }
      } else {
        // general path: every candidate's threshold, tasks of this queue only
        uint32_t thrs[MM];
#pragma unroll
        for (int m = 0; m < MM; ++m) thrs[m] = sg.bcast(thr, m);
        uint32_t K[MM];
        uint64_t U[MM];
#pragma unroll
        for (int m = 0; m < MM; ++m) {
          K[m] = 0u;
          U[m] = 0ull;
        }
        for (uint32_t p = c; p < len; ++p) {
          const uint32_t w = tt - ldg(Ah + p);
          const uint32_t gw = G_of(P, C, w);
#pragma unroll
          for (int m = 0; m < MM; ++m) {
            if (m == g && p < B) continue;  // own served tasks
            if (w >= thrs[m]) K[m] += 1u;
            else U[m] += gw;
          }
        }
        // always-clipped prefix [0, c) of this queue: clipped for every
        // candidate except where it is candidate g's own served range
        const uint32_t cB = c < B ? c : B;
        uint32_t k_own = 0;
        uint64_t u_own = 0;
#pragma unroll
        for (int m = 0; m < MM; ++m) {
          const uint32_t kk = sg.sum(K[m] + (m == g ? c - cB : c));
          const uint64_t uu = sg.sum64(U[m]);
          if (m == g) {
            k_own = kk;
            u_own = uu;
          }
        }
        if (len) {
          const uint64_t lo = H * u_own, hi = __umul64hi(H, u_own);
          Sq = C.C_q * (uint64_t)k_own + ((hi << (64 - F)) | (lo >> F));
        }
      }
      // ---- a7: Eq. 7 argmin of (S_q, m), lowest m on ties (Q3)
      uint32_t mkey = len ? (uint32_t)g : 0xFFu;
      if (!__any_sync(FULL, len > 0u && Sq >= (1ull << 61))) {
        uint64_t key = len ? ((Sq << 3) | (uint64_t)g) : ~0ull;
#pragma unroll
        for (int o = 1; o < MM; o <<= 1) {
          const uint64_t ko = __shfl_xor_sync(FULL, key, o, MM);
          key = ko < key ? ko : key;
        }
        Sq = key >> 3;
        mkey = key == ~0ull ? 0xFFu : (uint32_t)(key & 7u);
      } else {
#pragma unroll
        for (int o = 1; o < MM; o <<= 1) {
          const uint64_t So = __shfl_xor_sync(FULL, Sq, o, MM);
          const uint32_t mo = __shfl_xor_sync(FULL, mkey, o, MM);
          if (So < Sq || (So == Sq && mo < mkey)) {
            Sq = So;
            mkey = mo;
          }
        }
      }
      const int src = (int)(mkey & (MM - 1));
      const uint32_t pk = sg.bcast(e | (feas ? 0x80u : 0u) | (B << 8), src);
      const uint32_t Lw = sg.bcast(L, src);
      const uint64_t qb_w = sg.bcast(qb, src);
      const uint32_t head_w = sg.bcast(head, src);
      const uint32_t ncand = __popc(sg.sbits(__ballot_sync(FULL, len > 0u)));
      // ---- a8: commit
      if (dec) {
        const uint32_t Bw = pk >> 8, ew = pk & 0x7Fu;
        const uint64_t done64 = (uint64_t)t + Lw;
        if (done64 > 0xFFFFFFFFull) {
          status = ES_ERR_RANGE;
        } else {
          const uint32_t done = (uint32_t)done64;
          decisions++;
          candidates += ncand;
          if (!(pk & 0x80u)) infeasible++;
          if (len) {
            cells += nallow;
            live_sum += len - c;
            terms += (uint64_t)(len - c) * ncand;
          }
          for (uint32_t j = (uint32_t)g; j < Bw; j += MM) {
            const uint64_t i = qb_w + head_w + j;
            const uint32_t T = done - ldg(a.arrival + i);  // Eq. 1: T = w + t
            if (a.completion) a.completion[i] = done;
            if (a.exit_used) a.exit_used[i] = (uint8_t)ew;
            const uint32_t q = seq + j;
            a.lat[base0 + q] = T;
            if (q >= C.warmup) {  // reading Q14
              completed++;
              sum_lat += T;
              viol += T > C.tau ? 1u : 0u;  // Eq. 2, strict
            }
          }
          if (a.dec_cap && g == 0 && (int64_t)decisions <= a.dec_cap) {
            const int64_t o = s * a.dec_cap + (int64_t)decisions - 1;
            if (a.dec_t) a.dec_t[o] = t;
            if (a.dec_m) a.dec_m[o] = (uint8_t)mkey;
            if (a.dec_e) a.dec_e[o] = (uint8_t)ew;
            if (a.dec_B) a.dec_B[o] = (uint16_t)Bw;
            if (a.dec_L) a.dec_L[o] = Lw;
            if (a.dec_S) a.dec_S[o] = Sq;
            if (a.dec_f) a.dec_f[o] = (pk & 0x80u) ? 1 : 0;
          }
          if ((uint32_t)g == mkey) {
            head += Bw;
            if (head < tail) ahead = ldg(Aq + head);  // consumed next decision
          }
          seq += Bw;
          served += Bw;
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
      if (g == 0) {
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
        if (status) lreport(a.dstat, status, s);
      }
      active = false;
    }
  }
}

template <int MM>
cudaError_t launch_mm(const uint8_t *img, const ImgLayout &lay, const LaneArgs &a, cudaStream_t st, int sms) {
  auto kern = k2_lane<MM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.bytes);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, lay.bytes);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  constexpr int SEG_PER_BLOCK = 256 / MM;
  int64_t blocks = (a.n_scen + SEG_PER_BLOCK - 1) / SEG_PER_BLOCK;
  const int64_t cap = (int64_t)sms * occ;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, 256, lay.bytes, st>>>(img, lay, a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_replay_lane(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                               const es_replay_out &out, DevStatus *dstat, uint32_t *work_ctr, cudaStream_t st,
                               int sms) {
  LaneArgs a;
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
  if (lay.M <= 2) return launch_mm<2>(img, lay, a, st, sms);
  if (lay.M <= 4) return launch_mm<4>(img, lay, a, st, sms);
  return launch_mm<8>(img, lay, a, st, sms);
}

}  // namespace es
