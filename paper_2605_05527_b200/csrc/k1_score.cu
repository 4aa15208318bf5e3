// k1_score.cu -- K1: independent scheduling decisions on queue snapshots.
//
// One warp segment of LPS lanes per snapshot (grid-stride), model g's queue
// owned by lane group g (decide.cuh).  Per snapshot the segment reads the
// (M+1) CSR offsets, the head wait of every queue and the live window of every
// queue -- tasks whose wait is already >= x_c are clipped for every candidate
// (Eq. 3) and are counted from the index by a GL-ary search on the
// non-increasing waits (reading Q7), never read.  This is the HBM-streaming
// form of the stability-score evaluation: no loop-carried state between
// snapshots.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "decide.cuh"

namespace es {
namespace {

struct ScoreArgs {
  int64_t n;
  const uint16_t *cfg_idx;
  const uint64_t *q_off;
  const uint32_t *waits;
  uint8_t *m, *e;
  uint16_t *B;
  uint32_t *L;
  uint64_t *S;
  uint8_t *flags;
  uint64_t *cand;
  DevStatus *dstat;
};

template <int LPS, int MM, bool POL>
__global__ void __launch_bounds__(256) k1_score(const uint8_t *__restrict__ gimg, ImgLayout lay, ScoreArgs a) {
  constexpr int GL = Seg<LPS, MM>::GL;
  constexpr int SPW = 32 / LPS;  // segments per warp
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  stage_image(smem, gimg, lay.bytes, &mbar);
  const SmemProf P = smem_prof(smem, lay);
  const Seg<LPS, MM> sg;
  const int g = sg.grp;
  const int M = P.M;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s0 = wid * SPW; s0 < a.n; s0 += nw * SPW) {  // warp-uniform loop
    const int64_t s = s0 + sg.seg;
    const bool live_s = s < a.n;
    const int k = live_s ? (a.cfg_idx ? (int)a.cfg_idx[s] : 0) : 0;
    const bool cfg_ok = k < P.ncfg;
    const SmemCfg C = smem_cfg(P, cfg_ok ? k : 0);
    uint64_t lo = 0;
    uint32_t len = 0;
    if (live_s && cfg_ok && g < M) {
      lo = a.q_off[s * M + g];
      len = (uint32_t)(a.q_off[s * M + g + 1] - lo);
    }
    const uint32_t *W = a.waits + lo;
    const uint32_t wmax = len ? __ldg(W) : 0u;
    // clipped-for-everyone prefix [0, c): first position with w < x_c
    uint32_t plo = 0, phi = len;  // invariant: w[plo] >= x_c, w[phi] < x_c (phi == len: sentinel)
    const bool srch = len > 0u && wmax >= C.x_c;
    if (__any_sync(FULL, srch)) {
      while (__any_sync(FULL, srch && phi - plo > 1u)) {
        const bool act = srch && phi - plo > 1u;
        const uint32_t nin = phi - plo - 1u;  // candidates strictly between
        const uint32_t q = plo + 1u + (uint32_t)(((uint64_t)(sg.gl + 1) * nin) / (GL + 1));
        const bool pr = act && __ldg(W + (q < phi ? q : phi - 1u)) >= C.x_c;
        const uint32_t cnt = __popc(sg.gbits(__ballot_sync(FULL, pr)));
        const uint32_t q_lo = __shfl_sync(FULL, q, g * GL + (cnt ? cnt - 1 : 0), LPS);
        const uint32_t q_hi = __shfl_sync(FULL, q, g * GL + (cnt < GL ? cnt : GL - 1), LPS);
        if (act) {
          if (cnt) plo = q_lo;
          if (cnt < (uint32_t)GL) phi = q_hi;
        }
      }
    }
    const uint32_t c = srch ? phi : 0u;
    const Cand cand = cand_params<LPS, MM, POL>(sg, P, C, len, wmax);
    bool bad = false;
    const bool fast = !__any_sync(FULL, len > 0u && wmax >= C.fast_lim);
    auto wait_at = [&](uint32_t p) {
      const uint32_t w = __ldg(W + p);
      // read-window validation: head-first waits must not increase (Q7)
      if (p > c && w > __ldg(W + p - 1)) bad = true;
      if (w >= C.x_c) bad = true;
      return w;
    };
    // Eq. 7 on the stability score, or a baseline policy (Q26) / GRID (Q28):
    // each branch runs warp-wide when some segment of the warp needs it
    const bool sc = !POL || policy_scores(C.policy);
    const bool grid = POL && C.policy == ES_POLICY_GRID;
    Decision d{};
    uint64_t own_grid = ~0ull;
    if (!POL || __any_sync(FULL, sc)) d = decide<LPS, MM>(sg, P, C, len, c, fast, cand, wait_at);
    if (POL && __any_sync(FULL, !sc && !grid)) {
      const Decision ds = select_simple<LPS, MM>(sg, cand, len, wmax, C);
      if (!sc && !grid) {
        d = ds;
        for (uint32_t p = c + sg.gl; p < len; p += GL) (void)wait_at(p);  // the read window's Q24 check
      }
    }
    if (POL && __any_sync(FULL, grid)) {
      uint32_t ng = 0u;
      uint64_t own = ~0ull;
      const Decision dg = decide_grid<LPS, MM>(sg, P, C, len, c, wmax, wait_at, ng, own);
      if (grid) {
        d = dg;
        own_grid = own;
      }
    }
    const bool anybad = sg.seg_any(bad) || !cfg_ok;
    const bool nowork = !sg.seg_any(len > 0u);
    if (live_s && sg.sl == 0) {
      if (anybad || nowork) {
        a.m[s] = 0; a.e[s] = 0; a.B[s] = 0; a.L[s] = 0; a.S[s] = 0;
        a.flags[s] = anybad ? ES_FLAG_BAD_INPUT : ES_FLAG_NO_WORK;
        if (!cfg_ok && atomicCAS(&a.dstat->code, 0u, (uint32_t)ES_ERR_ARG) == 0u) a.dstat->item = s;
      } else {
        a.m[s] = (uint8_t)d.m;
        a.e[s] = (uint8_t)d.e;
        a.B[s] = (uint16_t)d.B;
        a.L[s] = d.L;
        a.S[s] = d.S;
        a.flags[s] = d.feas ? ES_FLAG_FEASIBLE : 0u;
      }
    }
    const uint64_t own_score = sc ? d.S_own : (grid ? own_grid : ~0ull);  // LQF / EDF policies score nothing
    if (live_s && a.cand && sg.gl == 0 && g < M) a.cand[s * M + g] = (anybad || len == 0u) ? ~0ull : own_score;
  }
}

template <int LPS, int MM>
cudaError_t launch_t(const uint8_t *img, const ImgLayout &lay, const ScoreArgs &a, cudaStream_t st, int sms) {
  auto kern = lay.pol_mask == (1u << ES_POLICY_EDGESERVING) ? k1_score<LPS, MM, false> : k1_score<LPS, MM, true>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.bytes);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, lay.bytes);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  constexpr int SEG_PER_BLOCK = 256 / LPS;
  int64_t blocks = (a.n + SEG_PER_BLOCK - 1) / SEG_PER_BLOCK;
  const int64_t cap = (int64_t)sms * occ;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, 256, lay.bytes, st>>>(img, lay, a);
  return cudaGetLastError();
}

template <int LPS>
cudaError_t launch_lps(const uint8_t *img, const ImgLayout &lay, const ScoreArgs &a, cudaStream_t st, int sms) {
  if (lay.M <= 2) return launch_t<LPS, 2>(img, lay, a, st, sms);
  if (lay.M <= 4) return launch_t<LPS, 4>(img, lay, a, st, sms);
  return launch_t<LPS, 8>(img, lay, a, st, sms);
}

// ---------------------------------------------------------------------------
// Deep snapshots: one CTA (256 threads) per snapshot streams every live wait
// with coalesced loads; per-queue state and the candidates live in shared
// memory.  Same integers as k1_score (decide.cuh); only the mapping differs.
constexpr int BT = 128;
constexpr int BW = BT / 32;

__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ uint32_t warp_sum32(uint32_t v) { return redux_add(v); }

template <int MM>
__global__ void __launch_bounds__(BT) k1_block(const uint8_t *__restrict__ gimg, ImgLayout lay, ScoreArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ uint64_t s_lo[MM], s_H[MM], s_srv[MM], s_S[MM];
  __shared__ uint32_t s_len[MM], s_wmax[MM], s_c[MM], s_B[MM], s_e[MM], s_L[MM], s_thr[MM], s_feas[MM];
  __shared__ uint64_t s_redU[BW][MM];
  __shared__ uint32_t s_redK[BW][MM];
  __shared__ int s_bad, s_fast;
  stage_image(smem, gimg, lay.bytes, &mbar);
  const SmemProf P = smem_prof(smem, lay);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int M = P.M;
  // the next snapshot's CSR entries and head waits are prefetched into
  // registers of threads 0..M-1 while the current one streams
  auto fetch = [&](int64_t ss, int &kk, uint64_t &lo, uint32_t &len, uint32_t &wm) {
    kk = 0;
    lo = 0;
    len = 0;
    wm = 0;
    if (ss < a.n && tid < M) {
      kk = a.cfg_idx ? (int)a.cfg_idx[ss] : 0;
      if (kk < P.ncfg) {
        lo = a.q_off[ss * M + tid];
        len = (uint32_t)(a.q_off[ss * M + tid + 1] - lo);
        wm = len ? __ldg(a.waits + lo) : 0u;
      }
    }
  };
  int nk;
  uint64_t nlo;
  uint32_t nlen, nwm;
  fetch(blockIdx.x, nk, nlo, nlen, nwm);
  for (int64_t s = blockIdx.x; s < a.n; s += gridDim.x) {
    const int k = a.cfg_idx ? (int)a.cfg_idx[s] : 0;
    const bool cfg_ok = k < P.ncfg;
    const SmemCfg C = smem_cfg(P, cfg_ok ? k : 0);
    if (tid < MM) {
      s_lo[tid] = nlo;
      s_len[tid] = nlen;
      s_wmax[tid] = nwm;
      s_c[tid] = 0;
      s_srv[tid] = 0;
    }
    fetch(s + gridDim.x, nk, nlo, nlen, nwm);  // consumed next iteration
    if (tid == 0) {
      s_bad = cfg_ok ? 0 : 1;
      s_fast = 1;
    }
    __syncthreads();
    // clipped-for-everyone prefix of queue `warp`: 32-ary search on the
    // non-increasing waits (counted, never read)
    for (int qs = warp; qs < M; qs += BW) {  // warp-uniform
      if (!(s_len[qs] && s_wmax[qs] >= C.x_c)) continue;
      const uint32_t *W = a.waits + s_lo[qs];
      uint32_t plo = 0, phi = s_len[qs];  // w[plo] >= x_c, w[phi] < x_c (phi == len: sentinel)
      while (phi - plo > 1u) {  // warp-uniform
        const uint32_t nin = phi - plo - 1u;
        const uint32_t q = plo + 1u + (uint32_t)(((uint64_t)(lane + 1) * nin) / 33u);
        const bool pr = __ldg(W + (q < phi ? q : phi - 1u)) >= C.x_c;
        const uint32_t cnt = __popc(__ballot_sync(FULL, pr));
        const uint32_t q_lo = __shfl_sync(FULL, q, cnt ? cnt - 1 : 0);
        const uint32_t q_hi = __shfl_sync(FULL, q, cnt < 32 ? cnt : 31);
        if (cnt) plo = q_lo;
        if (cnt < 32u) phi = q_hi;
      }
      if (lane == 0) s_c[qs] = phi;
    }
    // Eq. 5-6 per candidate
    if (tid < M && s_len[tid]) {
      const uint32_t len = s_len[tid];
      const uint32_t cap = len < C.b_max ? len : C.b_max;
      const uint32_t bi = P.sm[C.off_bidx + cap];
      const uint32_t mbits = P.mask[tid];
      const uint32_t *row = P.lat + (size_t)tid * P.E * P.nb + bi;
      int best = -1;
      for (int e = 0; e < P.E; ++e)
        if (((mbits >> e) & 1u) && (uint64_t)s_wmax[tid] + row[e * P.nb] <= (uint64_t)C.tau) best = e;
      const uint32_t e = best >= 0 ? (uint32_t)best : (uint32_t)(__ffs(mbits) - 1);
      const uint32_t L = row[e * P.nb];
      s_B[tid] = P.bs[bi];
      s_e[tid] = e;
      s_L[tid] = L;
      s_feas[tid] = best >= 0;
      s_thr[tid] = L < C.x_c ? C.x_c - L : 0u;
      s_H[tid] = L < C.x_c ? reinterpret_cast<const uint64_t *>(P.hb + C.off_H)[((size_t)tid * P.E + e) * P.nb + bi]
                           : 0ull;
      if (s_wmax[tid] >= C.fast_lim) s_fast = 0;
    }
    __syncthreads();
    const bool fast = s_fast != 0;
    uint64_t U[MM];
    uint32_t K[MM];
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      U[m] = 0ull;
      K[m] = 0u;
    }
    uint64_t tot = 0;
    bool bad = false;
    // the two loops are separate so the compiler cannot if-convert both bodies
    if (fast) {
    for (int q = 0; q < M; ++q) {
      const uint32_t len = s_len[q], c0 = s_c[q], Bq = s_B[q];
      const uint32_t *W = a.waits + s_lo[q];
      // each warp streams a contiguous slice of the live window, UNR coalesced
      // 32-wide loads in flight; the neighbour check carries lane 31's value
      constexpr int UNR = 4;
      const uint32_t nlive = len > c0 ? len - c0 : 0u;
      const uint32_t per = ((nlive + BW * 32u - 1u) / (BW * 32u)) * 32u;  // slice, multiple of 32
      const uint32_t beg = c0 + warp * per, end = min(beg + per, len);
      uint32_t carry = (beg > c0 && beg < end) ? __ldg(W + beg - 1) : 0xFFFFFFFFu;
      for (uint32_t p0 = beg; p0 < end; p0 += UNR * 32u) {  // warp-uniform trip count
        uint32_t wv[UNR];
#pragma unroll
        for (int jj = 0; jj < UNR; ++jj) {
          const uint32_t p = p0 + jj * 32u + lane;
          wv[jj] = p < end ? __ldg(W + p) : 0u;
        }
#pragma unroll
        for (int jj = 0; jj < UNR; ++jj) {
          const uint32_t p = p0 + jj * 32u + lane;
          const uint32_t w = wv[jj];
          const bool valid = p < end;
          uint32_t prev = __shfl_up_sync(FULL, w, 1);
          if (lane == 0) prev = carry;
          carry = __shfl_sync(FULL, w, 31);
          if (valid && (w > prev || w >= C.x_c)) bad = true;  // read-window validation (Q7, Q24)
          if (!valid) continue;
          const uint32_t gw = G_of(P, C, w);
          tot += gw;
          if (p < Bq) atomicAdd(reinterpret_cast<unsigned long long *>(&s_srv[q]), (unsigned long long)gw);
        }
      }
    }
    } else {
      uint32_t thr_r[MM];
#pragma unroll
      for (int m = 0; m < MM; ++m) thr_r[m] = m < M ? s_thr[m] : 0xFFFFFFFFu;
    for (int q = 0; q < M; ++q) {
      const uint32_t len = s_len[q], c0 = s_c[q], Bq = s_B[q];
      const uint32_t *W = a.waits + s_lo[q];
      // each warp streams a contiguous slice of the live window, UNR coalesced
      // 32-wide loads in flight; the neighbour check carries lane 31's value
      constexpr int UNR = 4;
      const uint32_t nlive = len > c0 ? len - c0 : 0u;
      const uint32_t per = ((nlive + BW * 32u - 1u) / (BW * 32u)) * 32u;  // slice, multiple of 32
      const uint32_t beg = c0 + warp * per, end = min(beg + per, len);
      uint32_t carry = (beg > c0 && beg < end) ? __ldg(W + beg - 1) : 0xFFFFFFFFu;
      for (uint32_t p0 = beg; p0 < end; p0 += UNR * 32u) {  // warp-uniform trip count
        uint32_t wv[UNR];
#pragma unroll
        for (int jj = 0; jj < UNR; ++jj) {
          const uint32_t p = p0 + jj * 32u + lane;
          wv[jj] = p < end ? __ldg(W + p) : 0u;
        }
#pragma unroll
        for (int jj = 0; jj < UNR; ++jj) {
          const uint32_t p = p0 + jj * 32u + lane;
          const uint32_t w = wv[jj];
          const bool valid = p < end;
          uint32_t prev = __shfl_up_sync(FULL, w, 1);
          if (lane == 0) prev = carry;
          carry = __shfl_sync(FULL, w, 31);
          if (valid && (w > prev || w >= C.x_c)) bad = true;  // read-window validation (Q7, Q24)
          if (!valid) continue;
          const uint32_t gw = G_of(P, C, w);
#pragma unroll
          for (int m = 0; m < MM; ++m) {
            if (m == q && p < Bq) continue;  // candidate m's own served tasks
            if (w >= thr_r[m]) K[m] += 1u;
            else U[m] += gw;
          }
        }
      }
    }
    }
    if (__any_sync(FULL, bad) && lane == 0) s_bad = 1;
    if (fast) {
      tot = warp_sum64(tot);
      if (lane == 0) s_redU[warp][0] = tot;
    } else {
#pragma unroll
      for (int m = 0; m < MM; ++m) {
        const uint64_t u = warp_sum64(U[m]);
        const uint32_t kk = warp_sum32(K[m]);
        if (lane == 0) {
          s_redU[warp][m] = u;
          s_redK[warp][m] = kk;
        }
      }
    }
    __syncthreads();
    if (tid < M) {
      uint64_t S = ~0ull;
      if (s_len[tid]) {
        uint64_t u = 0, kk = 0;
        if (fast) {
          for (int w = 0; w < BW; ++w) u += s_redU[w][0];
          u -= s_srv[tid];
        } else {
          for (int w = 0; w < BW; ++w) {
            u += s_redU[w][tid];
            kk += s_redK[w][tid];
          }
          uint32_t cpre = 0;
          for (int q = 0; q < M; ++q) cpre += s_c[q];
          const uint32_t cB = s_c[tid] < s_B[tid] ? s_c[tid] : s_B[tid];
          kk += cpre - cB;
        }
        const uint64_t H = s_H[tid];
        const uint64_t lo = H * u, hi = __umul64hi(H, u);
        S = C.C_q * kk + ((hi << (64 - F)) | (lo >> F));
      }
      s_S[tid] = S;
    }
    __syncthreads();
    if (tid == 0) {
      int best = -1;
      for (int m = 0; m < M; ++m)
        if (s_len[m] && (best < 0 || s_S[m] < s_S[best])) best = m;  // (S, m): lowest m on ties
      if (s_bad || best < 0) {
        a.m[s] = 0; a.e[s] = 0; a.B[s] = 0; a.L[s] = 0; a.S[s] = 0;
        a.flags[s] = s_bad ? ES_FLAG_BAD_INPUT : ES_FLAG_NO_WORK;
        if (!cfg_ok && atomicCAS(&a.dstat->code, 0u, (uint32_t)ES_ERR_ARG) == 0u) a.dstat->item = s;
      } else {
        a.m[s] = (uint8_t)best;
        a.e[s] = (uint8_t)s_e[best];
        a.B[s] = (uint16_t)s_B[best];
        a.L[s] = s_L[best];
        a.S[s] = s_S[best];
        a.flags[s] = s_feas[best] ? ES_FLAG_FEASIBLE : 0u;
      }
    }
    if (a.cand && tid < M) a.cand[s * M + tid] = (s_bad || !s_len[tid]) ? ~0ull : s_S[tid];
    __syncthreads();
  }
}

template <int MM>
cudaError_t launch_block(const uint8_t *img, const ImgLayout &lay, const ScoreArgs &a, cudaStream_t st, int sms) {
  auto kern = k1_block<MM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.bytes);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, BT, lay.bytes);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  int64_t blocks = a.n;
  const int64_t cap = (int64_t)sms * occ;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, BT, lay.bytes, st>>>(img, lay, a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_score(const uint8_t *img, const ImgLayout &lay, const es_snapshots &sn,
                         const es_decisions &out, DevStatus *dstat, cudaStream_t st, int sms) {
  ScoreArgs a;
  a.n = sn.n;
  a.cfg_idx = sn.cfg_idx;
  a.q_off = sn.q_off;
  a.waits = sn.waits_us;
  a.m = out.m;
  a.e = out.e;
  a.B = out.B;
  a.L = out.L_us;
  a.S = out.score_q;
  a.flags = out.flags;
  a.cand = out.cand_score_q;
  a.dstat = dstat;
  // deep snapshots (>= 1024 waits each on average): one CTA per snapshot
  const char *k1 = getenv("ES_K1");
  const bool deep = sn.n_waits > 0 && sn.n > 0 && sn.n_waits / sn.n >= 1024;
  // the baseline policies and GRID run on the warp-segment mapping only
  const bool pol = lay.pol_mask != (1u << ES_POLICY_EDGESERVING);
  if (!pol && (k1 ? strcmp(k1, "stream") == 0 : deep)) return launch_score_stream(img, lay, sn, out, dstat, st, sms);
  if (!pol && k1 && strcmp(k1, "block") == 0) {
    if (lay.M <= 2) return launch_block<2>(img, lay, a, st, sms);
    if (lay.M <= 4) return launch_block<4>(img, lay, a, st, sms);
    return launch_block<8>(img, lay, a, st, sms);
  }
  int lps = 16;
  if (const char *env = getenv("ES_K1_LPS")) {
    const int v = atoi(env);
    if (v == 8 || v == 16 || v == 32) lps = v;
  }
  if (lps == 8) return launch_lps<8>(img, lay, a, st, sms);
  if (lps == 16) return launch_lps<16>(img, lay, a, st, sms);
  return launch_lps<32>(img, lay, a, st, sms);
}

}  // namespace es
