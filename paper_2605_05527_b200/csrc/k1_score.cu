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

template <int LPS, int MM>
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
    const Cand cand = cand_params<LPS, MM>(sg, P, C, len, wmax);
    bool bad = false;
    const Decision d = decide<LPS, MM>(sg, P, C, len, c, wmax, cand, [&](uint32_t p) {
      const uint32_t w = __ldg(W + p);
      // read-window validation: head-first waits must not increase (Q7)
      if (p > c && w > __ldg(W + p - 1)) bad = true;
      if (w >= C.x_c) bad = true;
      return w;
    });
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
    if (live_s && a.cand && sg.gl == 0 && g < M) a.cand[s * M + g] = (anybad || len == 0u) ? ~0ull : d.S_own;
  }
}

template <int LPS, int MM>
cudaError_t launch_t(const uint8_t *img, const ImgLayout &lay, const ScoreArgs &a, cudaStream_t st, int sms) {
  auto kern = k1_score<LPS, MM>;
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
