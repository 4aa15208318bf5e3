// k1_score.cu -- K1: independent scheduling decisions on queue snapshots
// (Algorithm 1, on the system state of S:112-115).  Two mappings:
//
// k1_thread (Algorithm 1, short snapshots; the default below 1,024 waits per
//   snapshot): a lane pair per snapshot for the per-queue logic, one balanced
//   pass of the warp for the Eq. 3-4 sums (see the comment above it).
// k1_score (warp segments): one segment of LPS lanes per snapshot
//   (grid-stride), model g's queue owned by lane group g (decide.cuh); used
//   for the baseline policies and GRID, and for k1_thread's clip-path list.
//   Per snapshot the segment reads the (M+1) CSR offsets, the head wait of
//   every queue and the live window of every queue -- tasks whose wait is
//   already >= x_c are clipped for every candidate (Eq. 3) and are
//   counted from the index by a GL-ary search on the non-increasing waits
//   (reading Q7), never read.
// Deep snapshots (>= 1,024 waits on average) take the streamed mapping of
// k1_stream.cu.  All mappings compute the same integers (tested invariant).
#include <cuda_runtime.h>

#include <algorithm>
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
  uint32_t stage_bytes;  // image prefix staged per CTA (lay.bytes, or lay.core_bytes: H read from global)
  // clip-path hand-over from k1_thread to k1_score: list of snapshot indices
  // and its length (device); k1_score walks list[0 .. *list_n) when non-null
  uint32_t *list;
  unsigned long long *list_n;
};

template <int LPS, int MM, bool POL>
__global__ void __launch_bounds__(256) k1_score(const uint8_t *__restrict__ gimg, ImgLayout lay, ScoreArgs a) {
  constexpr int GL = Seg<LPS, MM>::GL;
  constexpr int SPW = 32 / LPS;  // segments per warp
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  stage_image(smem, gimg, a.stage_bytes, &mbar);
  SmemProf P = smem_prof(smem, lay);
  if (a.stage_bytes < lay.bytes) P.hb = gimg;  // H tables stay in global memory (L1-cached)
  const Seg<LPS, MM> sg;
  const int g = sg.grp;
  const int M = P.M;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nitems = a.list ? (int64_t)*a.list_n : a.n;  // k1_thread's clip-path list, or every snapshot
  for (int64_t s0 = wid * SPW; s0 < nitems; s0 += nw * SPW) {  // warp-uniform loop
    const bool live_s = s0 + sg.seg < nitems;
    const int64_t s = !live_s ? 0 : a.list ? (int64_t)a.list[s0 + sg.seg] : s0 + sg.seg;
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
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a.stage_bytes);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, a.stage_bytes);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  constexpr int SEG_PER_BLOCK = 256 / LPS;
  int64_t blocks = (a.n + SEG_PER_BLOCK - 1) / SEG_PER_BLOCK;
  const int64_t cap = (int64_t)sms * occ;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, 256, a.stage_bytes, st>>>(img, lay, a);
  return cudaGetLastError();
}

template <int LPS>
cudaError_t launch_lps(const uint8_t *img, const ImgLayout &lay, const ScoreArgs &a, cudaStream_t st, int sms) {
  if (lay.M <= 2) return launch_t<LPS, 2>(img, lay, a, st, sms);
  if (lay.M <= 4) return launch_t<LPS, 4>(img, lay, a, st, sms);
  return launch_t<LPS, 8>(img, lay, a, st, sms);
}

// ---------------------------------------------------------------------------
// Short snapshots under Algorithm 1: one or two LANES per snapshot (k1_thread).
// A warp segment spends warp-wide shuffles and reductions on a handful of
// waits (harvested cfg3 states: 33 waits over 8 queues on average, median
// queue 2), so here a lane (or a lane pair, each with half the queues) owns a
// snapshot's decision logic:
//   per queue q: Eq. 5 (bidx, Q8) and Eq. 6 (a count over the padded
//   exit-minor latency row, Q2); S_q(m) = floor(H(L_m) (tot - srv_m) /
//   2^28) and the Eq. 7 argmin (S, m) (Q3) -- the fast path of decide.cuh
//   (same integers), valid when every head wait is below x_c - max L.
// The sums come from one balanced pass of the whole warp: the waits of the
// warp's 16 (32) consecutive snapshots are one contiguous region, read as 16-byte
// vectors (8 waits per lane, 256 per trip) whatever the queue-length mix; G(w)
// (Q5) of every wait with the SLO's tables (a warp whose snapshots mix SLOs
// takes the per-lane loop below), an exclusive running sum E over the region
// into shared memory (chunks of `cap` positions), and each lane reads E at its
// queues' boundaries:  tot = E(end_M) - E(start_0),  srv_m = E(start_m +
// min(B*_m, len_m)) - E(start_m)  (own served head).  Read-window check
// (Q24): a wait above its predecessor inside a queue (queue starts marked in a
// per-chunk bitmap) sends the warp to the per-lane loop, which flags it.
// A snapshot with a head at or past x_c - max L (some task may clip) is
// appended to a list that the warp-segment kernel (k1_score, general clip
// path) scores afterwards.

__device__ __forceinline__ uint32_t lds32(uint32_t a) {  // read-only tables / bitmap after a __syncwarp
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds32_ro(uint32_t a) {  // staged profile tables (never written after staging)
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, uint64_t x) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(x) : "memory");
}
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}

// G(w) with 32-bit shared addresses: v4 = 4 (w + r) (exact: x_c + 1024 < 2^30
// for tau <= 2^20, Q25); the A index is clamped (an inverted input is flagged
// and its value unused)
struct GSh {
  uint32_t sA, sBt, r4, nA1;
  __device__ __forceinline__ uint32_t operator()(uint32_t w) const {
    const uint32_t v4 = w * 4u + r4;
    const uint32_t h = min(v4 >> (SBITS + 2), nA1);
    return (uint32_t)(((uint64_t)lds32_ro(sA + 4u * h) * (uint64_t)lds32_ro(sBt + (v4 & (4u * S - 4u)))) >> F);
  }
};

// LPN lanes per snapshot (1 or 2): lane h of a snapshot owns its queues
// q = h HQ + j, j < HQ = MM / LPN; the snapshot's total, the Eq. 7 argmin and
// the per-lane fallback combine over the LPN lanes with one xor-shuffle.
template <int MM, int LPN, int NT>
__global__ void __launch_bounds__(NT, 1) k1_thread(const uint8_t *__restrict__ gimg, ImgLayout lay, ScoreArgs a,
                                                  uint32_t cap) {
  constexpr int HQ = MM / LPN;       // queues per lane
  constexpr int SPI = 32 / LPN;      // snapshots per warp iteration
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  stage_image(smem, gimg, a.stage_bytes, &mbar);
  SmemProf P = smem_prof(smem, lay);
  if (a.stage_bytes < lay.bytes) P.hb = gimg;  // H tables stay in global memory (L1-cached)
  const int M = P.M;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int h = LPN == 1 ? 0 : (lane & (LPN - 1));  // this lane's half of the snapshot's queues
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  // this warp's scratch: E [cap + 4] u64, then the queue-start bitmap [cap / 32]
  const uint32_t sE = sbase + ((a.stage_bytes + 127u) & ~127u) + (uint32_t)wib * (cap * 8u + 32u + cap / 8u);
  const uint32_t sBits = sE + cap * 8u + 32u;
  const int64_t nwarps = (int64_t)gridDim.x * NW;
  auto out_empty = [&](int64_t s, uint8_t flag) {  // by lane h == 0
    a.m[s] = 0; a.e[s] = 0; a.B[s] = 0; a.L[s] = 0; a.S[s] = 0;
    a.flags[s] = flag;
    if (a.cand)
      for (int q = 0; q < M; ++q) a.cand[s * M + q] = ~0ull;
  };
  auto pair_or = [&](bool v) {  // OR over the snapshot's LPN lanes; whole warp (no shuffle is skipped)
    int x = v ? 1 : 0;
#pragma unroll
    for (int o = 1; o < LPN; o <<= 1) x |= __shfl_xor_sync(FULL, x, o);
    return x != 0;
  };
  // warps stride over groups of SPI snapshots (snapshot sizes are correlated
  // along the batch: strided groups balance the warps); the next group's CSR
  // rows and SLO indices are prefetched into L2 at the start of a group, its
  // waits region once its bounds (loaded early) are known
  const int64_t stride = nwarps * SPI;
  for (int64_t s0 = ((int64_t)blockIdx.x * NW + wib) * SPI; s0 < a.n; s0 += stride) {  // warp-uniform
    const int64_t s = s0 + lane / LPN;
    const bool live = s < a.n;
    const int64_t s1 = s0 + stride;  // the next group
    uint64_t nb = 0ull;  // lane 0: its region start, lane 31: its region end
    if (s1 < a.n) {
      const char *nq = reinterpret_cast<const char *>(a.q_off + s1 * M);
      if ((uint32_t)lane * 128u < (uint32_t)SPI * 8u * (uint32_t)M + 8u)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(nq + 128 * lane));
      if (lane == 30 && a.cfg_idx) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.cfg_idx + s1));
      if (lane == 0) nb = __ldg(a.q_off + s1 * M);
      if (lane == 31) nb = __ldg(a.q_off + min(s1 + SPI, a.n) * M);
    }
    const int k = live ? (a.cfg_idx ? (int)a.cfg_idx[s] : 0) : 0;
    const bool cfg_ok = k < P.ncfg;
    const SmemCfg C = smem_cfg(P, cfg_ok ? k : 0);
    // this lane's CSR boundaries (queues h HQ .. h HQ + HQ, clamped to M) and
    // head waits; offsets kept relative to the group's region start R0 (a
    // region of 2^31 waits or more goes to the warp segments whole)
    uint32_t rel[HQ + 1];
    uint64_t R0, R1;
    bool huge;
    {
      uint64_t off[HQ + 1];
#pragma unroll
      for (int j = 0; j <= HQ; ++j) off[j] = live ? __ldg(a.q_off + s * M + min(h * HQ + j, M)) : 0ull;
      R0 = __shfl_sync(FULL, off[0], 0);
      const int ll = 31 - __clz(__ballot_sync(FULL, live));  // the last live snapshot's last lane
      R1 = __shfl_sync(FULL, off[HQ], ll);
      huge = R1 - R0 >= (1ull << 31);
#pragma unroll
      for (int j = 0; j <= HQ; ++j) rel[j] = live ? (uint32_t)(off[j] - R0) : 0u;
    }
    {  // L2 prefetch of the next group's waits region (its bounds loaded at the top)
      const uint64_t n0 = __shfl_sync(FULL, nb, 0), n1 = __shfl_sync(FULL, nb, 31);
      const char *nw = reinterpret_cast<const char *>(a.waits + n0);
      for (uint64_t b = 128u * (uint64_t)lane; b < 4u * (n1 - n0); b += 4096u) asm volatile("prefetch.global.L2 [%0];" ::"l"(nw + b));
    }
    const uint32_t *Wr = a.waits + R0;  // the region's waits
    uint32_t pk[HQ];  // e | bi << 4 | feasible << 12 | min(B*, len) << 16; 0xFFFFFFFF: empty queue
    bool active = false;
    {
      uint32_t head[HQ];
      bool slow = false, any = false;
#pragma unroll
      for (int j = 0; j < HQ; ++j) {
        const bool has = rel[j + 1] > rel[j];
        head[j] = has ? __ldg(Wr + rel[j]) : 0u;
        slow |= has && head[j] >= C.fast_lim;
        any |= has;
      }
      slow = pair_or(slow);
      any = pair_or(any);
      if (live) {
        if (!cfg_ok) {
          if (h == 0) {
            out_empty(s, ES_FLAG_BAD_INPUT);
            if (atomicCAS(&a.dstat->code, 0u, (uint32_t)ES_ERR_ARG) == 0u) a.dstat->item = s;
          }
        } else if (slow || huge) {  // some task may clip: the general path (k1_score on the list)
          if (h == 0) a.list[atomicAdd(a.list_n, 1ull)] = (uint32_t)s;
        } else if (!any) {
          if (h == 0) out_empty(s, ES_FLAG_NO_WORK);
        } else {
          active = true;
        }
      }
      // Eq. 5 / Eq. 6 of this lane's queues
#pragma unroll
      for (int j = 0; j < HQ; ++j) {
        pk[j] = 0xFFFFFFFFu;
        const int q = h * HQ + j;
        const uint32_t len = rel[j + 1] - rel[j];
        if (!active || !len) continue;
        const uint32_t cap_b = len < C.b_max ? len : C.b_max;
        const uint32_t bi = P.sm[C.off_bidx + cap_b];
        const uint32_t nsv = min((uint32_t)P.bs[bi], len);
        const uint32_t mbits = P.mask[q];
        const unsigned bits = head[j] <= C.tau ? ((1u << eq6_count(P, q, bi, C.tau - head[j])) - 1u) & mbits : 0u;
        const uint32_t e = bits ? 31u - __clz(bits) : (uint32_t)(__ffs(mbits) - 1);
        pk[j] = e | (bi << 4) | (bits ? 0x1000u : 0u) | (nsv << 16);
      }
    }
    const unsigned b_act = __ballot_sync(FULL, active);
    if (b_act == 0u) continue;
    uint64_t tot = 0ull, srv[HQ];  // tot: this lane's part of the snapshot total
#pragma unroll
    for (int j = 0; j < HQ; ++j) srv[j] = 0ull;
    bool bad = false;
    // ---- the balanced pass: one SLO across the warp's active snapshots
    const int kf = __shfl_sync(FULL, k, __ffs(b_act) - 1);
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(Wr);
    const uint32_t mis = (uint32_t)((a0 & 15u) >> 2);  // waits before R0 in its 16-byte vector
    bool flat = __all_sync(FULL, !active || k == kf);
    if (flat) {
      const uint32_t *abase = reinterpret_cast<const uint32_t *>(a0 & ~(uintptr_t)15u);  // relative position 0
      const uint32_t nrel = (uint32_t)(R1 - R0) + mis;
      const SmemCfg Cf = smem_cfg(P, kf);
      const GSh G{sbase + Cf.off_A, sbase + Cf.off_Bt, 4u * Cf.r, Cf.nA1};
      uint64_t carry = 0ull;
      uint32_t pcarry = 0xFFFFFFFFu;
      bool inv = false;
      const uint32_t lo_x = rel[0] + mis, hi_x = rel[HQ] + mis;  // this lane's span of boundaries
      for (uint32_t cb = 0; cb < nrel; cb += cap) {  // warp-uniform chunks
        const uint32_t ce = min(cb + cap, nrel);
        for (uint32_t j = lane; j < cap / 32u; j += 32u) asm volatile("st.shared.u32 [%0], 0;" ::"r"(sBits + 4u * j));
        __syncwarp();
        if (live && hi_x >= cb && lo_x < ce) {  // queue starts of this chunk (no predecessor check, Q24)
#pragma unroll
          for (int j = 0; j < HQ; ++j) {
            const uint32_t x = rel[j] + mis;
            if (h * HQ + j < M && x >= cb && x < ce)
              asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(sBits + 4u * ((x - cb) >> 5)), "r"(1u << ((x - cb) & 31u)));
          }
        }
        __syncwarp();
        for (uint32_t tb = cb; tb < ce; tb += 256u) {  // warp-uniform trips of 8 waits per lane
          const uint32_t p = tb + 8u * (uint32_t)lane;
          uint32_t w[8];
          // positions outside [mis, nrel) (the region's edge vectors) are masked
          const uint32_t vm = p >= mis && p + 8u <= nrel
                                  ? 0xFFu
                                  : (p + 8u <= mis || p >= nrel ? 0u
                                                                : (0xFFu << (p < mis ? mis - p : 0u)) &
                                                                      (0xFFu >> (p + 8u > nrel ? p + 8u - nrel : 0u)));
          if (vm == 0xFFu) {
            const uint4 v0 = __ldg(reinterpret_cast<const uint4 *>(abase + p));
            const uint4 v1 = __ldg(reinterpret_cast<const uint4 *>(abase + p + 4u));
            w[0] = v0.x; w[1] = v0.y; w[2] = v0.z; w[3] = v0.w;
            w[4] = v1.x; w[5] = v1.y; w[6] = v1.z; w[7] = v1.w;
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = (vm >> i) & 1u ? __ldg(abase + p + i) : 0u;
          }
          // Q24: a wait above its predecessor, except at a queue start
          const uint32_t sb8 = (lds32(sBits + 4u * ((tb - cb) / 32u + (uint32_t)lane / 4u)) >> (8u * (lane & 3))) & 0xFFu;
          uint32_t prev = __shfl_up_sync(FULL, w[7], 1);
          if (lane == 0) prev = pcarry;
          pcarry = __shfl_sync(FULL, w[7], 31);
          uint32_t gt = w[0] > prev ? 1u : 0u;
#pragma unroll
          for (int i = 1; i < 8; ++i) gt |= w[i] > w[i - 1] ? 1u << i : 0u;
          inv |= (gt & vm & ~sb8) != 0u;
          // G of every loaded wait (masked positions hold 0: G(0) is in range)
          uint32_t g[8];
          uint64_t ls = 0ull;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            g[i] = G(w[i]) & (0u - ((vm >> i) & 1u));
            ls += g[i];
          }
          uint64_t sc = ls;  // warp inclusive scan of the lane sums
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint64_t t = __shfl_up_sync(FULL, sc, o);
            if (lane >= o) sc += t;
          }
          uint64_t e = carry + sc - ls;  // E at position p
          const uint32_t ea = sE + 8u * (p - cb);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            sts64(ea + 8u * i, e);
            e += g[i];
          }
          carry += __shfl_sync(FULL, sc, 31);
        }
        __syncwarp();
        if (active && hi_x >= cb && lo_x < ce) {  // this lane's queue boundaries inside the chunk
#pragma unroll
          for (int j = 0; j <= HQ; ++j) {
            const uint32_t x = rel[j] + mis;
            const bool first = h == 0 && j == 0, last = h == LPN - 1 && j == HQ;  // the snapshot's start / end
            const bool own = j < HQ && h * HQ + j < M;
            if ((first || last || own) && x >= cb && x < ce) {
              const uint64_t e = lds64(sE + 8u * (x - cb));
              if (first) tot -= e;
              if (last) tot += e;
              if (own) srv[j] -= e;
            }
            if (own) {
              const uint32_t x1 = x + (pk[j] >> 16);
              if (x1 >= cb && x1 < ce) srv[j] += lds64(sE + 8u * (x1 - cb));
            }
          }
        }
        __syncwarp();
      }
      if (active && hi_x == nrel) {  // boundaries at the region's end: E = the final sum
#pragma unroll
        for (int j = 0; j <= HQ; ++j) {
          const uint32_t x = rel[j] + mis;
          const bool first = h == 0 && j == 0, last = h == LPN - 1 && j == HQ;
          const bool own = j < HQ && h * HQ + j < M;
          if (x == nrel) {
            if (first) tot -= carry;
            if (last) tot += carry;
            if (own) srv[j] -= carry;
          }
          if (own && x + (pk[j] >> 16) == nrel) srv[j] += carry;
        }
      }
      flat = !__any_sync(FULL, inv);  // an inversion: redo the warp per lane (flags it exactly)
    }
    if (!flat) {
      // ---- per-lane loop (mixed SLOs or an inversion in the region)
      tot = 0ull;
      if (active) {
        const GSh G{sbase + C.off_A, sbase + C.off_Bt, 4u * C.r, C.nA1};
#pragma unroll
        for (int j = 0; j < HQ; ++j) {
          srv[j] = 0ull;
          const uint32_t len = rel[j + 1] - rel[j];
          if (!len) continue;
          const uint32_t *W = Wr + rel[j];
          uint32_t prev = __ldg(W);
          uint64_t Q = G(prev), sv = Q;  // nsv >= 1
          for (uint32_t p = 1; p < len; ++p) {
            const uint32_t w = __ldg(W + p);
            bad |= w > prev;
            prev = w;
            const uint64_t g = G(w);
            Q += g;
            if (p < (pk[j] >> 16)) sv += g;
          }
          tot += Q;
          srv[j] = sv;
        }
      }
      bad = pair_or(bad);
    }
#pragma unroll
    for (int o = 1; o < LPN; o <<= 1) tot += __shfl_xor_sync(FULL, tot, o);  // the snapshot's total over its lanes
    // Eq. 3-4 on each candidate's predicted state, Eq. 7 argmin (S, m)
    uint64_t bS = ~0ull;
    uint32_t bq = 0xFFu, bpk = 0u;
    if (active && !bad) {
      const uint64_t *Hq = reinterpret_cast<const uint64_t *>(P.hb + C.off_H);
#pragma unroll
      for (int j = 0; j < HQ; ++j) {
        const int q = h * HQ + j;
        if (q >= M) continue;
        uint64_t Sv = ~0ull;
        if (pk[j] != 0xFFFFFFFFu) {
          const uint32_t e = pk[j] & 15u, bi = (pk[j] >> 4) & 0xFFu;
          const uint64_t Hc = Hq[((size_t)q * P.E + e) * P.nb + bi];
          const uint64_t H = Hc == ~0ull ? 0ull : Hc;  // L >= x_c: every task clips (k_build_tables)
          const uint64_t u = tot - srv[j];
          const uint64_t lo = H * u, hi = __umul64hi(H, u);
          Sv = (hi << (64 - F)) | (lo >> F);
          if (Sv < bS || bq == 0xFFu) {
            bS = Sv;
            bq = (uint32_t)q;
            bpk = pk[j];
          }
        }
        if (a.cand) a.cand[s * M + q] = Sv;
      }
    }
#pragma unroll
    for (int o = 1; o < LPN; o <<= 1) {  // (S, m) argmin over the snapshot's lanes (lowest m on ties, Q3)
      const uint64_t oS = __shfl_xor_sync(FULL, bS, o);
      const uint32_t oq = __shfl_xor_sync(FULL, bq, o), opk = __shfl_xor_sync(FULL, bpk, o);
      if (oq != 0xFFu && (bq == 0xFFu || oS < bS || (oS == bS && oq < bq))) {
        bS = oS;
        bq = oq;
        bpk = opk;
      }
    }
    if (!active || h != 0) continue;
    if (bad) {
      out_empty(s, ES_FLAG_BAD_INPUT);
      continue;
    }
    const uint32_t e = bpk & 15u, bi = (bpk >> 4) & 0xFFu;
    a.m[s] = (uint8_t)bq;
    a.e[s] = (uint8_t)e;
    a.B[s] = P.bs[bi];
    a.L[s] = P.latT[((size_t)bq * P.nb + bi) * 8u + e];
    a.S[s] = bS;
    a.flags[s] = (bpk & 0x1000u) ? ES_FLAG_FEASIBLE : 0u;
  }
}

template <int MM, int LPN, int NT>
cudaError_t launch_thread_t(const uint8_t *img, const ImgLayout &lay, ScoreArgs a, cudaStream_t st, int sms) {
  // the clip-path list (u32 indices) and its counter: stream-ordered scratch
  void *scratch = nullptr;
  const size_t list_bytes = ((size_t)a.n * sizeof(uint32_t) + 15u) & ~(size_t)15u;
  cudaError_t e = cudaMallocAsync(&scratch, list_bytes + 16u, st);
  if (e != cudaSuccess) return e;
  a.list = static_cast<uint32_t *>(scratch);
  a.list_n = reinterpret_cast<unsigned long long *>(static_cast<uint8_t *>(scratch) + list_bytes);
  e = cudaMemsetAsync(a.list_n, 0, sizeof(unsigned long long), st);
  // one CTA of NT threads per SM; what shared memory the staged image leaves
  // becomes each warp's E chunk (cap positions, a multiple of 256)
  constexpr int NW = NT / 32;
  int dev = 0, optin = 0;
  if (e == cudaSuccess) e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t img_b = ((size_t)a.stage_bytes + 127u) & ~(size_t)127u;
  const int64_t room = (int64_t)optin - (int64_t)img_b - 256;
  int64_t capw = room / NW;  // bytes per warp: cap * 8 + 32 + cap / 8
  uint32_t cap = (uint32_t)std::min<int64_t>(std::max<int64_t>((capw - 32) * 8 / 65, 0) & ~255ll, 4096);
  if (e == cudaSuccess && cap < 256u) e = cudaErrorInvalidConfiguration;
  const size_t dyn = img_b + (size_t)NW * (cap * 8u + 32u + cap / 8u);
  auto kern = k1_thread<MM, LPN, NT>;
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e == cudaSuccess) {
    int64_t blocks = (a.n * LPN + NT - 1) / NT;
    if (blocks > sms) blocks = sms;
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, NT, dyn, st>>>(img, lay, a, cap);
    e = cudaGetLastError();
  }
  // the listed (clip-path) snapshots: the warp-segment kernel, general path
  if (e == cudaSuccess) e = launch_t<16, MM>(img, lay, a, st, sms);
  const cudaError_t f = cudaFreeAsync(scratch, st);
  return e != cudaSuccess ? e : f;
}

// two lanes per snapshot, 16 warps per SM (measured on the harvested cfg3
// batch: 1.36 ms; one lane per snapshot 1.42 ms; two lanes at 24 warps 1.39 ms;
// four lanes 1.60 ms at 16 warps, 1.40 ms at 24)
template <int MM>
cudaError_t launch_thread(const uint8_t *img, const ImgLayout &lay, ScoreArgs a, cudaStream_t st, int sms) {
  return launch_thread_t<MM, 2, 512>(img, lay, a, st, sms);
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
  a.list = nullptr;
  a.list_n = nullptr;
  // many SLOs (image above 48 KB, e.g. cfg3's nine): stage only the core so
  // that 4 CTAs fit per SM; each candidate's H is one L1-cached global load
  a.stage_bytes = lay.bytes > 48u * 1024u ? lay.core_bytes : lay.bytes;
  // deep snapshots (>= 1024 waits each on average): the three-phase stream;
  // Algorithm 1 on short snapshots: one thread per snapshot (clip-path ones
  // handed to the warp segments); the baseline policies and GRID: warp segments
  const char *k1 = getenv("ES_K1");
  const bool deep = sn.n_waits > 0 && sn.n > 0 && sn.n_waits / sn.n >= 1024;
  const bool pol = lay.pol_mask != (1u << ES_POLICY_EDGESERVING);
  if (!pol && (k1 ? strcmp(k1, "stream") == 0 : deep)) return launch_score_stream(img, lay, sn, out, dstat, st, sms);
  if (!pol && (k1 ? strcmp(k1, "thread") == 0 : true)) {
    if (lay.M <= 2) return launch_thread<2>(img, lay, a, st, sms);
    if (lay.M <= 4) return launch_thread<4>(img, lay, a, st, sms);
    return launch_thread<8>(img, lay, a, st, sms);
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
