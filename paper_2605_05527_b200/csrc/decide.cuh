// decide.cuh -- one scheduling decision (Algorithm 1) evaluated by
// a segment of LPS lanes of a warp, shared by K1 (snapshots) and K2 (replay).
//
// Lane layout: a warp holds 32/LPS independent segments (one scenario or
// snapshot each).  A segment's LPS lanes form MM groups of GL = LPS/MM lanes;
// group g owns model g's queue Q_g.  Per decision:
//   a3  Eq. 5: B*_g = largest profiled batch <= min(|Q_g|, B_max)
//       (reading Q8; SMEM table bidx).
//   a4  Eq. 6: the GL lanes of group g test one exit each against
//       w_max + L(g, e, B*) <= tau; the deepest passing exit is the top bit of
//       the group's ballot (reading Q2: none passes -> shallowest allowed,
//       infeasible).
//   a5  prediction: never materialised; candidate m with latency
//       L_m clips a remaining task iff its predicted wait w + L_m >= x_c, i.e.
//       w >= thr_m = x_c - L_m; candidate m's own B*_m head tasks are excluded
//       (P:364).
//   a6  Eq. 3-4 in fixed point (reading Q5): each lane walks its group's live
//       window, evaluates G(w) once per task (2 LDS + IMAD.WIDE + SHF) and
//       accumulates (K_m, U_m) for every candidate m; tasks with w >= x_c (the
//       clipped-for-everyone prefix) are counted from the index, never read.
//       S_q(m) = C_q K_m + floor(H(L_m) U_m / 2^28).
//   a7  Eq. 7: argmin of the key (S_q(m), m) -- lowest model index
//       on ties (reading Q3) -- by a shuffle butterfly across the groups.
// All integer; every reduction is exact, so any lane order gives the same bits.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "es_internal.cuh"

namespace es {

constexpr unsigned FULL = 0xffffffffu;

// per-cfg constants, held in registers by every lane of a segment
struct SmemCfg {
  uint32_t off_A, off_Bt, off_H, off_bidx;  // byte offsets into the staged image
  uint32_t tau, b_max, warmup, x_c, r, nA1;
  uint32_t fast_lim;  // head waits below it cannot clip for any candidate
  uint32_t policy;    // ES_POLICY_* (Q26)
  uint64_t C_q;
};

// policies that select by the stability score (Eq. 7) -- the others pick by
// queue length (LQF) or head wait (EDF) and score nothing
__device__ __forceinline__ bool policy_scores(uint32_t pol) {
  return pol == ES_POLICY_EDGESERVING || pol == ES_POLICY_ALLFINAL_DA || pol == ES_POLICY_OURS_BS1;
}

struct SmemProf {
  const uint8_t *sm;
  const uint8_t *hb;  // base of the H tables: the staged image, or the global one (core-only staging)
  const uint32_t *lat;
  const uint32_t *latT;  // [M][nb][8], exit-minor, padded (Eq. 6 by counting)
  const uint16_t *bs;
  const uint32_t *mask;
  const uint16_t *acc;  // [M][E] accuracy, basis points
  const CfgRec *cfg;
  int M, E, nb, ncfg;
};

__device__ __forceinline__ SmemProf smem_prof(const uint8_t *sm, const ImgLayout &lay) {
  SmemProf p;
  p.sm = sm;
  p.hb = sm;
  p.lat = reinterpret_cast<const uint32_t *>(sm + lay.off_lat);
  p.latT = reinterpret_cast<const uint32_t *>(sm + lay.off_latT);
  p.bs = reinterpret_cast<const uint16_t *>(sm + lay.off_bs);
  p.mask = reinterpret_cast<const uint32_t *>(sm + lay.off_mask);
  p.acc = reinterpret_cast<const uint16_t *>(sm + lay.off_acc);
  p.cfg = reinterpret_cast<const CfgRec *>(sm + lay.off_cfg);
  p.M = lay.M;
  p.E = lay.E;
  p.nb = lay.nb;
  p.ncfg = lay.ncfg;
  return p;
}

__device__ __forceinline__ SmemCfg smem_cfg(const SmemProf &p, int k) {
  const CfgRec &c = p.cfg[k];
  SmemCfg s;
  s.off_A = c.off_A;
  s.off_Bt = c.off_Bt;
  s.off_H = c.off_H;
  s.off_bidx = c.off_bidx;
  s.tau = c.tau;
  s.b_max = c.b_max;
  s.warmup = c.warmup;
  s.x_c = c.x_c;
  s.r = c.r;
  s.nA1 = c.nA - 1u;
  s.fast_lim = c.fast_lim;
  s.policy = c.policy;
  s.C_q = c.C_q;
  return s;
}

// G(w) = (A[(w+r)>>10] * Bt[(w+r)&1023]) >> 28 for w < x_c (reading Q5).
// w >= x_c is clamped (its value is never used: such a task clips for all).
__device__ __forceinline__ uint32_t G_of(const SmemProf &P, const SmemCfg &c, uint32_t w) {
  const uint32_t v = min(w, c.x_c) + c.r;
  const uint32_t h = min(v >> SBITS, c.nA1);
  const uint32_t a = *reinterpret_cast<const uint32_t *>(P.sm + c.off_A + 4u * h);
  const uint32_t b = *reinterpret_cast<const uint32_t *>(P.sm + c.off_Bt + 4u * (v & (S - 1u)));
  return (uint32_t)(((uint64_t)a * (uint64_t)b) >> F);
}

// Stage the profile image into shared memory with TMA 1-D bulk copies that
// complete on one mbarrier (cp.async.bulk -> SASS UBLKCP).  All threads wait.
__device__ __forceinline__ void stage_image(uint8_t *smem, const uint8_t *gimg, uint32_t bytes,
                                            uint64_t *mbar) {
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
                 : "memory");
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem);
    constexpr uint32_t CHUNK = 16384;
    for (uint32_t off = 0; off < bytes; off += CHUNK) {
      uint32_t n = bytes - off < CHUNK ? bytes - off : CHUNK;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              dst + off),
          "l"(gimg + off), "r"(n), "r"(mb)
          : "memory");
    }
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(mb)
        : "memory");
  }
}

__device__ __forceinline__ constexpr unsigned low_mask(int n) { return n >= 32 ? FULL : ((1u << n) - 1u); }

// Full-warp REDUX as volatile PTX: the compiler must not sink it into a
// lane-dependent branch (only the full warp may execute redux.sync).
__device__ __forceinline__ uint32_t redux_add(uint32_t v) {
  uint32_t r;
  asm volatile("redux.sync.add.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ uint32_t redux_min(uint32_t v) {
  uint32_t r;
  asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ uint32_t redux_max(uint32_t v) {
  uint32_t r;
  asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
  return r;
}

// Lane roles inside a warp: 32/LPS segments, MM groups of GL lanes each.
// Reductions use compile-time-constant masks (a runtime mask makes ptxas emit
// a collective loop): REDUX over the full warp when LPS == 32, xor-shuffle
// butterflies of width LPS / GL otherwise.
template <int LPS, int MM>
struct Seg {
  static_assert(LPS == 8 || LPS == 16 || LPS == 32, "LPS");
  static_assert(MM <= LPS && (LPS % MM) == 0, "MM");
  static constexpr int GL = LPS / MM;
  int lane, seg, sl, grp, gl, seg_base;
  __device__ __forceinline__ Seg() {
    lane = threadIdx.x & 31;
    seg = lane / LPS;
    sl = lane % LPS;
    grp = sl / GL;
    gl = sl % GL;
    seg_base = seg * LPS;
  }
  // this group's bits of a warp ballot, shifted to bit 0
  __device__ __forceinline__ unsigned gbits(unsigned ballot) const {
    return (ballot >> (seg_base + grp * GL)) & low_mask(GL);
  }
  // this segment's bits of a warp ballot
  __device__ __forceinline__ unsigned sbits(unsigned ballot) const {
    return LPS == 32 ? ballot : (ballot >> seg_base) & low_mask(LPS);
  }
  __device__ __forceinline__ bool seg_any(bool p) const { return sbits(__ballot_sync(FULL, p)) != 0u; }
  static constexpr int SPW = 32 / LPS;  // segments per warp
  // Segment reductions: one full-mask REDUX per segment with the other
  // segments' lanes contributing the identity, then each lane keeps its own.
  __device__ __forceinline__ uint32_t sum(uint32_t v) const {
    __syncwarp();  // segments may arrive from divergent paths: reconverge first
    if constexpr (LPS == 32) {
      return redux_add(v);
    } else {
      uint32_t r = 0;
#pragma unroll
      for (int k = 0; k < SPW; ++k) {
        const uint32_t x = redux_add(seg == k ? v : 0u);
        if (seg == k) r = x;
      }
      return r;
    }
  }
  __device__ __forceinline__ uint32_t vmin(uint32_t v) const {
    __syncwarp();  // segments may arrive from divergent paths: reconverge first
    if constexpr (LPS == 32) {
      return redux_min(v);
    } else {
      uint32_t r = 0;
#pragma unroll
      for (int k = 0; k < SPW; ++k) {
        const uint32_t x = redux_min(seg == k ? v : 0xFFFFFFFFu);
        if (seg == k) r = x;
      }
      return r;
    }
  }
  __device__ __forceinline__ uint32_t vmax(uint32_t v) const {
    __syncwarp();  // segments may arrive from divergent paths: reconverge first
    if constexpr (LPS == 32) {
      return redux_max(v);
    } else {
      uint32_t r = 0;
#pragma unroll
      for (int k = 0; k < SPW; ++k) {
        const uint32_t x = redux_max(seg == k ? v : 0u);
        if (seg == k) r = x;
      }
      return r;
    }
  }
  // exact segment sum of u64 values < 2^51 each (24 | 27-bit halves per REDUX)
  __device__ __forceinline__ uint64_t sum64(uint64_t v) const {
    const uint32_t lo = (uint32_t)(v & 0xFFFFFFu);
    const uint32_t hi = (uint32_t)(v >> 24);
    return ((uint64_t)sum(hi) << 24) + (uint64_t)sum(lo);
  }
  // exact group sum of u64 values
  __device__ __forceinline__ uint64_t gsum64(uint64_t v) const {
#pragma unroll
    for (int o = GL / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o, GL);
    return v;
  }
  template <typename T>
  __device__ __forceinline__ T bcast(T v, int src_sl) const {
    return __shfl_sync(FULL, v, src_sl, LPS);
  }
};

// Eq. 6 as a count: the number of exits e with L(m, e, bs[bi]) <=
// lim, i.e. the length of the feasible prefix (L strictly increasing in e;
// the padding 0xFFFFFFFF never counts).  lim < 2^32 - 1.
__device__ __forceinline__ uint32_t eq6_count(const SmemProf &P, int m, uint32_t bi, uint32_t lim) {
  const uint4 *row = reinterpret_cast<const uint4 *>(P.latT + ((size_t)m * P.nb + bi) * 8u);
  const uint4 x = row[0];
  uint32_t c = (x.x <= lim) + (x.y <= lim) + (x.z <= lim) + (x.w <= lim);
  if (P.E > 4) {
    const uint4 y = row[1];
    c += (y.x <= lim) + (y.y <= lim) + (y.z <= lim) + (y.w <= lim);
  }
  return c;
}

// per-group candidate (uniform across the group's lanes)
struct Cand {
  uint32_t B, e, L, thr;
  uint64_t H;
  bool feas;
};

// a3 + a4 for the group's own model g (valid when len > 0).  Whole warp.
// POL = false compiles Algorithm 1 only (C.policy ignored, no override code).
template <int LPS, int MM, bool POL = false>
__device__ __forceinline__ Cand cand_params(const Seg<LPS, MM> &sg, const SmemProf &P, const SmemCfg &C,
                                            uint32_t len, uint32_t wmax) {
  constexpr int GL = Seg<LPS, MM>::GL;
  Cand k;
  // Eq. 5 (OURS_BS1: B* = bs[0] = 1); fixed exits for ALL_FINAL / ALLFINAL_DA
  // (deepest allowed) and ALL_EARLY (shallowest allowed), else Eq. 6
  const uint32_t cap = POL && C.policy == ES_POLICY_OURS_BS1 ? 1u : (len < C.b_max ? len : C.b_max);
  const int fixed = !POL                                                                     ? 0
                    : (C.policy == ES_POLICY_ALL_FINAL || C.policy == ES_POLICY_ALLFINAL_DA ||
                       C.policy == ES_POLICY_SYMPHONY)                                       ? 1
                    : C.policy == ES_POLICY_ALL_EARLY                                        ? 2
                                                                                             : 0;
  const int gg = sg.grp < P.M ? sg.grp : 0;
  const uint32_t bi = P.sm[C.off_bidx + cap];
  k.B = P.bs[bi];
  const uint32_t mbits = P.mask[gg];
  const uint32_t *row = P.lat + (size_t)gg * P.E * P.nb + bi;  // row[e * nb]
  unsigned bits = 0;
  if (P.E <= GL) {  // warp-uniform: one exit per lane, L and H fetched in parallel
    const int e = sg.gl < P.E ? sg.gl : 0;
    const uint32_t Le = row[e * P.nb];
    const uint64_t He = reinterpret_cast<const uint64_t *>(P.hb + C.off_H)[((size_t)gg * P.E + e) * P.nb + bi];
    const bool ok = sg.gl < P.E && ((mbits >> sg.gl) & 1u) && (uint64_t)wmax + Le <= (uint64_t)C.tau;
    bits = sg.gbits(__ballot_sync(FULL, ok));
    k.feas = bits != 0u;
    k.e = k.feas ? 31u - __clz(bits) : (uint32_t)(__ffs(mbits) - 1);
    if (fixed) k.e = fixed == 1 ? 31u - __clz(mbits) : (uint32_t)(__ffs(mbits) - 1);
    const int src = sg.grp * GL + (int)k.e;
    k.L = __shfl_sync(FULL, Le, src, LPS);
    k.H = __shfl_sync(FULL, He, src, LPS);
    if (fixed) k.feas = (uint64_t)wmax + k.L <= (uint64_t)C.tau;
    k.thr = k.L < C.x_c ? C.x_c - k.L : 0u;
    if (k.L >= C.x_c) k.H = 0ull;
    return k;
  }
  // more exits than group lanes: every lane evaluates Eq. 6 for its group's
  // model itself.  L is strictly increasing in e (validated), so the exits
  // with wmax + L <= tau are the first c ones: c counted on the padded
  // exit-minor row (two independent 16-byte loads), then the mask keeps the
  // allowed ones.
  if (wmax <= C.tau) bits = ((1u << eq6_count(P, gg, bi, C.tau - wmax)) - 1u) & mbits;
  k.feas = bits != 0u;
  k.e = k.feas ? 31u - __clz(bits) : (uint32_t)(__ffs(mbits) - 1);
  if (fixed) k.e = fixed == 1 ? 31u - __clz(mbits) : (uint32_t)(__ffs(mbits) - 1);
  k.L = row[k.e * P.nb];
  if (fixed) k.feas = (uint64_t)wmax + k.L <= (uint64_t)C.tau;
  k.thr = k.L < C.x_c ? C.x_c - k.L : 0u;
  k.H = k.L < C.x_c ? reinterpret_cast<const uint64_t *>(P.hb + C.off_H)[((size_t)gg * P.E + k.e) * P.nb + bi]
                    : 0ull;
  return k;
}

struct Decision {
  uint64_t S;      // S_q(m*)
  uint64_t S_own;  // S_q of this lane's group model (~0 when its queue is empty)
  uint32_t m, e, B, L;
  bool feas;
};

// a7: Eq. 7 argmin of (S, m) across the segment's groups + winner broadcast
template <int LPS, int MM>
__device__ __forceinline__ Decision finish_decision(const Seg<LPS, MM> &sg, const Cand &cand, uint64_t Sq,
                                                   uint32_t mkey) {
  constexpr int GL = Seg<LPS, MM>::GL;
  const uint64_t S_own = Sq;
  constexpr uint64_t LIM = 1ull << 61;
  // key = S * 8 + m orders exactly like (S, m) while S < 2^61; empty -> max.
  // The packed argmin runs unconditionally (the vote on S >= 2^61 overlaps
  // it); the wide (S, m) argmin redoes it only if some score is that large.
  const bool wide = __any_sync(FULL, mkey != 0xFFu && Sq >= LIM);
  uint64_t key = mkey == 0xFFu ? ~0ull : ((Sq << 3) | mkey);
#pragma unroll
  for (int o = GL; o < LPS; o <<= 1) {
    const uint64_t ko = __shfl_xor_sync(FULL, key, o, LPS);
    key = ko < key ? ko : key;
  }
  if (!wide) {
    if (key != ~0ull) {
      Sq = key >> 3;
      mkey = (uint32_t)(key & 7u);
    } else {
      mkey = 0xFFu;
    }
  } else {
#pragma unroll
    for (int o = GL; o < LPS; o <<= 1) {
      const uint64_t So = __shfl_xor_sync(FULL, Sq, o, LPS);
      const uint32_t mo = __shfl_xor_sync(FULL, mkey, o, LPS);
      if (So < Sq || (So == Sq && mo < mkey)) {
        Sq = So;
        mkey = mo;
      }
    }
  }
  Decision d;
  d.S = Sq;
  d.S_own = S_own;
  d.m = mkey;
  const int src = (int)(mkey & (MM - 1)) * GL;
  const uint32_t pk = sg.bcast(cand.e | (cand.feas ? 0x80u : 0u) | (cand.B << 8), src);
  d.L = sg.bcast(cand.L, src);
  d.e = pk & 0x7Fu;
  d.feas = (pk & 0x80u) != 0u;
  d.B = pk >> 8;
  return d;
}

// LQF / EDF selection (ALL_FINAL, ALL_EARLY, EE_LQF: most queued tasks;
// EE_EDF: least slack tau - w_head, i.e. the largest head wait; ties lowest m)
// across the segment's groups; the winner's (e, B, L, feasible) from
// cand_params; S = 0 (nothing is scored).  Whole warp.
// SYMPHONY (Q27): only triggered queues (w_head + L >= tau or |Q| >= B_max)
// compete, by the largest w_head + L; none triggered -> d.m = 0xFF.
template <int LPS, int MM>
__device__ __forceinline__ Decision select_simple(const Seg<LPS, MM> &sg, const Cand &cand, uint32_t len,
                                                  uint32_t wmax, const SmemCfg &C) {
  constexpr int GL = Seg<LPS, MM>::GL;
  const uint32_t policy = C.policy;
  const uint64_t need = (uint64_t)wmax + cand.L;
  const bool trig = need >= C.tau || len >= C.b_max;
  const uint64_t prim = policy == ES_POLICY_EE_EDF ? (uint64_t)wmax : policy == ES_POLICY_SYMPHONY ? need : len;
  const bool cand_ok = len && (policy != ES_POLICY_SYMPHONY || trig);
  uint64_t key = cand_ok ? (((prim + 1u) << 3) | (uint64_t)(7 - sg.grp)) : 0ull;  // no candidate: 0
#pragma unroll
  for (int o = GL; o < LPS; o <<= 1) {
    const uint64_t ko = __shfl_xor_sync(FULL, key, o, LPS);
    key = ko > key ? ko : key;
  }
  Decision d;
  d.S = 0ull;
  d.S_own = 0ull;
  d.m = key ? 7u - (uint32_t)(key & 7u) : 0xFFu;
  const int src = (int)(d.m & (MM - 1)) * GL;
  const uint32_t pk = sg.bcast(cand.e | (cand.feas ? 0x80u : 0u) | (cand.B << 8), src);
  d.L = sg.bcast(cand.L, src);
  d.e = pk & 0x7Fu;
  d.feas = (pk & 0x80u) != 0u;
  d.B = pk >> 8;
  return d;
}

// positions per lane per step in the G loops: 2 when a segment is 8/16 lanes
// (short queues: fewer predicated-off loads on the chain), 4 for whole-warp
// segments (8 models; deep queues want more loads in flight); ES_WU overrides
template <int LPS>
__device__ __forceinline__ constexpr int wu_of() {
#ifdef ES_WU
  return ES_WU;
#else
  return LPS == 32 ? 4 : 2;
#endif
}

// f2 GRID (Q28): every admissible (m, e, b) of every segment, in a
// warp-uniform (m, e, b index) sweep with per-segment validity; per cell the
// segment's lanes count K / sum U over their group's live positions (own
// queue: the b served positions excluded), the clipped-for-everyone
// prefixes are counted from the indices; running argmin of (S, cell index).
// ncells = admissible cells of this segment.  Whole warp.
template <int LPS, int MM, class WaitAt>
__device__ __noinline__ Decision decide_grid(const Seg<LPS, MM> &sg, const SmemProf &P, const SmemCfg &C,
                                             uint32_t len, uint32_t c, uint32_t wmax, WaitAt wait_at,
                                             uint32_t &ncells, uint64_t &own_best) {
  constexpr int GL = Seg<LPS, MM>::GL;
  uint64_t bS = ~0ull;
  uint32_t bidx = 0xFFFFFFFFu, bm = 0xFFu, be = 0u, bB = 0u, bL = 0u;
  bool bfeas = false;
  ncells = 0u;
  own_best = ~0ull;  // best cell of this lane's group model (the candidate score K1 reports)
  const uint32_t cpre = sg.sum(sg.gl == 0 ? c : 0u);
  const uint64_t *Hq = reinterpret_cast<const uint64_t *>(P.hb + C.off_H);
  for (int m = 0; m < P.M; ++m) {
    const uint32_t len_m = sg.bcast(len, m * GL), c_m = sg.bcast(c, m * GL), wmax_m = sg.bcast(wmax, m * GL);
    const uint32_t cap = len_m < C.b_max ? len_m : C.b_max;
    for (int e = 0; e < P.E; ++e) {
      const bool ok_e = len_m > 0u && ((P.mask[m] >> e) & 1u);
      for (int bi = 0; bi < P.nb; ++bi) {
        const uint32_t b = P.bs[bi];
        const bool valid = ok_e && b <= cap;
        if (!__any_sync(FULL, valid)) continue;  // (bs increasing: no later bi either for this segment)
        const int cell = (m * P.E + e) * P.nb + bi;
        const uint32_t L = P.lat[cell];
        const uint32_t thr = L < C.x_c ? C.x_c - L : 0u;
        uint32_t K = 0u;
        uint64_t U = 0ull;
        if (valid)
          for (uint32_t p = c + sg.gl; p < len; p += GL) {
            if (sg.grp == m && p < b) continue;  // candidate m's own served tasks
            const uint32_t w = wait_at(p);
            if (w >= thr) K += 1u;
            else U += G_of(P, C, w);
          }
        K = sg.sum(K);
        U = sg.sum64(U);
        if (valid) {
          const uint64_t Kt = (uint64_t)K + (uint64_t)(cpre - (c_m < b ? c_m : b));
          uint64_t S = C.C_q * Kt;
          if (L < C.x_c) {
            const uint64_t H = Hq[cell], lo = H * U, hi = __umul64hi(H, U);
            S += (hi << (64 - F)) | (lo >> F);
          }
          ncells++;
          if (sg.grp == m && S < own_best) own_best = S;
          if (S < bS || (S == bS && (uint32_t)cell < bidx)) {
            bS = S;
            bidx = (uint32_t)cell;
            bm = (uint32_t)m;
            be = (uint32_t)e;
            bB = b;
            bL = L;
            bfeas = (uint64_t)wmax_m + L <= (uint64_t)C.tau;
          }
        }
      }
    }
  }
  Decision dd;
  dd.S = bS;
  dd.S_own = bS;
  dd.m = bm;
  dd.e = be;
  dd.B = bB;
  dd.L = bL;
  dd.feas = bfeas;
  return dd;
}

template <int LPS, int MM, class WaitAt>
__device__ __forceinline__ Decision decide_general(const Seg<LPS, MM> &sg, const SmemProf &P, const SmemCfg &C,
                                                uint32_t len, uint32_t c, const Cand &cand, uint32_t Bown,
                                                WaitAt wait_at) {
  constexpr int GL = Seg<LPS, MM>::GL;
  // every candidate's clip threshold thr_m = x_c - L_m
  uint32_t thr[MM];
#pragma unroll
  for (int m = 0; m < MM; ++m) thr[m] = sg.bcast(cand.thr, m * GL);
  uint32_t K[MM];
  uint64_t U[MM];
#pragma unroll
  for (int m = 0; m < MM; ++m) {
    K[m] = 0u;
    U[m] = 0ull;
  }
  uint32_t p = c + sg.gl;
  // own served head tasks (positions < B*_g): count for every candidate but g
  for (; p < len && p < Bown; p += GL) {
    const uint32_t w = wait_at(p);
    const uint32_t gw = G_of(P, C, w);
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      if (m == sg.grp) continue;
      if (w >= thr[m]) K[m] += 1u;
      else U[m] += gw;
    }
  }
  constexpr int WU = wu_of<LPS>();
  for (; p < len; p += WU * GL) {
    uint32_t w[WU];
#pragma unroll
    for (int k = 0; k < WU; ++k) w[k] = p + k * GL < len ? wait_at(p + k * GL) : 0u;
#pragma unroll
    for (int k = 0; k < WU; ++k) {
      if (p + k * GL < len) {
        const uint32_t gw = G_of(P, C, w[k]);
#pragma unroll
        for (int m = 0; m < MM; ++m) {
          if (w[k] >= thr[m]) K[m] += 1u;
          else U[m] += gw;
        }
      }
    }
  }
  __syncwarp();
  // exact segment reductions; each group keeps its own candidate's sums
  uint32_t k_own = 0u;
  uint64_t u_own = 0ull;
#pragma unroll
  for (int m = 0; m < MM; ++m) {
    if (m >= P.M) break;  // warp-uniform
    const uint32_t k = sg.sum(K[m]);
    const uint64_t u = sg.sum64(U[m]);
    if (m == sg.grp) {
      k_own = k;
      u_own = u;
    }
  }
  const uint32_t cpre = sg.sum(sg.gl == 0 ? c : 0u);
  // Eq. 4 on the predicted state of candidate g (served tasks excluded)
  const uint32_t cB = c < Bown ? c : Bown;
  const uint64_t Ktot = (uint64_t)k_own + (uint64_t)(cpre - cB);
  uint64_t Sq = ~0ull;
  uint32_t mkey = 0xFFu;
  if (len) {
    // floor(H * U / 2^28) via the 128-bit product
    const uint64_t lo = cand.H * u_own, hi = __umul64hi(cand.H, u_own);
    Sq = C.C_q * Ktot + ((hi << (64 - F)) | (lo >> F));
    mkey = (uint32_t)sg.grp;
  }
  return finish_decision<LPS, MM>(sg, cand, Sq, mkey);
}

// Fast path of a replay step with the queued positions of the WHOLE warp
// flattened (K2).  The per-group fast path below walks each queue with its
// own GL lanes, so a warp step costs its longest queue; K2's batches are
// heavy-tailed across scenarios (cfg3: queued tasks per decision p50 19, p99
// 300), so here the non-empty queues of every segment are concatenated and
// each trip evaluates G for 32 consecutive positions, one per lane.  Per
// queue q the sums come from a running inclusive scan Pf over the flat order:
//   S_q = Pf(start_q), E_q = Pf(start_q + B_q), T_q = Pf(end_q)
//   srv_q = E_q - S_q (own served head tasks), Q_q = T_q - S_q (whole queue),
// tot = sum over the segment's queues of Q_q.  Same integers as the fast path
// of decide(); exact in any order.  Whole warp; `fast` must be warp-uniform.
// Per-warp scratch (shared memory, FLAT_BYTES): one 16-byte descriptor per
// non-empty queue by rank {queue address minus 4 x its flat start, t + r, A and
// Bt word offsets}, and the running sums at each queue's start (slotS, by rank;
// slotS[nq] = the warp's total, so a queue's total is slotS[r + 1] - slotS[r])
// and after its served head (slotE).  A position's queue rank, and whether it
// starts a queue or ends a served head, come from per-trip bit words that the
// queue owners publish with one REDUX.OR each.
constexpr uint32_t FLAT_BYTES = 32 * 16 + 33 * 8 + 32 * 8 + 8;
#ifndef FLAT_WF
#define FLAT_WF 2  // flat positions per lane per trip
#endif

__device__ __forceinline__ uint32_t lds_ro(uint32_t saddr) {  // staged tables: never written after staging
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}

template <int LPS, int MM>
__device__ __forceinline__ Decision decide_fast_flat(const Seg<LPS, MM> &sg, const SmemProf &P, const SmemCfg &C,
                                                    uint32_t len, const Cand &cand, const uint32_t *Ah, uint32_t t,
                                                    uint8_t *scratch) {
  constexpr int GL = Seg<LPS, MM>::GL;
  uint4 *ent = reinterpret_cast<uint4 *>(scratch);           // by rank
  uint64_t *slotS = reinterpret_cast<uint64_t *>(ent + 32);  // [33]
  uint64_t *slotE = slotS + 33;                               // [32]
  const uint32_t lane = (uint32_t)sg.lane;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(P.sm);
  const bool own = sg.gl == 0 && len > 0u;  // queue owner: lane 0 of a non-empty group
  const uint32_t Bown = len ? cand.B : 0u;  // 1 <= B* <= len (Eq. 5)
  // exclusive scan of the owners' lengths over the warp
  uint32_t incl = own ? len : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(FULL, incl, o);
    if (lane >= (uint32_t)o) incl += v;
  }
  const uint32_t start = incl - (own ? len : 0u);
  const uint32_t send = start + Bown - 1u;  // last position of the own served head
  const uint32_t NW = __shfl_sync(FULL, incl, 31);
  const unsigned ne = __ballot_sync(FULL, own);
  const uint32_t orank = __popc(ne & ((1u << lane) - 1u));
  if (own) {
    const uint64_t ptr = reinterpret_cast<uint64_t>(Ah) - 4ull * start;  // address of flat position f: ptr + 4 f
    ent[orank] = make_uint4((uint32_t)ptr, (uint32_t)(ptr >> 32), t + C.r, (C.off_A >> 2) | ((C.off_Bt >> 2) << 16));
  }
  __syncwarp();
  uint64_t carry = 0ull;
  uint32_t cb = 0u;  // non-empty queues starting before this trip
  // a trip covers 32 WF consecutive flat positions; lane l takes positions
  // base + WF l + k (k < WF), all inside 32-position word l / (32 / WF)
  constexpr int WF = FLAT_WF;
  constexpr int LPW = 32 / WF;  // lanes per 32-position word
  const uint32_t lw = lane / LPW, lb = (lane % LPW) * WF;  // this lane's word, its first bit in it
  for (uint32_t base = 0; base < NW; base += 32u * WF) {
    // queue starts and served-head ends inside this trip: one bit per position
    const uint32_t rel = start - base, rel2 = send - base;
    const bool here = own && start >= base && rel < 32u * WF;
    const bool here2 = own && send >= base && rel2 < 32u * WF;
    uint32_t pre = 0u, word = 0u, word2 = 0u, tripc = 0u;
#pragma unroll
    for (int w = 0; w < WF; ++w) {
      const uint32_t bit = here && (rel >> 5) == (uint32_t)w ? 1u << (rel & 31u) : 0u;
      const uint32_t bit2 = here2 && (rel2 >> 5) == (uint32_t)w ? 1u << (rel2 & 31u) : 0u;
      uint32_t mw, mw2;
      asm volatile("redux.sync.or.b32 %0, %1, 0xffffffff;" : "=r"(mw) : "r"(bit));
      asm volatile("redux.sync.or.b32 %0, %1, 0xffffffff;" : "=r"(mw2) : "r"(bit2));
      const uint32_t c = __popc(mw);
      if ((uint32_t)w < lw) pre += c;
      if ((uint32_t)w == lw) {
        word = mw;
        word2 = mw2;
      }
      tripc += c;
    }
    // G of the lane's positions; boundary roles packed with the queue rank
    uint64_t gk[WF];
    uint32_t ik[WF];
    uint64_t lsum = 0ull;
#pragma unroll
    for (int k = 0; k < WF; ++k) {
      const uint32_t f = base + lane * WF + (uint32_t)k;
      gk[k] = 0ull;
      ik[k] = 0u;
      if (f < NW) {
        const uint32_t bk = lb + (uint32_t)k;
        const uint32_t le = bk == 31u ? FULL : ((2u << bk) - 1u);
        const uint32_t rk = cb + pre + __popc(word & le) - 1u;
        const uint4 e = ent[rk];
        const uint32_t *qa = reinterpret_cast<const uint32_t *>((uint64_t)e.x | ((uint64_t)e.y << 32));
        // v = w + r = (t + r) - a; w < fast_lim <= x_c, so v >> 10 < nA (the
        // clamps of G_of are no-ops on the fast path)
        const uint32_t v = e.z - __ldg(qa + f);
        const uint32_t A = lds_ro(sbase + 4u * ((e.w & 0xFFFFu) + (v >> SBITS)));
        const uint32_t Bt = lds_ro(sbase + 4u * ((e.w >> 16) + (v & (S - 1u))));
        gk[k] = ((uint64_t)A * (uint64_t)Bt) >> F;
        lsum += gk[k];
        ik[k] = rk | (((word >> bk) & 1u) << 8) | (((word2 >> bk) & 1u) << 9);
      }
    }
    // running prefix over the flat order: exclusive scan of the lane sums
    uint64_t s = lsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t v = __shfl_up_sync(FULL, s, o);
      if (lane >= (uint32_t)o) s += v;
    }
    uint64_t Pf = carry + s - lsum;
#pragma unroll
    for (int k = 0; k < WF; ++k) {
      Pf += gk[k];  // prefix through this position
      if (ik[k] >> 8) {
        const uint32_t r = ik[k] & 0xFFu;
        if (ik[k] & 0x100u) slotS[r] = Pf - gk[k];
        if (ik[k] & 0x200u) slotE[r] = Pf;
      }
    }
    carry += __shfl_sync(FULL, s, 31);
    cb += tripc;
  }
  if (lane == 0) slotS[__popc(ne)] = carry;
  __syncwarp();
  uint64_t srv = 0ull, Q = 0ull;
  if (own) {
    const uint64_t s0 = slotS[orank];
    srv = slotE[orank] - s0;
    Q = slotS[orank + 1u] - s0;
  }
  const uint64_t tot = sg.sum64(Q);
  srv = sg.bcast(srv, sg.grp * GL);
  uint64_t Sq = ~0ull;
  uint32_t mkey = 0xFFu;
  if (len) {
    const uint64_t u = tot - srv;
    const uint64_t lo = cand.H * u, hi = __umul64hi(cand.H, u);
    Sq = (hi << (64 - F)) | (lo >> F);
    mkey = (uint32_t)sg.grp;
  }
  __syncwarp();  // the scratch is reused by the next step
  return finish_decision<LPS, MM>(sg, cand, Sq, mkey);
}

// a5-a7.  Inputs per group g (uniform in the group): len = |Q_g|, c = number of
// head tasks with w >= x_c (clipped for everyone, never read), cand = a3/a4
// result, and wait_at(p) returning the wait of position p (c <= p < len; no
// warp-synchronous operation inside).  Returns the segment's decision
// (uniform across the segment).  Empty groups / inactive segments: len = 0.
// fast: no head wait of the warp reaches x_c - max L (warp-uniform; see below).
template <int LPS, int MM, class WaitAt>
__device__ __forceinline__ Decision decide(const Seg<LPS, MM> &sg, const SmemProf &P, const SmemCfg &C,
                                           uint32_t len, uint32_t c, bool fast, const Cand &cand,
                                           WaitAt wait_at) {
  constexpr int GL = Seg<LPS, MM>::GL;
  const uint32_t Bown = len ? cand.B : 0u;
  uint64_t Sq = ~0ull;
  uint32_t mkey = 0xFFu;
  // Fast path (same integers): when every head wait is below x_c - max L, no
  // task of any queue can reach x_c under any candidate's prediction, so
  // K_m = 0 and U_m = sum_all G - sum_{own served} G for every m.  The
  // per-candidate clip tests and 3 M reductions collapse to 4 reductions.
  if (fast) {
    uint64_t tot = 0ull, srv = 0ull;
    constexpr int WU = wu_of<LPS>();
    // WU positions per lane per step: their loads issue back to back (the
    // per-decision chain is latency-bound, one queue is a handful of steps)
    for (uint32_t p0 = sg.gl; p0 < len; p0 += WU * GL) {
      uint32_t w[WU];
#pragma unroll
      for (int k = 0; k < WU; ++k) {
        const uint32_t p = p0 + k * GL;
        w[k] = p < len ? wait_at(p) : 0u;
      }
#pragma unroll
      for (int k = 0; k < WU; ++k) {
        const uint32_t p = p0 + k * GL;
        if (p < len) {
          const uint64_t gw = G_of(P, C, w[k]);
          tot += gw;
          if (p < Bown) srv += gw;
        }
      }
    }
    __syncwarp();
    tot = sg.sum64(tot);
    srv = sg.gsum64(srv);
    if (len) {
      const uint64_t u = tot - srv;
      const uint64_t lo = cand.H * u, hi = __umul64hi(cand.H, u);
      Sq = (hi << (64 - F)) | (lo >> F);
      mkey = (uint32_t)sg.grp;
    }
    return finish_decision<LPS, MM>(sg, cand, Sq, mkey);
  }
  return decide_general<LPS, MM>(sg, P, C, len, c, cand, Bown, wait_at);
}

}  // namespace es
