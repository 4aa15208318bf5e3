// decide.cuh -- one scheduling decision (Algorithm 1) evaluated by
// one warp, shared by K1 (snapshots) and K2 (trace replay).
//
// Warp layout: the 32 lanes form MM groups of GL = 32/MM lanes; group g owns
// model g's queue Q_g.  Per decision:
//   a3  Eq. 5: B*_g = largest profiled batch <= min(|Q_g|, B_max)
//       (reading Q8; SMEM table bidx).
//   a4  Eq. 6: the GL lanes of group g test one exit each against
//       w_max + L(g, e, B*) <= tau; the deepest passing exit is the top bit of
//       the group's ballot (reading Q2: none passes -> shallowest allowed,
//       infeasible).
//   a5  prediction: never materialised; a candidate m with latency
//       L_m clips a remaining task iff its predicted wait w + L_m >= x_c, i.e.
//       w >= thr_m = x_c - L_m; candidate m's own B*_m head tasks are excluded
//       (P:364).
//   a6  Eq. 3-4 in fixed point (reading Q5): every lane walks its group's live
//       window once, evaluates G(w) once per task (2 LDS + IMAD.WIDE + SHF) and
//       accumulates (K_m, U_m) for all candidates m; tasks with w >= x_c (the
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

struct SmemCfg {  // per-cfg pointers into the staged SMEM image
  const uint32_t *A, *Bt;
  const uint64_t *H;
  const uint8_t *bidx;
  uint32_t tau, b_max, warmup, x_c, r, nA1;
  uint64_t C_q;
};

struct SmemProf {
  const uint32_t *lat;
  const uint16_t *bs;
  const uint32_t *mask;
  const CfgRec *cfg;
  int M, E, nb, ncfg;
};

__device__ __forceinline__ SmemProf smem_prof(const uint8_t *sm, const ImgLayout &lay) {
  SmemProf p;
  p.lat = reinterpret_cast<const uint32_t *>(sm + lay.off_lat);
  p.bs = reinterpret_cast<const uint16_t *>(sm + lay.off_bs);
  p.mask = reinterpret_cast<const uint32_t *>(sm + lay.off_mask);
  p.cfg = reinterpret_cast<const CfgRec *>(sm + lay.off_cfg);
  p.M = lay.M;
  p.E = lay.E;
  p.nb = lay.nb;
  p.ncfg = lay.ncfg;
  return p;
}

__device__ __forceinline__ SmemCfg smem_cfg(const uint8_t *sm, const SmemProf &p, int k) {
  const CfgRec &c = p.cfg[k];
  SmemCfg s;
  s.A = reinterpret_cast<const uint32_t *>(sm + c.off_A);
  s.Bt = reinterpret_cast<const uint32_t *>(sm + c.off_Bt);
  s.H = reinterpret_cast<const uint64_t *>(sm + c.off_H);
  s.bidx = sm + c.off_bidx;
  s.tau = c.tau;
  s.b_max = c.b_max;
  s.warmup = c.warmup;
  s.x_c = c.x_c;
  s.r = c.r;
  s.nA1 = c.nA - 1u;
  s.C_q = c.C_q;
  return s;
}

// G(w) = (A[(w+r)>>10] * Bt[(w+r)&1023]) >> 28 for w < x_c (reading Q5).
// w >= x_c is clamped (its value is never used: such a task clips for all).
__device__ __forceinline__ uint32_t G_of(const SmemCfg &c, uint32_t w) {
  uint32_t v = min(w, c.x_c) + c.r;
  uint32_t h = min(v >> SBITS, c.nA1);
  uint64_t prod = (uint64_t)c.A[h] * (uint64_t)c.Bt[v & (S - 1u)];
  return (uint32_t)(prod >> F);
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

template <int MM>
struct Lanes {
  static constexpr int GL = 32 / MM;
  int lane, grp, gl;
  unsigned gmask;  // this group's lanes
  __device__ __forceinline__ Lanes() {
    lane = threadIdx.x & 31;
    grp = lane / GL;
    gl = lane % GL;
    gmask = (GL == 32) ? FULL : (((1u << GL) - 1u) << (grp * GL));
  }
  // group-local bits of a warp ballot, shifted to bit 0
  __device__ __forceinline__ unsigned gbits(unsigned ballot) const {
    return (GL == 32) ? ballot : ((ballot >> (grp * GL)) & ((1u << GL) - 1u));
  }
};

__device__ __forceinline__ uint32_t red_u32(uint32_t v) { return __reduce_add_sync(FULL, v); }
// exact warp sum of u64 values < 2^51 each: split 24 | 27 bits into two u32 reductions
__device__ __forceinline__ uint64_t red_u64(uint64_t v) {
  uint32_t lo = (uint32_t)(v & 0xFFFFFFu);
  uint32_t hi = (uint32_t)(v >> 24);
  return ((uint64_t)__reduce_add_sync(FULL, hi) << 24) + (uint64_t)__reduce_add_sync(FULL, lo);
}
template <int GL>
__device__ __forceinline__ uint32_t grp_sum_u32(uint32_t v) {
#pragma unroll
  for (int o = GL / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o, GL);
  return v;
}
template <int GL>
__device__ __forceinline__ uint64_t grp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = GL / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o, GL);
  return v;
}

// per-group candidate (uniform across the group's lanes)
struct Cand {
  uint32_t B, bi, e, L, thr;
  uint64_t H;
  bool feas;
};

// a3 + a4 for the group's own model g (valid when len > 0).  Must be called
// by the whole warp (contains ballots).
template <int MM>
__device__ __forceinline__ Cand cand_params(const Lanes<MM> &ln, const SmemProf &P, const SmemCfg &C,
                                            int g, uint32_t len, uint32_t wmax) {
  constexpr int GL = Lanes<MM>::GL;
  Cand k;
  const uint32_t cap = len < C.b_max ? len : C.b_max;
  const int gg = g < P.M ? g : 0;
  k.bi = C.bidx[cap];
  k.B = P.bs[k.bi];
  const uint32_t mbits = P.mask[gg];
  const uint32_t *row = P.lat + (size_t)gg * P.E * P.nb + k.bi;  // row[e * nb]
  unsigned bits = 0;
  for (int e0 = 0; e0 < P.E; e0 += GL) {  // warp-uniform trip count
    const int e = e0 + ln.gl;
    bool ok = false;
    if (e < P.E && ((mbits >> e) & 1u)) ok = (uint64_t)wmax + row[e * P.nb] <= (uint64_t)C.tau;
    bits |= ln.gbits(__ballot_sync(FULL, ok)) << e0;
  }
  k.feas = bits != 0u;
  k.e = k.feas ? 31u - __clz(bits) : (uint32_t)(__ffs(mbits) - 1);
  k.L = row[k.e * P.nb];
  k.thr = k.L < C.x_c ? C.x_c - k.L : 0u;
  k.H = k.L < C.x_c ? C.H[((size_t)gg * P.E + k.e) * P.nb + k.bi] : 0ull;
  return k;
}

struct Decision {
  uint64_t S;      // S_q(m*)
  uint64_t S_own;  // S_q of this lane's group model (~0 when its queue is empty)
  uint32_t m, e, B, L;
  bool feas;
};

// a5-a7.  Inputs per group g (uniform in the group): len = |Q_g|, c = number of
// head tasks with w >= x_c (clipped for everyone, never read), cand = a3/a4
// result, and wait_at(p) returning the wait of position p (c <= p < len).
// Returns the decision (uniform across the warp).  Unused groups: len = 0.
template <int MM, class WaitAt>
__device__ __forceinline__ Decision decide(const Lanes<MM> &ln, const SmemCfg &C, uint32_t len, uint32_t c,
                                           const Cand &cand, WaitAt wait_at) {
  constexpr int GL = Lanes<MM>::GL;
  // broadcast every candidate's clip threshold thr_m = x_c - L_m
  uint32_t thr[MM];
#pragma unroll
  for (int m = 0; m < MM; ++m) thr[m] = __shfl_sync(FULL, cand.thr, m * GL);
  uint32_t K[MM];
  uint64_t U[MM];
#pragma unroll
  for (int m = 0; m < MM; ++m) {
    K[m] = 0u;
    U[m] = 0ull;
  }
  uint32_t Kx = 0u;  // own served tasks (positions < B*_g) -- excluded for candidate g
  uint64_t Ux = 0ull;
  const uint32_t Bown = len ? cand.B : 0u;
  for (uint32_t p = c + ln.gl; p < len; p += GL) {
    const uint32_t w = wait_at(p);
    const uint32_t gw = G_of(C, w);
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      if (w >= thr[m]) K[m] += 1u;
      else U[m] += gw;
    }
    if (p < Bown) {
      if (w >= cand.thr) Kx += 1u;
      else Ux += gw;
    }
  }
  // exact reductions
#pragma unroll
  for (int m = 0; m < MM; ++m) {
    K[m] = red_u32(K[m]);
    U[m] = red_u64(U[m]);
  }
  Kx = grp_sum_u32<GL>(Kx);
  Ux = grp_sum_u64<GL>(Ux);
  const uint32_t cpre = red_u32(ln.gl == 0 ? c : 0u);
  uint32_t k_own = 0u;
  uint64_t u_own = 0ull;
#pragma unroll
  for (int m = 0; m < MM; ++m)
    if (m == ln.grp) {
      k_own = K[m];
      u_own = U[m];
    }
  // Eq. 4 on the predicted state of candidate g (served tasks excluded)
  const uint32_t cB = c < Bown ? c : Bown;
  const uint64_t Ktot = (uint64_t)(k_own - Kx) + (uint64_t)(cpre - cB);
  const uint64_t Utot = u_own - Ux;
  uint64_t Sq = ~0ull;
  uint32_t mkey = 0xFFu;
  if (len) {
    // floor(H * U / 2^28) via the 128-bit product
    const uint64_t lo = cand.H * Utot, hi = __umul64hi(cand.H, Utot);
    Sq = C.C_q * Ktot + ((hi << (64 - F)) | (lo >> F));
    mkey = (uint32_t)ln.grp;
  }
  const uint64_t S_own = Sq;
  // Eq. 7: argmin of (S, m) across groups
#pragma unroll
  for (int o = GL; o < 32; o <<= 1) {
    const uint64_t So = __shfl_xor_sync(FULL, Sq, o);
    const uint32_t mo = __shfl_xor_sync(FULL, mkey, o);
    if (So < Sq || (So == Sq && mo < mkey)) {
      Sq = So;
      mkey = mo;
    }
  }
  Decision d;
  d.S = Sq;
  d.S_own = S_own;
  d.m = mkey;
  const int src = (int)(mkey & (MM - 1)) * GL;
  const uint32_t pk = __shfl_sync(FULL, cand.e | (cand.feas ? 0x80u : 0u) | (cand.B << 8), src);
  d.L = __shfl_sync(FULL, cand.L, src);
  d.e = pk & 0x7Fu;
  d.feas = (pk & 0x80u) != 0u;
  d.B = pk >> 8;
  return d;
}

}  // namespace es
