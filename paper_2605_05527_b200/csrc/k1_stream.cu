// k1_stream.cu -- K1 for deep snapshots as three stream-ordered phases.
//
// Same method and integers as k1_score.cu (Algorithm 1 on queue snapshots,
// decide.cuh); the work is re-partitioned so the bulk of it -- reading every
// live wait once and evaluating G(w) (Eq. 3-4, reading Q5) -- is a pure
// streaming reduction with no block-wide synchronisation:
//   A  k1s_prep    one thread per queue: CSR, head wait (Q7), clipped prefix
//                  by binary search (counted, never read), Eq. 5 / Eq. 6 of
//                  the queue's own candidate, "can clip" flag of the snapshot
//   B  k1s_stream_fast / k1s_stream_slow  one warp per queue, coalesced loads
//                  in flight per lane (double-buffered on the fast path):
//                  fast path   sum G over the live window (+ the own served
//                              head for the candidate's exclusion)
//                  clip path   (K_m, U_m) for every candidate m of the snapshot
//                  read-window validation (Q24); u64 atomics into the
//                  snapshot's accumulators
//   C  k1s_finish  one segment of 8 lanes per snapshot: S_q(m) for every
//                  candidate, Eq. 7 argmin (S, m) (Q3), outputs
// Scratch (records + accumulators) is stream-ordered (cudaMallocAsync).
#include <cuda_runtime.h>

#include "decide.cuh"

namespace es {
namespace {

struct QRec {  // per (snapshot, model) queue
  uint64_t lo;
  uint64_t H;
  uint32_t len, c, B, thr, L, ef;  // ef = e | feasible << 7
};

constexpr int ACC = 2 + 2 * MAXM;  // tot, flags, S-part[8] (srv or U), K[8]
constexpr uint64_t F_SLOW = 1, F_BAD = 2;
#ifndef ES_K1_MINB
#define ES_K1_MINB 4
#endif
constexpr uint32_t V4_LIM = (1u << 30) - 1024u;  // fast-stream G needs 4 (x_c + 1023) < 2^32

struct StreamArgs {
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
  QRec *rec;
  unsigned long long *acc;
  unsigned long long *slow_n;  // number of clip-path snapshots (appended by k1s_prep)
  int64_t *slow_list;          // their indices
};

// programmatic dependent launch (see launch_persistent)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__global__ void __launch_bounds__(256) k1s_prep(const uint8_t *__restrict__ gimg, ImgLayout lay, StreamArgs a) {
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  stage_image(smem, gimg, lay.bytes, &mbar);
  const SmemProf P = smem_prof(smem, lay);
  const int M = P.M;
  const int64_t nq = a.n * M;
  for (int64_t qi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; qi < nq; qi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = qi / M;
    const int g = (int)(qi - s * M);
    const int k = a.cfg_idx ? (int)a.cfg_idx[s] : 0;
    QRec r{};
    if (k >= P.ncfg) {
      atomicOr(a.acc + s * ACC + 1, F_BAD);
      a.rec[qi] = r;
      continue;
    }
    const SmemCfg C = smem_cfg(P, k);
    r.lo = a.q_off[qi];
    r.len = (uint32_t)(a.q_off[qi + 1] - r.lo);
    if (r.len) {
      const uint32_t *W = a.waits + r.lo;
      const uint32_t wmax = __ldg(W);
      if (wmax >= C.x_c) {  // clipped-for-everyone prefix: first position with w < x_c
        uint32_t plo = 0, phi = r.len;
        while (phi - plo > 1u) {
          const uint32_t mid = plo + (phi - plo) / 2u;
          if (__ldg(W + mid) >= C.x_c) plo = mid;
          else phi = mid;
        }
        r.c = phi;
      }
      const uint32_t cap = r.len < C.b_max ? r.len : C.b_max;
      const uint32_t bi = P.sm[C.off_bidx + cap];
      const uint32_t mbits = P.mask[g];
      const uint32_t *row = P.lat + (size_t)g * P.E * P.nb + bi;
      int best = -1;
      for (int e = 0; e < P.E; ++e)
        if (((mbits >> e) & 1u) && (uint64_t)wmax + row[e * P.nb] <= (uint64_t)C.tau) best = e;
      const uint32_t e = best >= 0 ? (uint32_t)best : (uint32_t)(__ffs(mbits) - 1);
      r.B = P.bs[bi];
      r.L = row[e * P.nb];
      r.ef = e | (best >= 0 ? 0x80u : 0u);
      r.thr = r.L < C.x_c ? C.x_c - r.L : 0u;
      r.H = r.L < C.x_c ? reinterpret_cast<const uint64_t *>(P.sm + C.off_H)[((size_t)g * P.E + e) * P.nb + bi] : 0ull;
      if (wmax >= C.fast_lim || C.x_c > V4_LIM) {
        const unsigned long long was = atomicOr(a.acc + s * ACC + 1, F_SLOW);
        if (!(was & F_SLOW)) a.slow_list[atomicAdd(a.slow_n, 1ull)] = s;
      }
    }
    a.rec[qi] = r;
  }
}

__device__ __forceinline__ uint64_t wsum64(uint64_t v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// shared-memory table lookup with 32-bit shared addresses
__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}

// G(w) for a live wait (w < x_c guaranteed by the prefix search; an inverted
// input is flagged and its value unused, the index is clamped for safety).
// v4 = 4 (w + r) in one IMAD: exact while x_c + 1024 <= 2^30 (k1s_prep routes
// other SLOs to the clip path, which uses the plain form).
struct GTab {
  uint32_t sA, sBt, r4, nA1;
  __device__ __forceinline__ uint32_t operator()(uint32_t w) const {
    const uint32_t v4 = w * 4u + r4;
    const uint32_t h = min(v4 >> (SBITS + 2), nA1);
    const uint32_t a = lds_u32(sA + 4u * h);
    const uint32_t b = lds_u32(sBt + (v4 & (4u * S - 4u)));
    return (uint32_t)(((uint64_t)a * (uint64_t)b) >> F);
  }
};

__device__ __forceinline__ void load_stage(const uint4 *__restrict__ V, uint32_t nv, uint32_t v0, int lane, uint4 &c0,
                                           uint4 &c1) {
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  c0 = v0 + lane < nv ? __ldg(V + v0 + lane) : z;
  c1 = v0 + 32u + lane < nv ? __ldg(V + v0 + 32u + lane) : z;
}

// vectors [v0, v0 + 64): lane holds v0 + lane (c0) and v0 + 32 + lane (c1);
// `carry` = last wait before v0 (0xFFFFFFFF: none)
__device__ __forceinline__ void sum_stage(const GTab &G, uint32_t nv, uint32_t v0, int lane, const uint4 &c0,
                                          const uint4 &c1, uint32_t &carry, uint64_t &tot, bool &bad) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const uint4 cur = k ? c1 : c0;
    uint32_t prev = __shfl_up_sync(FULL, cur.w, 1);
    if (lane == 0) prev = carry;
    carry = __shfl_sync(FULL, cur.w, 31);
    if (v0 + 32u * k + lane < nv) {
      bad |= (cur.x > prev) | (cur.y > cur.x) | (cur.z > cur.y) | (cur.w > cur.z);
      tot += (uint64_t)G(cur.x) + G(cur.y) + (uint64_t)G(cur.z) + G(cur.w);
    }
  }
}

// Sum of G over waits [ps, pe) of one queue (absolute positions in the waits
// array), with the read-window neighbour check (Q24).  16-byte vector loads
// (4 waits per lane, two vectors per lane per stage, next stage prefetched);
// scalar head up to 16-byte alignment and scalar tail; one shuffle per vector
// carries the predecessor across lanes.  `first` = position of the queue's
// first live wait (no predecessor check there).
__device__ __forceinline__ void stream_piece(const uint32_t *__restrict__ W, uint64_t ps, uint64_t pe, uint64_t first,
                                             uint64_t se, const GTab &G, int lane, uint64_t &tot, uint64_t &srv,
                                             bool &bad) {
  const uint32_t mis = (uint32_t)(((uintptr_t)(W + ps) >> 2) & 3u);
  const uint64_t pa = min(ps + (uint64_t)((4u - mis) & 3u), pe);
  const uint32_t nv = (uint32_t)((pe - pa) / 4u);
  const uint64_t pt = pa + 4ull * nv;
  const uint4 *V = reinterpret_cast<const uint4 *>(W + pa);
  // one round of loads: first stage, the body's predecessor, the scalar
  // head/tail waits with theirs, the first 32 served-head waits
  uint4 x0, x1, y0, y1;
  load_stage(V, nv, 0u, lane, x0, x1);
  uint32_t carry = pa > first ? __ldg(W + pa - 1) : 0xFFFFFFFFu;
  const uint32_t nh = (uint32_t)(pa - ps), ntl = (uint32_t)(pe - pt);
  uint64_t p = ~0ull;
  if (lane < (int)nh) p = ps + lane;
  else if (lane >= 8 && lane < 8 + (int)ntl) p = pt + (lane - 8);
  const uint32_t sw = p != ~0ull ? __ldg(W + p) : 0u;
  const uint32_t sp = (p != ~0ull && p > first) ? __ldg(W + p - 1) : 0xFFFFFFFFu;
  const uint64_t p_srv = ps + lane;
  const uint32_t ww = p_srv < se ? __ldg(W + p_srv) : 0u;
  if (p != ~0ull) {
    if (sw > sp) bad = true;
    tot += G(sw);
  }
  if (p_srv < se) srv += G(ww);
  for (uint64_t q2 = p_srv + 32u; q2 < se; q2 += 32u) srv += G(__ldg(W + q2));  // B > 32 only
  // stage X = vectors [v0, v0 + 64), stage Y = [v0 + 64, v0 + 128): two
  // vectors per lane each; one stage is in flight while the other is summed
  for (uint32_t v0 = 0; v0 < nv; v0 += 128u) {  // warp-uniform trip count
    load_stage(V, nv, v0 + 64u, lane, y0, y1);
    sum_stage(G, nv, v0, lane, x0, x1, carry, tot, bad);
    if (v0 + 64u >= nv) break;
    load_stage(V, nv, v0 + 128u, lane, x0, x1);
    sum_stage(G, nv, v0 + 64u, lane, y0, y1, carry, tot, bad);
  }
}

// fast path (snapshot cannot clip): sum of G over every live window.  The
// flat waits array [q_off[0], q_off[nq]) is cut into equal contiguous ranges,
// one per warp (balanced in bytes whatever the queue-length mix); a warp finds
// its first queue with a 32-ary search over q_off, then walks the queues that
// intersect its range.  Per piece: u64 atomics into the snapshot's total and
// into the candidate's own served-head sum (positions < B).
__global__ void __launch_bounds__(256, ES_K1_MINB) k1s_stream_fast(const uint8_t *__restrict__ gimg, ImgLayout lay,
                                                         StreamArgs a) {
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  stage_image(smem, gimg, lay.bytes, &mbar);
  const SmemProf P = smem_prof(smem, lay);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const int M = P.M;
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nq = a.n * M;
  if (nq == 0) return;
  const uint64_t base = __ldg(a.q_off), end = __ldg(a.q_off + nq);
  uint64_t per = ((end - base) + (uint64_t)nw - 1u) / (uint64_t)nw;
  per = max((per + 3u) & ~3ull, 512ull);
  const uint64_t x0 = base + (uint64_t)wid * per;
  if (x0 >= end) return;  // warp-uniform
  const uint64_t x1 = min(x0 + per, end);
  int64_t lo = 0, hi = nq;  // largest q < nq with q_off[q] <= x0
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t pr = lo + step * lane;
    const bool ok = pr < hi && __ldg(a.q_off + pr) <= x0;
    const int l = 31 - __clz(__ballot_sync(FULL, ok));  // lane 0 always ok
    lo += step * l;
    hi = min(hi, lo + step);
  }
  // queue descriptors spread over the lanes (lane l < 10: word l of the QRec,
  // lane 10: the snapshot's flag word, lane 11: its SLO index), fetched one
  // piece ahead so the next piece's record is in flight while this one streams
  static_assert(sizeof(QRec) == 40, "QRec");
  auto fetch = [&](int64_t q) -> uint32_t {
    if (q >= nq) return 0u;
    const int64_t s = q / M;
    if (lane < 10) return __ldg(reinterpret_cast<const uint32_t *>(a.rec + q) + lane);
    if (lane == 10) return (uint32_t)a.acc[s * ACC + 1];  // F_SLOW is final (set by k1s_prep)
    if (lane == 11) return a.cfg_idx ? (uint32_t)a.cfg_idx[s] : 0u;
    return 0u;
  };
  pdl_wait();  // k1s_prep's records and flags
  uint32_t dcur = fetch(lo);
  for (int64_t q = lo; q < nq; ++q) {  // warp-uniform
    const uint32_t dnext = fetch(q + 1);
    const uint64_t rlo = (uint64_t)__shfl_sync(FULL, dcur, 0) | ((uint64_t)__shfl_sync(FULL, dcur, 1) << 32);
    const uint32_t rlen = __shfl_sync(FULL, dcur, 4), rc = __shfl_sync(FULL, dcur, 5);
    const uint32_t rB = __shfl_sync(FULL, dcur, 6);
    const uint32_t flg = __shfl_sync(FULL, dcur, 10), k = __shfl_sync(FULL, dcur, 11);
    dcur = dnext;
    if (rlo >= x1) break;
    if (rlen <= rc || (flg & (uint32_t)F_SLOW)) continue;
    const uint64_t first = rlo + rc;
    const uint64_t ps = max(first, x0), pe = min(rlo + rlen, x1);
    if (ps >= pe) continue;
    const int64_t s = q / M;
    unsigned long long *acc = a.acc + s * ACC;
    const SmemCfg C = smem_cfg(P, (int)k);
    const GTab G{sbase + C.off_A, sbase + C.off_Bt, 4u * C.r, C.nA1};
    uint64_t tot = 0, srv = 0;
    bool bad = false;
    stream_piece(a.waits, ps, pe, first, min(pe, rlo + min(rB, rlen)), G, lane, tot, srv, bad);
    if (__any_sync(FULL, bad) && lane == 0) atomicOr(acc + 1, F_BAD);
    tot = wsum64(tot);
    srv = wsum64(srv);
    if (lane == 0) {
      atomicAdd(acc + 0, (unsigned long long)tot);
      if (srv) atomicAdd(acc + 2 + (q - s * M), (unsigned long long)srv);
    }
  }
}

// clip path (some head wait is within max L of x_c): (K_m, U_m) for every candidate
template <int MM>
__global__ void __launch_bounds__(256) k1s_stream_slow(const uint8_t *__restrict__ gimg, ImgLayout lay,
                                                       StreamArgs a) {
  pdl_trigger();
  pdl_wait();
  const int64_t n_slow = (int64_t)*a.slow_n;  // block-uniform
  if (n_slow == 0) return;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  stage_image(smem, gimg, lay.bytes, &mbar);
  const SmemProf P = smem_prof(smem, lay);
  const int M = P.M;
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int UNR = 4;
  for (int64_t li = wid; li < n_slow * M; li += nw) {  // warp-uniform
    const int64_t s = a.slow_list[li / M];
    const int g = (int)(li % M);
    const int64_t qi = s * M + g;
    const QRec r = a.rec[qi];
    if (r.len <= r.c) continue;
    unsigned long long *acc = a.acc + s * ACC;
    const SmemCfg C = smem_cfg(P, a.cfg_idx ? (int)a.cfg_idx[s] : 0);
    const uint32_t *W = a.waits + r.lo;
    uint64_t U[MM];
    uint32_t K[MM], thr[MM];
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      U[m] = 0ull;
      K[m] = 0u;
      thr[m] = m < M ? a.rec[s * M + m].thr : 0xFFFFFFFFu;
    }
    bool bad = false;
    uint32_t carry = 0xFFFFFFFFu;
    for (uint32_t p0 = r.c; p0 < r.len; p0 += UNR * 32u) {  // warp-uniform trip count
      uint32_t wv[UNR];
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const uint32_t p = p0 + j * 32u + lane;
        wv[j] = p < r.len ? __ldg(W + p) : 0u;
      }
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const uint32_t p = p0 + j * 32u + lane;
        const uint32_t w = wv[j];
        uint32_t prev = __shfl_up_sync(FULL, w, 1);
        if (lane == 0) prev = carry;
        carry = __shfl_sync(FULL, w, 31);
        if (p >= r.len) continue;
        bad |= w > prev || w >= C.x_c;
        const uint32_t gw = G_of(P, C, w);
#pragma unroll
        for (int m = 0; m < MM; ++m) {
          if (m == g && p < r.B) continue;  // candidate g's own served tasks
          if (w >= thr[m]) K[m] += 1u;
          else U[m] += gw;
        }
      }
    }
    if (__any_sync(FULL, bad) && lane == 0) atomicOr(acc + 1, F_BAD);
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      if (m >= M) break;
      const uint64_t u = wsum64(U[m]);
      const uint32_t kk = redux_add(K[m]);
      if (lane == 0) {
        if (u) atomicAdd(acc + 2 + m, (unsigned long long)u);
        if (kk) atomicAdd(acc + 2 + MAXM + m, (unsigned long long)kk);
      }
    }
  }
}

// one 8-lane group per snapshot, lane m = candidate m
__global__ void __launch_bounds__(256) k1s_finish(const uint8_t *__restrict__ gimg, ImgLayout lay, StreamArgs a) {
  pdl_wait();
  const CfgRec *cfg = reinterpret_cast<const CfgRec *>(gimg + lay.off_cfg);
  const int M = lay.M;
  const int lane = threadIdx.x & 31, sub = lane >> 3, m = lane & 7;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s0 = wid * 4; s0 < a.n; s0 += nw * 4) {  // warp-uniform
    const int64_t s = s0 + sub;
    const bool ok = s < a.n;
    const int k = ok ? (a.cfg_idx ? (int)a.cfg_idx[s] : 0) : 0;
    const bool cfg_ok = k < lay.ncfg;
    const unsigned long long *acc = a.acc + (ok ? s : 0) * ACC;
    const uint64_t flags = ok ? acc[1] : 0ull;
    QRec r{};
    if (ok && m < M) r = a.rec[s * M + m];
    const bool has = r.len > 0u;
    // always-clipped prefixes of all queues (for the clip path)
    uint32_t cs = has ? r.c : 0u;
#pragma unroll
    for (int o = 4; o >= 1; o >>= 1) cs += __shfl_xor_sync(FULL, cs, o, 8);
    uint64_t Sq = ~0ull;
    if (has && cfg_ok) {
      const CfgRec &C = cfg[k];
      uint64_t u, kk = 0;
      if (!(flags & F_SLOW)) {
        u = acc[0] - acc[2 + m];
      } else {
        u = acc[2 + m];
        const uint32_t cB = r.c < r.B ? r.c : r.B;
        kk = acc[2 + MAXM + m] + (uint64_t)(cs - cB);
      }
      const uint64_t lo = r.H * u, hi = __umul64hi(r.H, u);
      Sq = C.C_q * kk + ((hi << (64 - F)) | (lo >> F));
    }
    // Eq. 7: argmin (S, m) over the 8-lane group
    uint64_t bS = Sq;
    uint32_t bm = has ? (uint32_t)m : 0xFFu;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint64_t So = __shfl_xor_sync(FULL, bS, o, 8);
      const uint32_t mo = __shfl_xor_sync(FULL, bm, o, 8);
      if (So < bS || (So == bS && mo < bm)) {
        bS = So;
        bm = mo;
      }
    }
    const int src = (int)(bm & 7u);
    const uint32_t ef = __shfl_sync(FULL, r.ef, src, 8);
    const uint32_t Bw = __shfl_sync(FULL, r.B, src, 8);
    const uint32_t Lw = __shfl_sync(FULL, r.L, src, 8);
    if (!ok) continue;
    const bool bad = (flags & F_BAD) || !cfg_ok;
    if (m == 0) {
      if (bad || bm == 0xFFu) {
        a.m[s] = 0; a.e[s] = 0; a.B[s] = 0; a.L[s] = 0; a.S[s] = 0;
        a.flags[s] = bad ? ES_FLAG_BAD_INPUT : ES_FLAG_NO_WORK;
        if (!cfg_ok && atomicCAS(&a.dstat->code, 0u, (uint32_t)ES_ERR_ARG) == 0u) a.dstat->item = s;
      } else {
        a.m[s] = (uint8_t)bm;
        a.e[s] = (uint8_t)(ef & 0x7Fu);
        a.B[s] = (uint16_t)Bw;
        a.L[s] = Lw;
        a.S[s] = bS;
        a.flags[s] = (ef & 0x80u) ? ES_FLAG_FEASIBLE : 0u;
      }
    }
    if (a.cand && m < M) a.cand[s * M + m] = (bad || !has) ? ~0ull : Sq;
  }
}

// pdl: programmatic dependent launch -- the kernel may start while its
// predecessor drains; it runs its prologue (image staging, range search) and
// blocks in pdl_wait() before touching the predecessor's outputs
template <typename Kern>
cudaError_t launch_persistent(Kern kern, const uint8_t *img, const ImgLayout &lay, const StreamArgs &a, int64_t items,
                              int per_block, size_t dyn, cudaStream_t st, int sms, bool pdl = true) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, dyn);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  int64_t blocks = (items + per_block - 1) / per_block;
  const int64_t cap = (int64_t)sms * occ;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, img, lay, a);
}

}  // namespace

cudaError_t launch_score_stream(const uint8_t *img, const ImgLayout &lay, const es_snapshots &sn,
                                const es_decisions &out, DevStatus *dstat, cudaStream_t st, int sms) {
  StreamArgs a{};
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
  const int64_t nq = sn.n * lay.M;
  void *scratch = nullptr;
  // scratch: [acc | slow_n | slow_list | rec]; acc and slow_n zeroed
  const size_t acc_bytes = (size_t)sn.n * ACC * sizeof(uint64_t) + sizeof(uint64_t);
  const size_t list_bytes = (size_t)sn.n * sizeof(int64_t), rec_bytes = (size_t)nq * sizeof(QRec);
  cudaError_t e = cudaMallocAsync(&scratch, acc_bytes + list_bytes + rec_bytes, st);
  if (e != cudaSuccess) return e;
  uint8_t *sp = static_cast<uint8_t *>(scratch);
  a.acc = reinterpret_cast<unsigned long long *>(sp);
  a.slow_n = a.acc + (size_t)sn.n * ACC;
  a.slow_list = reinterpret_cast<int64_t *>(sp + acc_bytes);
  a.rec = reinterpret_cast<QRec *>(sp + acc_bytes + list_bytes);
  e = cudaMemsetAsync(a.acc, 0, acc_bytes, st);
  if (e == cudaSuccess) e = launch_persistent(k1s_prep, img, lay, a, nq, 256, lay.bytes, st, sms, false);
  if (e == cudaSuccess) e = launch_persistent(k1s_stream_fast, img, lay, a, nq, 8, lay.bytes, st, sms);
  if (e == cudaSuccess) {
    if (lay.M <= 2) e = launch_persistent(k1s_stream_slow<2>, img, lay, a, nq, 8, lay.bytes, st, sms);
    else if (lay.M <= 4) e = launch_persistent(k1s_stream_slow<4>, img, lay, a, nq, 8, lay.bytes, st, sms);
    else e = launch_persistent(k1s_stream_slow<8>, img, lay, a, nq, 8, lay.bytes, st, sms);
  }
  if (e == cudaSuccess) e = launch_persistent(k1s_finish, img, lay, a, sn.n, 32, 0, st, sms);
  const cudaError_t f = cudaFreeAsync(scratch, st);
  return e != cudaSuccess ? e : f;
}

}  // namespace es
