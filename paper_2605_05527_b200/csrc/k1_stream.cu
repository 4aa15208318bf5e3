// k1_stream.cu -- K1 for deep snapshots as three stream-ordered phases.
//
// Same method and integers as k1_score.cu (Algorithm 1 on queue snapshots,
// decide.cuh); the work is re-partitioned so the bulk of it -- reading every
// live wait once and evaluating G(w) (Eq. 3-4, reading Q5) -- is a pure
// streaming reduction with no block-wide synchronisation:
//   A  k1s_prep    one thread per queue: CSR, head wait (Q7), clipped prefix
//                  by binary search (counted, never read), Eq. 5 / Eq. 6 of
//                  the queue's own candidate, "can clip" flag of the snapshot
//   B  k1s_stream_tma  fast path (snapshot cannot clip): the flat waits array
//                  streamed through per-warp TMA rings, sum of G over every
//                  live window (+ the own served head), Q24 check
//      k1s_clip    clip path: one warp per clip-path snapshot, (K_m, U_m) for
//                  every candidate m, per-wait threshold tests only near the
//                  clip boundary and in served heads
//   C  k1s_finish  one segment of 8 lanes per snapshot: S_q(m) for every
//                  candidate, Eq. 7 argmin (S, m) (Q3), outputs
// Scratch (records + accumulators) is stream-ordered (cudaMallocAsync).
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "decide.cuh"

namespace es {
namespace {

struct QRec {  // per (snapshot, model) queue
  uint64_t lo;
  uint64_t H;
  uint32_t len, c, B, thr, L, ef;  // ef = e | feasible << 7
  uint64_t srv;                    // fast path: sum of G over the own served head [0, min(B*, len))
};

constexpr int ACC = 2 + 2 * MAXM;  // tot, flags, S-part[8] (srv or U), K[8]
constexpr uint64_t F_SLOW = 1, F_BAD = 2;
#ifndef ES_K1_MINB
#define ES_K1_MINB 4
#endif
constexpr uint32_t V4_LIM = (1u << 30) - 1024u;
  // fast-stream G needs 4 (x_c + 1023) < 2^32

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

// exact warp sum of u64 values whose total stays below 2^64 and whose high
// words sum below 2^32: three REDUX (the low word split into 16-bit halves)
__device__ __forceinline__ uint64_t wsum64_pre(uint64_t v) {
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  const uint64_t l0 = redux_add(lo & 0xFFFFu), l1 = redux_add(lo >> 16);
  return l0 + (l1 << 16) + ((uint64_t)redux_add(hi) << 32);
}

__global__ void __launch_bounds__(256, 6) k1s_prep(const uint8_t *__restrict__ gimg, ImgLayout lay, StreamArgs a) {
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  stage_image(smem, gimg, lay.core_bytes, &mbar);  // the core: H (one load per queue) stays in global memory
  SmemProf P = smem_prof(smem, lay);
  P.hb = gimg;
  const int M = P.M;
  const int64_t nq = a.n * M;
  const int lane = threadIdx.x & 31;
  // warp-uniform sweep: lane l of a warp prepares queue base + l
  for (int64_t q0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll; q0 < nq;
       q0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t qi = q0 + lane;
    const bool on = qi < nq;
    const int64_t s = qi / M;
    const int g = (int)(qi - s * M);
    const int k = on ? (a.cfg_idx ? (int)a.cfg_idx[s] : 0) : 0;
    QRec r{};
    uint32_t nsv = 0u;
    bool slowq = false;
    SmemCfg C{};
    if (on && k >= P.ncfg) atomicOr(a.acc + s * ACC + 1, F_BAD);
    if (on && k < P.ncfg) {
      C = smem_cfg(P, k);
      r.lo = a.q_off[qi];
      r.len = (uint32_t)(a.q_off[qi + 1] - r.lo);
    }
    if (on && k < P.ncfg && r.len) {
      const uint32_t *W = a.waits + r.lo;
      const uint32_t wmax = __ldg(W);
      if (wmax >= C.x_c) {  // clipped-for-everyone prefix: first position with w < x_c
        // interpolation on the waits (near-linear in position: Poisson
        // arrivals), alternated with bisection so the worst case stays
        // logarithmic; the bracket W[plo] >= x_c > W[phi] holds throughout, so
        // the result is the exact boundary (counted, never summed: Q24)
        const uint32_t wl = __ldg(W + r.len - 1u);
        if (wl >= C.x_c) {
          r.c = r.len;
        } else {
          uint32_t plo = 0, phi = r.len - 1u, wlo = wmax, whi = wl;
          bool interp = true;
          while (phi - plo > 1u) {
            uint32_t mid = plo + (phi - plo) / 2u;
            if (interp)  // wlo >= x_c > whi, so wlo > whi
              mid = plo + 1u + (uint32_t)((float)(wlo - C.x_c) / (float)(wlo - whi) * (float)(phi - plo));
            interp = !interp;
            mid = min(max(mid, plo + 1u), phi - 1u);
            const uint32_t v = __ldg(W + mid);
            if (v >= C.x_c) {
              plo = mid;
              wlo = v;
            } else {
              phi = mid;
              whi = v;
            }
          }
          r.c = phi;
        }
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
      r.H = r.L < C.x_c ? reinterpret_cast<const uint64_t *>(P.hb + C.off_H)[((size_t)g * P.E + e) * P.nb + bi] : 0ull;
      nsv = r.B < r.len ? r.B : r.len;
      if (wmax >= C.fast_lim || C.x_c > V4_LIM) {
        slowq = true;
        const unsigned long long was = atomicOr(a.acc + s * ACC + 1, F_SLOW);
        if (!(was & F_SLOW)) a.slow_list[atomicAdd(a.slow_n, 1ull)] = s;
      }
    }
    // the clip path excludes served tasks per wait: when a snapshot's queues
    // share this warp (M divides 32) and one of them clips, skip its served heads
    if ((32 % M) == 0) {
      const unsigned segm = (M == 32 ? FULL : ((1u << M) - 1u)) << ((lane / M) * M);
      if (__ballot_sync(FULL, slowq) & segm) nsv = 0u;
    }
    // own served heads for the fast path (the clip path excludes them
    // per task): the warp reads its 32 queues' first min(B*, len) waits with
    // coalesced loads, 8 queues' loads in flight at a time
    uint64_t mine = 0;
    if (__any_sync(FULL, nsv > 0u)) {
#pragma unroll 1
      for (int u0 = 0; u0 < 32; u0 += 8) {
        uint32_t wv[8], nn[8];
        uint64_t lo8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          lo8[u] = __shfl_sync(FULL, r.lo, u0 + u);
          nn[u] = __shfl_sync(FULL, nsv, u0 + u);
          wv[u] = (uint32_t)lane < nn[u] ? __ldg(a.waits + lo8[u] + lane) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const SmemCfg Cs = smem_cfg(P, __shfl_sync(FULL, k, u0 + u) < P.ncfg ? __shfl_sync(FULL, k, u0 + u) : 0);
          uint64_t sv = (uint32_t)lane < nn[u] ? (uint64_t)G_of(P, Cs, wv[u]) : 0ull;
          for (uint32_t j = 32u + lane; j < nn[u]; j += 32u) sv += G_of(P, Cs, __ldg(a.waits + lo8[u] + j));  // B* > 32
          sv = wsum64_pre(sv);
          if (lane == u0 + u) mine = sv;
        }
      }
    }
    r.srv = mine;
    if (on) a.rec[qi] = r;
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
  stage_image(smem, gimg, lay.core_bytes, &mbar);  // A and Bt: the core
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
  static_assert(sizeof(QRec) == 48, "QRec");  // words 0..9 fetched; srv is read by k1s_finish
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
    stream_piece(a.waits, ps, pe, first, ps, G, lane, tot, srv, bad);  // served heads: k1s_finish
    if (__any_sync(FULL, bad) && lane == 0) atomicOr(acc + 1, F_BAD);
    tot = wsum64(tot);
    srv = wsum64(srv);
    if (lane == 0) {
      atomicAdd(acc + 0, (unsigned long long)tot);
      if (srv) atomicAdd(acc + 2 + (q - s * M), (unsigned long long)srv);
    }
  }
}

// ---------------------------------------------------------------------------
// fast path, TMA form: the flat waits array is cut into one contiguous range of
// 16-byte vectors per warp (equal bytes per warp).  Each warp owns a ring of
// NSL shared-memory slots of PV vectors; its lane 0 keeps NSL-1 pieces of the
// range in flight with cp.async.bulk (one mbarrier per slot), so the HBM
// stream never restarts at queue boundaries and needs no registers for the
// bytes in flight.  The warp walks its range one 128-wait window at a time
// with a warp-uniform queue state (current queue record, the next one
// prefetched): a window strictly inside the live, unserved part of a fast
// queue takes the 4-waits-per-lane fast body; any other window (queue or
// snapshot boundary, served head, range end) goes through the
// element-wise handler.  Per-snapshot totals and per-queue served sums are
// warp-reduced and added with one u64 atomic per snapshot / queue.
constexpr uint32_t PV_MAX = 256;  // vectors (16 B) per piece: 4 KB (2 KB for large profile images)

struct TmaRing {
  uint32_t pv;        // vectors per piece (slot size 16 pv bytes)
  uint32_t nsl;       // slots per warp
  uint32_t ring_off;  // byte offset of the rings in dynamic smem
  uint32_t mbar_off;  // byte offset of the mbarriers
};

__device__ __forceinline__ void mbar_init(uint32_t mb, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(cnt));
}
__device__ __forceinline__ void mbar_wait(uint32_t mb, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(mb), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ uint4 lds_v4(uint32_t saddr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(saddr));
  return v;
}

__device__ __forceinline__ uint64_t wsum64_u(uint64_t v) {
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  // lo sum needs 37 bits: split into 16-bit halves to keep REDUX exact
  const uint64_t l0 = redux_add(lo & 0xFFFFu), l1 = redux_add(lo >> 16);
  const uint64_t h = redux_add(hi);
  return l0 + (l1 << 16) + (h << 32);
}

// G(w) of the single-SLO specialisation: the table bases are kernel
// parameters (uniform registers, folded into the LDS address), the A index is
// masked to the table's power-of-two capacity (exact for w < x_c; an inverted
// input reads an in-bounds garbage value and is flagged bad)
struct GOne {
  uint32_t sA, sBt, r4, amask;
  __device__ __forceinline__ uint32_t operator()(uint32_t w) const {
    const uint32_t v4 = w * 4u + r4;
    const uint32_t a = lds_u32(sA + ((v4 >> SBITS) & amask));
    const uint32_t b = lds_u32(sBt + (v4 & (4u * S - 4u)));
    return (uint32_t)(((uint64_t)a * (uint64_t)b) >> F);
  }
};

template <bool ONE, int TMA_NW>
__global__ void __launch_bounds__(TMA_NW * 32, 1) k1s_stream_tma(const uint8_t *__restrict__ gimg, ImgLayout lay,
                                                                 StreamArgs a, TmaRing rg) {
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t PV = rg.pv;
  const uint32_t ring = sbase + rg.ring_off + (uint32_t)wib * rg.nsl * (PV * 16u);
  const uint32_t bars = sbase + rg.mbar_off + (uint32_t)wib * rg.nsl * 8u;
  const int M = lay.M;
  const int64_t nq = a.n * M;
  // ---- this warp's vector range (vector 0 = the 16-byte unit holding waits[base])
  const uint64_t base = nq ? __ldg(a.q_off) : 0ull, end = nq ? __ldg(a.q_off + nq) : 0ull;
  const uintptr_t ga = reinterpret_cast<uintptr_t>(a.waits);
  const uintptr_t vaddr = (ga + 4u * base) & ~(uintptr_t)15u;
  const int64_t pv0 = (int64_t)base - (int64_t)(((ga + 4u * base) & 15u) >> 2);  // position of vector 0, lane 0
  const uint64_t bytes_end = ga + 4u * end - vaddr;
  const int64_t nvec = end > base ? (int64_t)((bytes_end + 15u) >> 4) : 0;
  const int64_t nfull = end > base ? (int64_t)(bytes_end >> 4) : 0;  // vectors wholly inside the array
  const int64_t nwarps = (int64_t)gridDim.x * TMA_NW;
  const int64_t vper = ((nvec + nwarps - 1) / nwarps + 31) & ~31ll;
  const int64_t gw = (int64_t)blockIdx.x * TMA_NW + wib;
  const int64_t v0 = gw * vper, v1 = min(v0 + vper, nvec);
  const int64_t npieces = v1 > v0 ? (v1 - v0 + PV - 1) / PV : 0;
  const uint8_t *gsrc = reinterpret_cast<const uint8_t *>(vaddr);
  // piece k into `slot`: executed by the whole warp with warp-uniform operands,
  // one elected lane arms the slot's mbarrier and issues the bulk copy
  auto issue = [&](int64_t k, uint32_t slot) {
    const int64_t vs = v0 + k * (int64_t)PV;
    const int64_t vf = min(min(vs + (int64_t)PV, v1), nfull);
    const uint32_t nb = vf > vs ? (uint32_t)(vf - vs) * 16u : 0u;
    const uint32_t mb = bars + 8u * slot;
    asm volatile(
        "{\n\t.reg .pred e, c;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
        "setp.ne.and.u32 c, %1, 0, e;\n\t"
        "@c cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], %1, [%0];\n\t}" ::"r"(mb),
        "r"(nb), "r"(ring + slot * (PV * 16u)), "l"(gsrc + vs * 16)
        : "memory");
  };
  if (lane == 0) {
    for (uint32_t i = 0; i < rg.nsl; ++i) mbar_init(bars + 8u * i, 1u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  for (int64_t k = 0; k < min((int64_t)rg.nsl - 1, npieces); ++k) issue(k, (uint32_t)k);
  stage_image(smem, gimg, lay.core_bytes, &mbar);  // A and Bt (also publishes the mbarrier inits)
  if (npieces == 0) return;
  const SmemProf P = smem_prof(smem, lay);
  // ---- initial queue: largest q < nq with q_off[q] <= first position of the range
  const int64_t R0 = pv0 + 4 * v0;  // range-relative positions are int32 offsets from R0
  const uint64_t x0 = (uint64_t)max(R0, (int64_t)base);
  int64_t lo = 0, hi = nq;
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t pr = lo + step * lane;
    const bool ok = pr < hi && __ldg(a.q_off + pr) <= x0;
    const int l = 31 - __clz(__ballot_sync(FULL, ok));
    lo += step * l;
    hi = min(hi, lo + step);
  }
  pdl_wait();  // k1s_prep's snapshot flags
  if ((int64_t)*a.slow_n == a.n) {
    // every snapshot takes the clip path (k1s_clip reads their live
    // windows): nothing to stream here; drain the pieces already in flight
    for (int64_t k = 0; k < min((int64_t)rg.nsl - 1, npieces); ++k) mbar_wait(bars + 8u * (uint32_t)k, 0u);
    return;
  }
  constexpr int32_t BIG = 0x3FFFFFFF;
  const int32_t rend_full = (int32_t)(4 * (min(v1, nfull) - v0));  // fast windows end here
  int64_t qi = lo, s_cur = lo / M;
  int m_cur = (int)(lo - s_cur * M);
  // queue and snapshot descriptors in warp-distributed register windows, the
  // next window loaded 32 entries ahead (no dependent load per queue):
  //   qw_*: lane l holds q_off[qb + l] (q_off[nq] past the end)
  //   fw_*: lane l holds F_SLOW | cfg << 1 of snapshot sb + l (final after k1s_prep)
  auto qload = [&](int64_t b) -> uint64_t { return b + lane <= nq ? __ldg(a.q_off + b + lane) : end; };
  auto fload = [&](int64_t b) -> uint32_t {
    const int64_t sx = b + lane;
    if (sx >= a.n) return 0u;
    const uint32_t k = a.cfg_idx ? (uint32_t)a.cfg_idx[sx] : 0u;
    return (uint32_t)(a.acc[sx * ACC + 1] & F_SLOW) | (k << 1);
  };
  int64_t qb = qi, sb = s_cur;
  uint64_t qw_cur = qload(qb), qw_nxt = qload(qb + 32);
  uint32_t fw_cur = fload(sb), fw_nxt = fload(sb + 32);
  auto qoff = [&](int64_t q) -> uint64_t {  // q in [qb, qb + 32]
    const int d = (int)(q - qb);
    const uint64_t x = __shfl_sync(FULL, qw_cur, d & 31), y = __shfl_sync(FULL, qw_nxt, 0);
    return d < 32 ? x : y;
  };
  // warp-uniform queue state (range-relative positions)
  int32_t qs_r = 0, qe_r = 0, lo_r = BIG, hi_r = -BIG;
  bool skip = true;
  GTab Gg{0u, 0u, 0u, 0u};
  const GOne G1{sbase + lay.c0_offA, sbase + lay.c0_offBt, lay.c0_r4, lay.c0_amask};
  auto clampr = [&](int64_t p) -> int32_t { return (int32_t)max(min(p - R0, (int64_t)BIG), -(int64_t)BIG); };
  auto set_queue = [&](bool new_snap) {
    if (qi - qb >= 32) {  // slide the queue window
      qb += 32;
      qw_cur = qw_nxt;
      qw_nxt = qload(qb + 32);
    }
    if (s_cur - sb >= 32) {  // slide the snapshot window
      sb += 32;
      fw_cur = fw_nxt;
      fw_nxt = fload(sb + 32);
    }
    const uint64_t rlo = qoff(qi), rhi = qoff(qi + 1);
    const uint32_t fk = __shfl_sync(FULL, fw_cur, (int)(s_cur - sb));
    const uint32_t k = fk >> 1;
    if (!ONE && new_snap && k < (uint32_t)P.ncfg) {
      const SmemCfg C = smem_cfg(P, (int)k);
      Gg = GTab{sbase + C.off_A, sbase + C.off_Bt, 4u * C.r, C.nA1};
    }
    skip = (fk & 1u) != 0u || rhi == rlo || k >= (uint32_t)P.ncfg;
    qs_r = clampr((int64_t)rlo);
    qe_r = clampr((int64_t)rhi);
    lo_r = skip ? BIG : qs_r;  // a window starting at the head: its first pair is cross-queue (qstart)
    hi_r = min(qe_r, rend_full) - 128;
  };
  set_queue(true);
  uint64_t tot = 0;
  uint32_t bad = 0u;
  auto Gv = [&](uint32_t w) -> uint32_t { return ONE ? G1(w) : Gg(w); };
  auto flush_snap = [&]() {
    const uint64_t v = wsum64_u(tot);
    const bool b = __any_sync(FULL, bad != 0u);
    if (lane == 0) {
      if (v) atomicAdd(a.acc + s_cur * ACC, (unsigned long long)v);
      if (b) atomicOr(a.acc + s_cur * ACC + 1, F_BAD);
    }
    tot = 0;
    bad = 0u;
  };
  auto advance = [&]() {
    ++qi;
    if (qi >= nq) {
      skip = true;
      qs_r = qe_r = BIG;
      lo_r = BIG;
      return;
    }
    const bool ns = ++m_cur == M;
    if (ns) {
      flush_snap();
      m_cur = 0;
      ++s_cur;
    }
    set_queue(ns);
  };
  // one fast window: 32 vectors (128 waits) of one live, unserved queue range
  auto fast_window = [&](const uint4 &x, uint32_t &carry, bool qstart) {
    uint32_t prev = __shfl_up_sync(FULL, x.w, 1);
    if (lane == 0) prev = qstart ? 0xFFFFFFFFu : carry;  // no predecessor check at the queue head
    carry = __shfl_sync(FULL, x.w, 31);
    // Q24 read-window check as one predicate chain: bad = 1 if any wait exceeds its predecessor
    asm("{\n\t.reg .pred p;\n\t"
        "setp.gt.u32 p, %1, %2;\n\t"
        "setp.gt.or.u32 p, %3, %1, p;\n\t"
        "setp.gt.or.u32 p, %4, %3, p;\n\t"
        "setp.gt.or.u32 p, %5, %4, p;\n\t"
        "selp.u32 %0, 1, %0, p;\n\t}"
        : "+r"(bad)
        : "r"(x.x), "r"(prev), "r"(x.y), "r"(x.z), "r"(x.w));
    tot += (uint64_t)Gv(x.x) + Gv(x.y) + (uint64_t)Gv(x.z) + Gv(x.w);
  };
  uint32_t carry = R0 > (int64_t)base ? __ldg(a.waits + R0 - 1) : 0u;  // the range's predecessor wait
  uint32_t slot = 0, phase = 0, rslot = rg.nsl - 1;  // slot of piece k, its parity, slot to refill
  for (int64_t k = 0; k < npieces; ++k) {
    if (k + rg.nsl - 1 < npieces) {
      // refill the slot consumed in the previous iteration (reads are complete:
      // every lane passed the __syncwarp at the end of that piece)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + rg.nsl - 1, rslot);
    }
    rslot = slot;
    mbar_wait(bars + 8u * slot, phase);
    const int64_t vs = v0 + k * (int64_t)PV;
    const uint32_t nv = (uint32_t)min((int64_t)PV, v1 - vs);
    const uint32_t sl = ring + slot * (PV * 16u) + 16u * lane;
    const int32_t pw0 = (int32_t)(4 * (vs - v0));
    for (uint32_t j = 0; j < nv; j += 32u) {  // windows of 32 vectors, warp-uniform
      const int32_t pw = pw0 + 4 * (int32_t)j;
      while (qe_r <= pw) advance();  // queues that ended before this window (or are empty)
      const bool qstart = pw == qs_r;
      if (pw >= lo_r && pw + 384 <= hi_r && j + 96u < nv) {  // four fast windows
        const uint32_t sa = sl + 16u * j;
        const uint4 x = lds_v4(sa), y = lds_v4(sa + 512u), z = lds_v4(sa + 1024u), u = lds_v4(sa + 1536u);
        fast_window(x, carry, qstart);
        fast_window(y, carry, false);
        fast_window(z, carry, false);
        fast_window(u, carry, false);
        j += 96u;
        continue;
      }
      if (pw >= lo_r && pw + 128 <= hi_r && j + 32u < nv) {  // two fast windows
        const uint4 x = lds_v4(sl + 16u * j), y = lds_v4(sl + 16u * (j + 32u));
        fast_window(x, carry, qstart);
        fast_window(y, carry, false);
        j += 32u;
        continue;
      }
      if (pw >= lo_r && pw <= hi_r) {
        fast_window(lds_v4(sl + 16u * j), carry, qstart);
        continue;
      }
      // ---- one queue boundary inside the window, same snapshot (so the same
      // SLO tables and slow flag), the next queue reaching past the window:
      // every wait is summed into the snapshot total; the Q24 pair check skips
      // only the next queue's head
      if (pw >= lo_r && qe_r > pw && qe_r < pw + 128 && pw + 128 <= rend_full && m_cur + 1 < M &&
          qi + 2 - qb <= 32 && clampr((int64_t)qoff(qi + 2)) >= pw + 128) {
        const uint4 x = lds_v4(sl + 16u * j);
        uint32_t prev = __shfl_up_sync(FULL, x.w, 1);
        if (lane == 0) prev = carry;
        carry = __shfl_sync(FULL, x.w, 31);
        const int32_t pl = pw + 4 * lane;  // position of x.x
        const bool inv = ((x.x > prev) & (pl != qe_r) & (pl != qs_r)) | ((x.y > x.x) & (pl + 1 != qe_r)) |
                         ((x.z > x.y) & (pl + 2 != qe_r)) | ((x.w > x.z) & (pl + 3 != qe_r));
        if (inv) bad = 1u;
        tot += (uint64_t)Gv(x.x) + Gv(x.y) + (uint64_t)Gv(x.z) + Gv(x.w);
        continue;  // the next window's catch-up advances to the next queue (same snapshot: no flush)
      }
      // ---- element-wise window: boundaries, served heads, skipped queues, range end
      const uint32_t vl = j + lane;
      const int64_t v = vs + vl;
      uint32_t xv[4] = {0u, 0u, 0u, 0u};
      if (vl < nv) {
        if (v < nfull) {
          const uint4 x = lds_v4(sl + 16u * j);
          xv[0] = x.x; xv[1] = x.y; xv[2] = x.z; xv[3] = x.w;
        } else {  // the partial last vector: its waits below `end` straight from global
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int64_t p = pv0 + 4 * v + i;
            if (p >= (int64_t)base && p < (int64_t)end) xv[i] = __ldg(a.waits + p);
          }
        }
      }
      uint32_t prev = __shfl_up_sync(FULL, xv[3], 1);
      if (lane == 0) prev = carry;
      carry = __shfl_sync(FULL, xv[3], 31);
      const int32_t pl = pw + 4 * lane;
      const int32_t wend = min(pw + 128, (int32_t)(4 * (v1 - v0)));
      // one SLO: G of every wait once; several SLOs: per queue pass (its snapshot's tables)
      uint32_t gv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) gv[i] = ONE ? G1(xv[i]) : 0u;
      for (;;) {
        if (!skip) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int32_t p = pl + i;
            if (p >= qs_r && p < qe_r && vl < nv) {
              tot += ONE ? gv[i] : Gg(xv[i]);
              if (p > qs_r && xv[i] > (i ? xv[i - 1] : prev)) bad = 1u;
            }
          }
        }
        if (qe_r >= wend) break;  // the current queue reaches past this window
        advance();
      }
    }
    __syncwarp();
    if (++slot == rg.nsl) {
      slot = 0;
      phase ^= 1u;
    }
  }
  flush_snap();
}

// clip path (some head wait is within max L of x_c): (K_m, U_m) for every
// candidate m of the snapshot, one warp per clip-path snapshot.  Lane g < M
// holds queue g's record; the warp walks the live windows [c_q, len_q) of the
// snapshot's queues in rows of 32 consecutive waits (eight rows' loads in
// flight; an L2 prefetch of the next snapshot's windows was measured to add
// 1.8 GB of DRAM reads per call for no time).  Waits are non-increasing from the head (checked, Q24), so a row
// whose first wait is below every candidate's threshold min_m thr_m and which
// lies past the queue's served head is below x_c - L_m for every m:
// its G values go to one running sum T that every U_m receives.  Only the
// rows near the clip boundary (w >= min thr) or in a served head compare each
// wait with the M thresholds.  One reduce-scatter per snapshot leaves (U_m,
// K_m) in the lanes that store them (plain stores: one writer per snapshot).
template <int MM>
__device__ __forceinline__ void reduce_scatter(uint64_t (&U)[MM], uint32_t (&K)[MM], int lane) {
  // step with offset o keeps half the remaining entries: the upper half in
  // lanes with bit o set; afterwards entry 0 holds m = lane >> (5 - log2 MM)
#pragma unroll
  for (int h = MM / 2, o = 16; h >= 1; h >>= 1, o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const uint64_t su = up ? U[i] : U[i + h], ku = up ? U[i + h] : U[i];
      const uint32_t sk = up ? K[i] : K[i + h], kk = up ? K[i + h] : K[i];
      U[i] = ku + __shfl_xor_sync(FULL, su, o);
      K[i] = kk + __shfl_xor_sync(FULL, sk, o);
    }
  }
#pragma unroll
  for (int o = 16 / MM; o >= 1; o >>= 1) {
    U[0] += __shfl_xor_sync(FULL, U[0], o);
    K[0] += __shfl_xor_sync(FULL, K[0], o);
  }
}

constexpr int CLIP_ROWS = 8;  // rows of 32 waits in flight per warp

template <int MM>
__global__ void __launch_bounds__(256) k1s_clip(const uint8_t *__restrict__ gimg, ImgLayout lay, StreamArgs a) {
  pdl_trigger();
  pdl_wait();
  const int64_t n_slow = (int64_t)*a.slow_n;  // block-uniform
  if (n_slow == 0) return;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  stage_image(smem, gimg, lay.core_bytes, &mbar);  // A and Bt (H comes with the records)
  const SmemProf P = smem_prof(smem, lay);
  const int M = P.M;
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t li = wid; li < n_slow; li += nw) {  // warp-uniform
    const int64_t s = a.slow_list[li];
    const SmemCfg C = smem_cfg(P, a.cfg_idx ? (int)a.cfg_idx[s] : 0);  // < ncfg (k1s_prep)
    uint64_t rlo = 0;
    uint32_t rlen = 0, rc = 0, rB = 0, rthr = 0xFFFFFFFFu;
    if (lane < M) {
      const QRec *r = a.rec + s * M + lane;
      rlo = r->lo;
      rlen = r->len;
      rc = r->c;
      rB = r->B;
      if (rlen) rthr = r->thr;  // empty queue: no candidate (its sums are unused)
    }
    uint32_t thr[MM], K[MM];
    uint64_t U[MM];
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      thr[m] = __shfl_sync(FULL, rthr, m);
      K[m] = 0u;
      U[m] = 0ull;
    }
    const uint32_t minthr = redux_min(rthr);
    uint64_t T = 0ull;  // G over the rows below every threshold
    bool bad = false;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    const GTab G{sbase + C.off_A, sbase + C.off_Bt, 4u * C.r, C.nA1};  // w < x_c in the read window (else flagged)
    for (int q = 0; q < M; ++q) {  // warp-uniform
      const uint32_t len = __shfl_sync(FULL, rlen, q), c = __shfl_sync(FULL, rc, q);
      if (len <= c) continue;
      const uint32_t B = __shfl_sync(FULL, rB, q);
      const uint32_t *W = a.waits + __shfl_sync(FULL, rlo, q);
      uint32_t carry = 0xFFFFFFFFu;  // no predecessor check at the first live wait
      for (uint32_t p0 = c; p0 < len; p0 += 32u * CLIP_ROWS) {  // warp-uniform
        const uint32_t *Wp = W + p0 + lane;
        const uint32_t nr = min((len - p0 + 31u) / 32u, (uint32_t)CLIP_ROWS);  // rows in this window
        uint32_t wv[CLIP_ROWS];
#pragma unroll
        for (int j = 0; j < CLIP_ROWS; ++j) {
          wv[j] = 0u;
          if ((uint32_t)j < nr && p0 + 32u * j + lane < len) wv[j] = __ldg(Wp + 32 * j);
        }
#pragma unroll
        for (int j = 0; j < CLIP_ROWS; ++j) {
          if ((uint32_t)j >= nr) break;
          const uint32_t r0 = p0 + 32u * j;
          const uint32_t p = r0 + lane, w = wv[j];
          uint32_t prev = __shfl_up_sync(FULL, w, 1);
          if (lane == 0) prev = carry;
          carry = __shfl_sync(FULL, w, 31);
          const uint32_t rowmax = __shfl_sync(FULL, w, 0);
          const bool valid = p < len;
          bad |= valid && (w > prev || w >= C.x_c);
          const uint32_t gw = valid ? G(w) : 0u;
          if (rowmax < minthr && r0 >= B) {  // below every threshold, no served task
            T += gw;
            continue;
          }
          if (!valid) continue;
#pragma unroll
          for (int m = 0; m < MM; ++m) {
            if (m == q && p < B) continue;  // candidate q's own served tasks
            if (w >= thr[m]) K[m] += 1u;
            else U[m] += gw;
          }
        }
      }
    }
#pragma unroll
    for (int m = 0; m < MM; ++m) U[m] += T;
    const bool anybad = __any_sync(FULL, bad);
    reduce_scatter<MM>(U, K, lane);
    unsigned long long *acc = a.acc + s * ACC;
    const int m = lane >> (5 - (MM == 8 ? 3 : MM == 4 ? 2 : 1));
    if ((lane & (32 / MM - 1)) == 0 && m < M) {
      acc[2 + m] = U[0];
      acc[2 + MAXM + m] = K[0];
    }
    if (anybad && lane == 0) atomicOr(acc + 1, F_BAD);
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
        u = acc[0] - r.srv;  // fast path: U_m = total G - own served head (k1s_prep)
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

// fast-path launcher: the TMA ring kernel (default) or the register-pipelined
// one (ES_K1_FAST=regs, or when the profile image leaves no room for 2 slots)
template <int NW>
cudaError_t launch_tma(const uint8_t *img, const ImgLayout &lay, const StreamArgs &a, int64_t nq, cudaStream_t st,
                       int sms, int optin, bool regs) {
  TmaRing rg{};
  rg.ring_off = (lay.core_bytes + 127u) & ~127u;
  const int64_t room = (int64_t)optin - 64 - rg.ring_off;
  for (uint32_t pv = PV_MAX; pv >= 128u && rg.nsl < 3u; pv >>= 1) {
    const int64_t per_slot = NW * (pv * 16 + 8);
    rg.pv = pv;
    rg.nsl = room > 0 ? (uint32_t)(room / per_slot < 6 ? room / per_slot : 6) : 0u;
  }
  if (regs || rg.nsl < 2) return launch_persistent(k1s_stream_fast, img, lay, a, nq, 8, lay.core_bytes, st, sms);
  rg.mbar_off = rg.ring_off + NW * rg.nsl * rg.pv * 16u;
  const size_t dyn = rg.mbar_off + NW * rg.nsl * 8u;
  // single SLO: table bases as parameters; the masked A index must stay inside dynamic smem
  const bool one = lay.ncfg == 1 && (size_t)lay.c0_offA + lay.c0_amask + 4u <= dyn;
  auto kern = one ? k1s_stream_tma<true, NW> : k1s_stream_tma<false, NW>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)sms);
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, img, lay, a, rg);
}

// fast-path launcher: the TMA ring kernel (default; ES_K1_NW = consumer warps
// per CTA) or the register-pipelined one (ES_K1_FAST=regs, or when the profile
// image leaves no room for 2 slots per warp)
cudaError_t launch_fast(const uint8_t *img, const ImgLayout &lay, const StreamArgs &a, int64_t nq, cudaStream_t st,
                        int sms) {
  const char *env = getenv("ES_K1_FAST");
  const bool regs = env && strcmp(env, "regs") == 0;
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  const char *nw = getenv("ES_K1_NW");
  const int w = nw ? atoi(nw) : 16;
  if (w == 32) return launch_tma<32>(img, lay, a, nq, st, sms, optin, regs);
  if (w == 24) return launch_tma<24>(img, lay, a, nq, st, sms, optin, regs);
  return launch_tma<16>(img, lay, a, nq, st, sms, optin, regs);
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
  if (e == cudaSuccess) e = launch_persistent(k1s_prep, img, lay, a, nq, 256, lay.core_bytes, st, sms, false);
  if (e == cudaSuccess) e = launch_fast(img, lay, a, nq, st, sms);
  if (e == cudaSuccess) {
    if (lay.M <= 2) e = launch_persistent(k1s_clip<2>, img, lay, a, sn.n, 8, lay.core_bytes, st, sms);
    else if (lay.M <= 4) e = launch_persistent(k1s_clip<4>, img, lay, a, sn.n, 8, lay.core_bytes, st, sms);
    else e = launch_persistent(k1s_clip<8>, img, lay, a, sn.n, 8, lay.core_bytes, st, sms);
  }
  if (e == cudaSuccess) e = launch_persistent(k1s_finish, img, lay, a, sn.n, 32, 0, st, sms);
  const cudaError_t f = cudaFreeAsync(scratch, st);
  return e != cudaSuccess ? e : f;
}

}  // namespace es
