// k3_stats.cu -- K3: per-scenario nearest-rank P95 and the per-group merge
// (steps a9, a10).
//
// P95 (reading Q15): the k-th smallest post-warmup latency, k = ceil(0.95 N),
// found by exact radix selection with 12-bit digits.  Per scenario (one CTA):
// the latencies are staged in shared memory when they fit (else re-read from
// global), the top significant 12 bits form the first digit (so the first
// histogram is spread, not piled into bin 0), and 1-3 histogram passes select
// the exact value.
//
// Groups (sweep points) use digits that are the same on every rank, so that
// histograms from any number of ranks can be summed (all_reduce) before each
// selection and the result is bit-identical for any rank count:
//   level 0  coarse 4.096 ms bins: min(T >> 12, 4095)     (fused into K3)
//   level 1  normal:   T & 0xFFF inside the selected coarse bin -> exact value
//            overflow (coarse bin 4095, T >= 16.77 s): T >> 20
//   level 2  overflow: (T >> 8) & 0xFFF inside the selected T >> 20
//   level 3  overflow: T & 0xFF inside the selected T >> 8
// Levels 2-3 are no-ops for groups resolved at level 1 (the common case).
#include <cuda_runtime.h>

#include <algorithm>

#include "es_internal.cuh"

namespace es {
namespace {

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int BINS = ES_HIST_BINS;  // 4096
constexpr uint32_t COARSE_OVF = 4095u;
// group state [g][2]: word 0 = selected digit prefix (low 32 bits) | MODE_OVF
// while the selection runs, the P95 itself once done; word 1 = the residual
// rank as a full u64 (a group may hold far more than 2^32 completions), or
// DONE.  Ranks are < 2^63, so neither flag bit can be taken by a value.
constexpr uint64_t MODE_OVF = 1ull << 63;  // word 0: the rank lies among T >= 16.77 s
constexpr uint64_t DONE = 1ull << 63;      // word 1: resolved (word 0 is the P95)

// block-wide: find the bin holding rank k (1-based) in hist[0..nbins);
// returns bin and writes the count strictly before it into *before.
template <typename T>
__device__ uint32_t find_bin(const T *hist, int nbins, uint64_t k, uint64_t *before) {
  __shared__ uint64_t s_warp[NW];
  __shared__ uint32_t s_bin;
  __shared__ uint64_t s_before;
  const int per = (nbins + NT - 1) / NT;
  const int b0 = threadIdx.x * per;
  uint64_t loc = 0;
  for (int i = 0; i < per; ++i)
    if (b0 + i < nbins) loc += (uint64_t)hist[b0 + i];
  // inclusive scan: warp shuffles, then the warp totals
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  uint64_t woff = 0;
  for (int w = 0; w < wid; ++w) woff += s_warp[w];
  incl += woff;
  const uint64_t excl = incl - loc;
  if (excl < k && k <= incl) {
    uint64_t run = excl;
    for (int i = 0; i < per && b0 + i < nbins; ++i) {
      const uint64_t h = (uint64_t)hist[b0 + i];
      if (run + h >= k) {
        s_bin = (uint32_t)(b0 + i);
        s_before = run;
        break;
      }
      run += h;
    }
  }
  __syncthreads();
  *before = s_before;
  const uint32_t b = s_bin;
  __syncthreads();
  return b;
}

struct StatsArgs {
  int64_t n_scen;
  int M;
  const uint16_t *cfg_idx;
  const uint32_t *group_id;
  const uint64_t *arr_off;
  const uint32_t *lat;
  const uint64_t *stats;
  uint32_t *p95;  // per-scenario P95 or NULL
  const CfgRec *cfg;  // global copy of the records
  uint32_t cap;       // values staged in shared memory when n <= cap
  uint32_t n_groups;  // 0: no group outputs
  uint64_t *counts;   // [G][ES_NGSTAT]
  uint64_t *hist0;    // [G][4096] coarse level
};

__global__ void __launch_bounds__(NT) k3_stats(StatsArgs a) {
  __shared__ uint32_t hist[BINS];
  __shared__ uint32_t s_max;
  extern __shared__ __align__(16) uint32_t vals[];
  __shared__ uint64_t mbar;
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
  uint32_t phase = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (int64_t s = blockIdx.x; s < a.n_scen; s += gridDim.x) {
    const uint64_t *st = a.stats + s * ES_NSTAT;
    const int k = a.cfg_idx ? (int)a.cfg_idx[s] : 0;
    if (st[ES_ST_STATUS] != 0ull) {
      if (a.p95 && threadIdx.x == 0) a.p95[s] = 0u;
      continue;
    }
    const uint32_t g = a.group_id ? a.group_id[s] : 0u;
    const bool grp = a.n_groups && g < a.n_groups;
    if (grp && threadIdx.x < ES_NGSTAT) {
      // group column -> scenario column: decisions .. infeasible, sum_lat, acc_bp, exit0 .. exit7
      static_assert(ES_ST_INFEASIBLE == 5 && ES_ST_EXIT0 == ES_ST_ACC_BP + 1 && ES_ST_EXIT7 + 1 == ES_NSTAT, "cols");
      const int t = (int)threadIdx.x;
      const int col = t < 6 ? t : t == 6 ? ES_ST_SUM_LAT : ES_ST_ACC_BP + (t - 7);
      atomicAdd(reinterpret_cast<unsigned long long *>(a.counts + (uint64_t)g * ES_NGSTAT + threadIdx.x),
                (unsigned long long)st[col]);
    }
    const uint32_t W = a.cfg[k].warmup;
    const uint64_t base = a.arr_off[s * a.M];
    const uint64_t total = a.arr_off[s * a.M + a.M] - base;
    const uint32_t n = total > W ? (uint32_t)(total - W) : 0u;
    if (n == 0u) {
      if (a.p95 && threadIdx.x == 0) a.p95[s] = 0u;
      continue;
    }
    const uint32_t *gsrc = a.lat + base + W;
    const bool staged = n + 3u <= a.cap;  // + up to 3 leading words of 16-byte alignment
    // stage the scenario's latencies into shared memory with TMA: one bulk copy
    // of the 16-byte aligned span [gsrc - off, ...) (off <= 3 leading words
    // ignored), the <= 3 trailing words loaded directly
    const uint32_t *src = gsrc;
    uint32_t off = 0u;  // staged: vals[off + i] holds latency i (vals 16-byte aligned)
    if (staged) {
      off = (uint32_t)(((uintptr_t)gsrc >> 2) & 3u);
      const uint32_t nv4 = (n + off) / 4u;
      if (threadIdx.x == 0 && nv4) {
        // the previous scenario's generic-proxy reads of vals precede these async writes
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(16u * nv4) : "memory");
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(vals);
        const uint8_t *gs = reinterpret_cast<const uint8_t *>(gsrc - off);
        for (uint32_t o = 0; o < 16u * nv4; o += 16384u)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  dst + o),
              "l"(gs + o), "r"(min(16384u, 16u * nv4 - o)), "r"(mb)
              : "memory");
      }
      for (uint32_t j = 4u * nv4 + threadIdx.x; j < n + off; j += NT) vals[j] = gsrc[j - off];
      if (nv4) {
        uint32_t done = 0;
        while (!done)
          asm volatile(
              "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
              "selp.u32 %0, 1, 0, p;\n\t}"
              : "=r"(done)
              : "r"(mb), "r"(phase)
              : "memory");
        phase ^= 1u;
      }
      src = vals + off;
    }
    // pass A: coarse histogram min(T >> 12, 4095) -- the group level-0 digit,
    // and the first digit of the scenario's own selection
    for (int i = threadIdx.x; i < BINS; i += NT) hist[i] = 0u;
    if (threadIdx.x == 0) s_max = 0u;
    __syncthreads();  // staged tail words and the zeroed histogram are visible
    uint32_t mx = 0;
    // staged: 16-byte shared loads; the quads strictly inside [off, n + off)
    // take no per-element test, the (at most two) edge quads do
    const uint4 *v4 = reinterpret_cast<const uint4 *>(vals);
    const uint32_t nq = (n + off + 3u) / 4u;
    // (warp-aggregated updates -- __match_any, or a ballot loop per distinct
    // bin -- measured 1.5x and 5.6x slower than plain shared atomics here)
    auto add_bin = [&](uint32_t bin) {  // bin = 0xFFFFFFFF: no value
      if (bin != 0xFFFFFFFFu) atomicAdd(&hist[bin], 1u);
    };
    if (staged) {
      for (uint32_t q0 = threadIdx.x & ~31u; q0 < nq; q0 += NT) {  // warp-uniform trip count
        const uint32_t q = q0 + (threadIdx.x & 31);
        const uint4 x = q < nq ? v4[q] : make_uint4(0u, 0u, 0u, 0u);
        const uint32_t j = 4u * q;
        const uint32_t e[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const bool in = q < nq && j + c >= off && j + c < n + off;
          if (in) mx = max(mx, e[c]);
          add_bin(in ? min(e[c] >> 12, COARSE_OVF) : 0xFFFFFFFFu);
        }
      }
    } else {
      for (uint32_t i0 = threadIdx.x & ~31u; i0 < n; i0 += NT) {
        const uint32_t i = i0 + (threadIdx.x & 31);
        const uint32_t v = i < n ? __ldg(gsrc + i) : 0u;
        if (i < n) mx = max(mx, v);
        add_bin(i < n ? min(v >> 12, COARSE_OVF) : 0xFFFFFFFFu);
      }
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) atomicMax(&s_max, mx);
    __syncthreads();
    const uint32_t vmax = s_max;
    const uint32_t top = min(vmax >> 12, COARSE_OVF);
    if (grp) {  // flush the coarse histogram into the group's level-0 histogram
      unsigned long long *gh = reinterpret_cast<unsigned long long *>(a.hist0 + (uint64_t)g * BINS);
      for (uint32_t i = threadIdx.x; i <= top; i += NT)
        if (hist[i]) atomicAdd(gh + i, (unsigned long long)hist[i]);
    }
    if (a.p95) {
      uint64_t kk = (95ull * n + 99ull) / 100ull;  // ceil(0.95 n), 1-based rank
      uint64_t before;
      const uint32_t cb = find_bin(hist, (int)top + 1, kk, &before);  // syncs: flush reads done
      uint32_t res;
      if (cb < COARSE_OVF) {  // pass B: T & 0xFFF inside the coarse bin -> exact value
        kk -= before;
        for (int i = threadIdx.x; i < BINS; i += NT) hist[i] = 0u;
        __syncthreads();
        if (staged) {
          for (uint32_t q = threadIdx.x; q < nq; q += NT) {
            const uint4 x = v4[q];
            const uint32_t j = 4u * q;
            // words outside [off, n + off) never match (masked to all ones)
            const uint32_t e0 = j >= off && j < n + off ? x.x : 0xFFFFFFFFu;
            const uint32_t e1 = j + 1u >= off && j + 1u < n + off ? x.y : 0xFFFFFFFFu;
            const uint32_t e2 = j + 2u >= off && j + 2u < n + off ? x.z : 0xFFFFFFFFu;
            const uint32_t e3 = j + 3u < n + off ? x.w : 0xFFFFFFFFu;
            const bool h0 = (e0 >> 12) == cb, h1 = (e1 >> 12) == cb, h2 = (e2 >> 12) == cb, h3 = (e3 >> 12) == cb;
            if (h0 | h1 | h2 | h3) {
              if (h0) atomicAdd(&hist[e0 & 0xFFFu], 1u);
              if (h1) atomicAdd(&hist[e1 & 0xFFFu], 1u);
              if (h2) atomicAdd(&hist[e2 & 0xFFFu], 1u);
              if (h3) atomicAdd(&hist[e3 & 0xFFFu], 1u);
            }
          }
        } else {
          for (uint32_t i = threadIdx.x; i < n; i += NT) {
            const uint32_t v = __ldg(gsrc + i);
            if ((v >> 12) == cb) atomicAdd(&hist[v & 0xFFFu], 1u);
          }
        }
        __syncthreads();
        const uint32_t fb = find_bin(hist, BINS, kk, &before);
        res = (cb << 12) | fb;
      } else {  // the rank falls among T >= 16.77 s: radix select from the top bit
        const uint32_t nbits = 32u - __clz(vmax);
        uint32_t prev = nbits;  // bits >= prev already selected (hv)
        uint32_t shift = nbits > 12u ? nbits - 12u : 0u;
        uint64_t hv = 0;
        for (;;) {
          const uint32_t nb = 1u << (prev - shift);
          for (uint32_t i = threadIdx.x; i < nb; i += NT) hist[i] = 0u;
          __syncthreads();
          const uint32_t dmask = nb - 1u;
          for (uint32_t i = threadIdx.x; i < n; i += NT) {
            const uint32_t v = src[i];
            if (((uint64_t)v >> prev) == hv) atomicAdd(&hist[(v >> shift) & dmask], 1u);
          }
          __syncthreads();
          const uint32_t bb = find_bin(hist, (int)nb, kk, &before);
          kk -= before;
          hv = (hv << (prev - shift)) | bb;
          if (shift == 0u) break;
          prev = shift;
          shift = shift > 12u ? shift - 12u : 0u;
        }
        res = (uint32_t)hv;
      }
      if (threadIdx.x == 0) a.p95[s] = res;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ groups

struct GroupArgs {
  int64_t n_scen;
  int M;
  const uint16_t *cfg_idx;
  const uint32_t *group_id;
  const uint64_t *arr_off;
  const uint32_t *lat;
  const uint64_t *stats;
  const CfgRec *cfg;
  uint32_t n_groups;
  int level;
  const uint64_t *state;  // [G][2]
  uint64_t *hist;         // [G][4096]
};

// level-1..3 digit of latency v for a group in state (ovf, prefix); false if
// v does not match the prefix selected so far
__device__ __forceinline__ bool level_digit(uint32_t v, int level, bool ovf, uint32_t prefix, uint32_t &bin) {
  if (!ovf) {  // level 1, normal: exact value inside the coarse bin
    bin = v & 0xFFFu;
    return (v >> 12) == prefix;
  }
  if (level == 1) {
    bin = v >> 20;
    return (v >> 12) >= COARSE_OVF;
  }
  if (level == 2) {
    bin = (v >> 8) & 0xFFFu;
    return (v >> 12) >= COARSE_OVF && (v >> 20) == prefix;
  }
  bin = v & 0xFFu;
  return (v >> 12) >= COARSE_OVF && (v >> 8) == prefix;
}

// levels 1-3: histogram of the digit selected by each group's state.  The
// scenarios come grouped (a device counting sort by group id, `order`), each
// CTA streams a contiguous run of them -- 16-byte loads of the latencies --
// into one shared-memory histogram that is flushed to the group's global
// histogram only when the run moves to another group (or ends).
__global__ void __launch_bounds__(NT) k_group_level(GroupArgs a, const uint32_t *order, int64_t per_cta) {
  __shared__ uint32_t hist[BINS];
  for (int i = threadIdx.x; i < BINS; i += NT) hist[i] = 0u;
  __syncthreads();
  const int64_t lo = (int64_t)blockIdx.x * per_cta, hi = ::min(lo + per_cta, a.n_scen);
  uint32_t cur = 0xFFFFFFFFu;  // group whose counts hist holds
  bool dirty = false;
  auto flush = [&]() {
    __syncthreads();
    if (dirty) {
      unsigned long long *gh = reinterpret_cast<unsigned long long *>(a.hist + (uint64_t)cur * BINS);
      for (int i = threadIdx.x; i < BINS; i += NT)
        if (hist[i]) {
          atomicAdd(gh + i, (unsigned long long)hist[i]);
          hist[i] = 0u;
        }
    }
    dirty = false;
    __syncthreads();
  };
  for (int64_t j = lo; j < hi; ++j) {
    const int64_t s = order[j];
    const uint64_t *st = a.stats + s * ES_NSTAT;
    if (st[ES_ST_STATUS] != 0ull) continue;
    const uint32_t g = a.group_id ? a.group_id[s] : 0u;
    if (g >= a.n_groups) continue;
    const uint64_t w1 = a.state[2 * g + 1];
    if ((w1 & DONE) || w1 == 0ull) continue;  // resolved or empty group
    const uint64_t w0 = a.state[2 * g];
    const bool ovf = (w0 & MODE_OVF) != 0ull;
    if (!ovf && a.level != 1) continue;
    const uint32_t prefix = (uint32_t)w0;
    const int k = a.cfg_idx ? (int)a.cfg_idx[s] : 0;
    const uint32_t W = a.cfg[k].warmup;
    const uint64_t base = a.arr_off[s * a.M];
    const uint64_t total = a.arr_off[s * a.M + a.M] - base;
    if (total <= W) continue;
    if (g != cur) {  // uniform across the CTA
      flush();
      cur = g;
    }
    dirty = true;
    // latencies [b0, b1): scalar head up to 16-byte alignment, uint4 body, scalar tail
    const uint64_t b0 = base + W, b1 = base + total;
    const uint64_t h1 = ::min((uint64_t)((b0 + 3u) & ~3ull), b1), t0 = ::max((uint64_t)(b1 & ~3ull), h1);
    uint32_t bin;
    if (threadIdx.x < h1 - b0 && level_digit(a.lat[b0 + threadIdx.x], a.level, ovf, prefix, bin))
      atomicAdd(&hist[bin], 1u);
    if (threadIdx.x < b1 - t0 && level_digit(a.lat[t0 + threadIdx.x], a.level, ovf, prefix, bin))
      atomicAdd(&hist[bin], 1u);
    const uint4 *body = reinterpret_cast<const uint4 *>(a.lat + h1);
    const uint64_t nv = (t0 - h1) / 4u;
    for (uint64_t i = threadIdx.x; i < nv; i += NT) {
      const uint4 q = __ldcs(body + i);  // streamed once per level: do not keep it in L1/L2
      if (level_digit(q.x, a.level, ovf, prefix, bin)) atomicAdd(&hist[bin], 1u);
      if (level_digit(q.y, a.level, ovf, prefix, bin)) atomicAdd(&hist[bin], 1u);
      if (level_digit(q.z, a.level, ovf, prefix, bin)) atomicAdd(&hist[bin], 1u);
      if (level_digit(q.w, a.level, ovf, prefix, bin)) atomicAdd(&hist[bin], 1u);
    }
  }
  flush();
}

// counting sort of the scenarios by group id (the grouped order k_group_level streams)
__global__ void k_group_count(int64_t n_scen, const uint32_t *group_id, uint32_t n_groups, unsigned *cnt) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_scen; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t g = group_id ? group_id[s] : 0u;
    atomicAdd(cnt + (g < n_groups ? g : n_groups), 1u);  // bucket n_groups: out-of-range ids
  }
}

__global__ void k_group_scan(uint32_t nb, unsigned *cnt) {  // one CTA: exclusive scan in place (nb buckets)
  __shared__ unsigned carry;
  if (threadIdx.x == 0) carry = 0u;
  __syncthreads();
  for (uint32_t b0 = 0; b0 < nb; b0 += NT) {
    const uint32_t i = b0 + threadIdx.x;
    const unsigned v = i < nb ? cnt[i] : 0u;
    unsigned x = v;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    __shared__ unsigned ws[NW];
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    unsigned off = carry;
    for (int w = 0; w < wid; ++w) off += ws[w];
    if (i < nb) cnt[i] = off + x - v;
    __syncthreads();
    if (threadIdx.x == NT - 1) carry = off + x;
    __syncthreads();
  }
}

__global__ void k_group_scatter(int64_t n_scen, const uint32_t *group_id, uint32_t n_groups, unsigned *pos,
                                uint32_t *order) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_scen; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t g = group_id ? group_id[s] : 0u;
    order[atomicAdd(pos + (g < n_groups ? g : n_groups), 1u)] = (uint32_t)s;
  }
}

__global__ void __launch_bounds__(NT) k_group_select(uint32_t n_groups, int level, const uint64_t *counts,
                                                     const uint64_t *hist, uint64_t *state) {
  const uint32_t g = blockIdx.x;
  if (g >= n_groups) return;
  uint64_t w0, w1;
  if (level == 0) {
    const uint64_t N = counts[(uint64_t)g * ES_NGSTAT + 3];  // completed
    w0 = 0;
    w1 = (95ull * N + 99ull) / 100ull;
    if (w1 == 0ull) {  // empty group: P95 = 0, done
      if (threadIdx.x == 0) {
        state[2 * g] = 0ull;
        state[2 * g + 1] = DONE;
      }
      return;
    }
  } else {
    w0 = state[2 * g];
    w1 = state[2 * g + 1];
    if ((w1 & DONE) || w1 == 0ull) return;
    if (!(w0 & MODE_OVF) && level != 1) return;
  }
  const bool ovf = (w0 & MODE_OVF) != 0ull;
  w0 &= ~MODE_OVF;        // the digit prefix selected so far
  const uint64_t rank = w1;  // full u64 residual rank
  const int nbins = (level == 3) ? 256 : BINS;
  uint64_t before;
  const uint32_t b = find_bin(hist + (uint64_t)g * BINS, nbins, rank, &before);
  if (threadIdx.x == 0) {
    const uint64_t r = rank - before;
    uint64_t v;
    bool done = false, ovf_next = ovf;
    if (level == 0) {
      v = b;
      ovf_next = b == COARSE_OVF;
    } else if (!ovf) {  // level 1 normal: exact value
      v = ((uint64_t)w0 << 12) | b;
      done = true;
    } else if (level == 1) {
      v = b;  // T >> 20
    } else if (level == 2) {
      v = ((uint64_t)w0 << 12) | b;  // T >> 8
    } else {
      v = ((uint64_t)w0 << 8) | b;  // T
      done = true;
    }
    state[2 * g] = done ? v : (v | (ovf_next ? MODE_OVF : 0ull));
    state[2 * g + 1] = done ? DONE : r;
  }
}

StatsArgs stats_args(const uint8_t *img, const ImgLayout &lay, const es_traces &tr, const es_replay_out &out) {
  StatsArgs a{};
  a.n_scen = tr.n_scen;
  a.M = lay.M;
  a.cfg_idx = tr.cfg_idx;
  a.group_id = tr.group_id;
  a.arr_off = tr.arr_off;
  a.lat = out.latency_us;
  a.stats = out.scen_stats;
  a.p95 = out.scen_p95_us;
  a.cfg = reinterpret_cast<const CfgRec *>(img + lay.off_cfg);
  a.cap = 12288;  // 48 KB of staged latencies per CTA
  return a;
}

cudaError_t launch_stats(const StatsArgs &a, cudaStream_t st, int sms) {
  const size_t dyn = (size_t)a.cap * sizeof(uint32_t);
  cudaError_t e = cudaFuncSetAttribute(k3_stats, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k3_stats, NT, dyn);
  if (e != cudaSuccess) return e;
  int64_t blocks = a.n_scen;
  const int64_t cap = (int64_t)sms * (occ > 0 ? occ : 1) * 4;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k3_stats<<<(unsigned)blocks, NT, dyn, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_scen_p95(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                            const es_replay_out &out, cudaStream_t st, int sms) {
  return launch_stats(stats_args(img, lay, tr, out), st, sms);
}

cudaError_t launch_stats_fused(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                               const es_replay_out &out, uint32_t n_groups, uint64_t *counts, uint64_t *hist0,
                               cudaStream_t st, int sms) {
  StatsArgs a = stats_args(img, lay, tr, out);
  a.n_groups = n_groups;
  a.counts = counts;
  a.hist0 = hist0;
  return launch_stats(a, st, sms);
}

cudaError_t launch_group_accumulate(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                                    const es_replay_out &out, uint32_t n_groups, uint64_t *counts,
                                    uint64_t *hist0, cudaStream_t st) {
  es_replay_out o = out;
  o.scen_p95_us = nullptr;  // group contributions only
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return launch_stats_fused(img, lay, tr, o, n_groups, counts, hist0, st, sms);
}

cudaError_t launch_group_hist(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                              const es_replay_out &out, uint32_t n_groups, int level,
                              const uint64_t *state, uint64_t *hist, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)n_groups * BINS * sizeof(uint64_t), st);
  if (e != cudaSuccess) return e;
  if (tr.n_scen >= (int64_t)0xFFFFFFFF) return cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  GroupArgs a{};
  a.n_scen = tr.n_scen;
  a.M = lay.M;
  a.cfg_idx = tr.cfg_idx;
  a.group_id = tr.group_id;
  a.arr_off = tr.arr_off;
  a.lat = out.latency_us;
  a.stats = out.scen_stats;
  a.cfg = reinterpret_cast<const CfgRec *>(img + lay.off_cfg);
  a.n_groups = n_groups;
  a.level = level;
  a.state = state;
  a.hist = hist;
  // grouped scenario order (stream-ordered scratch, per call)
  const size_t nb = (size_t)n_groups + 1;
  void *buf = nullptr;
  e = cudaMallocAsync(&buf, 4 * (nb + (size_t)tr.n_scen), st);
  if (e != cudaSuccess) return e;
  unsigned *cnt = static_cast<unsigned *>(buf);
  uint32_t *order = cnt + nb;
  const int blocks = (int)std::min<int64_t>((tr.n_scen + 255) / 256, (int64_t)sms * 8);
  e = cudaMemsetAsync(cnt, 0, 4 * nb, st);
  if (e == cudaSuccess) {
    k_group_count<<<blocks, 256, 0, st>>>(tr.n_scen, tr.group_id, n_groups, cnt);
    k_group_scan<<<1, NT, 0, st>>>((uint32_t)nb, cnt);
    k_group_scatter<<<blocks, 256, 0, st>>>(tr.n_scen, tr.group_id, n_groups, cnt, order);
    const int64_t ctas = std::min<int64_t>(tr.n_scen, (int64_t)sms * 8);
    const int64_t per = (tr.n_scen + ctas - 1) / ctas;
    k_group_level<<<(unsigned)((tr.n_scen + per - 1) / per), NT, 0, st>>>(a, order, per);
    e = cudaGetLastError();
  }
  const cudaError_t f = cudaFreeAsync(buf, st);
  return e != cudaSuccess ? e : f;
}

cudaError_t launch_group_select(uint32_t n_groups, int level, const uint64_t *counts,
                                const uint64_t *hist, uint64_t *state, cudaStream_t st) {
  k_group_select<<<n_groups, NT, 0, st>>>(n_groups, level, counts, hist, state);
  return cudaGetLastError();
}

}  // namespace es
