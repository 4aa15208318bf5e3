// k3_stats.cu -- K3: per-scenario nearest-rank P95 and the per-group merge
// (steps a9, a10).
//
// P95 (reading Q15): the k-th smallest post-warmup latency, k = ceil(0.95 N),
// found by exact radix selection with 12-bit digits.  Per scenario (one CTA,
// six per SM): the latencies are streamed from global memory with 16-byte
// loads, a coarse histogram of min(T >> 12, 4095) selects the 4.096 ms bin of
// the rank, and a second pass (an L2 re-read) histograms T & 0xFFF inside it
// -> the exact value.  Ranks among T >= 16.77 s take a radix select from the
// top significant bit instead (1-3 more passes).
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

// find_bin for a CTA's own shared-memory histogram (< 2^32 values): 32-bit
// scan, the warp offsets by one REDUX, the full 4096-bin case read as 16-byte
// words (4-way instead of 16-way bank conflicts)
__device__ uint32_t find_bin32(const uint32_t *hist, int nbins, uint32_t k, uint32_t *before) {
  __shared__ uint32_t s_warp[NW];
  __shared__ uint32_t s_bin, s_before;
  const int per = (nbins + NT - 1) / NT;
  const int b0 = threadIdx.x * per;
  uint32_t loc = 0;
  if (nbins == 16 * NT) {
    const uint4 *h4 = reinterpret_cast<const uint4 *>(hist + b0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 x = h4[i];
      loc += x.x + x.y + x.z + x.w;
    }
  } else {
    for (int i = 0; i < per; ++i)
      if (b0 + i < nbins) loc += hist[b0 + i];
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  incl += __reduce_add_sync(0xffffffffu, lane < wid ? s_warp[lane] : 0u);
  const uint32_t excl = incl - loc;
  if (excl < k && k <= incl) {
    uint32_t run = excl;
    for (int i = 0; i < per && b0 + i < nbins; ++i) {
      const uint32_t h = hist[b0 + i];
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

// L2 prefetch of the 4-byte words [p, q) by one bulk operation (the next
// scenario's latencies, fetched from HBM while this one is selected)
__device__ __forceinline__ void prefetch_l2(const uint32_t *p, const uint32_t *q) {
  const uintptr_t a = (uintptr_t)p & ~(uintptr_t)15, b = ((uintptr_t)q + 15) & ~(uintptr_t)15;
  if (b > a)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(b - a)) : "memory");
}

// apply f to each of the n words at g (global): 16-byte loads of the aligned
// interior, U per thread in flight, the (<= 3 + 3) edge words loaded singly
template <int U, typename F>
__device__ __forceinline__ void each_value(const uint32_t *g, uint32_t n, bool last_use, F f) {
  const uint32_t off = (uint32_t)(((uintptr_t)g >> 2) & 3u);
  const uint32_t lead = off ? min(4u - off, n) : 0u;
  const uint4 *q4 = reinterpret_cast<const uint4 *>(g + lead);
  const uint32_t nq = (n - lead) / 4u;
  const uint32_t tail0 = lead + 4u * nq;
  if (threadIdx.x < lead) f(__ldg(g + threadIdx.x));
  if (threadIdx.x >= 8u && threadIdx.x - 8u < n - tail0) f(__ldg(g + tail0 + (threadIdx.x - 8u)));
  for (uint32_t q = threadIdx.x; q < nq; q += U * NT) {
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q + u * NT < nq) x[u] = last_use ? __ldcs(q4 + q + u * NT) : __ldg(q4 + q + u * NT);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q + u * NT < nq) {
        f(x[u].x);
        f(x[u].y);
        f(x[u].z);
        f(x[u].w);
      }
  }
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
  uint32_t n_groups;  // 0: no group outputs
  uint64_t *counts;   // [G][ES_NGSTAT]
  uint64_t *hist0;    // [G][4096] coarse level
};

// shared layout of k3_stats: hist[4096] then priv[PRIV][32] -- the coarse bins
// below PRIV (T < 131 ms: 99.9 % of cfg3's latencies) counted per lane, so a
// warp's increments land in 32 distinct banks instead of piling onto the few
// addresses the coarse histogram concentrates them on (same-address atomics
// serialise: 129 M bank conflicts in the capture before this layout)
constexpr uint32_t PRIV = 32;

template <int U, int MINB>
__global__ void __launch_bounds__(NT, MINB) k3_stats(StatsArgs a) {
  __shared__ __align__(16) uint32_t hist[BINS + PRIV * 32];
  uint32_t *priv = hist + BINS;
  __shared__ uint32_t s_max;
  for (int i = threadIdx.x; i < BINS + (int)PRIV * 32; i += NT) hist[i] = 0u;
  // per-scenario metadata, fetched one scenario ahead: its chain of global
  // loads (status, config, group, trace span, the group columns) is in flight
  // during the previous scenario's histogram passes
  static_assert(ES_ST_INFEASIBLE == 5 && ES_ST_EXIT0 == ES_ST_ACC_BP + 1 && ES_ST_EXIT7 + 1 == ES_NSTAT, "cols");
  // group column t -> scenario column: decisions .. infeasible, sum_lat, acc_bp, exit0 .. exit7
  const int tcol = threadIdx.x < 6 ? (int)threadIdx.x : threadIdx.x == 6 ? ES_ST_SUM_LAT : ES_ST_ACC_BP + ((int)threadIdx.x - 7);
  struct Meta {
    uint64_t status, base, end, col;
    uint32_t k, g;
  };
  auto fetch = [&](int64_t s, Meta &m) {
    if (s >= a.n_scen) return;
    const uint64_t *st = a.stats + s * ES_NSTAT;
    m.status = st[ES_ST_STATUS];
    m.k = a.cfg_idx ? (uint32_t)a.cfg_idx[s] : 0u;
    m.g = a.group_id ? a.group_id[s] : 0u;
    m.base = a.arr_off[s * a.M];
    m.end = a.arr_off[s * a.M + a.M];
    m.col = threadIdx.x < ES_NGSTAT ? st[tcol] : 0ull;
  };
  Meta nxt;
  fetch(blockIdx.x, nxt);
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  __syncthreads();
  for (int64_t s = blockIdx.x; s < a.n_scen; s += gridDim.x) {
    const Meta m = nxt;
    fetch(s + gridDim.x, nxt);  // consumed on the next trip
    if (m.status != 0ull) {
      if (a.p95 && threadIdx.x == 0) a.p95[s] = 0u;
      continue;
    }
    const uint32_t g = m.g;
    const bool grp = a.n_groups && g < a.n_groups;
    if (grp && threadIdx.x < ES_NGSTAT)
      atomicAdd(reinterpret_cast<unsigned long long *>(a.counts + (uint64_t)g * ES_NGSTAT + threadIdx.x),
                (unsigned long long)m.col);
    const uint32_t W = a.cfg[m.k].warmup;
    const uint64_t total = m.end - m.base;
    const uint32_t n = total > W ? (uint32_t)(total - W) : 0u;
    if (n == 0u) {
      if (a.p95 && threadIdx.x == 0) a.p95[s] = 0u;
      continue;
    }
    // the latencies are streamed from global memory twice (pass B hits L2:
    // the scenario was read a moment before); hist is all zero here
    const uint32_t *gsrc = a.lat + m.base + W;
    if (threadIdx.x == 0) s_max = 0u;
    // pass A: coarse histogram min(T >> 12, 4095) -- the group level-0 digit,
    // and the first digit of the scenario's own selection
    uint32_t mx = 0;
    each_value<U>(gsrc, n, false, [&](uint32_t v) {
      mx = max(mx, v);
      const uint32_t b = min(v >> 12, COARSE_OVF);
      atomicAdd(b < PRIV ? priv + b * 32u + lane : hist + b, 1u);
    });
    mx = __reduce_max_sync(0xffffffffu, mx);
    // the next scenario's latencies: HBM -> L2 during this one's selection
    // (measured 1.10 -> 1.05 ms; issued at the top of the trip with the
    // records fetched two ahead: 1.10 ms)
    if (threadIdx.x == 0 && s + gridDim.x < a.n_scen && nxt.status == 0ull)
      prefetch_l2(a.lat + nxt.base, a.lat + nxt.end);
    __syncthreads();
    if (lane == 0) atomicMax(&s_max, mx);
    for (uint32_t b = wid; b < PRIV; b += NW) {  // fold the per-lane counts into hist
      const uint32_t c = __reduce_add_sync(0xffffffffu, priv[b * 32u + lane]);
      priv[b * 32u + lane] = 0u;
      if (lane == 0) hist[b] += c;
    }
    __syncthreads();
    const uint32_t vmax = s_max;
    const uint32_t top = min(vmax >> 12, COARSE_OVF);
    if (grp) {  // flush the coarse histogram into the group's level-0 histogram
      unsigned long long *gh = reinterpret_cast<unsigned long long *>(a.hist0 + (uint64_t)g * BINS);
      for (uint32_t i = threadIdx.x; i <= top; i += NT)
        if (hist[i]) atomicAdd(gh + i, (unsigned long long)hist[i]);
    }
    if (a.p95) {
      uint32_t kk = (uint32_t)((95ull * n + 99ull) / 100ull);  // ceil(0.95 n), 1-based rank
      uint32_t before;
      const uint32_t cb = find_bin32(hist, (int)top + 1, kk, &before);  // syncs: flush reads done
      uint32_t res;
      for (uint32_t i = threadIdx.x; i <= top; i += NT) hist[i] = 0u;
      __syncthreads();
      if (cb < COARSE_OVF) {  // pass B: T & 0xFFF inside the coarse bin -> exact value
        kk -= before;
        const uint32_t key = cb << 12;
        each_value<U>(gsrc, n, true, [&](uint32_t v) {
          const uint32_t d = v ^ key;
          if (d < 4096u) atomicAdd(&hist[d], 1u);
        });
        __syncthreads();
        const uint32_t fb = find_bin32(hist, BINS, kk, &before);
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
            const uint32_t v = __ldg(gsrc + i);
            if (((uint64_t)v >> prev) == hv) atomicAdd(&hist[(v >> shift) & dmask], 1u);
          }
          __syncthreads();
          const uint32_t bb = find_bin32(hist, (int)nb, kk, &before);
          kk -= before;
          hv = (hv << (prev - shift)) | bb;
          if (shift == 0u) break;
          prev = shift;
          shift = shift > 12u ? shift - 12u : 0u;
        }
        res = (uint32_t)hv;
      }
      if (threadIdx.x == 0) a.p95[s] = res;
      for (int i = threadIdx.x; i < BINS; i += NT) hist[i] = 0u;  // find_bin's reads are done
    } else {
      __syncthreads();  // flush reads done
      for (uint32_t i = threadIdx.x; i <= top; i += NT) hist[i] = 0u;
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
__global__ void __launch_bounds__(NT, 6) k_group_level(GroupArgs a, const uint32_t *order, int64_t per_cta) {
  __shared__ uint32_t hist[BINS];
  {  // nothing to do at this level (levels 2-3 when no group's rank lies among T >= 16.77 s)
    int need = 0;
    for (uint32_t g = threadIdx.x; g < a.n_groups; g += NT) {
      const uint64_t w1 = a.state[2 * g + 1];
      need |= !(w1 & DONE) && w1 != 0ull && (a.level == 1 || (a.state[2 * g] & MODE_OVF));
    }
    if (!__syncthreads_or(need)) return;
  }
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
  // per-scenario records fetched one scenario ahead (the scenario index two
  // ahead), so the chain order -> stats / group / span is in flight during the
  // previous scenario's stream; the group state and config are small tables
  struct Meta {
    uint64_t status, base, end;
    uint32_t g, k;
  };
  auto fetch = [&](int64_t s, Meta &m) {
    m.status = a.stats[s * ES_NSTAT + ES_ST_STATUS];
    m.g = a.group_id ? a.group_id[s] : 0u;
    m.k = a.cfg_idx ? (uint32_t)a.cfg_idx[s] : 0u;
    m.base = a.arr_off[s * a.M];
    m.end = a.arr_off[s * a.M + a.M];
  };
  Meta nxt{};
  if (lo < hi) fetch(order[lo], nxt);
  int64_t s_next = lo + 1 < hi ? (int64_t)order[lo + 1] : 0;
  for (int64_t j = lo; j < hi; ++j) {
    const Meta m = nxt;
    if (j + 1 < hi) fetch(s_next, nxt);
    if (j + 2 < hi) s_next = order[j + 2];
    if (m.status != 0ull) continue;
    const uint32_t g = m.g;
    if (g >= a.n_groups) continue;
    const uint64_t w1 = a.state[2 * g + 1];
    if ((w1 & DONE) || w1 == 0ull) continue;  // resolved or empty group
    const uint64_t w0 = a.state[2 * g];
    const bool ovf = (w0 & MODE_OVF) != 0ull;
    if (!ovf && a.level != 1) continue;
    const uint32_t prefix = (uint32_t)w0;
    const uint32_t W = a.cfg[m.k].warmup;
    const uint64_t base = m.base;
    const uint64_t total = m.end - base;
    if (total <= W) continue;
    if (g != cur) {  // uniform across the CTA
      flush();
      cur = g;
    }
    dirty = true;
    // latencies [base + W, base + total), streamed once per level (evict-first)
    const int lvl = a.level;
    each_value<2>(a.lat + base + W, (uint32_t)(total - W), true, [&](uint32_t v) {
      uint32_t bin;
      if (level_digit(v, lvl, ovf, prefix, bin)) atomicAdd(&hist[bin], 1u);
    });
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
  return a;
}

template <int U, int MINB>
cudaError_t launch_stats_t(const StatsArgs &a, cudaStream_t st, int sms) {
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k3_stats<U, MINB>, NT, 0);
  if (e != cudaSuccess) return e;
  int64_t blocks = a.n_scen;
  // 16 waves of resident CTAs over the grid-stride loop (measured on cfg3: 1 wave 1.10 ms, 4 1.05, 16 1.02,
  // 32 1.03, one CTA per scenario 1.08)
  const int64_t cap = (int64_t)sms * (occ > 0 ? occ : 1) * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k3_stats<U, MINB><<<(unsigned)blocks, NT, 0, st>>>(a);
  return cudaGetLastError();
}

// two 16-byte loads in flight per thread, six CTAs (48 warps) per SM: measured
// on cfg3 1.34 ms; four loads at five or four CTAs 1.42 / 1.49 ms, eight at
// three 1.77 ms (the per-scenario selection steps, not the load depth, bound it)
cudaError_t launch_stats(const StatsArgs &a, cudaStream_t st, int sms) { return launch_stats_t<2, 6>(a, st, sms); }

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
    int occ = 0;  // one wave of resident CTAs, each a contiguous run of grouped scenarios
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_group_level, NT, 0);
    const int64_t ctas = std::min<int64_t>(tr.n_scen, (int64_t)sms * std::max(occ, 1));  // (2-8 waves: same time)
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
