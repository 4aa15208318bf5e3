// k3_stats.cu -- K3: per-scenario nearest-rank P95 and the per-group merge
// (steps a9, a10).
//
// P95 (reading Q15): the k-th smallest post-warmup latency, k = ceil(0.95 N),
// found by exact radix selection with 12-bit digits.  Per scenario (one CTA):
// the latencies are staged in shared memory when they fit (else re-read from
// global), the top significant 12 bits form the first digit (so the first
// histogram is spread, not piled into bin 0), and 1-3 histogram passes select
// the exact value.  Groups (sweep points) use fixed digits [20,32), [8,20),
// [0,8) so that histograms from any number of ranks can be summed
// (all_reduce) before each selection: the result is bit-identical for any
// rank count.
#include <cuda_runtime.h>

#include "es_internal.cuh"

namespace es {
namespace {

constexpr int NT = 256;
constexpr int BINS = ES_HIST_BINS;  // 4096

// block-wide: find the bin holding rank k (1-based) in hist[0..nbins);
// returns bin and writes the count strictly before it into *before.
template <typename T>
__device__ uint32_t find_bin(const T *hist, int nbins, uint64_t k, uint64_t *before) {
  __shared__ uint64_t s_part[NT];
  __shared__ uint32_t s_bin;
  __shared__ uint64_t s_before;
  const int per = (nbins + NT - 1) / NT;
  const int b0 = threadIdx.x * per;
  uint64_t loc = 0;
  for (int i = 0; i < per; ++i)
    if (b0 + i < nbins) loc += (uint64_t)hist[b0 + i];
  s_part[threadIdx.x] = loc;
  __syncthreads();
  // inclusive scan of NT partials (Hillis-Steele in shared memory)
  for (int o = 1; o < NT; o <<= 1) {
    uint64_t v = threadIdx.x >= o ? s_part[threadIdx.x - o] : 0ull;
    __syncthreads();
    s_part[threadIdx.x] += v;
    __syncthreads();
  }
  const uint64_t incl = s_part[threadIdx.x];
  const uint64_t excl = incl - loc;
  if (excl < k && k <= incl) {
    uint64_t run = excl;
    for (int i = 0; i < per; ++i) {
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

struct P95Args {
  int64_t n_scen;
  int M;
  const uint16_t *cfg_idx;
  const uint64_t *arr_off;
  const uint32_t *lat;
  const uint64_t *stats;
  uint32_t *p95;
  const CfgRec *cfg;  // global copy of the records
  uint32_t cap;       // values staged in shared memory when n <= cap
};

__global__ void __launch_bounds__(NT) k3_scen_p95(P95Args a) {
  __shared__ uint32_t hist[BINS];
  __shared__ uint32_t s_max;
  extern __shared__ __align__(16) uint32_t vals[];
  for (int64_t s = blockIdx.x; s < a.n_scen; s += gridDim.x) {
    const uint64_t *st = a.stats + s * ES_NSTAT;
    const int k = a.cfg_idx ? (int)a.cfg_idx[s] : 0;
    if (st[ES_ST_STATUS] != 0ull) {
      if (threadIdx.x == 0) a.p95[s] = 0u;
      continue;
    }
    const uint32_t W = a.cfg[k].warmup;
    const uint64_t base = a.arr_off[s * a.M];
    const uint64_t total = a.arr_off[s * a.M + a.M] - base;
    const uint32_t n = total > W ? (uint32_t)(total - W) : 0u;
    if (n == 0u) {
      if (threadIdx.x == 0) a.p95[s] = 0u;
      continue;
    }
    const uint32_t *g = a.lat + base + W;
    const bool staged = n <= a.cap;
    if (threadIdx.x == 0) s_max = 0u;
    __syncthreads();
    uint32_t mx = 0;
    for (uint32_t i = threadIdx.x; i < n; i += NT) {
      const uint32_t v = g[i];
      if (staged) vals[i] = v;
      mx = max(mx, v);
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) atomicMax(&s_max, mx);
    __syncthreads();
    const uint32_t *src = staged ? vals : g;
    const uint32_t nbits = 32u - __clz(s_max);
    uint32_t prev = nbits;  // bits >= prev already selected (hv)
    uint32_t shift = nbits > 12u ? nbits - 12u : 0u;
    uint64_t kk = (95ull * n + 99ull) / 100ull;  // ceil(0.95 n), 1-based rank
    uint64_t hv = 0;
    for (;;) {
      for (int i = threadIdx.x; i < BINS; i += NT) hist[i] = 0u;
      __syncthreads();
      const uint32_t dmask = (1u << (prev - shift)) - 1u;
      for (uint32_t i = threadIdx.x; i < n; i += NT) {
        const uint32_t v = src[i];
        if (((uint64_t)v >> prev) == hv) atomicAdd(&hist[(v >> shift) & dmask], 1u);
      }
      __syncthreads();
      uint64_t before;
      const uint32_t b = find_bin(hist, (int)(dmask + 1u), kk, &before);
      kk -= before;
      hv = (hv << (prev - shift)) | b;
      if (shift == 0u) break;
      prev = shift;
      shift = shift > 12u ? shift - 12u : 0u;
    }
    if (threadIdx.x == 0) a.p95[s] = (uint32_t)hv;
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
  const uint64_t *state;  // [G][2] prefix, rank (levels 1, 2)
  uint64_t *counts;       // [G][ES_NGSTAT] (level 0) or NULL
  uint64_t *hist;         // [G][4096]
};

__global__ void __launch_bounds__(NT) k_group_level(GroupArgs a) {
  __shared__ uint32_t hist[BINS];
  for (int64_t s = blockIdx.x; s < a.n_scen; s += gridDim.x) {
    const uint64_t *st = a.stats + s * ES_NSTAT;
    if (st[ES_ST_STATUS] != 0ull) continue;
    const uint32_t g = a.group_id ? a.group_id[s] : 0u;
    if (g >= a.n_groups) continue;
    if (a.level == 0 && a.counts && threadIdx.x < ES_NGSTAT) {
      const int col[ES_NGSTAT] = {ES_ST_DECISIONS, ES_ST_CANDIDATES, ES_ST_CELLS, ES_ST_COMPLETED,
                                  ES_ST_VIOLATIONS, ES_ST_INFEASIBLE, ES_ST_SUM_LAT};
      atomicAdd(reinterpret_cast<unsigned long long *>(a.counts + (uint64_t)g * ES_NGSTAT + threadIdx.x),
                (unsigned long long)st[col[threadIdx.x]]);
    }
    uint64_t prefix = 0;
    if (a.level > 0) {
      if (a.state[2 * g + 1] == 0ull) continue;  // empty group: nothing to select
      prefix = a.state[2 * g];
    }
    const int k = a.cfg_idx ? (int)a.cfg_idx[s] : 0;
    const uint32_t W = a.cfg[k].warmup;
    const uint64_t base = a.arr_off[s * a.M];
    const uint64_t total = a.arr_off[s * a.M + a.M] - base;
    if (total <= W) continue;
    const uint32_t n = (uint32_t)(total - W);
    const uint32_t *src = a.lat + base + W;
    for (int i = threadIdx.x; i < BINS; i += NT) hist[i] = 0u;
    __syncthreads();
    for (uint32_t i0 = 0; i0 < n; i0 += NT) {  // whole warps iterate together (ballot below)
      const uint32_t i = i0 + threadIdx.x;
      const uint32_t v = i < n ? src[i] : 0u;
      uint32_t bin;
      bool take;
      if (i >= n) {
        bin = 0u;
        take = false;
      } else if (a.level == 0) {
        bin = v >> 20;
        take = true;
      } else if (a.level == 1) {
        bin = (v >> 8) & 0xFFFu;
        take = (v >> 20) == (uint32_t)prefix;
      } else {
        bin = v & 0xFFu;
        take = (v >> 8) == (uint32_t)prefix;
      }
      // warp-aggregated shared atomics: lanes with the same bin add once
      const unsigned act = __ballot_sync(0xffffffffu, take);
      if (take) {
        const unsigned peers = __match_any_sync(act, bin);
        if ((threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
      }
    }
    __syncthreads();
    unsigned long long *gh = reinterpret_cast<unsigned long long *>(a.hist + (uint64_t)g * BINS);
    for (int i = threadIdx.x; i < BINS; i += NT)
      if (hist[i]) atomicAdd(gh + i, (unsigned long long)hist[i]);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(NT) k_group_select(uint32_t n_groups, int level, const uint64_t *counts,
                                                     const uint64_t *hist, uint64_t *state) {
  const uint32_t g = blockIdx.x;
  if (g >= n_groups) return;
  uint64_t rank, prefix;
  if (level == 0) {
    const uint64_t N = counts[(uint64_t)g * ES_NGSTAT + 3];  // completed
    rank = (95ull * N + 99ull) / 100ull;
    prefix = 0;
  } else {
    prefix = state[2 * g];
    rank = state[2 * g + 1];
  }
  if (rank == 0ull) {  // empty group
    if (threadIdx.x == 0) {
      state[2 * g] = 0ull;
      state[2 * g + 1] = 0ull;
    }
    return;
  }
  const int nbins = level == 2 ? 256 : BINS;
  uint64_t before;
  const uint32_t b = find_bin(hist + (uint64_t)g * BINS, nbins, rank, &before);
  if (threadIdx.x == 0) {
    state[2 * g] = level == 0 ? b : (level == 1 ? ((prefix << 12) | b) : ((prefix << 8) | b));
    state[2 * g + 1] = rank - before;
  }
}

}  // namespace

cudaError_t launch_scen_p95(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                            const es_replay_out &out, cudaStream_t st, int sms) {
  P95Args a;
  a.n_scen = tr.n_scen;
  a.M = lay.M;
  a.cfg_idx = tr.cfg_idx;
  a.arr_off = tr.arr_off;
  a.lat = out.latency_us;
  a.stats = out.scen_stats;
  a.p95 = out.scen_p95_us;
  a.cfg = reinterpret_cast<const CfgRec *>(img + lay.off_cfg);
  a.cap = 12288;  // 48 KB of staged latencies per CTA
  const size_t dyn = (size_t)a.cap * sizeof(uint32_t);
  cudaError_t e = cudaFuncSetAttribute(k3_scen_p95, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k3_scen_p95, NT, dyn);
  if (e != cudaSuccess) return e;
  int64_t blocks = tr.n_scen;
  const int64_t cap = (int64_t)sms * (occ > 0 ? occ : 1) * 4;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k3_scen_p95<<<(unsigned)blocks, NT, dyn, st>>>(a);
  return cudaGetLastError();
}

static GroupArgs group_args(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                            const es_replay_out &out, uint32_t n_groups) {
  GroupArgs a;
  a.n_scen = tr.n_scen;
  a.M = lay.M;
  a.cfg_idx = tr.cfg_idx;
  a.group_id = tr.group_id;
  a.arr_off = tr.arr_off;
  a.lat = out.latency_us;
  a.stats = out.scen_stats;
  a.cfg = reinterpret_cast<const CfgRec *>(img + lay.off_cfg);
  a.n_groups = n_groups;
  a.state = nullptr;
  a.counts = nullptr;
  a.hist = nullptr;
  a.level = 0;
  return a;
}

static unsigned group_grid(int64_t n_scen) {
  int64_t b = n_scen < 148 * 16 ? n_scen : 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

cudaError_t launch_group_accumulate(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                                    const es_replay_out &out, uint32_t n_groups, uint64_t *counts,
                                    uint64_t *hist0, cudaStream_t st) {
  GroupArgs a = group_args(img, lay, tr, out, n_groups);
  a.level = 0;
  a.counts = counts;
  a.hist = hist0;
  k_group_level<<<group_grid(tr.n_scen), NT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_group_hist(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                              const es_replay_out &out, uint32_t n_groups, int level,
                              const uint64_t *state, uint64_t *hist, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)n_groups * BINS * sizeof(uint64_t), st);
  if (e != cudaSuccess) return e;
  GroupArgs a = group_args(img, lay, tr, out, n_groups);
  a.level = level;
  a.state = state;
  a.hist = hist;
  k_group_level<<<group_grid(tr.n_scen), NT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_group_select(uint32_t n_groups, int level, const uint64_t *counts,
                                const uint64_t *hist, uint64_t *state, cudaStream_t st) {
  k_group_select<<<n_groups, NT, 0, st>>>(n_groups, level, counts, hist, state);
  return cudaGetLastError();
}

}  // namespace es
