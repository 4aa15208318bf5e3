// es_internal.cuh -- shared device/host definitions of the CUDA path.
//
// The "profile image" is one contiguous, 16-byte aligned blob in device
// memory that every kernel stages into shared memory with a single TMA bulk
// copy (cp.async.bulk + mbarrier).  Layout (byte offsets in ImgLayout):
//   lat   u32 [M][E][nb]    L(m, e, bs[b]) in us
//   latT  u32 [M][nb][8]    the same, exit-minor, padded with 0xFFFFFFFF (one
//                           16-byte row pair per (m, b): Eq. 6 as a count)
//   bs    u16 [nb]          profiled batch sizes
//   mask  u32 [M]           allowed-exit bitmask per model  (P:517-527 ablation)
//   acc   u16 [M][E]        top-1 accuracy per (model, exit), basis points (Table I)
//   cfg   CfgRec [ncfg]     per-SLO constants (tau, x_c, r, C_q, b_max, W, ...)
//   per cfg c: A u32[nA_cap], Bt u32[1024], H u64[M*E*nb], bidx u8[b_max+1]
// A, Bt, H, x_c, bidx are written on the GPU by k_build_tables (k_tables.cu).
#pragma once
#include <cstdint>

#include "../../include/edgeserve.h"

namespace es {

constexpr int F = 28;         // fractional bits of the fixed-point score (Q5)
constexpr int SBITS = 10;     // Bt covers 2^SBITS us
constexpr uint32_t S = 1024;  // 2^SBITS
constexpr int MAXM = ES_MAX_MODELS;
constexpr int MAXE = ES_MAX_EXITS;

struct __align__(16) CfgRec {
  uint32_t tau, C, b_max, warmup;
  uint32_t x_c, r, nA, nA_cap;
  uint64_t C_q;
  uint32_t off_A, off_Bt, off_H, off_bidx;
  uint32_t status;    // ES_OK or ES_ERR_NUMERIC (set by k_build_tables)
  uint32_t fast_lim;  // x_c - max L over the profile (0 if <= 0): waits below it never clip
  uint32_t policy;    // ES_POLICY_* (selection rule, Q26)
  uint32_t pad[3];
};
static_assert(sizeof(CfgRec) == 80, "CfgRec layout");

struct ImgLayout {
  uint32_t bytes;       // total, multiple of 16
  uint32_t core_bytes;  // prefix without the per-cfg H tables (they form the tail)
  int32_t M, E, nb, ncfg;
  uint32_t off_lat, off_bs, off_mask, off_acc, off_cfg;
  uint32_t off_latT;  // latT u32 [M][nb][8]: L(m, e, bs[b]) for e < E, 0xFFFFFFFF past E (Eq. 6 by counting)
  // cfg 0's urgency-table constants (host-computed), kernel parameters for the
  // single-SLO specialisation of the K1 stream: byte offsets of A and Bt, 4 r,
  // and the A index mask 4 (2^k - 1) with 2^k >= nA_cap
  uint32_t c0_offA, c0_offBt, c0_r4, c0_amask;
  uint32_t pol_mask;  // bit p set iff some cfg uses policy p (ES_POLICY_*)
};

// device-side sticky error record (per profile handle)
struct DevStatus {
  unsigned long long item;  // first failing item
  uint32_t code;
  uint32_t pad;
};

// kernel launchers (defined in the .cu files, called from api.cu)
cudaError_t launch_build_tables(uint8_t *img, const ImgLayout &lay, cudaStream_t st);
cudaError_t launch_score(const uint8_t *img, const ImgLayout &lay, const es_snapshots &sn,
                         const es_decisions &out, DevStatus *dstat, cudaStream_t st, int sms);
cudaError_t launch_score_stream(const uint8_t *img, const ImgLayout &lay, const es_snapshots &sn,
                                const es_decisions &out, DevStatus *dstat, cudaStream_t st, int sms);
cudaError_t launch_replay(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                          const es_replay_out &out, DevStatus *dstat, cudaStream_t st, int sms, int *n_launch);
cudaError_t launch_scen_p95(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                            const es_replay_out &out, cudaStream_t st, int sms);
cudaError_t launch_stats_fused(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                               const es_replay_out &out, uint32_t n_groups, uint64_t *counts, uint64_t *hist0,
                               cudaStream_t st, int sms);
cudaError_t launch_group_accumulate(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                                    const es_replay_out &out, uint32_t n_groups, uint64_t *counts,
                                    uint64_t *hist0, cudaStream_t st);
cudaError_t launch_group_hist(const uint8_t *img, const ImgLayout &lay, const es_traces &tr,
                              const es_replay_out &out, uint32_t n_groups, int level,
                              const uint64_t *state, uint64_t *hist, cudaStream_t st);
cudaError_t launch_group_select(uint32_t n_groups, int level, const uint64_t *counts,
                                const uint64_t *hist, uint64_t *state, cudaStream_t st);

}  // namespace es
