// api.cu -- the C ABI (include/edgeserve.h): host-side validation, profile
// image layout, library-owned device memory and kernel launches.
//
// Nothing of the method is computed here: the host only checks the inputs the
// paper's problem statement fixes (M queues, L(m,e,B), tau, B_max;
// profile invariants S:26-34), lays out the profile image and launches
// K-tables (k_tables.cu), K1 (k1_score.cu), K2 (k2_replay.cu) and K3
// (k3_stats.cu) on the caller's stream.
#include <cuda_runtime.h>

#include <cmath>
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "es_internal.cuh"

using namespace es;

struct es_profile {
  int device = 0;
  int sms = 148;
  ImgLayout lay{};
  uint8_t *d_img = nullptr;
  DevStatus *d_status = nullptr;
  std::vector<es_sched_cfg> cfgs;
  std::vector<uint8_t> h_img;  // host copy (after table build)
  std::atomic<int64_t> launches{0};  // kernel launches (calls may come from several host threads)
  // scratch for es_replay_traces_host (double-buffered by the pipelined call)
  uint8_t *scratch = nullptr;
  size_t scratch_bytes = 0;
  uint8_t *scratch2 = nullptr;
  size_t scratch2_bytes = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr}, ev_start = nullptr;
};

namespace {

thread_local std::string g_err;

es_status fail(es_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

es_status cuda_fail(cudaError_t e, const char *where) {
  if (e == cudaErrorMemoryAllocation)
    return fail(ES_ERR_OOM, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
  return fail(ES_ERR_CUDA, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define CK(call, where)                      \
  do {                                       \
    cudaError_t _e = (call);                 \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

inline uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

es_status validate_profile(const es_profile_desc *d) {
  if (!d || !d->batch_sizes || !d->latency_us) return fail(ES_ERR_ARG, "null profile descriptor or array");
  if (d->M < 1 || d->M > ES_MAX_MODELS) return fail(ES_ERR_ARG, "M=%d outside 1..%d", d->M, ES_MAX_MODELS);
  if (d->E < 1 || d->E > ES_MAX_EXITS) return fail(ES_ERR_ARG, "E=%d outside 1..%d", d->E, ES_MAX_EXITS);
  if (d->nb < 1 || d->nb > ES_MAX_BATCHES) return fail(ES_ERR_ARG, "nb=%d outside 1..%d", d->nb, ES_MAX_BATCHES);
  if (d->batch_sizes[0] != 1) return fail(ES_ERR_PROFILE_GRID, "batch_sizes[0]=%d must be 1 (reading Q8)", d->batch_sizes[0]);
  for (int b = 1; b < d->nb; ++b)
    if (d->batch_sizes[b] <= d->batch_sizes[b - 1] || d->batch_sizes[b] > 65535)
      return fail(ES_ERR_PROFILE_GRID, "batch_sizes[%d]=%d not strictly increasing / above 65535", b,
                  d->batch_sizes[b]);
  for (int m = 0; m < d->M; ++m) {
    bool any = false;
    for (int e = 0; e < d->E; ++e) any |= d->exit_mask ? d->exit_mask[m * d->E + e] != 0 : true;
    if (!any) return fail(ES_ERR_PROFILE_GRID, "model %d has no allowed exit", m);
    for (int e = 0; e < d->E; ++e)
      if (d->accuracy_bp && d->accuracy_bp[m * d->E + e] > 10000)
        return fail(ES_ERR_ARG, "accuracy_bp(m=%d,e=%d)=%u above 10000 (100 %%)", m, e, d->accuracy_bp[m * d->E + e]);
    for (int e = 0; e < d->E; ++e)
      for (int b = 0; b < d->nb; ++b) {
        const uint32_t v = d->latency_us[((size_t)m * d->E + e) * d->nb + b];
        if (v == 0u) return fail(ES_ERR_PROFILE_MONOTONE, "L(m=%d,e=%d,b=%d) = 0", m, e, b);
        if (b > 0 && v < d->latency_us[((size_t)m * d->E + e) * d->nb + b - 1])
          return fail(ES_ERR_PROFILE_MONOTONE, "L(m=%d,e=%d,b=%d)=%u decreases in batch", m, e, b, v);
        if (e > 0 && v <= d->latency_us[((size_t)m * d->E + e - 1) * d->nb + b])
          return fail(ES_ERR_PROFILE_MONOTONE, "L(m=%d,e=%d,b=%d)=%u not above the shallower exit", m, e, b, v);
      }
  }
  return ES_OK;
}

es_status validate_cfg(const es_profile_desc *d, const es_sched_cfg &c, int k) {
  if (c.tau_us < 1024u || c.tau_us > (1u << 20))
    return fail(ES_ERR_ARG, "cfg %d: tau_us=%u outside [1024, 2^20]", k, c.tau_us);
  if (c.clip_C < 1u || c.clip_C > 15u) return fail(ES_ERR_ARG, "cfg %d: clip_C=%u outside 1..15", k, c.clip_C);
  if (c.b_max < 1u) return fail(ES_ERR_ARG, "cfg %d: b_max=0", k);
  if (c.b_max > (uint32_t)d->batch_sizes[d->nb - 1])
    return fail(ES_ERR_OUT_OF_GRID, "cfg %d: b_max=%u above the largest profiled batch %d", k, c.b_max,
                d->batch_sizes[d->nb - 1]);
  if (c.policy >= ES_POLICY_COUNT) return fail(ES_ERR_ARG, "cfg %d: unknown policy %u", k, c.policy);
  return ES_OK;
}

int max_dyn_smem(int dev) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v;
}

}  // namespace

extern "C" {

const char *es_last_error(void) { return g_err.c_str(); }
const char *es_version(void) { return "edgeserve-b200 0.1 (sm_100a)"; }

es_status es_load_profile(const es_profile_desc *desc, const es_sched_cfg *cfgs, int32_t ncfg, int32_t device,
                          es_profile **out) {
  if (!out) return fail(ES_ERR_ARG, "null output handle");
  *out = nullptr;
  es_status st = validate_profile(desc);
  if (st) return st;
  if (!cfgs || ncfg < 1 || ncfg > 65535) return fail(ES_ERR_ARG, "need 1..65535 cfgs (got %d)", ncfg);
  for (int k = 0; k < ncfg; ++k)
    if ((st = validate_cfg(desc, cfgs[k], k))) return st;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(ES_ERR_ARG, "device %d of %d", device, ndev);
  DeviceGuard guard(device);

  const int M = desc->M, E = desc->E, nb = desc->nb, cells = M * E * nb;
  ImgLayout lay{};
  lay.M = M;
  lay.E = E;
  lay.nb = nb;
  lay.ncfg = ncfg;
  uint32_t off = 0;
  lay.off_lat = off;
  off = align16(off + 4u * cells);
  lay.off_latT = off;
  off = align16(off + 32u * M * nb);
  lay.off_bs = off;
  off = align16(off + 2u * nb);
  lay.off_mask = off;
  off = align16(off + 4u * M);
  lay.off_acc = off;
  off = align16(off + 2u * M * E);
  lay.off_cfg = off;
  off = align16(off + (uint32_t)sizeof(CfgRec) * ncfg);
  std::vector<CfgRec> recs(ncfg);
  for (int k = 0; k < ncfg; ++k) {
    CfgRec &r = recs[k];
    memset(&r, 0, sizeof r);
    r.tau = cfgs[k].tau_us;
    r.C = cfgs[k].clip_C;
    r.b_max = cfgs[k].b_max;
    r.warmup = cfgs[k].warmup;
    r.policy = cfgs[k].policy;
    // capacity bound for A: x_c <= tau (1 + ln C) + 1 (+2 slack for rounding)
    const double xmax = std::floor((double)r.tau * (1.0 + std::log((double)r.C)) * (1.0 + 1e-12)) + 3.0;
    const uint32_t rr = (1024u - r.tau % 1024u) % 1024u;
    r.nA_cap = (uint32_t)(((uint64_t)xmax + rr) >> 10) + 2u;
    r.off_A = off;
    off = align16(off + 4u * r.nA_cap);
    r.off_Bt = off;
    off = align16(off + 4u * 1024u);
    r.off_bidx = off;
    off = align16(off + r.b_max + 1u);
    r.status = 0xFFFFFFFFu;
  }
  // the H tables of every cfg at the tail: kernels that need the urgency
  // tables in shared memory but can read H (one load per candidate) from
  // global memory stage only [0, core_bytes)
  lay.core_bytes = off;
  for (int k = 0; k < ncfg; ++k) {
    recs[k].off_H = off;
    off = align16(off + 8u * cells);
  }
  lay.bytes = off;
  lay.pol_mask = 0;
  for (int k = 0; k < ncfg; ++k) lay.pol_mask |= 1u << cfgs[k].policy;
  {
    uint32_t p2 = 1;
    while (p2 < recs[0].nA_cap) p2 <<= 1;
    lay.c0_offA = recs[0].off_A;
    lay.c0_offBt = recs[0].off_Bt;
    lay.c0_r4 = 4u * ((1024u - recs[0].tau % 1024u) % 1024u);
    lay.c0_amask = 4u * (p2 - 1u);
  }
  // kernels stage the image core (everything but the per-cfg H tables, read from
  // global memory) when the whole image would not fit or would cut residency
  const int smax = max_dyn_smem(device);
  if ((int)lay.core_bytes + 4096 > smax)
    return fail(ES_ERR_ARG,
                "profile image core of %u bytes (tables of %d cfgs) exceeds %d bytes of shared memory per CTA: "
                "split the cfgs over several handles",
                lay.core_bytes, ncfg, smax);

  std::vector<uint8_t> img(lay.bytes, 0);
  memcpy(img.data() + lay.off_lat, desc->latency_us, 4u * cells);
  for (int m = 0; m < M; ++m)
    for (int b = 0; b < nb; ++b)
      for (int e = 0; e < 8; ++e) {
        const uint32_t v = e < E ? desc->latency_us[(m * E + e) * nb + b] : 0xFFFFFFFFu;
        memcpy(img.data() + lay.off_latT + 4u * ((m * nb + b) * 8 + e), &v, 4);
      }
  for (int b = 0; b < nb; ++b) {
    const uint16_t v = (uint16_t)desc->batch_sizes[b];
    memcpy(img.data() + lay.off_bs + 2 * b, &v, 2);
  }
  for (int m = 0; m < M; ++m) {
    uint32_t bits = 0;
    for (int e = 0; e < E; ++e)
      if (!desc->exit_mask || desc->exit_mask[m * E + e]) bits |= 1u << e;
    memcpy(img.data() + lay.off_mask + 4 * m, &bits, 4);
  }
  if (desc->accuracy_bp) memcpy(img.data() + lay.off_acc, desc->accuracy_bp, 2u * M * E);
  memcpy(img.data() + lay.off_cfg, recs.data(), sizeof(CfgRec) * ncfg);

  {  // keep stream-ordered scratch (K1 streaming phases) cached in the pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  es_profile *p = new es_profile();
  p->device = device;
  p->lay = lay;
  p->cfgs.assign(cfgs, cfgs + ncfg);
  cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, device);
  auto cleanup = [&](es_status s) {
    es_free_profile(p);
    return s;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&p->d_img, lay.bytes)) != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc(image)"));
  if ((e = cudaMalloc(&p->d_status, sizeof(DevStatus))) != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc(status)"));
  if ((e = cudaMemset(p->d_status, 0, sizeof(DevStatus))) != cudaSuccess) return cleanup(cuda_fail(e, "memset"));
  if ((e = cudaMemcpy(p->d_img, img.data(), lay.bytes, cudaMemcpyHostToDevice)) != cudaSuccess)
    return cleanup(cuda_fail(e, "upload image"));
  if ((e = launch_build_tables(p->d_img, lay, 0)) != cudaSuccess) return cleanup(cuda_fail(e, "k_build_tables"));
  p->launches++;
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cleanup(cuda_fail(e, "k_build_tables sync"));
  p->h_img.resize(lay.bytes);
  if ((e = cudaMemcpy(p->h_img.data(), p->d_img, lay.bytes, cudaMemcpyDeviceToHost)) != cudaSuccess)
    return cleanup(cuda_fail(e, "download image"));
  for (int k = 0; k < ncfg; ++k) {
    CfgRec r;
    memcpy(&r, p->h_img.data() + lay.off_cfg + sizeof(CfgRec) * k, sizeof r);
    if (r.status == ES_ERR_NUMERIC)
      return cleanup(fail(ES_ERR_NUMERIC, "cfg %d (tau=%u, C=%u): a table value lies within 1e-7 of an integer", k,
                          r.tau, r.C));
    if (r.status != ES_OK) return cleanup(fail(ES_ERR_ARG, "cfg %d: table build status %u", k, r.status));
  }
  *out = p;
  return ES_OK;
}

es_status es_free_profile(es_profile *p) {
  if (!p) return ES_OK;
  DeviceGuard guard(p->device);
  cudaFree(p->d_img);
  cudaFree(p->d_status);
  cudaFree(p->scratch);
  cudaFree(p->scratch2);
  if (p->copy_stream) {
    cudaStreamSynchronize(p->copy_stream);
    cudaStreamDestroy(p->copy_stream);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(p->ev_copied[i]);
      cudaEventDestroy(p->ev_done[i]);
    }
    cudaEventDestroy(p->ev_start);
  }
  delete p;
  return ES_OK;
}

es_status es_get_tables(const es_profile *p, int32_t k, uint64_t *x_c_out, uint32_t *r_out, int32_t *nA_out,
                        uint32_t *A_out, int32_t A_cap, uint32_t *Bt_out, uint64_t *H_out) {
  if (!p) return fail(ES_ERR_ARG, "null profile");
  if (k < 0 || k >= p->lay.ncfg) return fail(ES_ERR_ARG, "cfg %d of %d", k, p->lay.ncfg);
  CfgRec r;
  memcpy(&r, p->h_img.data() + p->lay.off_cfg + sizeof(CfgRec) * k, sizeof r);
  if (x_c_out) *x_c_out = r.x_c;
  if (r_out) *r_out = r.r;
  if (nA_out) *nA_out = (int32_t)r.nA;
  if (A_out) {
    if (A_cap < (int32_t)r.nA) return fail(ES_ERR_ARG, "A_cap %d < nA %u", A_cap, r.nA);
    memcpy(A_out, p->h_img.data() + r.off_A, 4u * r.nA);
  }
  if (Bt_out) memcpy(Bt_out, p->h_img.data() + r.off_Bt, 4u * 1024u);
  if (H_out) memcpy(H_out, p->h_img.data() + r.off_H, 8u * p->lay.M * p->lay.E * p->lay.nb);
  return ES_OK;
}

es_status es_score_candidates(const es_profile *p, const es_snapshots *sn, es_decisions *out, es_stream stream) {
  if (!p || !sn || !out) return fail(ES_ERR_ARG, "null argument");
  if (sn->n < 0) return fail(ES_ERR_ARG, "n=%lld < 0", (long long)sn->n);
  if (sn->n == 0) return ES_OK;
  if (!sn->q_off || !sn->waits_us || !out->m || !out->e || !out->B || !out->L_us || !out->score_q || !out->flags)
    return fail(ES_ERR_ARG, "null snapshot input or decision output pointer");
  for (size_t k = 0; k < p->cfgs.size(); ++k)
    if (p->cfgs[k].policy == ES_POLICY_SYMPHONY)
      return fail(ES_ERR_ARG, "es_score_candidates: deferred batching (cfg %zu) needs a replay clock", k);
  DeviceGuard guard(p->device);
  CK(launch_score(p->d_img, p->lay, *sn, *out, p->d_status, (cudaStream_t)stream, p->sms), "k1_score");
  const_cast<es_profile *>(p)->launches++;
  return ES_OK;
}

es_status es_replay_traces(const es_profile *p, const es_traces *tr, es_replay_out *out, es_stream stream) {
  if (!p || !tr || !out) return fail(ES_ERR_ARG, "null argument");
  if (tr->n_scen < 0) return fail(ES_ERR_ARG, "n_scen < 0");
  if (tr->n_scen == 0) return ES_OK;
  if (!tr->arr_off || !tr->arrival_us || !out->latency_us || !out->scen_stats)
    return fail(ES_ERR_ARG, "null arr_off / arrival_us / latency_us / scen_stats");
  if (out->dec_cap < 0) return fail(ES_ERR_ARG, "dec_cap < 0");
  DeviceGuard guard(p->device);
  es_profile *pm = const_cast<es_profile *>(p);
  int nl = 0;
  CK(launch_replay(p->d_img, p->lay, *tr, *out, p->d_status, (cudaStream_t)stream, p->sms, &nl), "k2_replay");
  pm->launches += nl;
  if (out->scen_p95_us) {
    CK(launch_scen_p95(p->d_img, p->lay, *tr, *out, (cudaStream_t)stream, p->sms), "k3_scen_p95");
    pm->launches++;
  }
  return ES_OK;
}

es_status es_scen_p95(const es_profile *p, const es_traces *tr, es_replay_out *out, es_stream stream) {
  if (!p || !tr || !out) return fail(ES_ERR_ARG, "null argument");
  if (tr->n_scen <= 0) return tr->n_scen == 0 ? ES_OK : fail(ES_ERR_ARG, "n_scen < 0");
  if (!tr->arr_off || !out->latency_us || !out->scen_stats || !out->scen_p95_us)
    return fail(ES_ERR_ARG, "null arr_off / latency_us / scen_stats / scen_p95_us");
  DeviceGuard guard(p->device);
  CK(launch_scen_p95(p->d_img, p->lay, *tr, *out, (cudaStream_t)stream, p->sms), "k3_scen_p95");
  const_cast<es_profile *>(p)->launches++;
  return ES_OK;
}

namespace {

// device scratch layout of one host batch (es_replay_traces_host*)
struct HostLayout {
  size_t b_off, b_arr, b_cfg, b_grp, b_comp, b_exit, b_lat, b_st, b_p95, b_dec;
  size_t o_off, o_arr, o_cfg, o_grp, o_comp, o_exit, o_lat, o_st, o_p95, o_dec;
  size_t need;
  int64_t dc;
};

HostLayout host_layout(const es_profile *p, const es_traces *ht, const es_replay_out *ho) {
  HostLayout L{};
  const int M = p->lay.M;
  const int64_t n = ht->n_scen;
  const uint64_t total = ht->arr_off[n * M];
  L.b_off = 8u * (size_t)(n * M + 1);
  L.b_arr = 4u * total;
  L.b_cfg = ht->cfg_idx ? 2u * n : 0;
  L.b_grp = ht->group_id ? 4u * n : 0;
  L.b_comp = ho->completion_us ? 4u * total : 0;
  L.b_exit = ho->exit_used ? total : 0;
  L.b_lat = 4u * total;
  L.b_st = 8u * ES_NSTAT * n;
  L.b_p95 = ho->scen_p95_us ? 4u * n : 0;
  L.dc = ho->dec_cap;
  L.b_dec = L.dc > 0 ? (size_t)(n * L.dc) * (4 + 1 + 1 + 2 + 4 + 8 + 1) : 0;
  size_t need = 0;
  auto take = [&](size_t b) {
    size_t o = need;
    need += (b + 255) & ~(size_t)255;
    return o;
  };
  L.o_off = take(L.b_off);
  L.o_arr = take(L.b_arr);
  L.o_cfg = take(L.b_cfg);
  L.o_grp = take(L.b_grp);
  L.o_comp = take(L.b_comp);
  L.o_exit = take(L.b_exit);
  L.o_lat = take(L.b_lat);
  L.o_st = take(L.b_st);
  L.o_p95 = take(L.b_p95);
  L.o_dec = take(L.b_dec);
  L.need = need;
  return L;
}

es_status ensure_buf(uint8_t **buf, size_t *bytes, size_t need) {
  if (need <= *bytes) return ES_OK;
  cudaFree(*buf);
  *buf = nullptr;
  *bytes = 0;
  CK(cudaMalloc(buf, need), "cudaMalloc(scratch)");
  *bytes = need;
  return ES_OK;
}

// host -> device copies of one batch's inputs into scratch S
es_status host_in(const HostLayout &L, const es_traces *ht, uint8_t *S, cudaStream_t st) {
  CK(cudaMemcpyAsync(S + L.o_off, ht->arr_off, L.b_off, cudaMemcpyHostToDevice, st), "H2D arr_off");
  CK(cudaMemcpyAsync(S + L.o_arr, ht->arrival_us, L.b_arr, cudaMemcpyHostToDevice, st), "H2D arrival");
  if (L.b_cfg) CK(cudaMemcpyAsync(S + L.o_cfg, ht->cfg_idx, L.b_cfg, cudaMemcpyHostToDevice, st), "H2D cfg_idx");
  if (L.b_grp) CK(cudaMemcpyAsync(S + L.o_grp, ht->group_id, L.b_grp, cudaMemcpyHostToDevice, st), "H2D group_id");
  return ES_OK;
}

// K2 + K3 on the batch in scratch S, then device -> host copies of its outputs
es_status host_run(const es_profile *p, const HostLayout &L, const es_traces *ht, es_replay_out *ho, uint8_t *S,
                   cudaStream_t st) {
  es_traces dt = *ht;
  dt.arr_off = reinterpret_cast<const uint64_t *>(S + L.o_off);
  dt.arrival_us = reinterpret_cast<const uint32_t *>(S + L.o_arr);
  dt.cfg_idx = L.b_cfg ? reinterpret_cast<const uint16_t *>(S + L.o_cfg) : nullptr;
  dt.group_id = L.b_grp ? reinterpret_cast<const uint32_t *>(S + L.o_grp) : nullptr;
  es_replay_out dout{};
  dout.completion_us = L.b_comp ? reinterpret_cast<uint32_t *>(S + L.o_comp) : nullptr;
  dout.exit_used = L.b_exit ? S + L.o_exit : nullptr;
  dout.latency_us = reinterpret_cast<uint32_t *>(S + L.o_lat);
  dout.scen_stats = reinterpret_cast<uint64_t *>(S + L.o_st);
  dout.scen_p95_us = L.b_p95 ? reinterpret_cast<uint32_t *>(S + L.o_p95) : nullptr;
  const int64_t dc = L.dc;
  const int64_t n = ht->n_scen;
  dout.dec_cap = dc > 0 ? dc : 0;
  if (dc > 0) {
    uint8_t *q = S + L.o_dec;
    const size_t nd = (size_t)(n * dc);
    dout.dec_t_us = reinterpret_cast<uint32_t *>(q);
    q += 4 * nd;
    dout.dec_L_us = reinterpret_cast<uint32_t *>(q);
    q += 4 * nd;
    dout.dec_score_q = reinterpret_cast<uint64_t *>(q);
    q += 8 * nd;
    dout.dec_B = reinterpret_cast<uint16_t *>(q);
    q += 2 * nd;
    dout.dec_m = q;
    q += nd;
    dout.dec_e = q;
    q += nd;
    dout.dec_flags = q;
  }
  es_status s = es_replay_traces(p, &dt, &dout, (es_stream)st);
  if (s) return s;
  CK(cudaMemcpyAsync(ho->scen_stats, dout.scen_stats, L.b_st, cudaMemcpyDeviceToHost, st), "D2H stats");
  if (L.b_p95) CK(cudaMemcpyAsync(ho->scen_p95_us, dout.scen_p95_us, L.b_p95, cudaMemcpyDeviceToHost, st), "D2H p95");
  if (ho->latency_us)
    CK(cudaMemcpyAsync(ho->latency_us, dout.latency_us, L.b_lat, cudaMemcpyDeviceToHost, st), "D2H lat");
  if (L.b_comp)
    CK(cudaMemcpyAsync(ho->completion_us, dout.completion_us, L.b_comp, cudaMemcpyDeviceToHost, st), "D2H comp");
  if (L.b_exit) CK(cudaMemcpyAsync(ho->exit_used, dout.exit_used, L.b_exit, cudaMemcpyDeviceToHost, st), "D2H exit");
  if (dc > 0) {
    const size_t nd = (size_t)(n * dc);
    if (ho->dec_t_us) CK(cudaMemcpyAsync(ho->dec_t_us, dout.dec_t_us, 4 * nd, cudaMemcpyDeviceToHost, st), "D2H dec");
    if (ho->dec_L_us) CK(cudaMemcpyAsync(ho->dec_L_us, dout.dec_L_us, 4 * nd, cudaMemcpyDeviceToHost, st), "D2H dec");
    if (ho->dec_score_q)
      CK(cudaMemcpyAsync(ho->dec_score_q, dout.dec_score_q, 8 * nd, cudaMemcpyDeviceToHost, st), "D2H dec");
    if (ho->dec_B) CK(cudaMemcpyAsync(ho->dec_B, dout.dec_B, 2 * nd, cudaMemcpyDeviceToHost, st), "D2H dec");
    if (ho->dec_m) CK(cudaMemcpyAsync(ho->dec_m, dout.dec_m, nd, cudaMemcpyDeviceToHost, st), "D2H dec");
    if (ho->dec_e) CK(cudaMemcpyAsync(ho->dec_e, dout.dec_e, nd, cudaMemcpyDeviceToHost, st), "D2H dec");
    if (ho->dec_flags) CK(cudaMemcpyAsync(ho->dec_flags, dout.dec_flags, nd, cudaMemcpyDeviceToHost, st), "D2H dec");
  }
  return ES_OK;
}

es_status check_host_batch(const es_traces *ht, const es_replay_out *ho) {
  if (!ht || !ho) return fail(ES_ERR_ARG, "null argument");
  if (ht->n_scen < 0) return fail(ES_ERR_ARG, "n_scen < 0");
  if (ht->n_scen > 0 && (!ht->arr_off || !ht->arrival_us || !ho->scen_stats))
    return fail(ES_ERR_ARG, "null host input/stats");
  return ES_OK;
}

}  // namespace

es_status es_replay_traces_host(es_profile *p, const es_traces *ht, es_replay_out *ho, es_stream stream) {
  if (!p) return fail(ES_ERR_ARG, "null argument");
  es_status s = check_host_batch(ht, ho);
  if (s) return s;
  if (ht->n_scen == 0) return ES_OK;
  DeviceGuard guard(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  const HostLayout L = host_layout(p, ht, ho);
  if ((s = ensure_buf(&p->scratch, &p->scratch_bytes, L.need))) return s;
  if ((s = host_in(L, ht, p->scratch, st))) return s;
  if ((s = host_run(p, L, ht, ho, p->scratch, st))) return s;
  CK(cudaStreamSynchronize(st), "stream sync");
  return ES_OK;
}

es_status es_replay_traces_host_pipelined(es_profile *p, const es_traces *hts, es_replay_out *hos, int32_t nbatch,
                                          es_stream stream) {
  if (!p || !hts || !hos || nbatch < 0) return fail(ES_ERR_ARG, "null argument or nbatch < 0");
  size_t need = 0;
  for (int32_t k = 0; k < nbatch; ++k) {
    es_status s = check_host_batch(&hts[k], &hos[k]);
    if (s) return s;
    if (hts[k].n_scen > 0) need = std::max(need, host_layout(p, &hts[k], &hos[k]).need);
  }
  if (need == 0) return ES_OK;
  DeviceGuard guard(p->device);
  cudaStream_t st = (cudaStream_t)stream;
  es_status s;
  if ((s = ensure_buf(&p->scratch, &p->scratch_bytes, need))) return s;
  if ((s = ensure_buf(&p->scratch2, &p->scratch2_bytes, need))) return s;
  if (!p->copy_stream) {
    CK(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking), "copy stream");
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&p->ev_copied[i], cudaEventDisableTiming), "event");
      CK(cudaEventCreateWithFlags(&p->ev_done[i], cudaEventDisableTiming), "event");
    }
    CK(cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming), "event");
  }
  // the copy stream starts after the caller's prior work on `stream`
  CK(cudaEventRecord(p->ev_start, st), "event record");
  CK(cudaStreamWaitEvent(p->copy_stream, p->ev_start, 0), "stream wait");
  // batch k: inputs into buffer k % 2 on the copy stream (after batch k-2 is
  // done with it), K2 + K3 + output copies on `stream` after its inputs landed:
  // the input copy of batch k+1 overlaps the replay of batch k
  for (int32_t k = 0; k < nbatch; ++k) {
    if (hts[k].n_scen == 0) continue;
    const int b = k & 1;
    uint8_t *S = b ? p->scratch2 : p->scratch;
    const HostLayout L = host_layout(p, &hts[k], &hos[k]);
    if (k >= 2) CK(cudaStreamWaitEvent(p->copy_stream, p->ev_done[b], 0), "stream wait");
    if ((s = host_in(L, &hts[k], S, p->copy_stream))) return s;
    CK(cudaEventRecord(p->ev_copied[b], p->copy_stream), "event record");
    CK(cudaStreamWaitEvent(st, p->ev_copied[b], 0), "stream wait");
    if ((s = host_run(p, L, &hts[k], &hos[k], S, st))) return s;
    CK(cudaEventRecord(p->ev_done[b], st), "event record");
  }
  CK(cudaStreamSynchronize(st), "stream sync");
  return ES_OK;
}

es_status es_group_accumulate(const es_profile *p, const es_traces *tr, const es_replay_out *out, uint32_t n_groups,
                              uint64_t *counts, uint64_t *hist0, es_stream stream) {
  if (!p || !tr || !out || !counts || !hist0 || !out->latency_us || !out->scen_stats)
    return fail(ES_ERR_ARG, "null argument");
  if (n_groups == 0) return fail(ES_ERR_ARG, "n_groups == 0");
  if (tr->n_scen <= 0) return ES_OK;
  DeviceGuard guard(p->device);
  CK(launch_group_accumulate(p->d_img, p->lay, *tr, *out, n_groups, counts, hist0, (cudaStream_t)stream),
     "k_group_level(0)");
  const_cast<es_profile *>(p)->launches++;
  return ES_OK;
}

es_status es_scen_stats(const es_profile *p, const es_traces *tr, es_replay_out *out, uint32_t n_groups,
                        uint64_t *counts, uint64_t *hist0, es_stream stream) {
  if (!p || !tr || !out) return fail(ES_ERR_ARG, "null argument");
  if (tr->n_scen <= 0) return tr->n_scen == 0 ? ES_OK : fail(ES_ERR_ARG, "n_scen < 0");
  if (!tr->arr_off || !out->latency_us || !out->scen_stats) return fail(ES_ERR_ARG, "null arr_off / latency / stats");
  if (counts && (!hist0 || n_groups == 0)) return fail(ES_ERR_ARG, "group outputs need hist0 and n_groups > 0");
  DeviceGuard guard(p->device);
  CK(launch_stats_fused(p->d_img, p->lay, *tr, *out, counts ? n_groups : 0u, counts, hist0, (cudaStream_t)stream,
                        p->sms),
     "k3_stats");
  const_cast<es_profile *>(p)->launches++;
  return ES_OK;
}

es_status es_group_hist(const es_profile *p, const es_traces *tr, const es_replay_out *out, uint32_t n_groups,
                        int32_t level, const uint64_t *state, uint64_t *hist, es_stream stream) {
  if (!p || !tr || !out || !state || !hist || !out->latency_us || !out->scen_stats)
    return fail(ES_ERR_ARG, "null argument");
  if (level < 1 || level > 3) return fail(ES_ERR_ARG, "es_group_hist level %d (1..3)", level);
  if (n_groups == 0) return fail(ES_ERR_ARG, "n_groups == 0");
  DeviceGuard guard(p->device);
  if (tr->n_scen <= 0) {
    CK(cudaMemsetAsync(hist, 0, (size_t)n_groups * ES_HIST_BINS * 8, (cudaStream_t)stream), "memset hist");
    return ES_OK;
  }
  CK(launch_group_hist(p->d_img, p->lay, *tr, *out, n_groups, level, state, hist, (cudaStream_t)stream),
     "k_group_level");
  const_cast<es_profile *>(p)->launches++;
  return ES_OK;
}

es_status es_group_p95_select(uint32_t n_groups, int32_t level, const uint64_t *counts, const uint64_t *hist,
                              uint64_t *state, es_stream stream) {
  if (!hist || !state || (level == 0 && !counts)) return fail(ES_ERR_ARG, "null argument");
  if (level < 0 || level > 3) return fail(ES_ERR_ARG, "level %d", level);
  if (n_groups == 0) return fail(ES_ERR_ARG, "n_groups == 0");
  CK(launch_group_select(n_groups, level, counts, hist, state, (cudaStream_t)stream), "k_group_select");
  return ES_OK;
}

es_status es_device_status(es_profile *p, es_stream stream, uint32_t *code, int64_t *item) {
  if (!p) return fail(ES_ERR_ARG, "null profile");
  DeviceGuard guard(p->device);
  CK(cudaStreamSynchronize((cudaStream_t)stream), "stream sync");
  DevStatus h{};
  CK(cudaMemcpy(&h, p->d_status, sizeof h, cudaMemcpyDeviceToHost), "read status");
  CK(cudaMemset(p->d_status, 0, sizeof h), "clear status");
  if (code) *code = h.code;
  if (item) *item = (int64_t)h.item;
  return ES_OK;
}

int64_t es_launch_count(const es_profile *p) { return p ? p->launches.load() : 0; }

}  // extern "C"
