// k_tables.cu -- step a1: per-SLO fixed-point urgency tables, built on the GPU.
//
// Reading Q5 of Eq. 3: every table entry is the
// exact floor of a real number,
//   x_c   = ceil(tau (1 + ln C))                     (clip boundary)
//   A[h]  = floor(2^28 exp((h*1024 - r - tau)/tau))  (r = (1024 - tau%1024)%1024)
//   Bt[l] = floor(2^28 exp(l/tau))
//   H[c]  = floor(2^28 exp(L_c/tau))  for profile cell c with L_c < x_c
// evaluated here in double-double arithmetic (~106-bit significand, relative
// error < 1e-29), far below the 1e-7 distance-to-integer margin every value is
// checked against (ES_ERR_NUMERIC otherwise).  bidx[len] is Eq. 5 with reading
// Q8: the index of the largest profiled batch <= min(len, B_max).
#include <cuda_runtime.h>

#include <cmath>

#include "es_internal.cuh"

namespace es {
namespace {

struct dd {
  double hi, lo;
};

// error-free transformations; intrinsics forbid FMA contraction
__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  double bb = __dsub_rn(s, a);
  double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  double p = __dmul_rn(a, b);
  return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = quick_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo = __dadd_rn(p.lo, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo = __dadd_rn(p.lo, __dmul_rn(a.lo, b));
  return quick_two_sum(p.hi, p.lo);
}
// a / b for a double-double a and a double b (long division, 2 correction steps)
__device__ __forceinline__ dd dd_div_d(dd a, double b) {
  double q1 = __ddiv_rn(a.hi, b);
  dd r = dd_add(a, dd{-two_prod(q1, b).hi, -two_prod(q1, b).lo});
  double q2 = __ddiv_rn(r.hi, b);
  r = dd_add(r, dd{-two_prod(q2, b).hi, -two_prod(q2, b).lo});
  double q3 = __ddiv_rn(r.hi, b);
  dd q = quick_two_sum(q1, q2);
  return dd_add(q, dd{q3, 0.0});
}
__device__ __forceinline__ dd dd_ldexp(dd a, int k) { return {ldexp(a.hi, k), ldexp(a.lo, k)}; }

// exact rational num/den (|num|, den < 2^53) as a double-double
__device__ __forceinline__ dd dd_ratio(double num, double den) {
  double q = __ddiv_rn(num, den);
  double rem = __fma_rn(-q, den, num);  // exact remainder
  return quick_two_sum(q, __ddiv_rn(rem, den));
}

__device__ const dd LN2 = {6.93147180559945286e-01, 2.319046813846299558e-17};

// exp(x) in double-double: x = k ln2 + r, |r| <= ln2/2; expm1(r / 2^10) by
// Taylor (10 terms, truncation < 1e-40), undo the scaling with
// expm1(2y) = expm1(y) (expm1(y) + 2) ten times, then 1 + . and * 2^k.
__device__ dd dd_exp(dd x) {
  double k = rint(__ddiv_rn(x.hi, LN2.hi));
  dd r = dd_add(x, dd_mul_d(dd{-LN2.hi, -LN2.lo}, k));
  r = dd_ldexp(r, -10);
  dd term = r, sum = r;
  for (int i = 2; i <= 12; ++i) {
    term = dd_div_d(dd_mul(term, r), (double)i);
    sum = dd_add(sum, term);
  }
  for (int i = 0; i < 10; ++i) sum = dd_mul(sum, dd_add(sum, dd{2.0, 0.0}));
  dd e = dd_add(sum, dd{1.0, 0.0});
  return dd_ldexp(e, (int)k);
}

// floor of a double-double and the distance of its value to the nearest integer
__device__ __forceinline__ uint64_t dd_floor(dd v, double *dist) {
  double f = floor(v.hi);
  double frac;
  if (f == v.hi) {  // hi integral: the sign of lo decides
    if (v.lo < 0.0) {
      f -= 1.0;
      frac = 1.0 + v.lo;
    } else {
      frac = v.lo;
    }
  } else {
    frac = __dadd_rn(__dsub_rn(v.hi, f), v.lo);
  }
  *dist = fmin(frac, 1.0 - frac);
  return (uint64_t)f;
}

// floor(2^28 exp(num/den)); num == 0 is exactly 2^28
__device__ uint64_t fx_exp(double num, double den, double *min_dist) {
  if (num == 0.0) return 1ull << F;
  dd v = dd_ldexp(dd_exp(dd_ratio(num, den)), F);
  double d;
  uint64_t f = dd_floor(v, &d);
  *min_dist = fmin(*min_dist, d);
  return f;
}

constexpr double MARGIN = 1e-7;

// one block per cfg
__global__ void k_build_tables(uint8_t *img, ImgLayout lay) {
  const int c = blockIdx.x;
  CfgRec *rec = reinterpret_cast<CfgRec *>(img + lay.off_cfg) + c;
  const uint32_t *lat = reinterpret_cast<const uint32_t *>(img + lay.off_lat);
  const uint16_t *bs = reinterpret_cast<const uint16_t *>(img + lay.off_bs);
  __shared__ uint32_t s_xc, s_nA;
  __shared__ int s_bad;
  const uint32_t tau = rec->tau;
  if (threadIdx.x == 0) {
    s_bad = 0;
    uint32_t x_c;
    if (rec->C == 1u) {
      x_c = tau;  // ln 1 = 0 exactly
    } else {
      // ln C by one Newton step on exp: y1 = y0 + (C exp(-y0) - 1), error ~1e-32
      double y0 = log((double)rec->C);
      dd e = dd_exp(dd{-y0, 0.0});
      dd t = dd_add(dd_mul_d(e, (double)rec->C), dd{-1.0, 0.0});
      dd y = dd_add(dd{y0, 0.0}, t);
      dd v = dd_mul_d(dd_add(y, dd{1.0, 0.0}), (double)tau);  // tau (1 + ln C)
      double d;
      uint64_t f = dd_floor(v, &d);
      if (d < MARGIN) s_bad = 1;
      x_c = (uint32_t)f + 1u;  // ceil of a non-integer
    }
    uint32_t r = (S - tau % S) % S;
    uint32_t nA = ((x_c - 1u + r) >> SBITS) + 1u;
    uint32_t lmax = 0;
    for (int i = 0; i < lay.M * lay.E * lay.nb; ++i) lmax = lat[i] > lmax ? lat[i] : lmax;
    rec->fast_lim = x_c > lmax ? x_c - lmax : 0u;
    rec->x_c = x_c;
    rec->r = r;
    rec->nA = nA;
    rec->C_q = (uint64_t)rec->C << F;
    if (nA > rec->nA_cap) s_bad = 2;
    s_xc = x_c;
    s_nA = nA;
  }
  __syncthreads();
  if (s_bad == 2) {
    if (threadIdx.x == 0) rec->status = ES_ERR_ARG;
    return;
  }
  const uint32_t x_c = s_xc, nA = s_nA, r = rec->r;
  double dist = 1.0;
  uint32_t *A = reinterpret_cast<uint32_t *>(img + rec->off_A);
  uint32_t *Bt = reinterpret_cast<uint32_t *>(img + rec->off_Bt);
  uint64_t *H = reinterpret_cast<uint64_t *>(img + rec->off_H);
  uint8_t *bidx = img + rec->off_bidx;
  for (uint32_t h = threadIdx.x; h < rec->nA_cap; h += blockDim.x) {
    if (h < nA) {
      double num = (double)h * S - (double)r - (double)tau;
      A[h] = (uint32_t)fx_exp(num, (double)tau, &dist);
    } else {
      A[h] = 0u;
    }
  }
  for (uint32_t l = threadIdx.x; l < S; l += blockDim.x) Bt[l] = (uint32_t)fx_exp((double)l, (double)tau, &dist);
  const int cells = lay.M * lay.E * lay.nb;
  for (int i = threadIdx.x; i < cells; i += blockDim.x) {
    uint32_t L = lat[i];
    H[i] = (L < x_c) ? fx_exp((double)L, (double)tau, &dist) : ~0ull;
  }
  for (uint32_t len = threadIdx.x; len <= rec->b_max; len += blockDim.x) {
    uint32_t cap = len < rec->b_max ? len : rec->b_max;
    int bi = 0;
    for (int i = 0; i < lay.nb; ++i)
      if ((uint32_t)bs[i] <= cap) bi = i;
    bidx[len] = (uint8_t)bi;
  }
  if (dist < MARGIN) atomicExch(&s_bad, 1);
  __syncthreads();
  if (threadIdx.x == 0) rec->status = s_bad ? ES_ERR_NUMERIC : ES_OK;
}

}  // namespace

cudaError_t launch_build_tables(uint8_t *img, const ImgLayout &lay, cudaStream_t st) {
  k_build_tables<<<lay.ncfg, 256, 0, st>>>(img, lay);
  return cudaGetLastError();
}

}  // namespace es
