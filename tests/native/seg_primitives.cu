// Unit test of the Seg<LPS, MM> warp-segment primitives (decide.cuh) on the GPU.
// Each segment computes sum / min / max / sum64 / bcast / seg_any of lane
// values and writes them; the host checks against plain loops.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2605_05527_b200/csrc/decide.cuh"
using namespace es;

template <int LPS, int MM>
__global__ void k(const uint32_t *in, uint32_t *out, int flip) {
  const Seg<LPS, MM> sg;
  const uint32_t v = in[threadIdx.x];
  // emulate a divergent history: segment 1 lanes take a different branch first
  uint32_t w = v;
  if ((sg.seg & 1) == flip) w = v + 0;  // no-op branch
  const uint32_t s = sg.sum(w), mn = sg.vmin(w), mx = sg.vmax(w);
  const uint64_t s64 = sg.sum64((uint64_t)w << 20);
  const uint32_t b = sg.bcast(w, 3 % LPS);
  const uint64_t b64 = sg.bcast((uint64_t)w << 33, 5 % LPS);
  const uint32_t any = sg.seg_any(w == 77u) ? 1u : 0u;
  uint32_t *o = out + threadIdx.x * 8;
  o[0] = s; o[1] = mn; o[2] = mx; o[3] = (uint32_t)(s64 >> 20); o[4] = b; o[5] = (uint32_t)(b64 >> 33); o[6] = any;
  o[7] = (uint32_t)sg.gsum64((uint64_t)w);
}

template <int LPS, int MM>
int run(int flip) {
  std::vector<uint32_t> h(32), r(32 * 8);
  for (int i = 0; i < 32; ++i) h[i] = (i * 37 + 11) % 101 + (i == 9 ? 77 - ((9 * 37 + 11) % 101) : 0);
  uint32_t *din, *dout;
  cudaMalloc(&din, 32 * 4);
  cudaMalloc(&dout, 32 * 32);
  cudaMemcpy(din, h.data(), 128, cudaMemcpyHostToDevice);
  k<LPS, MM><<<1, 32>>>(din, dout, flip);
  cudaMemcpy(r.data(), dout, 32 * 32, cudaMemcpyDeviceToHost);
  int bad = 0;
  constexpr int GL = LPS / MM;
  for (int i = 0; i < 32; ++i) {
    int s0 = (i / LPS) * LPS, g0 = s0 + ((i % LPS) / GL) * GL;
    uint32_t s = 0, mn = ~0u, mx = 0, any = 0, gs = 0;
    for (int j = s0; j < s0 + LPS; ++j) { s += h[j]; mn = h[j] < mn ? h[j] : mn; mx = h[j] > mx ? h[j] : mx; any |= h[j] == 77; }
    for (int j = g0; j < g0 + GL; ++j) gs += h[j];
    uint32_t exp[8] = {s, mn, mx, s, h[s0 + 3 % LPS], h[s0 + 5 % LPS], any, gs};
    for (int q = 0; q < 8; ++q)
      if (r[i * 8 + q] != exp[q]) {
        if (bad < 10) printf("LPS %d MM %d lane %d field %d got %u exp %u\n", LPS, MM, i, q, r[i * 8 + q], exp[q]);
        bad++;
      }
  }
  printf("LPS %d MM %d flip %d: %s (%d bad)\n", LPS, MM, flip, bad ? "FAIL" : "ok", bad);
  return bad;
}

int main() {
  int bad = 0;
  for (int f = 0; f < 2; ++f) {
    bad += run<32, 4>(f) + run<32, 8>(f) + run<16, 4>(f) + run<16, 2>(f) + run<8, 4>(f) + run<8, 8>(f);
  }
  return bad ? 1 : 0;
}
