// Dependent-chain latency (cycles/op) of the warp primitives K2 is built from,
// one warp alone on the GPU.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t redux_add(uint32_t v) {
  uint32_t r;
  asm volatile("redux.sync.add.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
  return r;
}
__global__ void k(uint32_t *out, long long *cyc, int n) {
  uint32_t v = threadIdx.x;
  __shared__ uint32_t sm[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = i;
  __syncwarp();
  long long t0, t1;
#define BENCH(slot, expr)                      \
  t0 = clock64();                              \
  for (int i = 0; i < n; ++i) { expr; }        \
  t1 = clock64();                              \
  if (threadIdx.x == 0) cyc[slot] = (t1 - t0) / n;
  BENCH(0, v = __shfl_sync(0xffffffffu, v, (v + 1) & 31))
  BENCH(1, v = __shfl_xor_sync(0xffffffffu, v, 1) + 1)
  BENCH(2, v = redux_add(v) & 31)
  BENCH(3, v = __ballot_sync(0xffffffffu, v & 1) & 31)
  BENCH(4, v = __any_sync(0xffffffffu, v & 1) + v)
  BENCH(5, v = sm[v & 1023])
  BENCH(6, v = v * 3 + 1)
  BENCH(7, v = __popc(v) + v)
  BENCH(8, v = __shfl_sync(0xffffffffu, v, (v + 1) & 15, 16))
  BENCH(9, v = __match_any_sync(0xffffffffu, v & 3) & 31)
  out[threadIdx.x] = v;
}
int main() {
  uint32_t *o; long long *c;
  cudaMalloc(&o, 128); cudaMalloc(&c, 16 * 8);
  k<<<1, 32>>>(o, c, 1000);
  k<<<1, 32>>>(o, c, 1000);
  long long h[16];
  cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
  const char *nm[] = {"shfl.idx", "shfl.bfly+add", "redux.add+and", "ballot+and", "vote.any+add", "lds(dep)",
                      "imad", "popc+add", "shfl.idx w16", "match.any+and"};
  for (int i = 0; i < 10; ++i) printf("%-16s %lld cycles/iter\n", nm[i], h[i]);
  return 0;
}
