// Latency microbenchmarks (one warp): dependent chains of warp collectives.
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t seed, uint64_t *out, uint32_t *sink) {
  __shared__ uint32_t sm[1024];
  int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) sm[i] = (i * 7) & 1023;
  __syncwarp();
  uint32_t v = seed + lane;
  const int N = 4096;
  uint64_t t0, t1;
  // REDUX min chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) { v = __reduce_min_sync(0xffffffff, v) + lane; }
  t1 = clock64(); out[0] = t1 - t0;
  // ballot chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) { v = __ballot_sync(0xffffffff, (v >> (lane & 7)) & 1) + lane; }
  t1 = clock64(); out[1] = t1 - t0;
  // shfl chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) { v = __shfl_sync(0xffffffff, v, (v + 1) & 31) + 1; }
  t1 = clock64(); out[2] = t1 - t0;
  // LDS chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) { v = sm[v & 1023]; }
  t1 = clock64(); out[3] = t1 - t0;
  // IADD chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) { v = v * 3 + 1; }
  t1 = clock64(); out[4] = t1 - t0;
  // 64-bit add/max chain
  int64_t x = v;
  t0 = clock64();
  for (int i = 0; i < N; ++i) { x = max(x + 3, (int64_t)lane); }
  t1 = clock64(); out[5] = t1 - t0;
  // popc(ballot) -> uniform compare chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) { v = __popc(__ballot_sync(0xffffffff, v > (uint32_t)lane)); }
  t1 = clock64(); out[6] = t1 - t0;
  // branch on uniform value chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) { if (v & 1) v = v * 5 + 3; else v = v + 7; }
  t1 = clock64(); out[7] = t1 - t0;
  // reduce_min without the +lane (broadcast use)
  t0 = clock64();
  for (int i = 0; i < N; ++i) { v = __reduce_min_sync(0xffffffff, v ^ lane); }
  t1 = clock64(); out[8] = t1 - t0;
  sink[lane] = v + (uint32_t)x;
}
int main() {
  uint64_t *d; uint32_t *s; cudaMalloc(&d, 64 * 8); cudaMalloc(&s, 128);
  k<<<1, 32>>>(1, d, s); cudaDeviceSynchronize();
  k<<<1, 32>>>(1, d, s); cudaDeviceSynchronize();
  uint64_t h[9]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  const char *names[] = {"redux.min+iadd", "ballot+iadd", "shfl+iadd", "lds", "imad", "i64 add+max", "popc(ballot)", "uniform branch", "redux(x^lane)"};
  for (int i = 0; i < 9; ++i) printf("%-16s %.1f cycles/iter\n", names[i], h[i] / 4096.0);
  return 0;
}
