// Dependent-latency microbenchmark for the warp primitives on the scheduler's
// critical path (one warp, clock64 around chains of 256 dependent ops).
#include <cstdio>
#include <cstdint>
__global__ void k(unsigned long long* out, int seed) {
  __shared__ unsigned sm[64];
  __shared__ double smd[64];
  const int lane = threadIdx.x;
  sm[lane] = lane; sm[lane + 32] = lane; smd[lane] = lane + 1.5; smd[lane+32] = 2.0;
  __syncwarp();
  unsigned v = lane + seed; long long t0, t1; int idx = 0;
  double d = 1.0 + lane;
  constexpr int R = 256;
  // SHFL
  t0 = clock64();
  for (int i = 0; i < R; ++i) v = __shfl_sync(0xffffffffu, v, (v + i) & 31);
  t1 = clock64(); if (lane == 0) out[idx] = (t1 - t0); ++idx;
  // REDUX min
  t0 = clock64();
  for (int i = 0; i < R; ++i) v = __reduce_min_sync(0xffffffffu, v + lane) + 1;
  t1 = clock64(); if (lane == 0) out[idx] = (t1 - t0); ++idx;
  // VOTE ballot
  t0 = clock64();
  for (int i = 0; i < R; ++i) v = __ballot_sync(0xffffffffu, ((v >> (lane & 7)) & 1)) + i;
  t1 = clock64(); if (lane == 0) out[idx] = (t1 - t0); ++idx;
  // LDS dependent
  t0 = clock64();
  for (int i = 0; i < R; ++i) v = sm[(v + lane) & 63];
  t1 = clock64(); if (lane == 0) out[idx] = (t1 - t0); ++idx;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) d = d + 1.25;
  t1 = clock64(); if (lane == 0) out[idx] = (t1 - t0); ++idx;
  // DDIV chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) d = 3.0 / d + 1.0;
  t1 = clock64(); if (lane == 0) out[idx] = (t1 - t0); ++idx;
  // IADD chain
  unsigned u = v;
  t0 = clock64();
  for (int i = 0; i < R; ++i) u = u * 3u + (unsigned)i;
  t1 = clock64(); if (lane == 0) out[idx] = (t1 - t0); ++idx;
  // REDUX or
  t0 = clock64();
  for (int i = 0; i < R; ++i) v = __reduce_or_sync(0xffffffffu, v ^ lane) + 1;
  t1 = clock64(); if (lane == 0) out[idx] = (t1 - t0); ++idx;
  // syncwarp + STS/LDS round trip
  t0 = clock64();
  for (int i = 0; i < R; ++i) { sm[lane] = v + 1; __syncwarp(); v = sm[(lane + 1) & 31]; __syncwarp(); }
  t1 = clock64(); if (lane == 0) out[idx] = (t1 - t0); ++idx;
  // 64-bit shfl
  unsigned long long w = v;
  t0 = clock64();
  for (int i = 0; i < R; ++i) w = __shfl_sync(0xffffffffu, w, (unsigned)(w + i) & 31) + 1;
  t1 = clock64(); if (lane == 0) out[idx] = (t1 - t0); ++idx;
  if (lane == 0) out[31] = v + u + (unsigned)d + (unsigned)w;
}
int main() {
  unsigned long long* o; cudaMallocManaged(&o, 32 * 8);
  k<<<1, 32>>>(o, 1); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, 2); cudaDeviceSynchronize();
  const char* nm[] = {"shfl", "redux.min", "vote.ballot", "lds", "dadd", "ddiv+dadd", "imad", "redux.or", "sts+sync+lds+sync", "shfl64"};
  for (int i = 0; i < 10; ++i) printf("%-20s %6.1f cycles/op\n", nm[i], o[i] / 256.0);
  return 0;
}
