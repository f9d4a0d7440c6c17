// Integer-issue ceiling for the noisy router (MEASURED_PEAKS
// has no INT peak).  Measures rng::mix absorb steps per second on the whole
// GPU -- one absorb = the reference's per-word mix step (rng.h:43-51): a
// shift/add/xor combine plus splitmix64 (two u64 multiplies) -- with 8
// independent chains per thread so the pipes, not latency, bound it.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I../../paper_2511_20975_b200/csrc mix_peak.cu -o mix_peak
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__device__ __forceinline__ uint64_t splitmix_step(uint64_t x) {
  uint64_t z = x + kGamma;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t absorb(uint64_t state, uint64_t w) {
  state ^= w + kGamma + (state << 6) + (state >> 2);
  return splitmix_step(state);
}

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) k_absorb(uint64_t seed, int iters, uint64_t* sink) {
  uint64_t s[kChains];
  const uint64_t t = blockIdx.x * 256ull + threadIdx.x;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s[c] = seed ^ (t * kChains + c);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) s[c] = absorb(seed, s[c]);
  uint64_t x = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) x ^= s[c];
  if (x == 0x12345) sink[0] = x;  // keeps the work alive
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint64_t* sink;
  cudaMalloc(&sink, 8);
  const int blocks = sms * 8, iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_absorb<<<blocks, 256>>>(1, 64, sink);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_absorb<<<blocks, 256>>>(r + 2, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double n = (double)blocks * 256 * kChains * iters;
  printf("{\"absorbs_per_s\": %.6e, \"ms\": %.4f, \"sms\": %d, \"err\": \"%s\"}\n", n / (best * 1e-3), best, sms,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
