// Shared device/host definitions for the aragog_b200 CUDA library.
//
// Configurations are canonical indices over the mixed-radix space {0..M-1}^N,
// position 0 most significant (reference include/aragog/workflow.h:18-21,
// src/workflow.cpp:250-275).  The GPU path requires M^N <= 2^32 so every index
// fits a uint32 (the BASELINE's deepest space, 8x12, is 4.3e8).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "aragog_b200.h"

namespace agb {

constexpr int kMaxAgents = 32;
constexpr int kMaxModels = 255;
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kMixIV = 0x6a09e667f3bcc909ULL;
constexpr uint64_t kHashIV = 0x2545f4914f6cdd1dULL;
constexpr uint64_t kRouterSalt = 0xA3;

// ---- error plumbing --------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define AG_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t _e = (call);                                                 \
    if (_e != cudaSuccess)                                                   \
      return ::agb::fail(AG_ERR_CUDA, std::string(#call) + ": " +            \
                                          cudaGetErrorString(_e));           \
  } while (0)

// ---- rng (reference include/aragog/rng.h:34-51) ----------------------------
__host__ __device__ __forceinline__ uint64_t splitmix_step(uint64_t x) {
  uint64_t z = x + kGamma;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// one word of rng::mix: state ^= w + gamma + (state << 6) + (state >> 2),
// then state = splitmix64(copy)
__host__ __device__ __forceinline__ uint64_t absorb(uint64_t state, uint64_t w) {
  state ^= w + kGamma + (state << 6) + (state >> 2);
  return splitmix_step(state);
}

// ---- space description passed by value to kernels --------------------------
struct SpaceDev {
  int n, m;
  uint64_t size;        // M^N (<= 2^32)
  uint64_t div_m;       // ceil(2^64 / M): exact u32 division via __umul64hi
};

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t divm(uint32_t x, uint64_t magic) {
  return (uint32_t)__umul64hi((uint64_t)x, magic);
}
#endif

// Router thresholds: u = (key >> 11) * 2^-53 is compared exactly as integers
// (reference src/router.cpp:53-56): u >= fn <=> k >= ceil(fn * 2^53),
// u < fp <=> k < ceil(fp * 2^53).
struct RouterDev {
  int kind;             // AG_ROUTER_ORACLE / AG_ROUTER_NOISY
  uint64_t noise_seed;
  uint64_t t_fn;        // keep a true verdict iff k >= t_fn
  uint64_t t_fp;        // invent a member iff k < t_fp
};

struct TruthDev {
  int n_requests;
  const uint64_t* request_ids;
  const int32_t* seed_ptr;
  const uint8_t* seeds;
  const int32_t* removed_ptr;
  const uint64_t* removed;
};

}  // namespace agb
