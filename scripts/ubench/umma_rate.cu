// tcgen05.mma issue rate with the no-swizzle K-major operand layout used by
// ag_linear.cu: one CTA per SM issues ITER x (D/16) MMAs of M128 x N x K16
// (bf16 -> f32) from shared memory into TMEM; reports cycles per MMA and the
// aggregate TFLOP/s, for N = 128 and 256.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a umma_rate.cu -o umma_rate
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

template <int N>
__global__ void k(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  constexpr int M = 128, D = 128, KC = D / 8;
  unsigned char* sa = sm;
  unsigned char* sb = sm + M * D * 2;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  for (int i = threadIdx.x; i < (M + N) * D * 2 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int ks = 0; ks < D / 16; ++ks) {
        const uint64_t da = sdesc(su32(sa) + ks * 256, 128, KC * 128);
        const uint64_t db = sdesc(su32(sb) + ks * 256, 128, KC * 128);
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                     ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(1));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(su32(&mbar)), "r"(0));
    const long long t1 = clock64();
    if (blockIdx.x == 0) cyc[0] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int N>
void run(int sms) {
  const int iters = 2000, smem = (128 + N) * 128 * 2;
  cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  k<N><<<sms, 128, smem>>>(10, cyc);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<N><<<sms, 128, smem>>>(iters, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double mmas = (double)iters * 8;
  const double flops = 2.0 * 128 * N * 16 * mmas * sms;
  printf("{\"N\": %d, \"cycles_per_mma\": %.1f, \"tflops\": %.1f, \"err\": \"%s\"}\n", N, c / mmas,
         flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<128>(sms);
  run<256>(sms);
  return 0;
}
