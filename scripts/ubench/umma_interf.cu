// tcgen05.mma rate (M128 N128 K16, no-swizzle K-major operands in shared
// memory) alone and under interference that the learned-router kernel has:
// (1) epilogue warps streaming tcgen05.ld from the other TMEM half,
// (2) loader warps streaming cp.async into other shared memory.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a umma_interf.cu -o umma_interf
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

constexpr int M = 128, N = 128, D = 128, KC = D / 8;
// mode bit 0: tcgen05.ld interference (16 warps), bit 1: cp.async (8 warps)
__global__ void __launch_bounds__(800, 1) k(int iters, int mode, const uint4* gsrc, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* sa = sm;                 // 32 KB
  unsigned char* sb = sm + M * D * 2;     // 32 KB
  unsigned char* sc = sb + N * D * 2;     // 64 KB scratch for cp.async
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, wid = tid >> 5;
  // mode bit 2: random bf16 operands (power) instead of zeros
  for (int i = tid; i < (M + N) * D * 2 / 4; i += blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    // two bf16 in [-2, 2): sign, exponent 126..127, random mantissa
    const uint32_t h0 = ((x & 1u) << 15) | ((126u + ((x >> 1) & 1u)) << 7) | ((x >> 2) & 0x7Fu);
    const uint32_t h1 = (((x >> 9) & 1u) << 15) | ((126u + ((x >> 10) & 1u)) << 7) | ((x >> 11) & 0x7Fu);
    reinterpret_cast<uint32_t*>(sm)[i] = (mode & 4) ? (h0 | (h1 << 16)) : 0u;
  }
  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    stop = 0;
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (wid == 24) {
    if ((tid & 31) == 0) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
      const long long t0 = clock64();
      if (mode & 8) {
        // the learned-router issue pattern: per tile two accumulators (two A
        // halves), accumulate from k-step 1, stages alternating
        for (int it = 0; it < iters / 2; ++it)
          for (int hf = 0; hf < 2; ++hf)
            for (int ks = 0; ks < D / 16; ++ks) {
              const uint64_t da = sdesc(su32(sa) + (hf & 0) * 0 + ks * 256, 128, KC * 128);
              const uint64_t db = sdesc(su32(sb) + ks * 256, 128, KC * 128);
              const uint32_t acc = tmem + (uint32_t)((it & 1) * 256 + hf * 128);
              asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                           "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                           ::"r"(acc), "l"(da), "l"(db), "r"(idesc), "r"(ks > 0 ? 1 : 0));
            }
      } else
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
      stop = 1;
    }
  } else if (wid < 16) {
    if (mode & 1) {
      const int q = wid & 3;
      uint32_t acc = 0;
      while (!stop) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + 256 + (uint32_t)((wid >> 2) * 32);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 32; ++j) acc += v[j];
      }
      if (acc == 0x12345) cyc[1] = acc;
    }
  } else if (wid < 24) {
    if (mode & 2) {
      const int lt = tid - 512;
      size_t off = (size_t)blockIdx.x * 4096;
      while (!stop) {
        for (int i = lt; i < 4096; i += 256) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(sc + (i & 4095) * 16)),
                       "l"(gsrc + ((off + i) & ((1u << 19) - 1))) : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        off += 4096;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = (M + N) * D * 2 + 65536;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 16);
  uint4* g;
  cudaMalloc(&g, (size_t)16 << 19);
  cudaMemset(g, 0, (size_t)16 << 19);
  for (int mode = 0; mode < 16; mode += (mode < 8 ? 4 : 1)) {
    k<<<sms, 800, smem>>>(2000, mode, g, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"mode\": %d, \"tmem_ld\": %d, \"cp_async\": %d, \"random\": %d, \"pattern\": %d, \"cycles_per_mma\": %.1f, \"err\": \"%s\"}\n", mode,
           mode & 1, (mode >> 1) & 1, (mode >> 2) & 1, (mode >> 3) & 1, c / (2000.0 * 8), cudaGetErrorString(e));
  }
  return 0;
}
