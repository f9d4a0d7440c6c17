// Validates the hand-built tcgen05 (UMMA) descriptors used by ag_linear.cu:
// one CTA, D[128 x 256] (fp32, TMEM) = A[128 x 128] . B[256 x 128]^T, bf16,
// both operands K-major in the no-swizzle core-matrix layout.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 256, K = 128, KC = K / 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// byte offset of element (row, k) in the core-matrix layout: 8 rows x 16 B per
// core matrix, K-chunks adjacent (LBO = 128 B), row groups KC*128 B apart (SBO)
__device__ __forceinline__ uint32_t cm_off(int row, int k) {
  return (uint32_t)(((row >> 3) * KC + (k >> 3)) * 128 + (row & 7) * 16 + (k & 7) * 2);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__global__ void k(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* sa = sm;                 // 32 KB
  unsigned char* sb = sm + M * K * 2;     // 64 KB
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, kk = i % K;
    *(__nv_bfloat16*)(sa + cm_off(r, kk)) = A[i];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, kk = i % K;
    *(__nv_bfloat16*)(sb + cm_off(r, kk)) = B[i];
  }
  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
  }
  asm volatile("fence.proxy.async.shared::cta;");  // generic smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t da = sdesc(smem_u32(sa) + ks * 256, 128, KC * 128);
      const uint64_t db = sdesc(smem_u32(sb) + ks * 256, 128, KC * 128);
      const uint32_t acc = ks > 0 ? 1u : 0u;
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  // wait for the MMAs
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (wid < 4) {
    const int row = wid * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(wid * 32) << 16) + (uint32_t)c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                     "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                     "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 32; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
  std::vector<__nv_bfloat16> a(M * K), b(N * K);
  std::vector<float> fa(M * K), fb(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) { fa[i] = (float)(rand() % 7 - 3); a[i] = __float2bfloat16(fa[i]); }
  for (int i = 0; i < N * K; ++i) { fb[i] = (float)(rand() % 5 - 2); b[i] = __float2bfloat16(fb[i]); }
  __nv_bfloat16 *da, *db; float* dd;
  cudaMalloc(&da, a.size() * 2); cudaMalloc(&db, b.size() * 2); cudaMalloc(&dd, M * N * 4);
  cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(dd, 0, M * N * 4);
  const int smem = (M + N) * K * 2;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<1, 128, smem>>>(da, db, dd);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> d(M * N);
  cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0; int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int kk = 0; kk < K; ++kk) s += (double)fa[i * K + kk] * fb[j * K + kk];
      const double err = fabs(s - d[i * N + j]);
      if (err > maxerr) maxerr = err;
      if (err > 0.5 && bad < 5) { printf("mismatch (%d,%d): %f vs %f\n", i, j, d[i * N + j], s); ++bad; }
    }
  printf("max abs err %g\n", maxerr);
  return 0;
}
