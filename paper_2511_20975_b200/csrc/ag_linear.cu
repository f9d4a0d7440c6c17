// Learned binary router on the tensor cores (the
// paper's fused classifier heads, §4 "Efficient router inference").
// Not in the reference, so parity is against the numpy restatement in
// oracle/ within fp32 accumulation tolerance, not bit-exact.
//
//   verdict(r, c) = E[r] . H[c] + bias[c] > 0
//
// E: request embeddings [R][D] bf16; H: one linear head per canonical
// configuration [S][D] bf16; bias [S] fp32.  Scoring every configuration of a
// batch is the dense contraction E . H^T (2 R S D flops), run as tcgen05 tiles:
//   * one CTA owns a tile of 256 requests (the B operand, loaded once) and a
//     chunk of 8 configuration tiles of 128 (A operands, double buffered),
//     i.e. 1024 configurations = one 32-word bitmap group per request;
//   * operands sit in shared memory in the canonical no-swizzle K-major
//     layout (8-row x 16-byte core matrices, K-chunks 128 B apart); one thread
//     issues tcgen05.mma kind::f16 (M 128, N 256, K 16) into a TMEM
//     accumulator (two 256-column buffers) and commits to an mbarrier;
//   * the epilogue warps (TMEM lane quarters 0-3) read 32 accumulator columns
//     at a time with tcgen05.ld, threshold against the row's bias, and one
//     warp ballot per column turns 32 configurations into the request's
//     bitmap word -- the verdict bitmap comes out in the same [R][W] layout
//     as k_route_score, so the scans and k_route_compact finish the job.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "ag_internal.h"

namespace agb {
namespace {

constexpr int kLinM = 128;        // configurations per MMA tile
constexpr int kLinN = 256;        // requests per CTA
constexpr int kLinTiles = 8;      // configuration tiles per CTA (1024 configs)
constexpr int kLinThreads = 256;  // warps 0-3 epilogue, 4-7 loaders (+ MMA issue)
constexpr int kWbStride = 33;     // padded words per request row

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// canonical K-major, no swizzle: core matrix = 8 rows x 16 B; K-chunks of a
// row group 128 B apart (LBO); row groups KC * 128 B apart (SBO)
__device__ __forceinline__ uint32_t cm_off(int row, int kc, int KC) {
  return (uint32_t)(((row >> 3) * KC + kc) * 128 + (row & 7) * 16);
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);  // version 1 (sm100)
}

__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(su32(mb)), "r"(phase)
        : "memory");
}

struct LinArgs {
  const uint4* emb;     // [R][D] bf16, 16-byte rows chunks
  const uint4* heads;   // [S][D] bf16 (indexed by canonical index)
  const float* bias;    // [S]
  int R, D;
  uint64_t begin, end, top;
  uint32_t W, C;        // words per request, tasks (of 32 groups) per request
  uint32_t flags;
  uint32_t* bitmap;     // [R][W]
  uint32_t* task_counts;  // [R][C*32] popcount per 32-word group
};

__global__ void __launch_bounds__(kLinThreads, 1) k_linear_score(LinArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int KC = a.D / 8;                        // 16-byte K-chunks per row
  unsigned char* sb = smem;                      // [256 requests][D] core-matrix layout
  unsigned char* sa0 = sb + (size_t)kLinN * a.D * 2;
  unsigned char* sa1 = sa0 + (size_t)kLinM * a.D * 2;
  uint32_t* wbuf = reinterpret_cast<uint32_t*>(sa1 + (size_t)kLinM * a.D * 2);  // [256][33]
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t s_mbar[2];
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int rt = blockIdx.y;                      // request tile
  const uint32_t g = blockIdx.x;                  // 1024-configuration group
  const uint64_t cbase = a.begin + (uint64_t)g * (kLinM * kLinTiles);
  const int r0 = rt * kLinN;

  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&s_mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&s_mbar[1])));
  }
  // loaders: a configuration tile of heads into a core-matrix buffer
  auto load_a = [&](int t, unsigned char* sa) {
    const uint64_t c0 = cbase + (uint64_t)t * kLinM;
    for (int i = tid - 128; i < kLinM * KC; i += 128) {
      const int row = i / KC, kc = i - row * KC;
      const uint64_t c = c0 + row;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (c < a.end) v = __ldg(a.heads + c * KC + kc);
      *reinterpret_cast<uint4*>(sa + cm_off(row, kc, KC)) = v;
    }
  };
  if (wid >= 4) {
    for (int i = tid - 128; i < kLinN * KC; i += 128) {
      const int row = i / KC, kc = i - row * KC;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r0 + row < a.R) v = __ldg(a.emb + (size_t)(r0 + row) * KC + kc);
      *reinterpret_cast<uint4*>(sb + cm_off(row, kc, KC)) = v;
    }
    load_a(0, sa0);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core proxy
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  // instruction descriptor: bf16 x bf16 -> f32, K-major both, M 128, N 256
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kLinN >> 3) << 17) |
                         ((uint32_t)(kLinM >> 4) << 24);
  const uint32_t lbo = 128, sbo = (uint32_t)KC * 128;
  auto issue = [&](int t) {
    const unsigned char* sa = (t & 1) ? sa1 : sa0;
    const uint32_t acc_col = tmem + (uint32_t)((t & 1) * kLinN);
    for (int ks = 0; ks < a.D / 16; ++ks) {
      const uint64_t da = sdesc(su32(sa) + ks * 256, lbo, sbo);
      const uint64_t db = sdesc(su32(sb) + ks * 256, lbo, sbo);
      const uint32_t accumulate = ks > 0 ? 1u : 0u;
      asm volatile(
          "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(acc_col),
          "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     su32(&s_mbar[t & 1]))
                 : "memory");
  };
  if (tid == 128) issue(0);
  for (int t = 0; t < kLinTiles; ++t) {
    if (wid >= 4) {
      if (t + 1 < kLinTiles) load_a(t + 1, ((t + 1) & 1) ? sa1 : sa0);
    } else {
      // epilogue: rows = configurations (lane = configuration within the
      // warp's 32), columns = requests
      mbar_wait(&s_mbar[t & 1], (uint32_t)((t >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t c = cbase + (uint64_t)t * kLinM + (uint64_t)(wid * 32 + lane);
      const float thr = c < a.end ? -__ldg(a.bias + c) : INFINITY;  // acc + b > 0 <=> acc > -b
      const int widx = t * 4 + wid;  // word of the group
      for (int c0 = 0; c0 < kLinN; c0 += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(wid * 32) << 16) + (uint32_t)((t & 1) * kLinN + c0);
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
        uint32_t mine = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const uint32_t w = __ballot_sync(0xffffffffu, __uint_as_float(v[j]) > thr);
          if (lane == j) mine = w;
        }
        wbuf[(c0 + lane) * kWbStride + widx] = mine;
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 128 && t + 1 < kLinTiles) issue(t + 1);
  }
  // write the group: request rows of 32 words, top forced, tail masked
  const uint64_t wfirst = (uint64_t)g * 32;  // first word of the group
  for (int rr = wid; rr < kLinN; rr += kLinThreads / 32) {
    const int r = r0 + rr;
    if (r >= a.R) break;
    const uint64_t wi = wfirst + lane;
    uint32_t w = wbuf[rr * kWbStride + lane];
    const uint64_t i0 = a.begin + wi * 32;
    if (wi >= a.W) w = 0;
    else if (a.end - i0 < 32) w &= (1u << (uint32_t)(a.end - i0)) - 1u;
    if ((a.flags & AG_FORCE_TOP) && a.top >= i0 && a.top < i0 + 32 && wi < a.W) w |= 1u << (uint32_t)(a.top - i0);
    if (wi < a.W) a.bitmap[(size_t)r * a.W + wi] = w;
    uint32_t cnt = __popc(w);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) a.task_counts[(size_t)r * a.C * 32 + g] = cnt;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace

// scans + compaction of a verdict bitmap produced by a scoring kernel
// (ag_route.cu)
int finish_enumerate(ag_ctx* ctx, int R, uint32_t W, uint32_t C, uint64_t begin, uint32_t* bitmap,
                     uint64_t* offsets, const ag_route_out* out);

}  // namespace agb

using agb::fail;

extern "C" int ag_route_linear(ag_ctx* ctx, const void* emb, int32_t n_requests, const ag_linear_heads* heads,
                               uint64_t begin, uint64_t end, uint32_t flags, const ag_route_out* out) {
  if (!ctx || !heads || !out) return fail(AG_ERR_VALIDATION, "null argument");
  const ag_space* sp = ctx->space;
  if (!sp->gpu_ok) return fail(AG_ERR_VALIDATION, "GPU path needs M^N <= 2^32 and N <= 32");
  if (begin > end || end > sp->size) return fail(AG_ERR_VALIDATION, "configuration index out of range");
  if (n_requests < 0) return fail(AG_ERR_VALIDATION, "negative request count");
  if (heads->dim < 16 || heads->dim > 128 || heads->dim % 16)
    return fail(AG_ERR_VALIDATION, "head dimension must be a multiple of 16 in [16, 128]");
  if (!heads->heads || !heads->bias || (n_requests > 0 && !emb))
    return fail(AG_ERR_VALIDATION, "null embeddings / heads / bias");
  if (!out->counts) return fail(AG_ERR_VALIDATION, "counts output is required");
  if ((reinterpret_cast<uintptr_t>(emb) | reinterpret_cast<uintptr_t>(heads->heads)) & 15)
    return fail(AG_ERR_VALIDATION, "embeddings and heads must be 16-byte aligned");
  const int R = n_requests;
  cudaStream_t s = ctx->stream;
  if (R == 0) {
    if (out->offsets) AG_CUDA(cudaMemsetAsync(out->offsets, 0, 8, s));
    if (out->overflow) AG_CUDA(cudaMemsetAsync(out->overflow, 0, 4, s));
    return AG_OK;
  }
  const uint64_t range = end - begin;
  const uint32_t W = (uint32_t)((range + 31) / 32);
  const uint32_t C = (W + 1023) / 1024;  // k_route_score's task granularity
  const uint32_t G = (W + 31) / 32;      // 32-word groups per request
  int rc;
  if ((rc = ctx->chunk_counts.ensure((size_t)R * C * 32 * 4)) || (rc = ctx->chunk_off.ensure((size_t)R * C * 32 * 8)))
    return rc;
  AG_CUDA(cudaMemsetAsync(ctx->chunk_counts.p, 0, (size_t)R * C * 32 * 4, s));  // groups past G count 0
  uint32_t* bitmap = out->bitmap;
  if (!bitmap) {
    if ((rc = ctx->bitmap.ensure((size_t)R * W * 4 + 4))) return rc;
    bitmap = (uint32_t*)ctx->bitmap.p;
  }
  uint64_t* offsets = out->offsets;
  if (!offsets) {
    if ((rc = ctx->offsets.ensure(((size_t)R + 1) * 8))) return rc;
    offsets = (uint64_t*)ctx->offsets.p;
  }
  if (range > 0) {
    agb::LinArgs a;
    a.emb = (const uint4*)emb;
    a.heads = (const uint4*)heads->heads;
    a.bias = heads->bias;
    a.R = R;
    a.D = heads->dim;
    a.begin = begin;
    a.end = end;
    a.top = sp->size - 1;
    a.W = W;
    a.C = C;
    a.flags = flags;
    a.bitmap = bitmap;
    a.task_counts = (uint32_t*)ctx->chunk_counts.p;
    const size_t smem = (size_t)(agb::kLinN + 2 * agb::kLinM) * heads->dim * 2 +
                        (size_t)agb::kLinN * agb::kWbStride * 4;
    static bool attr = false;
    if (!attr) {
      const int max_smem = (agb::kLinN + 2 * agb::kLinM) * 128 * 2 + agb::kLinN * agb::kWbStride * 4;
      AG_CUDA(cudaFuncSetAttribute(agb::k_linear_score, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
      attr = true;
    }
    const dim3 grid(G, (R + agb::kLinN - 1) / agb::kLinN);
    {
      agb::Launch L(ctx, agb::K_LINEAR_SCORE);
      agb::k_linear_score<<<grid, agb::kLinThreads, smem, s>>>(a);
    }
    AG_CUDA(cudaGetLastError());
  }
  return agb::finish_enumerate(ctx, R, W, C, begin, bitmap, offsets, out);
}
