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
//   * one CTA owns a tile of 256 requests (two 128-row A operands, loaded
//     once) and a chunk of 16 configuration tiles of 128 (the B operand,
//     double buffered), i.e. 2048 configurations = two 32-word bitmap groups
//     per request;
//   * operands sit in shared memory in the canonical no-swizzle K-major
//     layout (8-row x 16-byte core matrices, K-chunks 128 B apart); one thread
//     issues tcgen05.mma kind::f16 (M 128, N 128, K 16), one per request half,
//     into TMEM accumulators (two stages x two halves x 128 columns) and
//     commits to an mbarrier;
//   * TMEM lane = request, column = configuration: an epilogue thread reads 32
//     consecutive configurations of its request with one tcgen05.ld and
//     thresholds them straight into that request's bitmap word (thresholds
//     broadcast from shared memory; no transpose) -- the verdict bitmap comes
//     out in the same [R][W] layout as k_route_score, so the scans and
//     k_route_compact finish the job.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "ag_internal.h"

namespace agb {
namespace {

constexpr int kLinM = 128;        // requests per MMA (one TMEM lane each)
constexpr int kLinR = 256;        // requests per CTA (two MMAs per K step)
constexpr int kLinN = 128;        // configurations per tile (MMA N)
constexpr int kLinTiles = 16;     // configuration tiles per CTA (2 groups of 1024)
constexpr int kEpiWarps = 16;     // epilogue: 4 per TMEM lane quarter
constexpr int kLdWarps = 8;       // cp.async loaders
constexpr int kBStages = 3;       // configuration-tile stages in shared memory
constexpr int kLinThreads = 32 * (kEpiWarps + kLdWarps + 1);  // + the MMA issuer
constexpr int kWbStride = 33;     // padded words per request row

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// canonical K-major, no swizzle: core matrix = 8 rows x 16 B; K-chunks of a
// row group 128 B apart (LBO); row groups KC * 128 B apart (SBO).  Core
// matrix cmi = (row / 8) * KC + kc starts at byte cmi * 128 (the loaders
// fill them in that order).

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);  // version 1 (sm100)
}

__device__ __forceinline__ void mbar_init(uint64_t* mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(mb)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* mb) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(su32(mb)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(su32(mb)), "r"(parity)
        : "memory");
}
// waiting roles that share a sub-partition with the MMA issuer back off, so
// their spins do not take its issue slots
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* mb, uint32_t parity) {
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(su32(mb)), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(64);
  }
}
__device__ __forceinline__ void umma_commit(uint64_t* mb) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(mb))
               : "memory");
}
// 16-byte async copy global -> shared (zero-filled when !valid)
__device__ __forceinline__ void cp16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}

struct LinArgs {
  const uint4* emb;     // [R][D] bf16, 16-byte row chunks
  const uint4* heads;   // [S][D] bf16 (indexed by canonical index)
  const float* bias;    // [S]
  int R, D;
  uint64_t begin, end, top;
  uint32_t W, C;        // words per request, tasks (of 32 groups) per request
  uint32_t G;           // 32-word groups per request
  uint32_t flags;
  uint32_t* bitmap;     // [R][W]
  uint32_t* task_counts;  // [R][C*32] popcount per 32-word group
};

// Warp-specialised: the loaders keep two B stages ahead (cp.async), the
// issuer runs the tensor core into two TMEM stages, the epilogue drains one
// stage while the other fills; full/empty mbarriers for both hand-offs.
// NKS = D / 16 MMA K steps per tile, unrolled (descriptors advance by a
// constant: the issue loop is the tensor core's feed rate)
template <int NKS>
__global__ void __launch_bounds__(kLinThreads, 1) k_linear_score(LinArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int KC = a.D / 8;                        // 16-byte K-chunks per row
  unsigned char* sa = smem;                      // [256 requests][D] core-matrix layout
  unsigned char* sb[kBStages];                   // [128 configurations][D] per stage
  sb[0] = sa + (size_t)kLinR * a.D * 2;
  for (int i = 1; i < kBStages; ++i) sb[i] = sb[i - 1] + (size_t)kLinN * a.D * 2;
  uint32_t* wbuf = reinterpret_cast<uint32_t*>(sb[kBStages - 1] + (size_t)kLinN * a.D * 2);  // [256][33]
  // thresholds of every configuration of the CTA (acc + b > 0 <=> acc > -b)
  __shared__ __align__(16) float s_thr[kLinN * kLinTiles];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t a_full, b_full[kBStages], b_empty[kBStages], t_full[2], t_empty[2];
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int r0 = blockIdx.y * kLinR;
  const uint64_t cbase = a.begin + (uint64_t)blockIdx.x * (kLinN * kLinTiles);
  // tiles of this CTA that hold any configuration of [begin, end)
  const int T = (int)min((uint64_t)kLinTiles, (a.end - cbase + kLinN - 1) / kLinN);

  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&a_full, 32 * kLdWarps);
    for (int i = 0; i < kBStages; ++i) {
      mbar_init(&b_full[i], 32 * kLdWarps);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 32 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;

  constexpr int kLd = 32 * kLdWarps;
  if (wid >= kEpiWarps && wid < kEpiWarps + kLdWarps) {
    // ---------------------------------------------------------- loaders
    const int lt = tid - 32 * kEpiWarps;
    // thread i fills row i % 8 of core matrix i / 8: a warp writes 512
    // contiguous bytes of shared memory (conflict-free) and reads 64-byte
    // runs of 8 rows
    for (int i = lt; i < kLinR * KC; i += kLd) {
      const int cmi = i >> 3, g = cmi / KC, kc = cmi - g * KC, row = g * 8 + (i & 7);
      const bool ok = r0 + row < a.R;
      cp16(sa + cmi * 128 + (i & 7) * 16, a.emb + (size_t)(ok ? r0 + row : 0) * KC + kc, ok);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive(&a_full);
    // two tiles' copies in flight per thread: tile t is issued before tile
    // t - 1 is waited for and published
    for (int t = 0; t < T; ++t) {
      const int s = t % kBStages;
      mbar_wait_sleep(&b_empty[s], ((t / kBStages) & 1) ^ 1);
      const uint64_t c0 = cbase + (uint64_t)t * kLinN;
      for (int i = lt; i < kLinN * KC; i += kLd) {
        const int cmi = i >> 3, g = cmi / KC, kc = cmi - g * KC;
        const uint64_t c = c0 + (uint64_t)(g * 8 + (i & 7));
        const bool ok = c < a.end;
        cp16(sb[s] + cmi * 128 + (i & 7) * 16, a.heads + (ok ? c : 0) * KC + kc, ok);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (t > 0) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&b_full[(t - 1) % kBStages]);
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (T > 0) mbar_arrive(&b_full[(T - 1) % kBStages]);
  } else if (wid == kEpiWarps + kLdWarps) {
    // ---------------------------------------------------------- MMA issue
    if (lane == 0) {
      // bf16 x bf16 -> f32, K-major both, M 128, N 128
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kLinN >> 3) << 17) |
                             ((uint32_t)(kLinM >> 4) << 24);
      const uint32_t lbo = 128, sbo = (uint32_t)KC * 128;
      const uint32_t half = (uint32_t)kLinM * KC * 16;  // byte offset of request rows 128..255
      // descriptors precomputed; K step ks adds 256 bytes = 16 to the
      // start-address field (addresses stay below 256 KB: no carry out)
      const uint64_t da0 = sdesc(su32(sa), lbo, sbo), da1 = sdesc(su32(sa) + half, lbo, sbo);
      const uint64_t db0 = sdesc(su32(sb[0]), lbo, sbo);
      const uint64_t b_stage = ((uint64_t)kLinN * KC * 16) >> 4;
      mbar_wait(&a_full, 0);
      for (int t = 0; t < T; ++t) {
        const int s = t & 1, bs = t % kBStages;
        mbar_wait(&b_full[bs], (t / kBStages) & 1);
        mbar_wait(&t_empty[s], ((t >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t db = db0 + (uint64_t)bs * b_stage;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const uint32_t acc = tmem + (uint32_t)(s * 2 * kLinN + hf * kLinN);
          const uint64_t da = hf ? da1 : da0;
#pragma unroll
          for (int ks = 0; ks < NKS; ++ks) {
            asm volatile(
                "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(acc),
                "l"(da + 16u * ks), "l"(db + 16u * ks), "r"(idesc), "r"(ks > 0 ? 1u : 0u));
          }
        }
        umma_commit(&b_empty[bs]);  // stage bs may be refilled once these MMAs are done
        umma_commit(&t_full[s]);   // and the accumulators are ready
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue
    // TMEM lane = request (warp w reads lane quarter w % 4), columns =
    // configurations: warp w takes request half (w / 8) and the 64 columns
    // ((w / 4) & 1) * 64 .. of it; a thread's 32 columns make one word
    const int q = wid & 3, hf = wid >> 3, ch = (wid >> 2) & 1;
    const int row = hf * kLinM + q * 32 + lane;  // request row in the CTA
    for (int i = tid; i < kLinN * kLinTiles; i += 32 * kEpiWarps) {
      const uint64_t c = cbase + (uint64_t)i;
      s_thr[i] = c < a.end ? -__ldg(a.bias + c) : INFINITY;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
    for (int t = 0; t < T; ++t) {
      const int s = t & 1;
      const float* thr = s_thr + t * kLinN + ch * 64;
      mbar_wait_sleep(&t_full[s], (t >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) +
                               (uint32_t)(s * 2 * kLinN + hf * kLinN + ch * 64 + k * 32);
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
        if (k == 1) {  // this warp's part of the stage is drained
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          mbar_arrive(&t_empty[s]);
        }
        uint32_t x = 0;
        const float4* th = reinterpret_cast<const float4*>(thr + 32 * k);
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 tv = th[j4];  // broadcast
          x |= (__uint_as_float(v[4 * j4 + 0]) > tv.x ? 1u : 0u) << (4 * j4 + 0);
          x |= (__uint_as_float(v[4 * j4 + 1]) > tv.y ? 1u : 0u) << (4 * j4 + 1);
          x |= (__uint_as_float(v[4 * j4 + 2]) > tv.z ? 1u : 0u) << (4 * j4 + 2);
          x |= (__uint_as_float(v[4 * j4 + 3]) > tv.w ? 1u : 0u) << (4 * j4 + 3);
        }
        wbuf[row * kWbStride + (t & 7) * 4 + ch * 2 + k] = x;
      }
      if ((t & 7) == 7 || t + 1 == T) {
        // the group is complete: 256 request rows of 32 words, top forced,
        // tail masked; per-group counts for the scans
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
        const uint32_t grp = blockIdx.x * (kLinTiles / 8) + (uint32_t)(t >> 3);
        const uint64_t wi = (uint64_t)grp * 32 + lane;
        const uint64_t i0 = a.begin + wi * 32;
        const int nw = ((t & 7) + 1) * 4;  // words of the group written by the tiles
        for (int rr = wid; rr < kLinR; rr += kEpiWarps) {
          const int r = r0 + rr;
          if (r >= a.R) break;
          uint32_t w = lane < nw ? wbuf[rr * kWbStride + lane] : 0u;
          if (wi >= a.W) w = 0;
          else if (a.end - i0 < 32) w &= (1u << (uint32_t)(a.end - i0)) - 1u;
          if ((a.flags & AG_FORCE_TOP) && wi < a.W && a.top >= i0 && a.top < i0 + 32) w |= 1u << (uint32_t)(a.top - i0);
          if (wi < a.W) a.bitmap[(size_t)r * a.W + wi] = w;
          uint32_t cnt = __popc(w);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
          if (lane == 0 && grp < a.G) a.task_counts[(size_t)r * a.C * 32 + grp] = cnt;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace


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
    a.G = G;
    a.bitmap = bitmap;
    a.task_counts = (uint32_t*)ctx->chunk_counts.p;
    const size_t smem = (size_t)(agb::kLinR + agb::kBStages * agb::kLinN) * heads->dim * 2 +
                        (size_t)agb::kLinR * agb::kWbStride * 4;
    typedef void (*lin_fn)(agb::LinArgs);
    static const lin_fn fns[8] = {agb::k_linear_score<1>, agb::k_linear_score<2>, agb::k_linear_score<3>,
                                  agb::k_linear_score<4>, agb::k_linear_score<5>, agb::k_linear_score<6>,
                                  agb::k_linear_score<7>, agb::k_linear_score<8>};
    const lin_fn fn = fns[heads->dim / 16 - 1];
    static bool attr = false;
    if (!attr) {
      const int max_smem = (agb::kLinR + agb::kBStages * agb::kLinN) * 128 * 2 + agb::kLinR * agb::kWbStride * 4;
      for (int i = 0; i < 8; ++i)
        AG_CUDA(cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
      attr = true;
    }
    const uint32_t per_cta = agb::kLinTiles / 8;  // groups per CTA
    const dim3 grid((G + per_cta - 1) / per_cta, (R + agb::kLinR - 1) / agb::kLinR);
    {
      agb::Launch L(ctx, agb::K_LINEAR_SCORE);
      fn<<<grid, agb::kLinThreads, smem, s>>>(a);
    }
    AG_CUDA(cudaGetLastError());
  }
  return agb::finish_enumerate(ctx, R, W, C, begin, bitmap, offsets, out);
}
