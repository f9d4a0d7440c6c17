// Learned binary router on the tensor cores (the
// paper's fused classifier heads, §4 "Efficient router inference").
// Not in the reference, so parity is against the numpy restatement in
// oracle/ within fp32 accumulation tolerance, not bit-exact.
//
//   verdict(r, c) = E[r] . H[c] + bias[c] > 0
//
// E: request embeddings [R][D] bf16; H: one linear head per canonical
// configuration [S][D] bf16; bias [S] fp32.  Scoring every configuration of a
// batch is the dense contraction E . H^T (2 R S D flops), run as tcgen05 tiles
// by a persistent grid (one CTA per SM):
//   * work item = (256 requests, one 1024-configuration bitmap group = 8
//     tiles of 128 configurations); a CTA walks a contiguous run of items in
//     request-block-major order, so the A operand (256 x D embeddings, two
//     M-128 halves) is loaded once per request block it touches;
//   * one thread moves A and the B tiles with TMA (2-D tensor maps, 128-byte
//     swizzle, boxes of 64 elements x 128 rows; D is padded to a multiple of
//     64 by the map's zero fill, only the D / 16 real K steps are issued),
//     three B stages in flight;
//   * one thread issues tcgen05.mma kind::f16 (M 128, N 128, K 16), one per
//     request half per K step, into TMEM (two stages x two halves x 128
//     columns) and commits to mbarriers;
//   * TMEM lane = request, column = configuration: an epilogue thread reads 64
//     consecutive configurations of its request (two tcgen05.ld x32) and
//     makes each bitmap word with one packed f32x2 subtract (threshold -
//     accumulator) per two configurations and one funnel shift per
//     configuration that moves the sign bit in: sign(thr - acc) == (acc >
//     thr) for every non-NaN accumulator once the threshold -0 is made +0.
//     The verdict bitmap comes out in k_route_score's [R][W] layout, so the
//     scans and k_route_compact finish the job.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "ag_internal.h"

namespace agb {
namespace {

#ifndef AG_LIN_EXP
// Diagnostic variants (scripts/linexp.sh; results are wrong by design except
// 0 and 3): 1 = no threshold work, 2 = no TMEM loads either (the MMA pipeline
// alone), 3 = spinning epilogue waits, 4 = B tiles loaded once (stale),
// 5 = 2 with one request half's MMAs only, 6 = 2 with half the K steps,
// 9 = 2 + 4, 10 = 2 without the TMEM-empty wait.
#define AG_LIN_EXP 0
#endif
constexpr int kLinM = 128;        // requests per MMA (one TMEM lane each)
constexpr int kLinR = 256;        // requests per work item (two MMAs per K step)
constexpr int kLinN = 128;        // configurations per tile (MMA N)
constexpr int kGroupTiles = 8;    // tiles per work item (one 32-word bitmap group)
constexpr int kEpiWarps = 16;     // epilogue: 4 per TMEM lane quarter
constexpr int kBStages = 3;       // configuration-tile stages in shared memory
constexpr int kLinThreads = 32 * (kEpiWarps + 2);  // + TMA producer + MMA issuer
constexpr int kWbStride = 33;     // padded words per request row
constexpr int kBox = 128 * 128;   // bytes per TMA box (64 bf16 x 128 rows)
constexpr int kMaxKB = 2;         // 64-element K boxes for D <= 128

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major operand, 128-byte swizzle (the TMA box layout): rows 128 B apart,
// 8-row groups 1024 B apart (SBO); a K step of 16 elements advances the start
// address by 32 B inside the swizzle atom.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ void mbar_init(uint64_t* mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(mb)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* mb) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(su32(mb)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mb, uint32_t bytes) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(su32(mb)),
               "r"(bytes)
               : "memory");
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
// epilogue waits back off, so their spins do not take the single-thread
// roles' issue slots
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* mb, uint32_t parity) {
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(su32(mb)), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(32);
  }
}
__device__ __forceinline__ void umma_commit_elect(uint64_t* mb) {
  asm volatile(
      "{ .reg .pred e; elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }" ::"r"(su32(mb))
      : "memory");
}
// one 64-element x 128-row box of a 2-D bf16 tensor map into shared memory
__device__ __forceinline__ void tma_box(void* dst, const CUtensorMap* map, int k0, int row, uint64_t* mb) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(k0), "r"(row), "r"(su32(mb))
      : "memory");
}

struct LinArgs {
  const float* bias;    // [S]
  int R, D, KB;         // KB = 64-element K boxes per row
  uint64_t begin, end, top;
  uint32_t W, C;        // words per request, tasks (of 32 groups) per request
  uint32_t G;           // 32-word groups per request = work items per request block
  uint32_t items;       // request blocks x G
  uint32_t flags;
  uint32_t* bitmap;     // [R][W]
  uint32_t* task_counts;  // [R][C*32] popcount per 32-word group
};

// NKS = D / 16 MMA K steps per tile, unrolled (descriptors advance by
// constants: the issue loop is the tensor core's feed rate)
template <int NKS>
__global__ void __launch_bounds__(kLinThreads, 1)
    k_linear_score(const __grid_constant__ CUtensorMap emb_map, const __grid_constant__ CUtensorMap head_map,
                   LinArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the 128-byte swizzle
  unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sa = smem;                                   // [half][kb] boxes
  unsigned char* sb = sa + 2 * kMaxKB * kBox;                 // [stage][kb] boxes
  uint32_t* wbuf = reinterpret_cast<uint32_t*>(sb + kBStages * kMaxKB * kBox);  // [256][33]
  float* s_thr = reinterpret_cast<float*>(wbuf + kLinR * kWbStride);            // [1024]
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_thr + kLinN * kGroupTiles);   // [256][2]
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t a_full, a_empty, b_full[kBStages], b_empty[kBStages], t_full[2], t_empty[2];
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  // this CTA's contiguous run of work items
  const uint32_t it0 = (uint32_t)(((uint64_t)blockIdx.x * a.items) / gridDim.x);
  const uint32_t it1 = (uint32_t)(((uint64_t)(blockIdx.x + 1) * a.items) / gridDim.x);

  if (wid == kEpiWarps + 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&a_full, 1);
    mbar_init(&a_empty, 1);
    for (int i = 0; i < kBStages; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;

  // tiles of an item holding any configuration of [begin, end)
  auto item_tiles = [&](uint32_t grp) -> int {
    const uint64_t c0 = a.begin + (uint64_t)grp * (kLinN * kGroupTiles);
    return (int)min((uint64_t)kGroupTiles, (a.end - c0 + kLinN - 1) / kLinN);
  };

  if (wid == kEpiWarps) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&emb_map)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&head_map)) : "memory");
      uint32_t cur_rb = ~0u, na = 0, gt = 0;
      for (uint32_t it = it0; it < it1; ++it) {
        const uint32_t rb = it / a.G, grp = it - rb * a.G;
        if (rb != cur_rb) {
          if (na > 0) mbar_wait(&a_empty, (na - 1) & 1);  // the previous block's MMAs are done
          mbar_expect_tx(&a_full, 2 * a.KB * kBox);
          for (int h = 0; h < 2; ++h)
            for (int kb = 0; kb < a.KB; ++kb)
              tma_box(sa + (h * kMaxKB + kb) * kBox, &emb_map, kb * 64, (int)(rb * kLinR + h * kLinM), &a_full);
          ++na;
          cur_rb = rb;
        }
        const int T = item_tiles(grp);
        const uint64_t cb = a.begin + (uint64_t)grp * (kLinN * kGroupTiles);
        for (int t = 0; t < T; ++t, ++gt) {
          const int s = gt % kBStages;
          mbar_wait(&b_empty[s], ((gt / kBStages) & 1) ^ 1);
#if AG_LIN_EXP == 4 || AG_LIN_EXP == 9
          if (gt >= kBStages) {
            mbar_arrive(&b_full[s]);
            continue;
          }
#endif
          mbar_expect_tx(&b_full[s], a.KB * kBox);
          for (int kb = 0; kb < a.KB; ++kb)
            tma_box(sb + (s * kMaxKB + kb) * kBox, &head_map, kb * 64, (int)(cb + (uint64_t)t * kLinN), &b_full[s]);
        }
      }
    }
  } else if (wid == kEpiWarps + 1) {
    // ---------------------------------------------------------- MMA issue
    {  // the whole warp runs the loop (uniform descriptors); one elected lane issues
      // bf16 x bf16 -> f32, K-major both, M 128, N 128
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kLinN >> 3) << 17) |
                             ((uint32_t)(kLinM >> 4) << 24);
      const uint64_t da0 = sdesc_sw128(su32(sa)), db0 = sdesc_sw128(su32(sb));
      uint32_t cur_rb = ~0u, na = 0, gt = 0;
      for (uint32_t it = it0; it < it1; ++it) {
        const uint32_t rb = it / a.G, grp = it - rb * a.G;
        if (rb != cur_rb) {
          mbar_wait(&a_full, na & 1);
          ++na;
          cur_rb = rb;
        }
        const int T = item_tiles(grp);
        for (int t = 0; t < T; ++t, ++gt) {
          const int ts = gt & 1, bs = gt % kBStages;
          mbar_wait(&b_full[bs], (gt / kBStages) & 1);
          if (AG_LIN_EXP != 10) mbar_wait(&t_empty[ts], ((gt >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t db = db0 + (uint64_t)((bs * kMaxKB * kBox) >> 4);
#pragma unroll
          for (int hf = 0; hf < (AG_LIN_EXP == 5 ? 1 : 2); ++hf) {
            const uint32_t acc = tmem + (uint32_t)(ts * 2 * kLinN + hf * kLinN);
            const uint64_t da = da0 + (uint64_t)((hf * kMaxKB * kBox) >> 4);
#pragma unroll
            for (int ks = 0; ks < (AG_LIN_EXP == 6 ? NKS / 2 : NKS); ++ks) {
              // K step ks: box ks / 4, 32 bytes per step inside the atom
              const uint64_t off = (uint64_t)(((ks >> 2) * kBox + (ks & 3) * 32) >> 4);
              asm volatile(
                  "{ .reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0;\n"
                  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(acc),
                  "l"(da + off), "l"(db + off), "r"(idesc), "r"(ks > 0 ? 1u : 0u));
            }
          }
          umma_commit_elect(&b_empty[bs]);  // stage bs may be refilled once these MMAs are done
          umma_commit_elect(&t_full[ts]);   // and the accumulators are ready
        }
        // A may be replaced once every MMA of this request block is done
        if (it + 1 == it1 || (it + 1) / a.G != rb) umma_commit_elect(&a_empty);
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue
    // TMEM lane = request (warp w reads lane quarter w % 4), columns =
    // configurations: warp w takes request half (w / 8) and the 64 columns
    // ((w / 4) & 1) * 64 .. of a tile; a thread's 32 columns make one word
    const int q = wid & 3, hf = wid >> 3, ch = (wid >> 2) & 1;
    const int row = hf * kLinM + q * 32 + lane;  // request row in the block
    uint32_t gt = 0, cnt = 0;
    for (uint32_t it = it0; it < it1; ++it) {
      const uint32_t rb = it / a.G, grp = it - rb * a.G;
      const int T = item_tiles(grp);
      const uint64_t cb = a.begin + (uint64_t)grp * (kLinN * kGroupTiles);
      // an item needs word masks only at the end of the range or around top
      const bool edge = cb + kLinN * kGroupTiles > a.end ||
                        ((a.flags & AG_FORCE_TOP) && a.top >= cb && a.top < cb + kLinN * kGroupTiles);
      // thresholds of the item (acc + b > 0 <=> acc > -b; -0 made +0, tail +inf)
      for (int i = tid; i < kLinN * kGroupTiles; i += 32 * kEpiWarps) {
        const uint64_t c = cb + (uint64_t)i;
        s_thr[i] = c < a.end ? 0.0f - __ldg(a.bias + c) : INFINITY;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      for (int t = 0; t < T; ++t, ++gt) {
        const int ts = gt & 1;
        const float4* th = reinterpret_cast<const float4*>(s_thr + t * kLinN + ch * 64);
#if AG_LIN_EXP == 3
        mbar_wait(&t_full[ts], (gt >> 1) & 1);
#else
        mbar_wait_sleep(&t_full[ts], (gt >> 1) & 1);
#endif
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint32_t v[64];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ts * 2 * kLinN + hf * kLinN + ch * 64);
#if AG_LIN_EXP == 2 || AG_LIN_EXP == 5 || AG_LIN_EXP == 6 || AG_LIN_EXP >= 9
        for (int k = 0; k < 64; ++k) v[k] = 0;
#else
#pragma unroll
        for (int k = 0; k < 2; ++k)
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(v[32 * k + 0]), "=r"(v[32 * k + 1]), "=r"(v[32 * k + 2]), "=r"(v[32 * k + 3]),
                "=r"(v[32 * k + 4]), "=r"(v[32 * k + 5]), "=r"(v[32 * k + 6]), "=r"(v[32 * k + 7]),
                "=r"(v[32 * k + 8]), "=r"(v[32 * k + 9]), "=r"(v[32 * k + 10]), "=r"(v[32 * k + 11]),
                "=r"(v[32 * k + 12]), "=r"(v[32 * k + 13]), "=r"(v[32 * k + 14]), "=r"(v[32 * k + 15]),
                "=r"(v[32 * k + 16]), "=r"(v[32 * k + 17]), "=r"(v[32 * k + 18]), "=r"(v[32 * k + 19]),
                "=r"(v[32 * k + 20]), "=r"(v[32 * k + 21]), "=r"(v[32 * k + 22]), "=r"(v[32 * k + 23]),
                "=r"(v[32 * k + 24]), "=r"(v[32 * k + 25]), "=r"(v[32 * k + 26]), "=r"(v[32 * k + 27]),
                "=r"(v[32 * k + 28]), "=r"(v[32 * k + 29]), "=r"(v[32 * k + 30]), "=r"(v[32 * k + 31])
              : "r"(taddr + 32u * k));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#endif
        // this warp's part of the stage is drained
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&t_empty[ts]);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          uint32_t x = 0;
#if AG_LIN_EXP == 1 || AG_LIN_EXP == 2 || AG_LIN_EXP == 5 || AG_LIN_EXP == 6 || AG_LIN_EXP >= 9
          x = v[32 * k] ^ v[32 * k + 31];
#else
          // highest configuration first: after 32 shifts configuration j sits at bit j
#pragma unroll
          for (int j4 = 7; j4 >= 0; --j4) {
            const float4 tv = th[8 * k + j4];  // broadcast
            uint64_t t01, t23, a01, a23, d01, d23;
            asm("mov.b64 %0, {%1,%2};" : "=l"(t01) : "f"(tv.x), "f"(tv.y));
            asm("mov.b64 %0, {%1,%2};" : "=l"(t23) : "f"(tv.z), "f"(tv.w));
            asm("mov.b64 %0, {%1,%2};" : "=l"(a01) : "r"(v[32 * k + 4 * j4 + 0]), "r"(v[32 * k + 4 * j4 + 1]));
            asm("mov.b64 %0, {%1,%2};" : "=l"(a23) : "r"(v[32 * k + 4 * j4 + 2]), "r"(v[32 * k + 4 * j4 + 3]));
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d01) : "l"(t01), "l"(a01));
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d23) : "l"(t23), "l"(a23));
            uint32_t y0, y1, y2, y3;
            asm("mov.b64 {%0,%1}, %2;" : "=r"(y0), "=r"(y1) : "l"(d01));
            asm("mov.b64 {%0,%1}, %2;" : "=r"(y2), "=r"(y3) : "l"(d23));
            x = __funnelshift_l(y3, x, 1);
            x = __funnelshift_l(y2, x, 1);
            x = __funnelshift_l(y1, x, 1);
            x = __funnelshift_l(y0, x, 1);
          }
#endif
          // tail mask and forced top (warp-uniform: the word index is)
          const uint64_t wi = (uint64_t)grp * 32 + t * 4 + ch * 2 + k, i0 = a.begin + wi * 32;
          if (edge) {
            if (wi >= a.W) {
              x = 0;
            } else {
              if (a.end - i0 < 32) x &= (1u << (uint32_t)(a.end - i0)) - 1u;
              if ((a.flags & AG_FORCE_TOP) && a.top >= i0 && a.top < i0 + 32) x |= 1u << (uint32_t)(a.top - i0);
            }
          }
          wbuf[row * kWbStride + t * 4 + ch * 2 + k] = x;
          cnt += __popc(x);
        }
      }
      // the group is complete: 256 request rows of 32 words written out
      // coalesced (a warp per row), per-group counts for the scans
      s_cnt[row * 2 + ch] = cnt;
      cnt = 0;
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      const uint64_t wi = (uint64_t)grp * 32 + lane;
      if (lane < T * 4 && wi < a.W) {
        const int nr = min(kLinR, a.R - (int)(rb * kLinR));
        uint32_t* dst = a.bitmap + (size_t)rb * kLinR * a.W + wi;
        for (int rr = wid; rr < nr; rr += kEpiWarps) dst[(size_t)rr * a.W] = wbuf[rr * kWbStride + lane];
      }
      if (tid < kLinR && (int)(rb * kLinR) + tid < a.R && grp < a.G)
        a.task_counts[((size_t)rb * kLinR + tid) * a.C * 32 + grp] = s_cnt[2 * tid] + s_cnt[2 * tid + 1];
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (wid == kEpiWarps + 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// cuTensorMapEncodeTiled from the driver (no -lcuda at link time)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int encode_rows(CUtensorMap* map, const void* base, uint64_t rows, int dim) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return fail(AG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)p;
  }
  const cuuint64_t gdim[2] = {(cuuint64_t)dim, (cuuint64_t)rows};
  const cuuint64_t gstride[1] = {(cuuint64_t)dim * 2};
  const cuuint32_t box[2] = {64, 128};
  const cuuint32_t estride[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride, box,
                        estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(AG_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return AG_OK;
}

}  // namespace

}  // namespace agb

using agb::fail;

extern "C" int ag_route_linear(ag_ctx* ctx, const void* emb, int32_t n_requests, const ag_linear_heads* heads,
                               uint64_t begin, uint64_t end, uint32_t flags, const ag_route_out* out) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
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
    CUtensorMap emb_map, head_map;
    if ((rc = agb::encode_rows(&emb_map, emb, (uint64_t)R, heads->dim)) ||
        (rc = agb::encode_rows(&head_map, heads->heads, sp->size, heads->dim)))
      return rc;
    agb::LinArgs a;
    a.bias = heads->bias;
    a.R = R;
    a.D = heads->dim;
    a.KB = (heads->dim + 63) / 64;
    a.begin = begin;
    a.end = end;
    a.top = sp->size - 1;
    a.W = W;
    a.C = C;
    a.flags = flags;
    a.G = G;
    a.items = (uint32_t)((R + agb::kLinR - 1) / agb::kLinR) * G;
    a.bitmap = bitmap;
    a.task_counts = (uint32_t*)ctx->chunk_counts.p;
    // A (two halves) + B stages + word buffer + thresholds + alignment slack
    const size_t smem = (size_t)(2 + agb::kBStages) * agb::kMaxKB * agb::kBox +
                        (size_t)agb::kLinR * agb::kWbStride * 4 + agb::kLinN * agb::kGroupTiles * 4 +
                        agb::kLinR * 2 * 4 + 1024;
    typedef void (*lin_fn)(const CUtensorMap, const CUtensorMap, agb::LinArgs);
    static const lin_fn fns[8] = {agb::k_linear_score<1>, agb::k_linear_score<2>, agb::k_linear_score<3>,
                                  agb::k_linear_score<4>, agb::k_linear_score<5>, agb::k_linear_score<6>,
                                  agb::k_linear_score<7>, agb::k_linear_score<8>};
    const lin_fn fn = fns[heads->dim / 16 - 1];
    int& n_sms = ctx->linear_sms;
    if (!n_sms) {
      for (int i = 0; i < 8; ++i)
        AG_CUDA(cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      AG_CUDA(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, ctx->device));
    }
    const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)n_sms, a.items);
    {
      agb::Launch L(ctx, agb::K_LINEAR_SCORE);
      fn<<<grid, agb::kLinThreads, smem, s>>>(emb_map, head_map, a);
    }
    AG_CUDA(cudaGetLastError());
  }
  return agb::finish_enumerate(ctx, R, W, C, begin, bitmap, offsets, out);
}
