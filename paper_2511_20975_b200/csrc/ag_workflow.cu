// Per-workflow baseline on the GPU: select_per_workflow_config
// (reference src/workload.cpp:99-127) without the reference's 4096-config
// guard.
//
//   needed = (1 - tolerance) * |sample|
//   choice = the first configuration in (static cost, canonical index) order
//            whose accurate count over the sample reaches needed
//          = min over {c : hits(c) >= needed} of (static_cost(c), c)
//
// 1. K1 (k_route_score, oracle router) scores every configuration of every
//    sample set into the bitmap [R][W].
// 2. k_column_hits: one thread per bitmap word column and chunk of sample
//    rows; the column's 32 per-configuration counts are kept bit-sliced (a
//    ripple-carry counter over bit planes: ~3 logic ops per plane per word
//    instead of 32 adds), extracted once, added to hits[S].
// 3. k_workflow_best: every configuration with enough hits is costed
//    (static_cost's left fold in agent order, fp64, no FMA -- workflow.cpp:
//    291-296) and the (cost, index) minimum is reduced per block, then over
//    blocks.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "ag_internal.h"

namespace agb {
namespace {

constexpr int kHitThreads = 256;
constexpr int kChunkRows = 2048;  // sample rows per bit-sliced counter
constexpr int kPlanes = 12;       // counts up to 4095 >= kChunkRows
constexpr int kBestThreads = 256;

__global__ void __launch_bounds__(kHitThreads)
    k_column_hits(const uint32_t* __restrict__ bitmap, int R, uint32_t W, uint32_t* __restrict__ hits,
                  uint64_t S, int single_chunk) {
  const uint32_t w = blockIdx.x * kHitThreads + threadIdx.x;
  if (w >= W) return;
  const int r0 = blockIdx.y * kChunkRows, r1 = min(R, r0 + kChunkRows);
  uint32_t plane[kPlanes];
#pragma unroll
  for (int p = 0; p < kPlanes; ++p) plane[p] = 0;
  const uint32_t* col = bitmap + w;
  int r = r0;
  for (; r + 4 <= r1; r += 4) {
    uint32_t x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = __ldg(col + (size_t)(r + u) * W);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint32_t carry = x[u];
#pragma unroll
      for (int p = 0; p < kPlanes; ++p) {
        const uint32_t t = plane[p] & carry;
        plane[p] ^= carry;
        carry = t;
      }
    }
  }
  for (; r < r1; ++r) {
    uint32_t carry = __ldg(col + (size_t)r * W);
#pragma unroll
    for (int p = 0; p < kPlanes; ++p) {
      const uint32_t t = plane[p] & carry;
      plane[p] ^= carry;
      carry = t;
    }
  }
  const uint64_t c0 = (uint64_t)w * 32;
#pragma unroll 4
  for (int b = 0; b < 32; ++b) {
    if (c0 + b >= S) break;
    uint32_t cnt = 0;
#pragma unroll
    for (int p = 0; p < kPlanes; ++p) cnt |= ((plane[p] >> b) & 1u) << p;
    if (single_chunk) hits[c0 + b] = cnt;
    else if (cnt) atomicAdd(hits + c0 + b, cnt);
  }
}

struct Best {
  double cost;
  uint32_t idx;
  uint32_t pad;
};

__device__ __forceinline__ bool best_less(double c1, uint32_t i1, double c2, uint32_t i2) {
  return c1 < c2 || (c1 == c2 && i1 < i2);
}

struct BestArgs {
  SpaceDev sp;
  double cost[kMaxModels + 1];
  const uint32_t* hits;
  double needed;
  Best* block_best;
};

__global__ void __launch_bounds__(kBestThreads) k_workflow_best(const BestArgs* __restrict__ Ap) {
  const BestArgs& A = *Ap;
  __shared__ Best s_w[kBestThreads / 32];
  const int n = A.sp.n;
  const uint32_t m = (uint32_t)A.sp.m;
  double bc = INFINITY;
  uint32_t bi = 0xffffffffu;
  const uint64_t stride = (uint64_t)gridDim.x * kBestThreads;
  for (uint64_t c = (uint64_t)blockIdx.x * kBestThreads + threadIdx.x; c < A.sp.size; c += stride) {
    if ((double)__ldg(A.hits + c) < A.needed) continue;
    uint32_t d[kMaxAgents];
    uint32_t x = (uint32_t)c;
    for (int a = n - 1; a >= 0; --a) {
      const uint32_t q = divm(x, A.sp.div_m);
      d[a] = x - q * m;
      x = q;
    }
    double cost = 0.0;
    for (int a = 0; a < n; ++a) cost += A.cost[d[a]];
    if (best_less(cost, (uint32_t)c, bc, bi)) bc = cost, bi = (uint32_t)c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (best_less(oc, oi, bc, bi)) bc = oc, bi = oi;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_w[wid] = Best{bc, bi, 0};
  __syncthreads();
  if (threadIdx.x == 0) {
    Best b = s_w[0];
    for (int k = 1; k < kBestThreads / 32; ++k)
      if (best_less(s_w[k].cost, s_w[k].idx, b.cost, b.idx)) b = s_w[k];
    A.block_best[blockIdx.x] = b;
  }
}

__global__ void k_best_reduce(const Best* __restrict__ in, int n, Best* __restrict__ out) {
  double bc = INFINITY;
  uint32_t bi = 0xffffffffu;
  for (int k = threadIdx.x; k < n; k += 32)
    if (best_less(in[k].cost, in[k].idx, bc, bi)) bc = in[k].cost, bi = in[k].idx;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (best_less(oc, oi, bc, bi)) bc = oc, bi = oi;
  }
  if (threadIdx.x == 0) *out = Best{bc, bi, 0};
}

}  // namespace
}  // namespace agb

using agb::fail;

extern "C" int ag_select_per_workflow_host(ag_ctx* ctx, const ag_truth* th, double tolerance,
                                           uint64_t* chosen, uint64_t* hits_out) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  if (!ctx || !th || !chosen) return fail(AG_ERR_VALIDATION, "null argument");
  const int R = th->n_requests;
  if (R < 0) return fail(AG_ERR_VALIDATION, "negative request count");
  // validation in the reference's order (workload.cpp:102-108)
  if (R == 0) return fail(AG_ERR_VALIDATION, "per-workflow sample is empty");
  if (!(tolerance >= 0 && tolerance <= 1)) return fail(AG_ERR_VALIDATION, "tolerance outside [0, 1]");
  const ag_space* sp = ctx->space;
  if (!sp->gpu_ok) return fail(AG_ERR_VALIDATION, "GPU path needs M^N <= 2^32 and N <= 32");
  const uint64_t S = sp->size;
  const uint32_t W = (uint32_t)((S + 31) / 32);
  ag_truth td;
  int rc = agb::upload_truth(ctx, th, &td);
  if (rc) return rc;
  const int chunks = (R + agb::kChunkRows - 1) / agb::kChunkRows;
  const int best_blocks = (int)std::min<uint64_t>((S + agb::kBestThreads - 1) / agb::kBestThreads, 148 * 16);
  if ((rc = ctx->counts.ensure(8 * (size_t)R)) || (rc = ctx->offsets.ensure(8 * ((size_t)R + 1))) ||
      (rc = ctx->bitmap.ensure((size_t)R * W * 4 + 4)) || (rc = ctx->wf_hits.ensure(4 * (size_t)S + 4)) ||
      (rc = ctx->wf_best.ensure(sizeof(agb::Best) * ((size_t)best_blocks + 1) + sizeof(agb::BestArgs) + 64)))
    return rc;
  cudaStream_t s = ctx->stream;
  // 1. verdicts of every sample set (AccurateSet::contains, accuracy.cpp:116-124)
  const ag_router oracle{AG_ROUTER_ORACLE, 0.0, 0.0, 0, 0.0};
  ag_route_out o1{(uint32_t*)ctx->bitmap.p, (uint64_t*)ctx->counts.p, nullptr, nullptr, 0, nullptr};
  if ((rc = agb::route_enumerate(ctx, &td, &oracle, 0, S, 0, &o1))) return rc;
  // 2. per-configuration hit counts
  uint32_t* hits = (uint32_t*)ctx->wf_hits.p;
  if (chunks > 1) AG_CUDA(cudaMemsetAsync(hits, 0, 4 * (size_t)S, s));
  {
    agb::Launch L(ctx, agb::K_COST_ARGMIN);
    const dim3 grid((W + agb::kHitThreads - 1) / agb::kHitThreads, chunks);
    agb::k_column_hits<<<grid, agb::kHitThreads, 0, s>>>((const uint32_t*)ctx->bitmap.p, R, W, hits, S,
                                                        chunks == 1 ? 1 : 0);
  }
  // 3. the cheapest configuration with enough hits
  agb::BestArgs A;
  A.sp = sp->dev();
  for (int i = 0; i <= agb::kMaxModels; ++i) A.cost[i] = i < sp->m ? sp->cost[i] : 0.0;
  A.hits = hits;
  A.needed = (1.0 - tolerance) * (double)R;
  char* d = (char*)ctx->wf_best.p;
  A.block_best = (agb::Best*)d;
  agb::Best* final_best = A.block_best + best_blocks;
  agb::BestArgs* dA = (agb::BestArgs*)(d + sizeof(agb::Best) * ((size_t)best_blocks + 1));
  AG_CUDA(cudaMemcpyAsync(dA, &A, sizeof A, cudaMemcpyHostToDevice, s));
  {
    agb::Launch L(ctx, agb::K_COST_ARGMIN);
    agb::k_workflow_best<<<best_blocks, agb::kBestThreads, 0, s>>>(dA);
    agb::k_best_reduce<<<1, 32, 0, s>>>(A.block_best, best_blocks, final_best);
  }
  AG_CUDA(cudaGetLastError());
  agb::Best b;
  AG_CUDA(cudaMemcpyAsync(&b, final_best, sizeof b, cudaMemcpyDeviceToHost, s));
  AG_CUDA(cudaStreamSynchronize(s));
  // found <=> a finite static cost: index 0xffffffff is a valid configuration
  // when M^N == 2^32, so the index cannot double as the not-found sentinel
  if (!(b.cost < INFINITY)) return fail(AG_ERR_VALIDATION, "per-workflow scan found no configuration");
  *chosen = b.idx;
  if (hits_out) {
    uint32_t h = 0;
    AG_CUDA(cudaMemcpy(&h, hits + b.idx, 4, cudaMemcpyDeviceToHost));
    *hits_out = h;
  }
  return AG_OK;
}
