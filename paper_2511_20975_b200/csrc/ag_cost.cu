// Runtime-cost re-cost + argmin (the per-input-runtime-cost policy):
// estimate_completion over every member of a request's set and the arg-min
// with the reference's tie order (reference src/workload.cpp:129-176).
//
//   est(c)  = sum over agents a (in order) of
//             ((occupancy[m] + queued_ahead[m]) / slots[m]) * mean[m] + mean[m]
//   cost(c) = sum over agents a (in order) of cost[m]          (static_cost)
// The reference sorts members by (cost, canonical index) and keeps the first
// strict minimum of est, i.e. the minimum of the key (est, cost, index).  The
// per-tier term is the same expression for every agent using that tier, so it
// is computed once; the sums are left folds in agent order, fp64, no FMA.
//
// One warp per request over its member list (canonical indices, the routing
// CSR); lanes keep their best key, a shuffle reduction picks the winner.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "ag_internal.h"

namespace agb {
namespace {

constexpr int kCostWarps = 8;

struct CostArgs {
  SpaceDev sp;
  const uint32_t* members;
  const uint64_t* offsets;  // [R+1]
  int R;
  int kind;                 // 0 static, 1 runtime
  double term[kMaxModels + 1];  // per-tier estimate term (NaN: tier missing)
  double cost[kMaxModels + 1];
  uint32_t* chosen;
  double* est;
  int32_t* status;
};

__global__ void __launch_bounds__(kCostWarps * 32) k_cost_argmin(const CostArgs* __restrict__ Ap) {
  const CostArgs& A = *Ap;
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * kCostWarps + (threadIdx.x >> 5);
  if (r >= A.R) return;
  const uint64_t b0 = A.offsets[r], b1 = A.offsets[r + 1];
  const int n = A.sp.n;
  const uint32_t m = (uint32_t)A.sp.m;
  double be = INFINITY, bc = INFINITY;
  uint32_t bi = 0xffffffffu;
  bool missing = false;
  for (uint64_t k = b0 + lane; k < b1; k += 32) {
    const uint32_t idx = A.members[k];
    uint32_t d[kMaxAgents];
    uint32_t x = idx;
    for (int a = n - 1; a >= 0; --a) {
      const uint32_t q = divm(x, A.sp.div_m);
      d[a] = x - q * m;
      x = q;
    }
    double e = 0.0, c = 0.0;
    for (int a = 0; a < n; ++a) {
      const double t = A.term[d[a]];
      missing |= isnan(t);
      e += t;
      c += A.cost[d[a]];
    }
    if (A.kind == 0) e = 0.0;
    const bool better = e < be || (e == be && (c < bc || (c == bc && idx < bi)));
    if (better) be = e, bc = c, bi = idx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double oe = __shfl_xor_sync(0xffffffffu, be, o);
    const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (oe < be || (oe == be && (oc < bc || (oc == bc && oi < bi)))) be = oe, bc = oc, bi = oi;
  }
  if (__any_sync(0xffffffffu, missing) && lane == 0) atomicExch(A.status, AG_ERR_VALIDATION);
  if (lane == 0) {
    if (b1 == b0) atomicExch(A.status, AG_ERR_VALIDATION + 1);  // empty set
    A.chosen[r] = bi;
    if (A.est) A.est[r] = be;
  }
}

}  // namespace
}  // namespace agb

using agb::fail;

extern "C" int ag_select_per_input(ag_ctx* ctx, const uint32_t* members, const uint64_t* offsets,
                                   int32_t n_requests, int32_t kind, const ag_load* load,
                                   uint32_t* chosen, double* est) {
  if (!ctx || !members || !offsets || !chosen) return fail(AG_ERR_VALIDATION, "null argument");
  if (kind != AG_POLICY_PER_INPUT_STATIC && kind != AG_POLICY_PER_INPUT_RUNTIME_COST)
    return fail(AG_ERR_VALIDATION, "per-input selection needs a per-input policy kind");
  if (kind == AG_POLICY_PER_INPUT_RUNTIME_COST && !load)
    return fail(AG_ERR_VALIDATION, "runtime-cost selection needs a load context");
  const ag_space* sp = ctx->space;
  if (!sp->gpu_ok) return fail(AG_ERR_VALIDATION, "GPU path needs M^N <= 2^32 and N <= 32");
  if (n_requests <= 0) return n_requests == 0 ? AG_OK : fail(AG_ERR_VALIDATION, "negative request count");
  agb::CostArgs A;
  A.sp = sp->dev();
  A.members = members;
  A.offsets = offsets;
  A.R = n_requests;
  A.kind = kind == AG_POLICY_PER_INPUT_RUNTIME_COST ? 1 : 0;
  for (int i = 0; i <= agb::kMaxModels; ++i) {
    A.term[i] = 0.0;
    A.cost[i] = i < sp->m ? sp->cost[i] : 0.0;
  }
  if (A.kind == 1) {
    // estimate_completion (workload.cpp:129-147): the context arrays must agree
    if (load->n_tiers < 0) return fail(AG_ERR_VALIDATION, "estimator context arrays disagree on tier count");
    for (int i = 0; i < sp->m; ++i) {
      if (i >= load->n_tiers || load->slots[i] <= 0) {
        A.term[i] = NAN;  // only an error if a member uses the tier
        continue;
      }
      const double ld = (double)(load->occupancy[i] + load->queued_ahead[i]);
      const double mean = load->mean[i];
      A.term[i] = (ld / (double)load->slots[i]) * mean + mean;
    }
  }
  int rc;
  if ((rc = ctx->cost_args.ensure(sizeof(A))) || (rc = ctx->cost_status.ensure(8))) return rc;
  int32_t* dstat = (int32_t*)ctx->cost_status.p;
  A.chosen = chosen;
  A.est = est;
  A.status = dstat;
  // the argument block (per-tier tables) is too large for kernel parameters
  AG_CUDA(cudaMemcpyAsync(ctx->cost_args.p, &A, sizeof(A), cudaMemcpyHostToDevice, ctx->stream));
  AG_CUDA(cudaMemsetAsync(dstat, 0, 8, ctx->stream));
  const int blocks = (n_requests + agb::kCostWarps - 1) / agb::kCostWarps;
  {
    agb::Launch L(ctx, agb::K_COST_ARGMIN);
    agb::k_cost_argmin<<<blocks, agb::kCostWarps * 32, 0, ctx->stream>>>(
        (const agb::CostArgs*)ctx->cost_args.p);
  }
  AG_CUDA(cudaGetLastError());
  int32_t st[2] = {0, 0};
  AG_CUDA(cudaMemcpyAsync(st, dstat, 8, cudaMemcpyDeviceToHost, ctx->stream));
  AG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (st[0] == AG_ERR_VALIDATION + 1) return fail(AG_ERR_VALIDATION, "accurate set is empty");
  if (st[0]) return fail(AG_ERR_VALIDATION, "estimator context missing a model tier");
  return AG_OK;
}
