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
// Stage 1: one warp per task (a slice of at most kTask members of one
// request), lanes keep their best key, a shuffle reduction writes the task's
// best.  Stage 2: one warp per request reduces its tasks.  Requests with
// hundreds of millions of members (the deep config-4 space) spread over many
// SMs; small requests are one task each.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "ag_internal.h"

namespace agb {
namespace {

constexpr int kCostWarps = 8;
constexpr uint64_t kTask = 1 << 16;

struct Key {
  double e, c;
  uint32_t i;
};

__device__ __forceinline__ bool key_less(double e1, double c1, uint32_t i1, double e2, double c2,
                                         uint32_t i2) {
  return e1 < e2 || (e1 == e2 && (c1 < c2 || (c1 == c2 && i1 < i2)));
}

struct CostArgs {
  SpaceDev sp;
  const uint32_t* members;
  int n_tasks;
  const uint64_t* t_begin;  // [n_tasks]
  const uint64_t* t_end;
  int kind;                     // 0 static, 1 runtime
  double term[kMaxModels + 1];  // per-tier estimate term (NaN: tier missing)
  double cost[kMaxModels + 1];
  Key* task_best;               // [n_tasks]
  int R;
  const int32_t* r_task;        // [R+1] task range per request
  uint32_t* chosen;
  double* est;
  int32_t* status;
};

__global__ void __launch_bounds__(kCostWarps * 32) k_cost_tasks(const CostArgs* __restrict__ Ap) {
  const CostArgs& A = *Ap;
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * kCostWarps + (threadIdx.x >> 5);
  if (t >= A.n_tasks) return;
  const uint64_t b0 = A.t_begin[t], b1 = A.t_end[t];
  const int n = A.sp.n;
  const uint32_t m = (uint32_t)A.sp.m;
  double be = INFINITY, bc = INFINITY;
  uint32_t bi = 0xffffffffu;
  bool missing = false;
  for (uint64_t k = b0 + lane; k < b1; k += 32) {
    const uint32_t idx = __ldg(A.members + k);
    uint32_t d[kMaxAgents];
    uint32_t x = idx;
    for (int a = n - 1; a >= 0; --a) {
      const uint32_t q = divm(x, A.sp.div_m);
      d[a] = x - q * m;
      x = q;
    }
    double e = 0.0, c = 0.0;
    for (int a = 0; a < n; ++a) {
      const double tv = A.term[d[a]];
      missing |= isnan(tv);
      e += tv;
      c += A.cost[d[a]];
    }
    if (A.kind == 0) e = 0.0;
    if (key_less(e, c, idx, be, bc, bi)) be = e, bc = c, bi = idx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double oe = __shfl_xor_sync(0xffffffffu, be, o);
    const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (key_less(oe, oc, oi, be, bc, bi)) be = oe, bc = oc, bi = oi;
  }
  if (__any_sync(0xffffffffu, missing) && lane == 0) atomicExch(A.status, AG_ERR_VALIDATION);
  if (lane == 0) A.task_best[t] = Key{be, bc, bi};
}

__global__ void __launch_bounds__(kCostWarps * 32) k_cost_reduce(const CostArgs* __restrict__ Ap) {
  const CostArgs& A = *Ap;
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * kCostWarps + (threadIdx.x >> 5);
  if (r >= A.R) return;
  double be = INFINITY, bc = INFINITY;
  uint32_t bi = 0xffffffffu;
  for (int t = A.r_task[r] + lane; t < A.r_task[r + 1]; t += 32) {
    const Key k = A.task_best[t];
    if (key_less(k.e, k.c, k.i, be, bc, bi)) be = k.e, bc = k.c, bi = k.i;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double oe = __shfl_xor_sync(0xffffffffu, be, o);
    const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (key_less(oe, oc, oi, be, bc, bi)) be = oe, bc = oc, bi = oi;
  }
  if (lane == 0) {
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
  cudaStream_t st = ctx->stream;
  const int R = n_requests;
  // task table from the request offsets (one slice of <= kTask members each)
  std::vector<uint64_t> off(R + 1);
  AG_CUDA(cudaMemcpyAsync(off.data(), offsets, 8 * (size_t)(R + 1), cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaStreamSynchronize(st));
  std::vector<uint64_t> tb, te;
  std::vector<int32_t> rt(R + 1, 0);
  for (int r = 0; r < R; ++r) {
    if (off[r + 1] <= off[r]) return fail(AG_ERR_VALIDATION, "accurate set is empty");
    for (uint64_t b = off[r]; b < off[r + 1]; b += agb::kTask) {
      tb.push_back(b);
      te.push_back(std::min(off[r + 1], b + agb::kTask));
    }
    rt[r + 1] = (int32_t)tb.size();
  }
  const int T = (int)tb.size();
  agb::CostArgs A;
  A.sp = sp->dev();
  A.members = members;
  A.n_tasks = T;
  A.kind = kind == AG_POLICY_PER_INPUT_RUNTIME_COST ? 1 : 0;
  for (int i = 0; i <= agb::kMaxModels; ++i) {
    A.term[i] = 0.0;
    A.cost[i] = i < sp->m ? sp->cost[i] : 0.0;
  }
  if (A.kind == 1) {
    // estimate_completion (workload.cpp:129-147)
    if (load->n_tiers < 0) return fail(AG_ERR_VALIDATION, "estimator context arrays disagree on tier count");
    for (int i = 0; i < sp->m; ++i) {
      if (i >= load->n_tiers || load->slots[i] <= 0) {
        A.term[i] = NAN;  // an error only if a member uses the tier
        continue;
      }
      const double ld = (double)(load->occupancy[i] + load->queued_ahead[i]);
      const double mean = load->mean[i];
      A.term[i] = (ld / (double)load->slots[i]) * mean + mean;
    }
  }
  A.R = R;
  A.chosen = chosen;
  A.est = est;
  int rc;
  const size_t tbytes = (size_t)T * 16 + (size_t)(R + 1) * 4 + (size_t)T * sizeof(agb::Key) + 64;
  if ((rc = ctx->cost_args.ensure(sizeof(A))) || (rc = ctx->cost_status.ensure(tbytes))) return rc;
  char* d = (char*)ctx->cost_status.p;
  A.status = (int32_t*)d;
  A.t_begin = (const uint64_t*)(d + 16);
  A.t_end = A.t_begin + T;
  A.r_task = (const int32_t*)(A.t_end + T);
  A.task_best = (agb::Key*)(((uintptr_t)(A.r_task + R + 1) + 15) & ~(uintptr_t)15);
  AG_CUDA(cudaMemsetAsync(d, 0, 16, st));
  AG_CUDA(cudaMemcpyAsync((void*)A.t_begin, tb.data(), 8 * (size_t)T, cudaMemcpyHostToDevice, st));
  AG_CUDA(cudaMemcpyAsync((void*)A.t_end, te.data(), 8 * (size_t)T, cudaMemcpyHostToDevice, st));
  AG_CUDA(cudaMemcpyAsync((void*)A.r_task, rt.data(), 4 * (size_t)(R + 1), cudaMemcpyHostToDevice, st));
  // the argument block (per-tier tables) is too large for kernel parameters
  AG_CUDA(cudaMemcpyAsync(ctx->cost_args.p, &A, sizeof(A), cudaMemcpyHostToDevice, st));
  const agb::CostArgs* dA = (const agb::CostArgs*)ctx->cost_args.p;
  {
    agb::Launch L(ctx, agb::K_COST_ARGMIN);
    agb::k_cost_tasks<<<(T + agb::kCostWarps - 1) / agb::kCostWarps, agb::kCostWarps * 32, 0, st>>>(dA);
  }
  {
    agb::Launch L(ctx, agb::K_COST_ARGMIN);
    agb::k_cost_reduce<<<(R + agb::kCostWarps - 1) / agb::kCostWarps, agb::kCostWarps * 32, 0, st>>>(dA);
  }
  AG_CUDA(cudaGetLastError());
  int32_t stv = 0;
  AG_CUDA(cudaMemcpyAsync(&stv, d, 4, cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaStreamSynchronize(st));
  if (stv) return fail(AG_ERR_VALIDATION, "estimator context missing a model tier");
  return AG_OK;
}
