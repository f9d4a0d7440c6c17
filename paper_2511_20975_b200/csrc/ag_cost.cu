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
// Stage 0: the folds over the first k digits of every prefix q (k <= N - 1,
// M^k <= kPrefixMax) are tabulated once per call -- (e, c) after agents
// 0..k-1, the same adds in the same order -- so a member costs one 16-byte
// table load (members are sorted, so a warp's lanes share one or two
// prefixes) plus the N - k remaining terms from shared memory.
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
constexpr uint64_t kPrefixMax = 1u << 22;  // prefix-table entries (64 MB)

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
  int k;                        // digits folded into the prefix table
  uint32_t mk;                  // M^(N-k): members per prefix
  uint64_t div_mk;              // ceil(2^64 / mk)
  const double2* prefix;        // [M^k] (e, c) after agents 0..k-1
};

// Stage 0: prefix folds (estimate_completion / static_cost, left to right)
__global__ void __launch_bounds__(256) k_cost_prefix(const CostArgs* __restrict__ Ap, uint64_t n_pre,
                                                     double2* __restrict__ out) {
  const CostArgs& A = *Ap;
  const uint64_t q = (uint64_t)blockIdx.x * 256 + threadIdx.x;
  if (q >= n_pre) return;
  const uint32_t m = (uint32_t)A.sp.m;
  uint32_t d[kMaxAgents];
  uint32_t x = (uint32_t)q;
  for (int a = A.k - 1; a >= 0; --a) {
    const uint32_t qq = divm(x, A.sp.div_m);
    d[a] = x - qq * m;
    x = qq;
  }
  double e = 0.0, c = 0.0;
  for (int a = 0; a < A.k; ++a) {
    e += A.term[d[a]];
    c += A.cost[d[a]];
  }
  out[q] = make_double2(e, c);
}

// SFX = N - k suffix digits per member (1..4 specialised; 0 = runtime, <= 16:
// M^N <= 2^32 and M^k <= kPrefixMax leave at most 16).
template <int SFX>
__global__ void __launch_bounds__(kCostWarps * 32) k_cost_tasks(const CostArgs* __restrict__ Ap) {
  const CostArgs& A = *Ap;
  __shared__ double s_term[kMaxModels + 1], s_cost[kMaxModels + 1];
  const int m_ = A.sp.m;
  for (int i = threadIdx.x; i < m_; i += blockDim.x) {
    s_term[i] = A.term[i];
    s_cost[i] = A.cost[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * kCostWarps + (threadIdx.x >> 5);
  if (t >= A.n_tasks) return;
  const uint64_t b0 = A.t_begin[t];
  const uint32_t len = (uint32_t)(A.t_end[t] - b0);  // <= kTask
  const uint32_t* mem = A.members + b0;
  const int sfx = SFX > 0 ? SFX : A.sp.n - A.k;
  const uint32_t m = (uint32_t)m_, mk = A.mk;
  const uint64_t div_m = A.sp.div_m, div_mk = A.div_mk;
  const double2* __restrict__ prefix = A.prefix;
  const bool runtime = A.kind != 0;
  double be = INFINITY, bc = INFINITY;
  uint32_t bi = 0xffffffffu;
  bool missing = false;
  // four members per lane per pass: their loads are in flight together
  constexpr int kU = 4;
  for (uint32_t j = lane; j < len; j += 32 * kU) {
    uint32_t idx[kU], q[kU];
    double2 pre[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) idx[u] = j + 32 * u < len ? __ldg(mem + j + 32 * u) : 0u;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      q[u] = divm(idx[u], div_mk);
      pre[u] = __ldg(prefix + (j + 32 * u < len ? q[u] : 0u));
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (j + 32 * u >= len) break;
      // suffix digits, last first, packed one per byte (two words: <= 16)
      uint32_t x = idx[u] - q[u] * mk;
      uint64_t pk[2] = {0, 0};
#pragma unroll
      for (int a = (SFX > 0 ? SFX : 16) - 1; a >= 0; --a) {
        if (SFX == 0 && a >= sfx) continue;
        const uint32_t qq = a > 0 ? divm(x, div_m) : 0u;
        pk[a >> 3] |= (uint64_t)(x - qq * m) << (8 * (a & 7));
        x = qq;
      }
      double e = pre[u].x, c = pre[u].y;
#pragma unroll
      for (int a = 0; a < (SFX > 0 ? SFX : 16); ++a) {
        if (SFX == 0 && a >= sfx) break;
        const uint32_t dg = (uint32_t)(pk[a >> 3] >> (8 * (a & 7))) & 0xFFu;
        e += s_term[dg];
        c += s_cost[dg];
      }
      missing |= isnan(e);  // a NaN term (missing tier) anywhere in the fold
      if (!runtime) e = 0.0;
      if (key_less(e, c, idx[u], be, bc, bi)) be = e, bc = c, bi = idx[u];
    }
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
  // prefix table: the largest k <= N - 1 with M^k <= kPrefixMax
  {
    int k = 0;
    uint64_t np = 1;
    while (k + 1 <= sp->n - 1 && np * (uint64_t)sp->m <= agb::kPrefixMax) np *= (uint64_t)sp->m, ++k;
    uint64_t mk = 1;
    for (int a = k; a < sp->n; ++a) mk *= (uint64_t)sp->m;
    A.k = k;
    A.mk = (uint32_t)mk;  // <= M^N <= 2^32 (gpu_ok); M^N == 2^32 needs k >= 1
    A.div_mk = mk > 1 ? (~0ULL) / mk + 1 : 0;
    if (mk <= 1) return fail(AG_ERR_INTERNAL, "prefix table covers every digit");
    if (sp->n - k > 16) return fail(AG_ERR_INTERNAL, "more than 16 digits outside the prefix table");
  }
  uint64_t n_pre = 1;
  for (int a = 0; a < A.k; ++a) n_pre *= (uint64_t)sp->m;
  int rc;
  const size_t tbytes = (size_t)T * 16 + (size_t)(R + 1) * 4 + (size_t)T * sizeof(agb::Key) + 64;
  if ((rc = ctx->cost_args.ensure(sizeof(A))) || (rc = ctx->cost_status.ensure(tbytes)) ||
      (rc = ctx->cost_prefix.ensure(16 * n_pre)))
    return rc;
  A.prefix = (const double2*)ctx->cost_prefix.p;
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
    agb::k_cost_prefix<<<(unsigned)((n_pre + 255) / 256), 256, 0, st>>>(dA, n_pre, (double2*)ctx->cost_prefix.p);
  }
  {
    agb::Launch L(ctx, agb::K_COST_ARGMIN);
    const dim3 g((T + agb::kCostWarps - 1) / agb::kCostWarps), b(agb::kCostWarps * 32);
    switch (sp->n - A.k) {
      case 1: agb::k_cost_tasks<1><<<g, b, 0, st>>>(dA); break;
      case 2: agb::k_cost_tasks<2><<<g, b, 0, st>>>(dA); break;
      case 3: agb::k_cost_tasks<3><<<g, b, 0, st>>>(dA); break;
      case 4: agb::k_cost_tasks<4><<<g, b, 0, st>>>(dA); break;
      default: agb::k_cost_tasks<0><<<g, b, 0, st>>>(dA); break;
    }
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
