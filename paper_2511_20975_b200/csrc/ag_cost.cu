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

#include <algorithm>
#include <cmath>
#include <vector>

#include "ag_internal.h"

namespace agb {
namespace {

constexpr int kCostWarps = 8;
// members per task: a power of two from kTask up to kTaskMax, the largest
// that still leaves about kTaskTarget tasks (2^15 members at config 4,
// 2^11 at config 3; the fixed-size sweep is in DESIGN.md §5)
constexpr uint64_t kTask = 1 << 11;
constexpr uint64_t kTaskMax = 1 << 16;
constexpr uint64_t kTaskTarget = 1 << 15;
constexpr int kPlanSmemReq = 24 * 1024;  // requests whose offsets the plan stages in shared memory
constexpr uint64_t kTaskCap = 1 << 20;  // tasks per call beyond one per request
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
  const uint64_t* offsets;      // [R+1] member CSR
  int kind;                     // 0 static, 1 runtime
  double term[kMaxModels + 1];  // per-tier estimate term (NaN: tier missing)
  double cost[kMaxModels + 1];
  Key* task_best;               // [tasks]
  int R;
  int32_t* r_task;              // [R+1] task range per request (k_cost_plan)
  uint64_t* tsize;              // members per task (k_cost_plan)
  int32_t* t_req;               // [tasks] request of each task (k_cost_plan)
  uint64_t* rec;                // [R][4] shard records (ag_shard_records) or null
  uint32_t m_magic;             // ceil(2^32 / M): exact x / M for x < 2^32 / M (suffix digits)
  int any_missing;              // some tier's estimate term is NaN (a missing tier)
  int allow_empty;              // shard records: an empty shard is not an error
  uint32_t* chosen;
  double* est;
  int32_t* status;
  int k;                        // digits folded into the prefix table
  uint32_t mk;                  // M^(N-k): members per prefix
  uint64_t div_mk;              // ceil(2^64 / mk)
  const double2* prefix;        // [M^k] (e, c) after agents 0..k-1
};

// Stage 0: prefix folds (estimate_completion / static_cost, left to right)
__global__ void __launch_bounds__(256) k_cost_prefix(const __grid_constant__ CostArgs A, uint64_t n_pre,
                                                     double2* __restrict__ out) {
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

// The task plan on the device (no host round trip): request r owns tasks
// [r_task[r], r_task[r+1]), one per tsize members (see kTask; more when the
// batch holds over kTaskCap * tsize members, so at most R + kTaskCap tasks);
// an empty set latches "accurate set is empty" (workload.cpp:151-156) and
// gets no task.
__global__ void __launch_bounds__(1024) k_cost_plan(const __grid_constant__ CostArgs A) {
  __shared__ int32_t s_wsum[32];
  extern __shared__ uint64_t s_off[];  // [R+1] when R < kPlanSmemReq
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const bool staged = A.R < kPlanSmemReq;
  if (staged)
    for (int i = tid; i <= A.R; i += 1024) s_off[i] = A.offsets[i];  // coalesced
  __syncthreads();
  auto off = [&](int i) -> uint64_t { return staged ? s_off[i] : A.offsets[i]; };
  // tasks of ts members, ts a power of two >= total / kTaskCap
  const uint64_t total = off(A.R) - off(0);
  const uint64_t tq = (total + kTaskCap - 1) / kTaskCap;
  uint64_t ts = kTask;
  while (ts < kTaskMax && total / (2 * ts) >= kTaskTarget) ts <<= 1;
  while (ts < tq) ts <<= 1;
  const int sh = __ffsll((long long)ts) - 1;
  if (tid == 0) *A.tsize = ts;
  // thread tid plans the contiguous requests [r0, r1): one pass, one scan
  const int per = (A.R + 1023) / 1024;
  const int r0 = min(A.R, tid * per), r1 = min(A.R, r0 + per);
  int32_t mine = 0;
  for (int r = r0; r < r1; ++r) {
    const uint64_t len = off(r + 1) - off(r);
    if (len == 0 && !A.allow_empty) atomicOr(A.status, 2);
    mine += (int32_t)((len + ts - 1) >> sh);
  }
  int32_t x = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    const int32_t v = s_wsum[lane];
    int32_t z = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    s_wsum[lane] = z - v;
    if (lane == 31) A.r_task[A.R] = z;
  }
  __syncthreads();
  int32_t acc = s_wsum[w] + x - mine;
  for (int r = r0; r < r1; ++r) {
    A.r_task[r] = acc;
    const int32_t nt = (int32_t)((off(r + 1) - off(r) + ts - 1) >> sh);
    for (int32_t k = 0; k < nt; ++k) A.t_req[acc + k] = r;
    acc += nt;
  }
}

// SFX = N - k suffix digits per member (1..4 specialised; 0 = runtime, <= 16:
// M^N <= 2^32 and M^k <= kPrefixMax leave at most 16).
template <int SFX>
__global__ void __launch_bounds__(kCostWarps * 32) k_cost_tasks(const __grid_constant__ CostArgs A) {
  // per tier: (estimate term, static cost), one 16-byte load per digit
  __shared__ double2 s_tc[kMaxModels + 1];
  const int m_ = A.sp.m;
  for (int i = threadIdx.x; i < m_; i += blockDim.x) s_tc[i] = make_double2(A.term[i], A.cost[i]);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int n_tasks = A.r_task[A.R];
  const uint64_t ts = *A.tsize;
  const int sfx = SFX > 0 ? SFX : A.sp.n - A.k;
  const uint32_t m = (uint32_t)m_, mk = A.mk, mg = A.m_magic;
  const uint64_t div_mk = A.div_mk;
  const double2* __restrict__ prefix = A.prefix;
  const bool runtime = A.kind != 0, check_nan = A.any_missing != 0;
  // persistent warps over the tasks (their number is only known on the device)
  for (int t = blockIdx.x * kCostWarps + (threadIdx.x >> 5); t < n_tasks; t += gridDim.x * kCostWarps) {
  const int r = A.t_req[t];  // the task's request
  const uint64_t b0 = A.offsets[r] + (uint64_t)(t - A.r_task[r]) * ts;
  const uint64_t rest = A.offsets[r + 1] - b0;
  const uint32_t len = (uint32_t)(rest < ts ? rest : ts);
  const uint32_t* mem = A.members + b0;
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
      // suffix digits, last first: x < mk <= 2^32 / M, so x / M is one
      // 32-bit high multiply (mg = ceil(2^32 / M) is exact below 2^32 / M)
      uint32_t x = idx[u] - q[u] * mk;
      uint32_t d[SFX > 0 ? SFX : 16];
#pragma unroll
      for (int a = (SFX > 0 ? SFX : 16) - 1; a >= 0; --a) {
        if (SFX == 0 && a >= sfx) continue;
        const uint32_t qq = a > 0 ? __umulhi(x, mg) : 0u;
        d[a] = x - qq * m;
        x = qq;
      }
      // the folds continue from the prefix, agent order, no contraction
      double e = pre[u].x, c = pre[u].y;
#pragma unroll
      for (int a = 0; a < (SFX > 0 ? SFX : 16); ++a) {
        if (SFX == 0 && a >= sfx) break;
        const double2 tc = s_tc[d[a]];
        e = __dadd_rn(e, tc.x);
        c = __dadd_rn(c, tc.y);
      }
      if (check_nan) missing |= isnan(e);  // a NaN term (missing tier) anywhere in the fold
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
  if (check_nan && __any_sync(0xffffffffu, missing) && lane == 0) atomicOr(A.status, 1);
  if (lane == 0) A.task_best[t] = Key{be, bc, bi};
  }
}

__global__ void __launch_bounds__(kCostWarps * 32) k_cost_reduce(const __grid_constant__ CostArgs A) {
  // few requests (deep spaces: thousands of tasks each): one block per
  // request and a block reduction; many requests: one warp per request
  __shared__ Key s_k[kCostWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool per_block = A.R <= 1024;
  const int r = per_block ? (int)blockIdx.x : (int)blockIdx.x * kCostWarps + wid;
  if (!per_block && r >= A.R) return;
  double be = INFINITY, bc = INFINITY;
  uint32_t bi = 0xffffffffu;
  const int t0 = A.r_task[r] + (per_block ? (int)threadIdx.x : lane), dt = per_block ? kCostWarps * 32 : 32;
  for (int t = t0; t < A.r_task[r + 1]; t += dt) {
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
  if (per_block) {
    if (lane == 0) s_k[wid] = Key{be, bc, bi};
    __syncthreads();
    if (wid != 0) return;
    if (lane < kCostWarps) {
      const Key k = s_k[lane];
      be = k.e, bc = k.c, bi = k.i;
    } else {
      be = INFINITY, bc = INFINITY, bi = 0xffffffffu;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double oe = __shfl_xor_sync(0xffffffffu, be, o);
      const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
      const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (key_less(oe, oc, oi, be, bc, bi)) be = oe, bc = oc, bi = oi;
    }
  }
  if (lane == 0) {
    if (A.chosen) A.chosen[r] = bi;
    if (A.est) A.est[r] = be;
    if (A.rec) {
      // {count, estimate, static cost, index}; an empty shard carries +inf keys
      const uint64_t cnt = A.offsets[r + 1] - A.offsets[r];
      A.rec[4 * r] = cnt;
      A.rec[4 * r + 1] = (uint64_t)__double_as_longlong(cnt ? be : INFINITY);
      A.rec[4 * r + 2] = (uint64_t)__double_as_longlong(cnt ? bc : INFINITY);
      A.rec[4 * r + 3] = cnt ? (uint64_t)bi : ~0ULL;
    }
  }
}

// Merge of the all-gathered shard records [world][R][4] (rank order is
// canonical order): per request the global member count, the members of the
// shards before `rank` (this rank's global offset into the request's list),
// and the lexicographic minimum of (estimate, static cost, index) over the
// non-empty shards -- the whole-space select_per_input_config choice
// (workload.cpp:149-176), since the minimum of shard minima is the minimum.
__global__ void __launch_bounds__(256) k_merge_records(const uint64_t* __restrict__ g, int world, int rank, int R,
                                                       uint64_t* total, uint64_t* before, uint64_t* best_idx,
                                                       double* best_est, double* best_cost) {
  const int r = blockIdx.x * 256 + threadIdx.x;
  if (r >= R) return;
  uint64_t tot = 0, bef = 0, bi = ~0ULL;
  double be = INFINITY, bc = INFINITY;
  for (int w = 0; w < world; ++w) {
    const uint64_t* x = g + ((size_t)w * R + r) * 4;
    const uint64_t cnt = x[0];
    if (w < rank) bef += cnt;
    tot += cnt;
    if (!cnt) continue;
    const double e = __longlong_as_double((long long)x[1]), c = __longlong_as_double((long long)x[2]);
    const uint64_t i = x[3];
    if (e < be || (e == be && (c < bc || (c == bc && i < bi)))) be = e, bc = c, bi = i;
  }
  if (total) total[r] = tot;
  if (before) before[r] = bef;
  if (best_idx) best_idx[r] = bi;
  if (best_est) best_est[r] = be;
  if (best_cost) best_cost[r] = bc;
}

// ---- argmin straight from the verdict bitmap (no member list) --------------
// The key's primary term p (the estimate; the static cost for the static
// policy) is a left fold of per-tier terms, and round-to-nearest addition is
// monotone in each operand, so lb[q] = fold(p of prefix q, tmin, ..., tmin)
// is a lower bound of p over every configuration under prefix q.  Exact keys
// of sampled members (the first of every run of words) give a per-request
// threshold T = the p of an actual member; only the members of words whose
// prefix bound is <= T are re-costed, exactly.  A member that is skipped has
// p > T >= the optimum's p, so the result is the exact minimum of
// (p, static cost, index) over the set -- the same choice as k_cost_tasks --
// and the bitmap (1/8 B per configuration) is read once instead of the
// member list (4 B per member).
// The prefix level k is chosen so that a 32-bit word spans at most two
// prefixes (M^(N-k) >= 32).
//
// Words per warp task: a power of two between kBmTaskMin and kBmTaskMax
// chosen per call so that the batch is about kBmTasksTarget tasks -- long
// tasks amortise the per-task start (a deep space: 2,048 words at config 4),
// short ones spread a batch of small rows over more warps (256 at config 3)
constexpr uint32_t kBmTaskMin = 256, kBmTaskMax = 4096;
constexpr uint64_t kBmTasksTarget = 1 << 16;
#ifndef AG_BM_MINB
#define AG_BM_MINB 3
#endif
#ifndef AG_BM_L2PF
#define AG_BM_L2PF 0
#endif
#ifndef AG_BM_RUN
#define AG_BM_RUN 8
#endif
constexpr int kBmRun = AG_BM_RUN;   // consecutive words per lane per step (a multiple of 4)
constexpr int kBmSampleSteps = 2;   // steps of a task that sample exact keys (T is shared after)

struct BmArgs {
  SpaceDev sp;
  const uint32_t* bitmap;  // [R][W]
  const uint64_t* counts;  // [R]
  uint64_t begin, end;
  uint32_t W, n_pre;
  uint32_t task_words;      // words per warp task (a multiple of 32 * kBmRun)
  int vec;                 // rows 16-byte aligned (vector loads)
  int R, tpr;              // tasks per request
  int kind, any_missing, allow_empty;
  double term[kMaxModels + 1];
  double cost[kMaxModels + 1];
  double tmin;             // min over tiers of the primary term
  uint64_t pw_magic[kMaxAgents];  // ceil(2^64 / M^(k-1-a)); 0 for M^0
  int k;
  uint32_t mk, m_magic;
  uint64_t div_mk;
  double2* prefix;         // [M^k] (e, c) after agents 0..k-1
  double* lb;              // [M^k] lower bound of p under the prefix
  uint64_t* thr;           // [R] order-preserving bits of T
  Key* task_best;          // [R * tpr]
  uint32_t* chosen;
  double* est;
  uint64_t* rec;
  int32_t* status;
  uint32_t* stats;         // optional [2]: words evaluated, members evaluated
};

__device__ __forceinline__ uint64_t ord_bits(double x) {
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_double(uint64_t o) {
  return __longlong_as_double((long long)((o >> 63) ? (o & 0x7fffffffffffffffull) : ~o));
}

// prefix folds + lower bounds; also initialises the thresholds to +inf
__global__ void __launch_bounds__(256) k_bm_prefix(const __grid_constant__ BmArgs A, uint64_t n_pre) {
  __shared__ double2 s_tc[kMaxModels + 1];
  for (int i = threadIdx.x; i < A.sp.m; i += blockDim.x) s_tc[i] = make_double2(A.term[i], A.cost[i]);
  __syncthreads();
  const uint64_t q = (uint64_t)blockIdx.x * 256 + threadIdx.x;
  if (q < (uint64_t)A.R) A.thr[q] = ord_bits(INFINITY);
  if (q >= n_pre) return;
  const uint32_t m = (uint32_t)A.sp.m;
  // digits most significant first (q / M^(k-1-a), then mod M), folded in
  // agent order: the same adds as estimate_completion's
  double e = 0.0, c = 0.0;
  for (int a = 0; a < A.k; ++a) {
    const uint32_t y = A.pw_magic[a] ? divm((uint32_t)q, A.pw_magic[a]) : (uint32_t)q;
    const double2 tc = s_tc[y - divm(y, A.sp.div_m) * m];
    e = __dadd_rn(e, tc.x);
    c = __dadd_rn(c, tc.y);
  }
  A.prefix[q] = make_double2(e, c);
  double p = A.kind != 0 ? e : c;
  for (int a = A.k; a < A.sp.n; ++a) p = __dadd_rn(p, A.tmin);
  A.lb[q] = p;
}

// exact (e, c) of canonical index idx = q * mk + x (x < mk)
template <int SFX>
__device__ __forceinline__ void bm_key(const BmArgs& A, const double2* s_tc, uint32_t q, uint32_t x, double& e,
                                       double& c) {
  const uint32_t m = (uint32_t)A.sp.m;
  const int sfx = SFX > 0 ? SFX : A.sp.n - A.k;
  uint32_t d[SFX > 0 ? SFX : 16];
#pragma unroll
  for (int a = (SFX > 0 ? SFX : 16) - 1; a >= 0; --a) {
    if (SFX == 0 && a >= sfx) continue;
    const uint32_t qq = a > 0 ? __umulhi(x, A.m_magic) : 0u;
    d[a] = x - qq * m;
    x = qq;
  }
  const double2 pre = A.prefix[q];
  e = pre.x, c = pre.y;
#pragma unroll
  for (int a = 0; a < (SFX > 0 ? SFX : 16); ++a) {
    if (SFX == 0 && a >= sfx) break;
    const double2 tc = s_tc[d[a]];
    e = __dadd_rn(e, tc.x);
    c = __dadd_rn(c, tc.y);
  }
}

// One pass: a warp takes runs of kBmRun consecutive words per lane (256
// words per step).  Per step each lane re-costs the first member of its run
// exactly; the warp minimum tightens the request's threshold T (published by
// an atomic on order-preserving bits, read back by every step of every warp:
// any member's p bounds the optimum, so every value seen is a valid T).  A
// word then qualifies when one of its (at most two) prefixes has lb <= T, and
// qualifying words are re-costed bit-parallel (lane j = bit j), exactly.
template <int SFX>
__global__ void __launch_bounds__(kCostWarps * 32, AG_BM_MINB) k_bm_eval(const __grid_constant__ BmArgs A) {
  __shared__ double2 s_tc[kMaxModels + 1];
  __shared__ uint2 s_q[kCostWarps][32 * kBmRun];  // per warp: qualifying (word, word index)
  for (int i = threadIdx.x; i < A.sp.m; i += blockDim.x) s_tc[i] = make_double2(A.term[i], A.cost[i]);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int t = blockIdx.x * kCostWarps + wid;
  if (t >= A.R * A.tpr) return;
  const int r = t / A.tpr;
  const uint32_t w0 = (uint32_t)(t - r * A.tpr) * A.task_words, w1 = min(A.W, w0 + A.task_words);
  const uint32_t* row = A.bitmap + (size_t)r * A.W;
  const bool runtime = A.kind != 0, check_nan = A.any_missing != 0;
  const uint32_t mk = A.mk;
  const double* __restrict__ lb = A.lb;
  uint2* q_ = s_q[wid];
  double T = INFINITY;  // stays +inf with a missing tier: every member is checked
  double be = INFINITY, bc = INFINITY;
  uint32_t bi = 0xffffffffu;
  bool missing = false;
  uint32_t n_words = 0;
  auto load_run = [&](uint32_t sub, uint32_t(&v)[kBmRun]) {
    const uint32_t ws = sub + kBmRun * lane;
    // streaming (evict-first) loads: the bitmap is read once and must not
    // push the prefix tables out of L2
    if (A.vec && ws + kBmRun <= w1) {  // 16-byte aligned rows: vector loads
#pragma unroll
      for (int h = 0; h < kBmRun / 4; ++h) {
        const uint4 a = __ldcs((const uint4*)(row + ws + 4 * h));
        v[4 * h] = a.x, v[4 * h + 1] = a.y, v[4 * h + 2] = a.z, v[4 * h + 3] = a.w;
      }
    } else {
#pragma unroll
      for (int u = 0; u < kBmRun; ++u) v[u] = ws + u < w1 ? __ldcs(row + ws + u) : 0u;
    }
  };
  // the next step's words, shared threshold and first two prefix bounds are
  // loaded one step ahead (the threshold through L2: a stale value is still
  // a valid bound)
  auto run_q = [&](uint32_t sub) {
    return (uint32_t)__umul64hi(A.begin + 32ull * (sub + kBmRun * lane), A.div_mk);
  };
  const uint32_t qmax = A.n_pre - 1;
#if AG_BM_L2PF
  if (lane == 0 && A.vec) {  // the whole task toward L2 in one bulk prefetch
    const uint32_t bytes = ((w1 - w0) * 4u) & ~15u;
    if (bytes)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(row + w0), "r"(bytes) : "memory");
  }
#endif
  uint32_t v[kBmRun], vn[kBmRun];
  load_run(w0, v);
  uint64_t tn = __ldcg((const unsigned long long*)(A.thr + r));
  uint32_t qn = min(run_q(w0), qmax);
  double lbn0 = lb[qn], lbn1 = lb[min(qn + 1, qmax)];
  int step = 0;  // non-empty steps so far (the first kBmSampleSteps sample)
  for (uint32_t sub = w0; sub < w1; sub += 32 * kBmRun) {
    const uint64_t tcur = tn;
    const double lb0 = lbn0, lb1 = lbn1;
    if (sub + 32 * kBmRun < w1) {  // next run in flight
      load_run(sub + 32 * kBmRun, vn);
      tn = __ldcg((const unsigned long long*)(A.thr + r));
      qn = min(run_q(sub + 32 * kBmRun), qmax);
      lbn0 = lb[qn], lbn1 = lb[min(qn + 1, qmax)];
    }
    const uint32_t ws = sub + kBmRun * lane;
    if (sub + 32 * kBmRun >= A.W) {  // the row's last word: bits past `end` are not members
      const uint64_t tail = (A.end - A.begin) - 32ull * (A.W - 1);
#pragma unroll
      for (int u = 0; u < kBmRun; ++u)
        if (ws + u == A.W - 1 && tail < 32) v[u] &= (1u << tail) - 1u;
    }
    const uint64_t base = A.begin + 32ull * ws;
    uint32_t any = 0;
#pragma unroll
    for (int u = 0; u < kBmRun; ++u) any |= v[u];
    if (!__any_sync(0xffffffffu, any != 0)) {  // an empty step (most of a sparse row)
#pragma unroll
      for (int u = 0; u < kBmRun; ++u) v[u] = vn[u];
      continue;
    }
    if (!check_nan) {
      if (step++ < kBmSampleSteps) {
        // the run's first member, exactly
        uint32_t fv = 0, fu = 0;
#pragma unroll
        for (int u = kBmRun - 1; u >= 0; --u)
          if (v[u]) fv = v[u], fu = (uint32_t)u;
        double ps = INFINITY;
        if (fv) {
          const uint64_t idx = base + 32u * fu + (uint32_t)(__ffs(fv) - 1);
          const uint32_t q = (uint32_t)__umul64hi(idx, A.div_mk);
          double e, c;
          bm_key<SFX>(A, s_tc, q, (uint32_t)(idx - (uint64_t)q * mk), e, c);
          ps = runtime ? e : c;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ps = fmin(ps, __shfl_xor_sync(0xffffffffu, ps, o));
        const double tg = ord_double(tcur);
        if (ps < tg && lane == 0) atomicMin((unsigned long long*)(A.thr + r), (unsigned long long)ord_bits(ps));
        T = fmin(T, fmin(ps, tg));
      } else {
        T = fmin(T, ord_double(tcur));
      }
    }
    // the run's prefixes first: most runs have none with lb <= T
    uint32_t q = (uint32_t)__umul64hi(base, A.div_mk);
    bool alive = false;
    if (any) {
      const uint32_t qe = min((uint32_t)__umul64hi(base + 32 * kBmRun - 1, A.div_mk), qmax);
      alive = !(lb0 > T) || (qe > q && !(lb1 > T));
      for (uint32_t qq = q + 2; qq <= qe; ++qq) alive |= !(lb[qq] > T);
    }
    // qualifying words of a live run (prefix q below split, q + 1 above) go
    // to the warp's queue
    uint32_t qmask = 0;
    if (alive) {
      uint32_t rr = (uint32_t)(base - (uint64_t)q * mk);
#pragma unroll
      for (int u = 0; u < kBmRun; ++u) {
        const uint32_t split = mk - rr;
        const uint32_t lo = split >= 32 ? 0xffffffffu : (1u << split) - 1u;
        const bool qual = ((v[u] & lo) && !(lb[q] > T)) || ((v[u] & ~lo) && !(lb[q + 1] > T));
        qmask |= (qual ? 1u : 0u) << u;
        rr += 32;
        if (rr >= mk) rr -= mk, ++q;  // mk >= 32 whenever a run has a second word
      }
    }
    if (!__any_sync(0xffffffffu, qmask != 0)) {
#pragma unroll
      for (int u = 0; u < kBmRun; ++u) v[u] = vn[u];
      continue;
    }
    const int nq = __popc(qmask);
    int incl = nq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total) {
      int pos = incl - nq;
#pragma unroll
      for (int u = 0; u < kBmRun; ++u)
        if ((qmask >> u) & 1u) q_[pos++] = make_uint2(v[u], ws + (uint32_t)u);
      __syncwarp();
      n_words += (uint32_t)total;
      // lane j re-costs bit j of four queued words at a time (four
      // independent folds in flight); an unset bit re-costs the word's first
      // index and is not compared
      for (int i = 0; i < total; i += 4) {
        double e[4], c[4];
        uint32_t idx[4];
        bool on[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint2 wd = i + k < total ? q_[i + k] : make_uint2(0u, q_[i].y);
          on[k] = (wd.x >> lane) & 1u;
          const uint64_t ix = A.begin + 32ull * wd.y + (on[k] ? (uint32_t)lane : 0u);
          idx[k] = (uint32_t)ix;
          const uint32_t qi = (uint32_t)__umul64hi(ix, A.div_mk);
          bm_key<SFX>(A, s_tc, qi, (uint32_t)(ix - (uint64_t)qi * mk), e[k], c[k]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (!on[k]) continue;
          if (check_nan) missing |= isnan(e[k]);
          const double ek = runtime ? e[k] : 0.0;
          if (key_less(ek, c[k], idx[k], be, bc, bi)) be = ek, bc = c[k], bi = idx[k];
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int u = 0; u < kBmRun; ++u) v[u] = vn[u];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double oe = __shfl_xor_sync(0xffffffffu, be, o);
    const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (key_less(oe, oc, oi, be, bc, bi)) be = oe, bc = oc, bi = oi;
  }
  if (check_nan && __any_sync(0xffffffffu, missing) && lane == 0) atomicOr(A.status, 1);
  if (lane == 0) {
    A.task_best[t] = Key{be, bc, bi};
    if (A.stats) atomicAdd(A.stats, n_words);
  }
}

// per request: the minimum over its tasks; outputs as k_cost_reduce
__global__ void __launch_bounds__(kCostWarps * 32) k_bm_reduce(const __grid_constant__ BmArgs A) {
  // few requests (thousands of tasks each): a block per request; many: a warp
  __shared__ Key s_k[kCostWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool per_block = A.R <= 1024;
  const int r = per_block ? (int)blockIdx.x : (int)blockIdx.x * kCostWarps + wid;
  if (!per_block && r >= A.R) return;
  double be = INFINITY, bc = INFINITY;
  uint32_t bi = 0xffffffffu;
  const int dt = per_block ? kCostWarps * 32 : 32;
  for (int t = r * A.tpr + (per_block ? (int)threadIdx.x : lane); t < (r + 1) * A.tpr; t += dt) {
    const Key k = A.task_best[t];
    if (key_less(k.e, k.c, k.i, be, bc, bi)) be = k.e, bc = k.c, bi = k.i;
  }
  auto warp_min = [&]() {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double oe = __shfl_xor_sync(0xffffffffu, be, o);
      const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
      const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (key_less(oe, oc, oi, be, bc, bi)) be = oe, bc = oc, bi = oi;
    }
  };
  warp_min();
  if (per_block) {
    if (lane == 0) s_k[wid] = Key{be, bc, bi};
    __syncthreads();
    if (wid != 0) return;
    const Key k = lane < kCostWarps ? s_k[lane] : Key{INFINITY, INFINITY, 0xffffffffu};
    be = k.e, bc = k.c, bi = k.i;
    warp_min();
  }
  if (lane != 0) return;
  const uint64_t cnt = A.counts[r];
  if (cnt == 0 && !A.allow_empty) atomicOr(A.status, 2);
  if (A.chosen) A.chosen[r] = bi;
  if (A.est) A.est[r] = be;
  if (A.rec) {
    A.rec[4 * r] = cnt;
    A.rec[4 * r + 1] = (uint64_t)__double_as_longlong(cnt ? be : INFINITY);
    A.rec[4 * r + 2] = (uint64_t)__double_as_longlong(cnt ? bc : INFINITY);
    A.rec[4 * r + 3] = cnt ? (uint64_t)bi : ~0ULL;
  }
}

}  // namespace
}  // namespace agb

using agb::fail;

namespace agb {
namespace {

// select_per_input_config over a member CSR, asynchronous: the chosen index /
// estimate per request, or (rec) the 32-byte shard record per request
int select_impl(ag_ctx* ctx, const uint32_t* members, const uint64_t* offsets, int32_t n_requests,
                int32_t kind, const ag_load* load, uint32_t* chosen, double* est, uint64_t* rec) {
  if (!ctx || !members || !offsets || (!chosen && !rec)) return fail(AG_ERR_VALIDATION, "null argument");
  if (kind != AG_POLICY_PER_INPUT_STATIC && kind != AG_POLICY_PER_INPUT_RUNTIME_COST)
    return fail(AG_ERR_VALIDATION, "per-input selection needs a per-input policy kind");
  if (kind == AG_POLICY_PER_INPUT_RUNTIME_COST && !load)
    return fail(AG_ERR_VALIDATION, "runtime-cost selection needs a load context");
  const ag_space* sp = ctx->space;
  if (!sp->gpu_ok) return fail(AG_ERR_VALIDATION, "GPU path needs M^N < 2^32 and N <= 32");
  if (n_requests <= 0) return n_requests == 0 ? AG_OK : fail(AG_ERR_VALIDATION, "negative request count");
  cudaStream_t st = ctx->stream;
  const int R = n_requests;
  agb::CostArgs A;
  A.sp = sp->dev();
  A.members = members;
  A.offsets = offsets;
  A.kind = kind == AG_POLICY_PER_INPUT_RUNTIME_COST ? 1 : 0;
  for (int i = 0; i <= agb::kMaxModels; ++i) {
    A.term[i] = 0.0;
    A.cost[i] = i < sp->m ? sp->cost[i] : 0.0;
  }
  A.m_magic = (uint32_t)((0x100000000ull + (uint64_t)sp->m - 1) / (uint64_t)sp->m);
  A.any_missing = 0;
  if (A.kind == 1) {
    // estimate_completion (workload.cpp:129-147)
    if (load->n_tiers < 0) return fail(AG_ERR_VALIDATION, "estimator context arrays disagree on tier count");
    for (int i = 0; i < sp->m; ++i) {
      if (i >= load->n_tiers || load->slots[i] <= 0) {
        A.term[i] = NAN;  // an error only if a member uses the tier
        A.any_missing = 1;
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
  A.rec = rec;
  A.allow_empty = rec != nullptr;
  // prefix table: the largest k <= N - 1 with M^k <= kPrefixMax
  {
    int k = 0;
    uint64_t np = 1;
    while (k + 1 <= sp->n - 1 && np * (uint64_t)sp->m <= agb::kPrefixMax) np *= (uint64_t)sp->m, ++k;
    uint64_t mk = 1;
    for (int a = k; a < sp->n; ++a) mk *= (uint64_t)sp->m;
    A.k = k;
    A.mk = (uint32_t)mk;  // <= M^N < 2^32 (gpu_ok)
    A.div_mk = mk > 1 ? (~0ULL) / mk + 1 : 0;
    if (mk <= 1) return fail(AG_ERR_INTERNAL, "prefix table covers every digit");
    if (sp->n - k > 16) return fail(AG_ERR_INTERNAL, "more than 16 digits outside the prefix table");
  }
  uint64_t n_pre = 1;
  for (int a = 0; a < A.k; ++a) n_pre *= (uint64_t)sp->m;
  // task bests: at most R + kTaskCap tasks (k_cost_plan sizes the tasks)
  int rc;
  const size_t tcap = (size_t)R + agb::kTaskCap;
  if (!ctx->async_status.p) {
    if ((rc = ctx->async_status.ensure(16))) return rc;
    AG_CUDA(cudaMemsetAsync(ctx->async_status.p, 0, 16, st));
  }
  const size_t rt_bytes = (((size_t)(R + 1) * 4 + 15) & ~(size_t)15) + 16;
  if ((rc = ctx->cost_status.ensure(rt_bytes + 4 * tcap)) ||
      (rc = ctx->cost_tasks.ensure(tcap * sizeof(agb::Key))) || (rc = ctx->cost_prefix.ensure(16 * n_pre)))
    return rc;
  A.prefix = (const double2*)ctx->cost_prefix.p;
  A.status = (int32_t*)ctx->async_status.p;
  A.r_task = (int32_t*)ctx->cost_status.p;
  A.tsize = (uint64_t*)((char*)ctx->cost_status.p + (((size_t)(R + 1) * 4 + 15) & ~(size_t)15));
  A.t_req = (int32_t*)((char*)ctx->cost_status.p + rt_bytes);
  A.task_best = (agb::Key*)ctx->cost_tasks.p;
  {
    agb::Launch L(ctx, agb::K_COST_ARGMIN);
    const size_t psm = R < agb::kPlanSmemReq ? 8 * ((size_t)R + 1) : 0;
    if (psm > 48 * 1024 && !ctx->cost_plan_attr) {
      AG_CUDA(cudaFuncSetAttribute(agb::k_cost_plan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   8 * agb::kPlanSmemReq));
      ctx->cost_plan_attr = true;
    }
    agb::k_cost_plan<<<1, 1024, psm, st>>>(A);
  }
  {
    agb::Launch L(ctx, agb::K_COST_ARGMIN);
    agb::k_cost_prefix<<<(unsigned)((n_pre + 255) / 256), 256, 0, st>>>(A, n_pre, (double2*)ctx->cost_prefix.p);
  }
  {
    agb::Launch L(ctx, agb::K_COST_ARGMIN);
    // grid = the resident capacity of the variant launched (occupancy differs
    // by suffix length: the generic variant keeps 16 digits in registers)
    const int sfx = sp->n - A.k;
    const int vi = sfx >= 1 && sfx <= 4 ? sfx : 0;
    if (!ctx->cost_grid[vi]) {
      static void (*const fns[5])(agb::CostArgs) = {agb::k_cost_tasks<0>, agb::k_cost_tasks<1>, agb::k_cost_tasks<2>,
                                                   agb::k_cost_tasks<3>, agb::k_cost_tasks<4>};
      int sms = 0, per_sm = 0;
      AG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
      AG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fns[vi], agb::kCostWarps * 32, 0));
      ctx->cost_grid[vi] = std::max(1, sms * per_sm);
    }
    const dim3 g(ctx->cost_grid[vi]), b(agb::kCostWarps * 32);
    switch (vi) {
      case 1: agb::k_cost_tasks<1><<<g, b, 0, st>>>(A); break;
      case 2: agb::k_cost_tasks<2><<<g, b, 0, st>>>(A); break;
      case 3: agb::k_cost_tasks<3><<<g, b, 0, st>>>(A); break;
      case 4: agb::k_cost_tasks<4><<<g, b, 0, st>>>(A); break;
      default: agb::k_cost_tasks<0><<<g, b, 0, st>>>(A); break;
    }
  }
  {
    agb::Launch L(ctx, agb::K_COST_ARGMIN);
    const unsigned rb = R <= 1024 ? (unsigned)R : (unsigned)((R + agb::kCostWarps - 1) / agb::kCostWarps);
    agb::k_cost_reduce<<<rb, agb::kCostWarps * 32, 0, st>>>(A);
  }
  AG_CUDA(cudaGetLastError());
  return AG_OK;
}

int select_bitmap_impl(ag_ctx* ctx, const uint32_t* bitmap, const uint64_t* counts, uint64_t begin, uint64_t end,
                       int32_t n_requests, int32_t kind, const ag_load* load, uint32_t* chosen, double* est,
                       uint64_t* rec) {
  if (!ctx || !bitmap || !counts || (!chosen && !rec)) return fail(AG_ERR_VALIDATION, "null argument");
  if (kind != AG_POLICY_PER_INPUT_STATIC && kind != AG_POLICY_PER_INPUT_RUNTIME_COST)
    return fail(AG_ERR_VALIDATION, "per-input selection needs a per-input policy kind");
  if (kind == AG_POLICY_PER_INPUT_RUNTIME_COST && !load)
    return fail(AG_ERR_VALIDATION, "runtime-cost selection needs a load context");
  const ag_space* sp = ctx->space;
  if (!sp->gpu_ok) return fail(AG_ERR_VALIDATION, "GPU path needs M^N < 2^32 and N <= 32");
  if (begin > end || end > sp->size) return fail(AG_ERR_VALIDATION, "configuration index out of range");
  if (n_requests <= 0) return n_requests == 0 ? AG_OK : fail(AG_ERR_VALIDATION, "negative request count");
  cudaStream_t st = ctx->stream;
  const int R = n_requests;
  BmArgs A;
  A.sp = sp->dev();
  A.bitmap = bitmap;
  A.counts = counts;
  A.begin = begin;
  A.end = end;
  const uint64_t W = (end - begin + 31) / 32;
  A.W = (uint32_t)W;
  {
    uint32_t tw = kBmTaskMin;
    while (tw < kBmTaskMax && (uint64_t)R * W / (2 * tw) >= kBmTasksTarget) tw *= 2;
    A.task_words = tw;
  }
  A.tpr = (int)std::max<uint64_t>(1, (W + A.task_words - 1) / A.task_words);
  if ((uint64_t)R * (uint64_t)A.tpr >= (1ull << 31)) return fail(AG_ERR_VALIDATION, "batch too large for one launch");
  A.R = R;
  A.kind = kind == AG_POLICY_PER_INPUT_RUNTIME_COST ? 1 : 0;
  A.any_missing = 0;
  for (int i = 0; i <= kMaxModels; ++i) {
    A.term[i] = 0.0;
    A.cost[i] = i < sp->m ? sp->cost[i] : 0.0;
  }
  if (A.kind == 1) {
    // estimate_completion (workload.cpp:129-147)
    if (load->n_tiers < 0) return fail(AG_ERR_VALIDATION, "estimator context arrays disagree on tier count");
    for (int i = 0; i < sp->m; ++i) {
      if (i >= load->n_tiers || load->slots[i] <= 0) {
        A.term[i] = NAN;
        A.any_missing = 1;
        continue;
      }
      const double ld = (double)(load->occupancy[i] + load->queued_ahead[i]);
      const double mean = load->mean[i];
      A.term[i] = (ld / (double)load->slots[i]) * mean + mean;
    }
  }
  A.tmin = INFINITY;
  for (int i = 0; i < sp->m; ++i) {
    const double p = A.kind ? A.term[i] : A.cost[i];
    if (!std::isnan(p)) A.tmin = std::min(A.tmin, p);
  }
  A.allow_empty = rec != nullptr;
  A.chosen = chosen;
  A.est = est;
  A.rec = rec;
  A.m_magic = (uint32_t)((0x100000000ull + (uint64_t)sp->m - 1) / (uint64_t)sp->m);
  // prefix level: the largest k <= N - 1 with M^k <= kPrefixMax and a word
  // spanning at most two prefixes (M^(N-k) >= 32)
  int k = 0;
  uint64_t n_pre = 1;
  {
    uint64_t mk = sp->size;
    while (k + 1 <= sp->n - 1 && n_pre * (uint64_t)sp->m <= kPrefixMax && mk / (uint64_t)sp->m >= 32)
      n_pre *= (uint64_t)sp->m, mk /= (uint64_t)sp->m, ++k;
    if (sp->n - k > 16) return fail(AG_ERR_VALIDATION, "more than 16 digits outside the prefix table");
    A.k = k;
    A.mk = (uint32_t)mk;
    A.div_mk = mk > 1 ? (~0ULL) / mk + 1 : 0;
    if (mk <= 1) return fail(AG_ERR_VALIDATION, "bitmap selection needs at least two configurations");
    uint64_t pw = 1;
    for (int a = k - 1; a >= 0; --a) {
      A.pw_magic[a] = pw > 1 ? (~0ULL) / pw + 1 : 0;
      pw *= (uint64_t)sp->m;
    }
  }
  int rc;
  if (!ctx->async_status.p) {
    if ((rc = ctx->async_status.ensure(16))) return rc;
    AG_CUDA(cudaMemsetAsync(ctx->async_status.p, 0, 16, st));
  }
  const size_t ntask = (size_t)R * A.tpr;
  if ((rc = ctx->cost_prefix.ensure(16 * n_pre)) || (rc = ctx->cost_bm.ensure(8 * n_pre + 8 * (size_t)R)) ||
      (rc = ctx->cost_tasks.ensure(ntask * sizeof(Key))))
    return rc;
  A.prefix = (double2*)ctx->cost_prefix.p;
  A.lb = (double*)ctx->cost_bm.p;
  A.thr = (uint64_t*)((char*)ctx->cost_bm.p + 8 * n_pre);
  A.task_best = (Key*)ctx->cost_tasks.p;
  A.status = (int32_t*)ctx->async_status.p;
  A.n_pre = (uint32_t)n_pre;
  A.vec = (W % 4 == 0 && ((uintptr_t)bitmap & 15) == 0) ? 1 : 0;
  A.stats = ctx->bm_stats_on ? (uint32_t*)ctx->bm_stats.p : nullptr;
  const int sfx = sp->n - k;
  const int vi = sfx >= 1 && sfx <= 4 ? sfx : 0;
  {
    Launch L(ctx, K_COST_ARGMIN);
    const uint64_t nth = std::max<uint64_t>(n_pre, (uint64_t)R);
    k_bm_prefix<<<(unsigned)((nth + 255) / 256), 256, 0, st>>>(A, n_pre);
  }
  const unsigned tb = (unsigned)((ntask + kCostWarps - 1) / kCostWarps);
  {
    Launch L(ctx, K_COST_ARGMIN);
    switch (vi) {
      case 1: k_bm_eval<1><<<tb, kCostWarps * 32, 0, st>>>(A); break;
      case 2: k_bm_eval<2><<<tb, kCostWarps * 32, 0, st>>>(A); break;
      case 3: k_bm_eval<3><<<tb, kCostWarps * 32, 0, st>>>(A); break;
      case 4: k_bm_eval<4><<<tb, kCostWarps * 32, 0, st>>>(A); break;
      default: k_bm_eval<0><<<tb, kCostWarps * 32, 0, st>>>(A); break;
    }
  }
  {
    Launch L(ctx, K_COST_ARGMIN);
    const unsigned rb = R <= 1024 ? (unsigned)R : (unsigned)((R + kCostWarps - 1) / kCostWarps);
    k_bm_reduce<<<rb, kCostWarps * 32, 0, st>>>(A);
  }
  AG_CUDA(cudaGetLastError());
  return AG_OK;
}

}  // namespace
}  // namespace agb

extern "C" int ag_select_bitmap(ag_ctx* ctx, const uint32_t* bitmap, const uint64_t* counts, uint64_t begin,
                                uint64_t end, int32_t n_requests, int32_t kind, const ag_load* load,
                                uint32_t* chosen, double* est, uint64_t* records) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  return agb::select_bitmap_impl(ctx, bitmap, counts, begin, end, n_requests, kind, load, chosen, est, records);
}

extern "C" int ag_select_bitmap_stats(ag_ctx* ctx, int32_t enable, uint64_t* words_evaluated) {
  // diagnostics: count the queued words ag_select_bitmap re-costs exactly
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  if (!ctx) return fail(AG_ERR_VALIDATION, "null argument");
  if (enable) {
    if (int rc = ctx->bm_stats.ensure(8)) return rc;
    AG_CUDA(cudaMemsetAsync(ctx->bm_stats.p, 0, 8, ctx->stream));
    ctx->bm_stats_on = true;
    return AG_OK;
  }
  uint32_t v = 0;
  if (ctx->bm_stats_on) {
    AG_CUDA(cudaMemcpyAsync(&v, ctx->bm_stats.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
    AG_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->bm_stats_on = false;
  }
  if (words_evaluated) *words_evaluated = v;
  return AG_OK;
}

extern "C" int ag_select_per_input(ag_ctx* ctx, const uint32_t* members, const uint64_t* offsets,
                                   int32_t n_requests, int32_t kind, const ag_load* load,
                                   uint32_t* chosen, double* est) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  if (!chosen) return fail(AG_ERR_VALIDATION, "null argument");
  return agb::select_impl(ctx, members, offsets, n_requests, kind, load, chosen, est, nullptr);
}

extern "C" int ag_shard_records(ag_ctx* ctx, const uint32_t* members, const uint64_t* offsets,
                                int32_t n_requests, int32_t kind, const ag_load* load, uint64_t* records) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  if (!records) return fail(AG_ERR_VALIDATION, "null argument");
  return agb::select_impl(ctx, members, offsets, n_requests, kind, load, nullptr, nullptr, records);
}

extern "C" int ag_merge_records(ag_ctx* ctx, const uint64_t* gathered, int32_t world, int32_t rank,
                                int32_t n_requests, uint64_t* total, uint64_t* before, uint64_t* best_index,
                                double* best_est, double* best_cost) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  if (!ctx || !gathered) return fail(AG_ERR_VALIDATION, "null argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(AG_ERR_VALIDATION, "rank outside the world");
  if (n_requests <= 0) return n_requests == 0 ? AG_OK : fail(AG_ERR_VALIDATION, "negative request count");
  {
    agb::Launch L(ctx, agb::K_COST_ARGMIN);
    agb::k_merge_records<<<(n_requests + 255) / 256, 256, 0, ctx->stream>>>(gathered, world, rank, n_requests, total,
                                                                          before, best_index, best_est, best_cost);
  }
  AG_CUDA(cudaGetLastError());
  return AG_OK;
}
