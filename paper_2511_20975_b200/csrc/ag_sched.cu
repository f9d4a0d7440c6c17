// Per-stage just-in-time scheduler (hot path 2): beam_schedule on the GPU.
//
// Reference: src/scheduler.cpp:29-378 (RoundContext, BeamState, state_better,
// extend_state, beam_schedule, finalize/score_assignment), src/request.cpp
// (candidate_models :60-68, mark_dispatched :70-86, mark_complete :88-107).
//
// Data layout (a resident session, ag_sched): every in-flight Request lives
// in HBM as
//   pool[voff[s] .. +nviable[s])  its viable list (canonical indices), pruned
//                                 in place on dispatch (order preserved)
//   hist[s][a][m]                 #viable configs with c[a] == m
//   cand[s][a]                    model mask = {m : hist[s][a][m] > 0}
//                                 (Request::candidate_models)
//   ready[s]                      ready-agent mask
// so a round never rescans viable lists except on the rare re-touch of a
// request with parallel ready branches.
//
// One round = one launch of k_sched_round (one CTA of 512 threads):
//   * producer warps (every warp not on the walker's SM sub-partition: wid %
//     4 != 0) scan the FIFO queue chunk by chunk -- RoundContext
//     (scheduler.cpp:36-72): pairs in (arrival, id) x (depth desc,
//     declaration asc) order, validation, and the compacted list of
//     "candidate" pairs, those whose candidate models meet the engines free
//     at round start.  Every other pair is a whole-beam skip in every branch
//     (scheduler.cpp:317-329), so the walk never looks at it.  Candidates
//     (pair position, engine mask, request details and, for the head of the
//     list, the model histogram row with the first-touch flexibility ratios
//     surv / initial already divided) are published through a
//     release/acquire counter in shared memory;
//   * warp 0 walks the candidates as beam_schedule walks pairs, starting as
//     soon as the first chunk is published: skipped runs are fast-forwarded
//     with one ballot scan; beam state w lives in the registers of lane w; at
//     a step lane c builds child c (extend_state), ranks it against the other
//     children under the exact state_better order, and nested retention
//     (scheduler.cpp:351-370) is B warp min-reductions over those ranks; a
//     child's triple list is a node of a history tree (triples_less compares
//     two tree paths through a per-step LCP structure).  The walk stops as
//     soon as every branch is full or the candidates are exhausted; the
//     queue's pair count comes from the host mirror, so the producers stop
//     scanning once the walker is done (unless validation needs every pair);
//   * the fast walker (B <= 4, <= 8 pools; ag_sched_fast.cuh) is fed by a
//     lookahead warp (warp 1) instead: it reads the first 64 positions' pair
//     records itself (a head start before the producers' first chunk), then
//     follows the producers' list, and hands the walker the candidates that
//     meet its current free-engine union through a 64-entry shared-memory
//     ring together with their histogram rows -- the walker's steps read
//     shared memory only;
//   * finalize: the winner's triples from the tree (written in parallel),
//     score_assignment's utilization and flexibility folded in the
//     reference's order;
//   * the round's input deltas (ready masks, FIFO tail) are read by the
//     kernel from mapped pinned host memory and the assignment is written
//     straight back into it: one launch per round, the host spinning on the
//     round's sequence number in the mapped result.  Large record batches
//     (a FIFO compaction, an arrival batch) are applied when they happen by
//     k_sched_refresh, outside the decision.
// Also here: k_sched_prune (mark_dispatched's prefix prune + histograms),
// k_sched_audit (audit_round_fairness, scheduler.cpp:456-480), the viable
// pool compaction (k_pool_scan / k_pool_copy) and k_queued_ahead.
// All fp64 arithmetic repeats the reference's operations in the same order
// (the library builds with --fmad=false).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include "ag_internal.h"

// Per-step phase timers of the walker (find / build / rank / adopt cycles,
// ag_sched_round_timing slots 5-8): diagnostics, compiled in on request only
// (-DAG_SCHED_PHASE_TIMERS=1) -- four clock reads per beam step otherwise.
#ifndef AG_SCHED_WAITPROD
#define AG_SCHED_WAITPROD 0
#endif
#ifndef AG_SCHED_PHASE_TIMERS
#define AG_SCHED_PHASE_TIMERS 0
#endif
#if AG_SCHED_PHASE_TIMERS
#define AG_PHASE_TICK(k)            \
  do {                              \
    const long long t_ = clock64(); \
    tw[k] += t_ - tp;               \
    tp = t_;                        \
  } while (0)
#else
#define AG_PHASE_TICK(k) \
  do {                   \
  } while (0)
#endif

namespace agb {

namespace {

// CTA shape of k_sched_round<BM>: warp 0 walks, the warps on its SM
// sub-partition (wid % 4 == 0) stay idle, the others produce.  The fast
// walker for B <= 4 keeps four beam states in every lane's registers, so its
// CTA has 12 warps (168 registers per thread) instead of 16 (128).
template <int BM>
struct RoundShape {
  static constexpr int threads = 512;
  // warps 1-3, 5-7, 9-11, 13-15; the fast walker (BM > 0) gives warp 1 to
  // its lookahead (candidate records and histogram rows fetched ahead)
  static constexpr int producers = threads / 4 * 3 - (BM > 0 ? 32 : 0);
};
constexpr int kLookahead = 64;  // lookahead ring entries (a power of two)
constexpr int kMaxBeam = 32;
constexpr int kMaxEng = 32;
constexpr int kPruneInline = 768;
constexpr int kInlineRec = 48;  // refresh records carried in the round's parameter block  // int32 words of small dispatch data carried in the parameter block
constexpr int kSmemNodes = 1024;
constexpr int kPer = 4;  // FIFO positions per producer thread per chunk
constexpr unsigned kFull = 0xffffffffu;

struct Node {  // one AssignmentTriple in the beam history tree
  int32_t qi;
  int32_t am;  // agent << 8 | model
  int32_t prev;
  int32_t depth;
  int32_t nsurv;  // survivors of request qi after this triple
  uint32_t nvia;  // round-start viable size of request qi
  int32_t slot;
  int32_t pad;
};

struct Cand {  // one candidate pair
  uint32_t pos;         // pair position in the round's two-level order
  int32_t qi;           // request index (queue container order)
  uint32_t slot_agent;  // slot | agent << 26
  uint32_t nvia;        // round-start viable size
};

// Engine pools in the kernel's internal order: weight descending, ties by
// the caller's index (so the children of one state come out of a mask in
// utilization order, fl(u + w) being monotone in w); inv[k] maps the caller's
// engine k to its internal index for the order-sensitive folds
// (initial_state and score_assignment sum over the caller's order) and the
// occupancy output.
struct EngDev {
  int E;
  int model[kMaxEng];
  int slots[kMaxEng];
  int occ[kMaxEng];
  double weight[kMaxEng];
  int8_t m2e[32];  // model -> engine, -1 none
  int8_t inv[kMaxEng];
  uint32_t mapped;  // models with a pool
};

struct RoundArgs {
  int N, M, B;
  int Q;                 // FIFO length (dead slots have ready 0)
  long long npairs;      // ready pairs in the queue (host mirror)
  int32_t* order;        // [Q] slots in FIFO order (device)
  int32_t* cidx;         // [Q] container index per FIFO position (device), or null
  uint64_t* ready;
  const uint32_t* cand;
  const uint32_t* hist;
  const uint64_t* voff;
  const uint32_t* pool;
  const uint32_t* nviable;
  const uint64_t* ids;
  const uint32_t* ever;  // OR of every candidate-model mask ever installed
  // round input deltas in mapped pinned host memory (or a DMA'd copy)
  const int4* h_rec;      // refresh records {pos (-1: none), slot, ready lo, ready hi}
  int n_rec;
  int n_inl;              // 1: the records are inl_rec (a small batch in the parameter block:
  int4 inl_rec[kInlineRec];  // no PCIe read on the round's critical path)
  const int32_t* h_cidx;  // [Q] or null
  uint4* pinfo;           // [Q] per-position pair records (see the setup)
  int8_t prio[64];
  int8_t prio_rank[64];
  uint32_t place[kMaxAgents];
  uint64_t place_magic[kMaxAgents];
  uint64_t div_m;
  EngDev eng;
  // scratch
  uint32_t* gmask;  // candidates beyond shared memory
  Cand* grec;
  int cand_cap, hist_cap;
  int rows_alloc;  // ratio / count rows allocated (>= hist_cap, >= the lookahead ring)
  int la_rows;     // lookahead ring entries (power of two, <= kLookahead; 0: no lookahead)
  int wor_cap;  // 32-candidate windows: the union of their engine masks
  Node* gnodes;
  int max_nodes;
  int max_children;
  // outputs (mapped pinned host memory): [0] status [1] aux | ag_assignment |
  // occ[32] | triples
  int32_t* out;
  uint32_t seq;  // round sequence number, written last (round_done)
  int triples_cap;
  unsigned long long* timing;  // [13]: globaltimer marks, walk/scan cycle buckets
  int32_t* async_status;       // errors latched by earlier dispatch / add kernels
};

constexpr int kOutHeader = 16;  // bytes before the ag_assignment: status, aux, round seq, pad

// The round's last act: status (and aux) into the mapped result header, then
// the round's sequence number, which the host spins on instead of a stream
// synchronisation (the assignment is visible before the number).
__device__ __forceinline__ void round_done(const RoundArgs& A, int status, int aux) {
  A.out[1] = aux;
  A.out[0] = status;
  __threadfence_system();
  *(volatile int32_t*)(A.out + 2) = (int32_t)A.seq;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];"
               : "=r"(v)
               : "r"((unsigned)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v)
               : "memory");
}

template <int P>
__device__ __forceinline__ void bar_producers() { asm volatile("bar.sync 1, %0;" ::"n"(P) : "memory"); }

__device__ __forceinline__ uint32_t digit_at(uint32_t c, int a, const RoundArgs& A) {
  const uint32_t q = A.place[a] == 1 ? c : (uint32_t)__umul64hi(c, A.place_magic[a]);
  return q - divm(q, A.div_m) * (uint32_t)A.M;
}

// ------------------------------------------------------------ comparisons
struct NodeView {
  const Node* s;  // shared-memory nodes [0, kSmemNodes)
  const Node* g;  // global overflow
  __device__ const Node& operator[](int i) const {
    return i < kSmemNodes ? s[i] : g[i - kSmemNodes];
  }
};

// triples_less (scheduler.cpp:95-105) between the beam states' triple lists,
// kept as a relation per ordered pair of states instead of the lists: rel[i][j]
// is LESS / GREATER when the lists differ at a position both have, P1 when
// list i is a proper prefix of list j (then the low bits hold list j's element
// at that position), P2 when list j is a proper prefix of list i (low bits:
// list i's element there).  A triple key orders (request_index, agent, model)
// lexicographically; kEnd sorts below every key.  Every pair (request, agent)
// is visited once per walk, so a step's key never equals an element of an
// earlier list, and distinct states never hold equal lists.  Adopting children
// updates the relation in O(B^2) without touching the lists.
constexpr uint64_t kEnd = 0;
constexpr uint64_t kRelLess = 0, kRelGreater = 1ull << 62, kRelP1 = 2ull << 62, kRelP2 = 3ull << 62;
constexpr uint64_t kRelCode = 3ull << 62, kRelThr = ~kRelCode;

__device__ __forceinline__ uint64_t tkey(int qi, int agent, int model) {
  return ((uint64_t)(uint32_t)(qi + 1) << 32) | ((uint64_t)(uint32_t)agent << 16) |
         (uint64_t)(uint32_t)model;
}

// relation of (list p1 + k1) to (list p2 + k2); k = kEnd for "no extra";
// r12 = rel[p1][p2] (unused when p1 == p2)
__device__ __forceinline__ uint64_t rel_extend(bool same, uint64_t r12, uint64_t k1, uint64_t k2) {
  if (same) {  // one parent: its children differ in the extra key
    if (k1 == kEnd) return kRelP1 | k2;
    if (k2 == kEnd) return kRelP2 | k1;
    return k1 < k2 ? kRelLess : kRelGreater;
  }
  const uint64_t code = r12 & kRelCode, thr = r12 & kRelThr;
  if (code == kRelP1) return k1 == kEnd ? r12 : (k1 < thr ? kRelLess : kRelGreater);
  if (code == kRelP2) return k2 == kEnd ? r12 : (thr < k2 ? kRelLess : kRelGreater);
  return r12;
}

// list 1 before list 2 (triples_less); lists of distinct items never compare equal
__device__ __forceinline__ bool rel_before(uint64_t r) {
  const uint64_t code = r & kRelCode;
  return code == kRelLess || code == kRelP1;
}

// (list p1 + k1) strictly before (list p2 + k2), branch-free: the common
// case of rel_before(rel_extend(...)).  kEnd = 0 sorts below every threshold.
__device__ __forceinline__ bool lex_before(bool same, uint64_t r12, uint64_t k1, uint64_t k2) {
  const uint64_t code = r12 & kRelCode, thr = r12 & kRelThr;
  const bool by_rel = (code == kRelLess) | ((code == kRelP1) & (k1 < thr)) | ((code == kRelP2) & (thr < k2));
  return same ? (k1 < k2) : by_rel;
}

// rel_extend without branches
__device__ __forceinline__ uint64_t rel_extend_sel(bool same, uint64_t r12, uint64_t k1, uint64_t k2) {
  const uint64_t code = r12 & kRelCode, thr = r12 & kRelThr;
  const uint64_t lg = k1 < k2 ? kRelLess : kRelGreater;
  const uint64_t s_res = k1 == kEnd ? (kRelP1 | k2) : (k2 == kEnd ? (kRelP2 | k1) : lg);
  const uint64_t p1 = k1 == kEnd ? r12 : (k1 < thr ? kRelLess : kRelGreater);
  const uint64_t p2 = k2 == kEnd ? r12 : (thr < k2 ? kRelLess : kRelGreater);
  const uint64_t o_res = code == kRelP1 ? p1 : (code == kRelP2 ? p2 : r12);
  return same ? s_res : o_res;
}


// order-preserving u64 image of an f64 (no NaNs here; -0 == +0)
__device__ __forceinline__ uint64_t okey(double d) {
  uint64_t b = (uint64_t)__double_as_longlong(d);
  if (b == 0x8000000000000000ull) b = 0;
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// rank record of a child: state_better keys (scheduler.cpp:109-115)
struct RankKey {
  uint64_t ku, kf;  // okey(util), okey(flexibility): larger is better
  uint32_t sk;      // skips: fewer is better
  uint32_t pk;      // parent | (model + 1) << 8, 0 for the skip child
  uint64_t pad;
};

struct Child {  // a BeamState child in shared memory (wide beams)
  double util, flex_sum, flex;
  long long skips;
  int flex_count, nsurv;
  int16_t parent, eng;  // eng < 0: skip child
  int pad;
};

// ------------------------------------------------------------ round kernel
// Applies refresh records {FIFO position, slot, ready mask}: ready[slot],
// order[pos] and the position's pair record pinfo[pos] = {slot | first ready
// agent << 26, that agent's candidate-model mask, viable size, ready-agent
// count}.  Loads are issued kU at a time so latency (PCIe for mapped host
// memory) is paid once per batch.  prank(agent): priority rank (depth desc,
// declaration asc, scheduler.cpp:238-242).
template <typename PRank>
__device__ __forceinline__ void apply_records(const int4* __restrict__ rec, int n_rec, int first, int stride, int N,
                                              uint64_t* ready, const uint32_t* cand, const uint32_t* nviable,
                                              int32_t* order, uint4* pinfo, PRank prank) {
  constexpr int kU = 4;
  for (int i0 = first; i0 < n_rec; i0 += stride * kU) {
    int4 rc[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * stride;
      rc[u] = i < n_rec ? rec[i] : make_int4(-1, -1, 0, 0);
    }
    uint32_t cm[kU], nvv[kU];
    int best[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int pos = rc[u].x, slot = rc[u].y;
      const uint64_t r = (uint64_t)(uint32_t)rc[u].z | ((uint64_t)(uint32_t)rc[u].w << 32);
      if (slot >= 0) ready[slot] = r;
      int bst = -1, br = 1 << 30;
      for (uint64_t b = r; b; b &= b - 1) {
        const int ag = __ffsll((long long)b) - 1;
        const int pr = prank(ag);
        if (pr < br) br = pr, bst = ag;
      }
      best[u] = bst;
      // the union of the ready agents' candidate models (one agent: its mask)
      uint32_t c = 0;
      if (pos >= 0 && slot >= 0)
        for (uint64_t b = r; b; b &= b - 1) c |= cand[(size_t)slot * N + (__ffsll((long long)b) - 1)];
      cm[u] = c;
      nvv[u] = pos >= 0 && slot >= 0 ? nviable[slot] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int pos = rc[u].x, slot = rc[u].y;
      if (pos < 0) continue;
      const uint64_t r = (uint64_t)(uint32_t)rc[u].z | ((uint64_t)(uint32_t)rc[u].w << 32);
      const uint32_t nr = slot >= 0 ? (uint32_t)__popcll(r) : 0u;
      order[pos] = slot;
      pinfo[pos] = make_uint4((uint32_t)(slot >= 0 ? slot : 0) | ((uint32_t)(best[u] & 63) << 26), cm[u], nvv[u], nr);
    }
  }
}

// Viable-pool compaction: the live requests' lists (pruned in place, so only
// the device knows their lengths) are packed into a fresh pool in slot-list
// order, and voff is rewritten.  The pool is then a capacity, not a lifetime
// budget for every request a session ever adds.
__global__ void __launch_bounds__(1024) k_pool_scan(const int32_t* __restrict__ live, int n_live,
                                                    const uint32_t* __restrict__ nviable, uint64_t* new_off,
                                                    uint64_t* total) {
  __shared__ uint64_t s_w[32];
  __shared__ uint64_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < n_live; base += 1024) {
    const int i = base + tid;
    const uint64_t len = i < n_live ? nviable[live[i]] : 0;
    uint64_t x = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    if (w == 0) {
      const uint64_t v = s_w[lane];
      uint64_t z = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += y;
      }
      s_w[lane] = z - v;
    }
    __syncthreads();
    const uint64_t carry = s_carry;
    if (i < n_live) new_off[i] = carry + s_w[w] + x - len;
    __syncthreads();
    if (tid == 1023) s_carry = carry + s_w[31] + x;
    __syncthreads();
  }
  if (tid == 0) *total = s_carry;
}

__global__ void __launch_bounds__(256) k_pool_copy(const int32_t* __restrict__ live, const uint64_t* __restrict__ new_off,
                                                   const uint32_t* __restrict__ nviable, uint64_t* voff,
                                                   const uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
  const int s = live[blockIdx.x];
  const uint64_t from = voff[s], to = new_off[blockIdx.x];
  const uint32_t len = nviable[s];
  for (uint32_t q = threadIdx.x; q < len; q += 256) dst[to + q] = src[from + q];
  __syncthreads();
  if (threadIdx.x == 0) voff[s] = to;
}

// Large record batches (a FIFO compaction, a big arrival batch) are applied
// when they happen, by this kernel, instead of inside the next round's
// decision latency.
struct RefreshArgs {
  int N;
  uint64_t* ready;
  const uint32_t* cand;
  const uint32_t* nviable;
  int32_t* order;
  uint4* pinfo;
  int8_t prio_rank[64];
};

__global__ void __launch_bounds__(256) k_sched_refresh(const int4* __restrict__ rec, int n_rec,
                                                       const __grid_constant__ RefreshArgs A) {
  __shared__ int8_t s_pr[64];
  if (threadIdx.x < 64) s_pr[threadIdx.x] = A.prio_rank[threadIdx.x];
  __syncthreads();
  apply_records(rec, n_rec, blockIdx.x * 256 + threadIdx.x, gridDim.x * 256, A.N, A.ready, A.cand, A.nviable,
                A.order, A.pinfo, [&](int ag) { return (int)s_pr[ag]; });
}

template <int BM>
__global__ void __launch_bounds__(RoundShape<BM>::threads, 1) k_sched_round(const __grid_constant__ RoundArgs A) {
  constexpr int kRoundThreads = RoundShape<BM>::threads, kProducers = RoundShape<BM>::producers;
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ int s_occ[2][kMaxBeam][kMaxEng];
  __shared__ uint64_t s_rel[2][kMaxBeam][kMaxBeam];
  __shared__ __align__(16) RankKey s_rk[32];
  __shared__ int s_cnt[kMaxBeam][32];
  // fast walker: re-touch flex deltas, relevant-child keys, exact child order
  __shared__ double s_rdelta[BM > 0 ? BM : 1][32];
  __shared__ double2 s_fkey[32];
  __shared__ unsigned long long s_fmeta[32];
  __shared__ int8_t s_fe[32];
  __shared__ int8_t s_order[BM > 0 ? BM : 1][8];
  __shared__ int s_picked[kMaxBeam];
  __shared__ int s_cons[kMaxAgents][2];
  __shared__ int s_ncons;
  __shared__ long long s_scan[kProducers / 32][3];
  __shared__ long long s_carry[3];
  __shared__ int s_chunk[2];     // candidates of the current chunk: [first, end)
  __shared__ int s_status;       // producer-detected validation error
  __shared__ int s_stop;         // producers: snapshot of s_walk_done
  __shared__ unsigned s_produced;  // candidates published (release/acquire)
  __shared__ unsigned s_rows;      // candidates whose histogram rows are staged
  __shared__ unsigned s_prod_done;
  __shared__ unsigned s_walk_done;
  __shared__ int e_model[kMaxEng], e_slots[kMaxEng];
  __shared__ double e_weight[kMaxEng];
  __shared__ int8_t e_m2e[32], s_prio[64], s_prank[64];
  __shared__ uint32_t s_emtab[4][256];  // model mask -> engine mask, one byte at a time
  // lookahead ring (BM > 0): candidate records and engine masks; their count
  // / ratio rows live in the staging rows below
  __shared__ __align__(16) Cand s_la_rec[BM > 0 ? kLookahead : 1];
  __shared__ uint32_t s_la_mask[BM > 0 ? kLookahead : 1];
  __shared__ int32_t s_la_idx[BM > 0 ? kLookahead : 1];
  __shared__ unsigned s_la_head, s_la_tail, s_la_done;
  __shared__ uint32_t s_U;  // the walker's current free-engine union (shrinks)
  // dynamic: nodes | children (wide beams) | ratio rows | cand records | cand masks | count rows
  Node* s_nodes = reinterpret_cast<Node*>(dsm);
  Child* children = reinterpret_cast<Child*>(s_nodes + kSmemNodes);
  double* h_rat = reinterpret_cast<double*>(children + A.max_children);
  Cand* c_rec = reinterpret_cast<Cand*>(h_rat + (size_t)A.rows_alloc * A.M);
  uint32_t* c_mask = reinterpret_cast<uint32_t*>(c_rec + A.cand_cap);
  uint32_t* h_cnt = c_mask + A.cand_cap;
  // per window of 32 candidates, the union of their masks: the walker skips
  // a published window whose union misses every free engine without reading
  // its candidates
  uint32_t* s_wor = h_cnt + (size_t)A.rows_alloc * A.M;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int N = A.N, M = A.M, B = A.B;
  if (tid == 0) {
    s_status = 0;
    s_stop = 0;
    s_produced = 0;
    s_rows = 0;
    s_prod_done = 0;
    s_walk_done = 0;
    s_la_head = s_la_tail = s_la_done = 0;
    uint32_t u0 = 0;
    for (int e = 0; e < A.eng.E; ++e)
      if (A.eng.slots[e] - A.eng.occ[e] > 0) u0 |= 1u << e;
    s_U = u0;
    s_carry[0] = s_carry[1] = s_carry[2] = 0;
    if (A.timing) A.timing[0] = gtimer();
    if (*A.async_status) {
      s_status = AG_ERR_VALIDATION + 600;  // a dispatch pruned a request to nothing
      *A.async_status = 0;
    }
  }
  for (int i = tid; i < A.wor_cap; i += kRoundThreads) s_wor[i] = 0u;
  if (tid < kMaxEng) {
    e_model[tid] = A.eng.model[tid];
    e_slots[tid] = A.eng.slots[tid];
    e_weight[tid] = A.eng.weight[tid];
    e_m2e[tid] = A.eng.m2e[tid];
  }
  if (tid < 64) {
    s_prio[tid] = A.prio[tid];
    s_prank[tid] = A.prio_rank[tid];
  }
  for (int i = tid; i < 1024; i += kRoundThreads) {
    uint32_t em = 0;
    for (int b = 0; b < 8; ++b) {
      const int e = A.eng.m2e[(i >> 8) * 8 + b];
      if (((i >> b) & 1) && e >= 0) em |= 1u << e;
    }
    s_emtab[i >> 8][i & 255] = em;
  }
  // The round's deltas (mapped host memory, small; one DMA copy when large):
  // refresh records {FIFO position, slot, ready mask} for the rewritten FIFO
  // range and for every other slot whose ready mask changed, and the
  // container indices of a stateless call.  A record rewrites ready[slot],
  // order[pos] and the position's pair record pinfo[pos] = {slot | first
  // ready agent << 26, that agent's candidate-model mask, viable size,
  // ready-agent count}, so the producers read one coalesced 16-byte record
  // per FIFO position instead of the order -> ready -> cand gather chain.
  // Loads are issued in batches so PCIe latency is paid once per batch.
  {
    constexpr int kU = 4;
    if (A.h_cidx)
      for (int i0 = 0; i0 < A.Q; i0 += kRoundThreads * kU) {
        int32_t v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int i = i0 + u * kRoundThreads + tid;
          v[u] = i < A.Q ? A.h_cidx[i] : 0;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int i = i0 + u * kRoundThreads + tid;
          if (i < A.Q) A.cidx[i] = v[u];
        }
      }
    apply_records(A.n_inl ? A.inl_rec : A.h_rec, A.n_rec, tid, kRoundThreads, N, A.ready, A.cand, A.nviable,
                  A.order, A.pinfo,
                  [&](int ag) { return (int)A.prio_rank[ag]; });
  }
  __syncthreads();
  if (s_status) {
    if (tid == 0) round_done(A, s_status, 0);
    return;
  }
  if (tid == 0 && A.timing) A.timing[1] = gtimer();
  // engines / models with a free slot at round start
  uint32_t U0 = 0, U0m = 0;
  for (int e = 0; e < A.eng.E; ++e)
    if (e_slots[e] - A.eng.occ[e] > 0) {
      U0 |= 1u << e;
      if (e_model[e] < 32) U0m |= 1u << e_model[e];
    }
  // every pair must be scanned for RoundContext validation only if some
  // installed candidate model has no pool
  const bool check_all = (*A.ever & ~A.eng.mapped) != 0u;

  if (wid != 0) {
    if ((wid & 3) == 0) return;  // the walker's SM sub-partition stays quiet
    if constexpr (BM > 0) {
      if (wid == 1) {
        // ============================================= lookahead (warp 1)
        // Runs ahead of the walker over the published candidate list: the
        // next candidates whose engine mask meets the walker's current
        // free-engine union (a superset of the union when the walker gets
        // there: it only shrinks) go into a ring with their records and
        // their histogram rows (surv counts, first-touch ratios surv /
        // initial): up to 16 windows are scanned per pass and up to 32 hits
        // fetched together, so the walker's steps read shared memory only.
        const int LA = A.la_rows;
        unsigned head = 0, have_l = 0;
        int jl = 0;
        bool exhausted = false;
        // Head start: the first 64 FIFO positions straight from their pair
        // records (the producers' first chunk takes several microseconds
        // longer) -- the candidate records the producers will publish for
        // them, in the same order, so the list is then followed from the
        // number of candidates found here.  Only when every such position
        // has at most one ready agent (chains; otherwise the producers' path).
        {
          constexpr int kHead = 64;
          uint4 inf[2];
          int npair[2], nq[2], nc[2];
          bool multi = false;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int p = lane * 2 + i;
            inf[i] = p < A.Q && p < kHead ? A.pinfo[p] : make_uint4(0u, 0u, 0u, 0u);
            multi |= inf[i].w > 1u;
            npair[i] = (int)inf[i].w;
            nq[i] = inf[i].w ? 1 : 0;
            nc[i] = inf[i].w == 1u && (inf[i].y & U0m) != 0u ? 1 : 0;
          }
          if (!__any_sync(kFull, multi)) {
            // exclusive prefixes over positions: pairs, ready requests, candidates
            int xp = npair[0] + npair[1], xq = nq[0] + nq[1], xc = nc[0] + nc[1];
            int ip = xp, iq = xq, ic = xc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int a1 = __shfl_up_sync(kFull, ip, o), a2 = __shfl_up_sync(kFull, iq, o),
                        a3 = __shfl_up_sync(kFull, ic, o);
              if (lane >= o) ip += a1, iq += a2, ic += a3;
            }
            const int n_cand = __shfl_sync(kFull, ic, 31);
            int bp = ip - xp, bq = iq - xq, bc = ic - xc;
            const uint32_t U = *(volatile uint32_t*)&s_U;
            // ring entries for the candidates meeting U, in order
            int hits[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const uint32_t em = nc[i] ? (s_emtab[0][inf[i].y & 255] | s_emtab[1][(inf[i].y >> 8) & 255] |
                                           s_emtab[2][(inf[i].y >> 16) & 255] | s_emtab[3][inf[i].y >> 24]) & U0
                                        : 0u;
              hits[i] = (em & U) != 0u ? 1 : 0;
              inf[i].y = em;
            }
            int xh = hits[0] + hits[1], ih = xh;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int a = __shfl_up_sync(kFull, ih, o);
              if (lane >= o) ih += a;
            }
            const int n_hit = __shfl_sync(kFull, ih, 31);
            int bh = ih - xh;
            if (n_hit <= LA) {
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const int p = lane * 2 + i;
                if (hits[i]) {
                  const int sl = bh & (LA - 1);
                  s_la_rec[sl] = Cand{(uint32_t)bp, A.cidx ? A.cidx[p] : bq, inf[i].x, inf[i].z};
                  s_la_mask[sl] = inf[i].y;
                  ++bh;
                }
                bp += npair[i];
                bq += nq[i];
                bc += nc[i];
              }
              __syncwarp();
              for (int e = lane; e < n_hit * M; e += 32) {
                const int k = e / M, mdl = e - k * M;
                const Cand r = s_la_rec[k];
                const int a = (int)(r.slot_agent >> 26), slt = (int)(r.slot_agent & 0x3ffffffu);
                const uint32_t sv = __ldg(A.hist + ((size_t)slt * N + a) * M + mdl);
                h_cnt[k * M + mdl] = sv;
                h_rat[k * M + mdl] = (double)sv / (double)r.nvia;
              }
              __syncwarp();
              if (lane == 0 && n_hit) {
                __threadfence_block();
                st_release(&s_la_head, (unsigned)n_hit);
              }
              head = (unsigned)n_hit;
              jl = n_cand;  // the producers' candidates of these positions are covered
            }
          }
        }
        while (!exhausted) {
          // room in the ring (entries below the walker's tail are consumed)
          unsigned tail = 0;
          if (lane == 0) {
            for (;;) {
              tail = *(volatile unsigned*)&s_la_tail;
              if (head - tail < (unsigned)LA || *(volatile unsigned*)&s_walk_done) break;
              __nanosleep(32);
            }
          }
          tail = __shfl_sync(kFull, tail, 0);
          if (*(volatile unsigned*)&s_walk_done) break;
          const int want = min(32, LA - (int)(head - tail));
          const uint32_t U = *(volatile uint32_t*)&s_U;
          int cnt = 0;
          for (int scanned = 0; cnt < want && scanned < 16; ++scanned) {
            if ((unsigned)jl >= have_l) {  // published candidates beyond jl, or the final count
              unsigned v = 0;
              if (lane == 0) {
                for (;;) {
                  const unsigned done = *(volatile unsigned*)&s_prod_done;
                  v = *(volatile unsigned*)&s_produced;
                  // with hits in hand, fetch them rather than wait for more
                  if (v > (unsigned)jl || done || cnt > 0 || *(volatile unsigned*)&s_walk_done) break;
                  __nanosleep(32);
                }
                v = ld_acquire(&s_produced);
              }
              have_l = __shfl_sync(kFull, v, 0);
              if ((unsigned)jl >= have_l) {
                if (cnt > 0) break;  // fetch first
                exhausted = true;
                break;
              }
            }
            if ((jl & 31) == 0) {  // skip published 32-candidate windows whose union misses U
              const int w0 = jl >> 5, wl = w0 + lane;
              const bool pub = (unsigned)(wl + 1) * 32u <= have_l;
              const unsigned sb = __ballot_sync(kFull, !pub || (s_wor[pub ? wl : 0] & U) != 0u);
              if (sb == 0u) {
                jl = (w0 + 32) * 32;
                continue;
              }
              jl = (w0 + __ffs(sb) - 1) * 32;
              if ((unsigned)jl >= have_l) continue;
            }
            const int lim = min((int)have_l, (jl & ~31) + 32);
            const int idx = jl + lane;
            const uint32_t mk = idx < lim ? (idx < A.cand_cap ? c_mask[idx] : A.gmask[idx - A.cand_cap]) : 0u;
            unsigned hit = __ballot_sync(kFull, (mk & U) != 0u);
            const int nh = __popc(hit);
            const int take = min(nh, want - cnt);
            if (take < nh) {  // keep the first `take` hits
              unsigned h2 = hit;
              for (int k = 0; k < take; ++k) h2 &= h2 - 1;
              hit &= ~h2;
            }
            if ((hit >> lane) & 1u) {
              const int sl = (int)((head + (unsigned)(cnt + __popc(hit & ((1u << lane) - 1u)))) & (unsigned)(LA - 1));
              s_la_idx[sl] = idx;
              s_la_mask[sl] = mk;
            }
            cnt += take;
            // next unexamined candidate: after the last taken hit, or the window end
            jl = take < nh ? jl + (32 - __clz(hit)) : lim;
          }
          __syncwarp();
          if (cnt) {
            // fetch: the records, then the histogram rows (cnt * M loads in flight)
            if (lane < cnt) {
              const int sl = (int)((head + (unsigned)lane) & (unsigned)(LA - 1));
              const int idx = s_la_idx[sl];
              s_la_rec[sl] = idx < A.cand_cap ? c_rec[idx] : A.grec[idx - A.cand_cap];
            }
            __syncwarp();
            for (int e = lane; e < cnt * M; e += 32) {
              const int k = e / M, mdl = e - k * M;
              const int sl = (int)((head + (unsigned)k) & (unsigned)(LA - 1));
              const Cand r = s_la_rec[sl];
              const int a = (int)(r.slot_agent >> 26), slt = (int)(r.slot_agent & 0x3ffffffu);
              const uint32_t sv = __ldg(A.hist + ((size_t)slt * N + a) * M + mdl);
              h_cnt[sl * M + mdl] = sv;
              h_rat[sl * M + mdl] = (double)sv / (double)r.nvia;
            }
            __syncwarp();
            if (lane == 0) {
              __threadfence_block();
              st_release(&s_la_head, head + (unsigned)cnt);
            }
            head += (unsigned)cnt;
          }
        }
        if (lane == 0) {
          __threadfence_block();
          st_release(&s_la_done, 1u);
        }
        return;
      }
    }
    // ================================================= producers
    // producer index 0 .. kProducers-1 over the producer warps
    const int pt = tid - 32 * (1 + (wid >> 2) + (BM > 0 && wid > 1 ? 1 : 0));
    const int pw = pt >> 5;
    // the next chunk's pair records are loaded while this one is processed
    uint4 inf[kPer], nxt[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int p = pt * kPer + i;
      nxt[i] = p < A.Q ? A.pinfo[p] : make_uint4(0u, 0u, 0u, 0u);
    }
    for (int base = 0; base < A.Q; base += kProducers * kPer) {
      if (s_stop) break;  // uniform: written before the previous barrier
      const int p0 = base + pt * kPer;
      int slot[kPer], a1[kPer];
      uint64_t rdy[kPer];
      uint32_t cm1[kPer], nvia[kPer];
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        inf[i] = nxt[i];
        const int p = p0 + kProducers * kPer + i;
        nxt[i] = p < A.Q ? A.pinfo[p] : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        slot[i] = (int)(inf[i].x & 0x3ffffffu);
        a1[i] = (int)(inf[i].x >> 26);
        cm1[i] = inf[i].y;
        nvia[i] = inf[i].z;
        // the full ready mask only for requests with parallel ready agents
        rdy[i] = inf[i].w > 1u ? A.ready[slot[i]] : (inf[i].w ? 1ull << a1[i] : 0ull);
      }
      // pass 1: counts (pairs, requests, candidates) of this thread's positions
      int np = 0, nq = 0, nc = 0;
      bool bad = false;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        if (!rdy[i]) continue;
        np += __popcll(rdy[i]);
        nq += 1;
        if ((rdy[i] & (rdy[i] - 1)) == 0) {  // one ready agent (chains): no more loads
          bad |= (cm1[i] & ~A.eng.mapped) != 0;
          nc += (cm1[i] & U0m) != 0;
        } else {
          for (uint64_t b = rdy[i]; b; b &= b - 1) {
            const int a = __ffsll((long long)b) - 1;
            const uint32_t cm = A.cand[(size_t)slot[i] * N + a];
            bad |= (cm & ~A.eng.mapped) != 0;
            nc += (cm & U0m) != 0;
          }
        }
      }
      if (bad) s_status = AG_ERR_VALIDATION + 100;  // viable tier without a pool
      if (base == 0 && pt == 0 && A.timing) A.timing[11] = gtimer();
      int x[3] = {np, nq, nc};
#pragma unroll
      for (int o = 1; o < 32; o <<= 1)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int y = __shfl_up_sync(kFull, x[k], o);
          if (lane >= o) x[k] += y;
        }
      if (lane == 31)
#pragma unroll
        for (int k = 0; k < 3; ++k) s_scan[pw][k] = x[k];
      bar_producers<kProducers>();
      if (pw == 0) {
        constexpr int NW = kProducers / 32;
        int v[3], z[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) v[k] = z[k] = lane < NW ? (int)s_scan[lane][k] : 0;
#pragma unroll
        for (int o = 1; o < NW; o <<= 1)
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const int y = __shfl_up_sync(kFull, z[k], o);
            if (lane >= o) z[k] += y;
          }
        if (lane < NW)
#pragma unroll
          for (int k = 0; k < 3; ++k) s_scan[lane][k] = z[k] - v[k] + s_carry[k];
        __syncwarp();
        if (lane == NW - 1) {
          s_chunk[0] = (int)s_carry[2];
#pragma unroll
          for (int k = 0; k < 3; ++k) s_carry[k] += z[k];
          s_chunk[1] = (int)s_carry[2];
        }
      }
      bar_producers<kProducers>();
      if (base == 0 && pt == 0 && A.timing) A.timing[12] = gtimer();
      // pass 2: this thread's candidates (position, engine mask, details) in pair order
      int pos = (int)(s_scan[pw][0] + x[0] - np);
      int qr = (int)(s_scan[pw][1] + x[1] - nq);
      int cw = (int)(s_scan[pw][2] + x[2] - nc);
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        if (!rdy[i]) continue;
        const int qi = A.cidx ? A.cidx[p0 + i] : qr;
        ++qr;
        const bool single = (rdy[i] & (rdy[i] - 1)) == 0;
        for (int t = 0; t < N; ++t) {
          const int a = single ? a1[i] : s_prio[t];
          if (!single && !((rdy[i] >> a) & 1ull)) continue;
          const uint32_t cm = single ? cm1[i] : A.cand[(size_t)slot[i] * N + a];
          if (cm & U0m) {
            // engine mask of the candidate models
            const uint32_t em = s_emtab[0][cm & 255] | s_emtab[1][(cm >> 8) & 255] |
                                s_emtab[2][(cm >> 16) & 255] | s_emtab[3][cm >> 24];
            const Cand r{(uint32_t)pos, qi, (uint32_t)slot[i] | ((uint32_t)a << 26), nvia[i]};
            if (cw < A.cand_cap) {
              c_mask[cw] = em & U0;
              c_rec[cw] = r;
            } else {
              A.gmask[cw - A.cand_cap] = em & U0;
              A.grec[cw - A.cand_cap] = r;
            }
            atomicOr(&s_wor[cw >> 5], em & U0);  // before the chunk's release
            ++cw;
          }
          ++pos;
          if (single) break;
        }
      }
      bar_producers<kProducers>();
      if (base == 0 && pt == 0 && A.timing) A.timing[13] = gtimer();
      // pass 3: for the head of the list, the histogram rows with the
      // first-touch flexibility ratios (extend_state, scheduler.cpp:182-191)
      // -- one (candidate, model) entry per thread, loads in parallel.  The
      // first rows of the chunk are published with its records, the rest
      // right after.
      const int c_lo = s_chunk[0], c_hi = BM > 0 ? c_lo : min(s_chunk[1], A.hist_cap);
      const int c_mid = min(c_hi, c_lo + 32);
      auto stage_rows = [&](int from, int to) {
        constexpr int kU = 4;
        for (int e0 = from * M; e0 < to * M; e0 += kProducers * kU) {
          uint32_t sv[kU], nvv[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int e = e0 + u * kProducers + pt;
            sv[u] = 0;
            nvv[u] = 1;
            if (e < to * M) {
              const int c = e / M, mdl = e - c * M;
              const Cand r = c_rec[c];
              const int a = (int)(r.slot_agent >> 26), sl = (int)(r.slot_agent & 0x3ffffffu);
              sv[u] = __ldg(A.hist + ((size_t)sl * N + a) * M + mdl);
              nvv[u] = r.nvia;
            }
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int e = e0 + u * kProducers + pt;
            if (e < to * M) {
              h_cnt[e] = sv[u];
              h_rat[e] = (double)sv[u] / (double)nvv[u];
            }
          }
        }
      };
      stage_rows(c_lo, c_mid);
      bar_producers<kProducers>();
      if (pt == 0) {
        if (base == 0 && A.timing) A.timing[14] = gtimer();
        __threadfence_block();
        if (c_mid > c_lo) st_release(&s_rows, (unsigned)c_mid);
        st_release(&s_produced, (unsigned)s_carry[2]);
      }
      if (c_hi > c_mid) {
        stage_rows(c_mid, c_hi);
        bar_producers<kProducers>();
        if (pt == 0) {
          __threadfence_block();
          st_release(&s_rows, (unsigned)c_hi);
        }
      }
      if (pt == 0) s_stop = check_all ? 0 : (int)*(volatile unsigned*)&s_walk_done;
      bar_producers<kProducers>();
    }
    if (pt == 0) {
      if (A.timing) A.timing[15] = gtimer();  // producers done
      __threadfence_block();
      st_release(&s_prod_done, 1u);
    }
    return;
  }

  // =================================================== walker (warp 0)
  const NodeView nv{s_nodes, A.gnodes};
  const int E = A.eng.E;
  const int lgE = E <= 1 ? 0 : 32 - __clz(E - 1);  // engines padded to a power of two
  const unsigned lt = (1u << lane) - 1u;
  const unsigned le = lt | (1u << lane);
  int wstatus = 0;
  // BeamState w lives in lane w (initial_state, scheduler.cpp:117-128)
  double st_u = 0.0, st_fs = 0.0;
  int st_fc = 0, st_nd = -1, st_ns = 0, st_lq = -1, st_ln = 0;
  long long st_sk = 0;
  uint32_t st_fm = 0;
  if (lane == 0) {
    for (int k = 0; k < E; ++k) {  // the caller's engine order (utilization fold)
      const int e = A.eng.inv[k];
      const int occ = A.eng.occ[e];
      if (occ > e_slots[e]) wstatus = AG_ERR_VALIDATION + 200;  // engine over capacity
      s_occ[0][0][e] = occ;
      st_u += occ * e_weight[e];
      if (e_slots[e] - occ > 0) st_fm |= 1u << e;
    }
  }
  wstatus = __shfl_sync(kFull, wstatus, 0);
  __syncwarp();
  // occupancy of state w, engine e in lane (w << lgE) + e when every state's
  // row fits the warp (B * E padded <= 32); shared-memory rows otherwise
  const bool regocc = BM == 0 && (B << lgE) <= 32;
  const int ow = lane >> lgE, oe = lane & ((1 << lgE) - 1);
  int occ_r = (ow == 0 && oe < E) ? A.eng.occ[oe] : 0;
  int cur = 0, nst = 1, nnodes = 0;
  unsigned long long explored = 1;
  long long pi = 0;  // next pair position not yet accounted for
  int j = 0;         // next candidate index
  int last_q = -1;   // request of the last visited candidate
  unsigned have = 0; // candidates known to be published
  int rows = 0;      // candidates known to have staged histogram rows
  long long tw[4] = {0, 0, 0, 0};
  unsigned long long n_steps = 0, n_child = 0;
  long long tp = clock64();
  // published count once it exceeds idx, or the final count
  auto wait_for = [&](unsigned idx) -> unsigned {
    if (idx < have) return have;
    unsigned v = 0;
    if (lane == 0) {
      // relaxed spin, then one acquire of the published count
      for (;;) {
        const unsigned done = *(volatile unsigned*)&s_prod_done;
        v = *(volatile unsigned*)&s_produced;
        if (v > idx || done) break;
        __nanosleep(32);
      }
      v = ld_acquire(&s_produced);
      __threadfence_block();
      if (have == 0 && v && A.timing) A.timing[2] = gtimer();
    }
    have = __shfl_sync(kFull, v, 0);
    return have;
  };
  auto maskf = [&](int i) -> uint32_t { return i < A.cand_cap ? c_mask[i] : A.gmask[i - A.cand_cap]; };
  auto recf = [&](int i) -> Cand { return i < A.cand_cap ? c_rec[i] : A.grec[i - A.cand_cap]; };

  if constexpr (BM > 0) {
#if AG_SCHED_WAITPROD  // diagnostics: walk only after the producers are done
    if (lane == 0)
      while (!ld_acquire(&s_prod_done)) __nanosleep(64);
    __syncwarp();
#endif
#include "ag_sched_fast.cuh"
  } else
  while (!wstatus) {
    const uint32_t U = __reduce_or_sync(kFull, lane < nst ? st_fm : 0u);
    if (!U) break;  // all-full early exit (scheduler.cpp:303-315)
    // the next candidate of the current request is visited unconditionally;
    // otherwise the next candidate whose mask meets a free engine
    int found = -1;
    uint32_t base = 0;
    for (int j0 = j;;) {
      const unsigned h = wait_for((unsigned)j0);
      if (h <= (unsigned)j0) break;  // producers done, list exhausted
      const int jj = j0 + lane;
      const uint32_t mm = jj < (int)h ? maskf(jj) : 0u;
      const bool cont = lane == 0 && j0 == j && last_q >= 0 && recf(j).qi == last_q;
      const uint32_t b = __ballot_sync(kFull, (mm & U) != 0 || cont);
      if (b) {
        const int src = __ffs(b) - 1;
        found = j0 + src;
        base = __shfl_sync(kFull, mm, src);
        break;
      }
      j0 = min(j0 + 32, (int)h);
      // skip published windows whose mask union misses U, 32 windows per
      // ballot; stop at the first window that may match or is not complete
      for (;;) {
        const int w0 = j0 >> 5, wl = w0 + lane;
        const bool pub = (unsigned)(wl + 1) * 32u <= have;
        const unsigned sb = __ballot_sync(kFull, !pub || (s_wor[pub ? wl : 0] & U) != 0u);
        if (sb == 0u) {
          j0 = (w0 + 32) * 32;
          continue;
        }
        const int first = __ffs(sb) - 1;
        if (first > 0) j0 = (w0 + first) * 32;
        break;
      }
    }
    AG_PHASE_TICK(0);
    if (found < 0) break;
    j = found;
    const Cand cr = recf(j);
    {  // whole-beam skips before this pair
      const long long k = (long long)cr.pos - pi;
      if (k > 0) {
        if (lane < nst) st_sk += k;
        explored += (unsigned long long)nst * (unsigned long long)k;
      }
      pi = (long long)cr.pos + 1;
    }
    const int qcur = cr.qi, a = (int)(cr.slot_agent >> 26), slot = (int)(cr.slot_agent & 0x3ffffffu);
    const double initial = (double)cr.nvia;
    const int hrow = j;
    if (hrow >= rows && hrow < A.hist_cap) rows = ld_acquire(&s_rows);  // uniform
    const bool tch = lane < nst && st_lq == qcur;
    // allowed_engines (scheduler.cpp:140-156)
    uint32_t mk = (lane < nst && !tch) ? (base & st_fm) : 0u;
    const uint32_t tmask = __ballot_sync(kFull, tch);
    // re-touch: counts per model of this agent over the request's viable
    // configurations consistent with the state's earlier triples for it
    for (uint32_t tb = tmask; tb; tb &= tb - 1) {
      const int si = __ffs(tb) - 1;
      const int snode = __shfl_sync(kFull, st_nd, si);
      if (lane == 0) {
        int n = snode, nc = 0;
        while (n >= 0 && nv[n].qi == qcur) {
          s_cons[nc][0] = nv[n].am >> 8;
          s_cons[nc][1] = nv[n].am & 0xFF;
          ++nc;
          n = nv[n].prev;
        }
        s_ncons = nc;
      }
      s_cnt[si][lane] = 0;
      __syncwarp();
      const int ncons = s_ncons;
      const uint32_t* vl = A.pool + A.voff[slot];
      const uint32_t nv_len = A.nviable[slot];
      for (uint32_t q = lane; q < nv_len; q += 32) {
        const uint32_t c = vl[q];
        bool ok = true;
        for (int t = 0; t < ncons && ok; ++t) ok = (int)digit_at(c, s_cons[t][0], A) == s_cons[t][1];
        if (ok) atomicAdd(&s_cnt[si][digit_at(c, a, A)], 1);
      }
      __syncwarp();
      if (lane == si) {
        uint32_t em = 0;
        for (int mdl = 0; mdl < M; ++mdl)
          if (s_cnt[si][mdl] > 0) em |= 1u << e_m2e[mdl];
        mk = em & st_fm;
      }
      __syncwarp();
    }
    last_q = qcur;
    ++j;
    if (!__any_sync(kFull, lane < nst && mk != 0)) {  // whole-beam skip (scheduler.cpp:317-329)
      if (lane < nst) st_sk += 1;
      explored += (unsigned long long)nst;
      continue;
    }
    // children in (state, engine ascending) order; a state with no free
    // candidate contributes one skip child (scheduler.cpp:331-349).
    // Exclusive offsets of the per-state child counts (<= 33) by bit slices.
    const int my_n = lane < nst ? (mk ? __popc(mk) : 1) : 0;
    int off = 0, nchild = 0;
#pragma unroll
    for (int bit = 0; bit < 6; ++bit) {
      const uint32_t bb = __ballot_sync(kFull, (my_n >> bit) & 1);
      off += __popc(bb & lt) << bit;
      nchild += __popc(bb) << bit;
    }
    explored += (unsigned long long)nchild;
    ++n_steps;
    n_child += nchild;
    const uint64_t(*R)[kMaxBeam] = s_rel[cur];
    const uint64_t key_base = tkey(qcur, a, 0);
    const bool fast = nchild <= 32;
    int npick = 0;
    // the picked child's values (lane w: the child adopted as state w)
    double c_u = 0.0, c_fs = 0.0;
    long long c_sk = 0;
    int c_fc = 0, c_ns = 0, c_par = 0, c_eng = -1;
    if (fast) {
      // lane c builds child c (extend_state, scheduler.cpp:158-206)
      const unsigned starts = __reduce_or_sync(kFull, lane < nst ? (1u << off) : 0u);
      const unsigned sl = starts & le;
      const bool valid = lane < nchild;
      const int par = valid ? __popc(sl) - 1 : 0;
      const int poff = valid ? 31 - __clz(sl) : 0;
      const double pu = __shfl_sync(kFull, st_u, par);
      const double pfs = __shfl_sync(kFull, st_fs, par);
      const int pfc = __shfl_sync(kFull, st_fc, par);
      const long long psk = __shfl_sync(kFull, st_sk, par);
      const int pns = __shfl_sync(kFull, st_ns, par);
      const uint32_t pm = __shfl_sync(kFull, mk, par);
      const bool ptch = ((tmask >> par) & 1u) != 0;
      double cu = pu, cfs = pfs, cf = 1.0;
      long long csk = psk;
      int cfc = pfc, cns = pns, ce = -1, cm1 = 0;  // cm1: model + 1, 0 for the skip child
      if (!pm) {
        csk = psk + 1;
      } else {
        ce = __fns(pm, 0, lane - poff + 1);
        const int mdl = e_model[ce];
        cm1 = mdl + 1;
        cu = pu + e_weight[ce];
        if (!ptch) {
          uint32_t surv;
          double r;
          if (hrow < rows) {
            surv = h_cnt[hrow * M + mdl];
            r = h_rat[hrow * M + mdl];
          } else {
            surv = __ldg(A.hist + ((size_t)slot * N + a) * M + mdl);
            r = (double)surv / initial;
          }
          cfs = pfs + r;
          cfc = pfc + 1;
          cns = (int)surv;
        } else {
          const int surv = s_cnt[par][mdl];
          const double before = (double)pns / initial;
          cfs = pfs + ((double)surv / initial - before);
          cns = surv;
        }
      }
      cf = cfc > 0 ? cfs / cfc : 1.0;
      const uint64_t ku = okey(cu), kf = okey(cf);
      const uint32_t sk = (uint32_t)csk;
      const uint64_t ck = cm1 ? key_base | (uint64_t)(cm1 - 1) : kEnd;
      if (valid) {
        RankKey rk;
        rk.ku = ku;
        rk.kf = kf;
        rk.sk = sk;
        rk.pk = (uint32_t)par | ((uint32_t)cm1 << 8);
        rk.pad = 0;
        s_rk[lane] = rk;
      }
      __syncwarp();
      AG_PHASE_TICK(1);
      // rank under state_better, then the lower child index (never reached:
      // distinct children hold distinct lists).  Pass 1 counts the children
      // with a strictly higher utilization (one 64-bit compare each, keys
      // read four at a time); pass 2 compares the remaining keys only
      // against the children with the same utilization (match_any group).
      const unsigned vmask = __ballot_sync(kFull, valid);
      const unsigned tie = __match_any_sync(kFull, ku) & vmask & ~(1u << lane);
      unsigned rank = 0xffffffffu;
      if (valid) {
        rank = 0;
        for (int c0 = 0; c0 < nchild; c0 += 4) {
          uint64_t yu[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) yu[u] = s_rk[min(c0 + u, 31)].ku;
#pragma unroll
          for (int u = 0; u < 4; ++u) rank += (c0 + u < nchild) & (yu[u] > ku);
        }
        for (unsigned tb = tie; tb; tb &= tb - 1) {
          const RankKey y = s_rk[__ffs(tb) - 1];
          const uint64_t rr = R[y.pk & 31u][par];
          const uint32_t ym1 = y.pk >> 8;
          const uint64_t yk = ym1 ? key_base | (uint64_t)(ym1 - 1) : kEnd;
          const bool lexb = lex_before((int)(y.pk & 31u) == par, rr, yk, ck);
          rank += (y.kf > kf) | ((y.kf == kf) & ((y.sk < sk) | ((y.sk == sk) & lexb)));
        }
      }
      // nested retention (scheduler.cpp:351-370): level w adopts the best
      // unused child of parents < w -- the lowest rank not yet taken in the
      // union of the parents' rank masks
      if (valid) s_picked[rank] = lane;  // rank -> child lane
      uint32_t avail_ranks = 0, taken = 0;
      int myrank = 0;
#pragma unroll 4
      for (int w = 1; w <= B && npick < nchild; ++w) {
        avail_ranks |= __reduce_or_sync(kFull, (valid && par == w - 1) ? 1u << rank : 0u);
        const uint32_t av = avail_ranks & ~taken;
        if (!av) continue;
        const int r = __ffs(av) - 1;
        taken |= 1u << r;
        if (lane == npick) myrank = r;
        ++npick;
      }
      __syncwarp();
      const int src = lane < npick ? s_picked[myrank] : 0;
      c_u = __shfl_sync(kFull, cu, src);
      c_fs = __shfl_sync(kFull, cfs, src);
      c_fc = __shfl_sync(kFull, cfc, src);
      c_sk = __shfl_sync(kFull, csk, src);
      c_ns = __shfl_sync(kFull, cns, src);
      c_par = __shfl_sync(kFull, par, src);
      c_eng = __shfl_sync(kFull, ce, src);
    } else {
      // wide beams: lane w writes its children, per level a warp arg-max
      if (lane < nst) {
        int c = off;
        if (!mk) {
          Child& chd = children[c];
          chd.parent = (int16_t)lane;
          chd.eng = -1;
          chd.util = st_u;
          chd.flex_sum = st_fs;
          chd.flex_count = st_fc;
          chd.skips = st_sk + 1;
          chd.nsurv = st_ns;
          chd.flex = st_fc > 0 ? st_fs / st_fc : 1.0;
        } else {
          for (uint32_t b = mk; b; b &= b - 1, ++c) {
            const int e = __ffs(b) - 1;
            const int mdl = e_model[e];
            Child& chd = children[c];
            chd.parent = (int16_t)lane;
            chd.eng = (int16_t)e;
            chd.util = st_u + e_weight[e];
            chd.skips = st_sk;
            if (!tch) {
              const uint32_t surv = hrow < rows ? h_cnt[hrow * M + mdl]
                                                : A.hist[((size_t)slot * N + a) * M + mdl];
              chd.flex_sum = st_fs + (hrow < rows ? h_rat[hrow * M + mdl] : (double)surv / initial);
              chd.flex_count = st_fc + 1;
              chd.nsurv = (int)surv;
            } else {
              const int surv = s_cnt[lane][mdl];
              const double before = (double)st_ns / initial;
              chd.flex_sum = st_fs + ((double)surv / initial - before);
              chd.flex_count = st_fc;
              chd.nsurv = surv;
            }
            chd.flex = chd.flex_count > 0 ? chd.flex_sum / chd.flex_count : 1.0;
          }
        }
      }
      __syncwarp();
      AG_PHASE_TICK(1);
      auto keyf = [&](int c) -> uint64_t {
        return children[c].eng >= 0 ? key_base | (uint64_t)(uint32_t)e_model[children[c].eng] : kEnd;
      };
      auto before = [&](int c1, int c2) -> bool {  // c1 strictly before c2
        if (c1 < 0) return false;
        if (c2 < 0) return true;
        const Child &x = children[c1], &y = children[c2];
        if (x.util != y.util) return x.util > y.util;
        if (x.flex != y.flex) return x.flex > y.flex;
        if (x.skips != y.skips) return x.skips < y.skips;
        const uint64_t k1 = keyf(c1), k2 = keyf(c2);
        if (x.parent == y.parent && k1 == k2) return c1 < c2;
        return rel_before(rel_extend(x.parent == y.parent, R[x.parent][y.parent], k1, k2));
      };
      constexpr int kUsedWords = (kMaxBeam * (kMaxEng + 1) + 31) / 32;
      uint32_t used[kUsedWords];
      for (int i = 0; i < kUsedWords; ++i) used[i] = 0;
      for (int w = 1; w <= B; ++w) {
        int best = -1;
        for (int c = lane; c < nchild; c += 32) {
          if ((used[c >> 5] >> (c & 31)) & 1u) continue;
          if (children[c].parent >= w) continue;
          if (before(c, best)) best = c;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const int other = __shfl_xor_sync(kFull, best, o);
          if (before(other, best)) best = other;
        }
        if (best < 0) continue;
        used[best >> 5] |= 1u << (best & 31);
        if (lane == 0) s_picked[npick] = best;
        ++npick;
      }
      __syncwarp();
      if (lane < npick) {
        const Child& chd = children[s_picked[lane]];
        c_u = chd.util;
        c_fs = chd.flex_sum;
        c_fc = chd.flex_count;
        c_sk = chd.skips;
        c_ns = chd.nsurv;
        c_par = chd.parent;
        c_eng = chd.eng;
      }
    }
    AG_PHASE_TICK(2);
    // adopt: picked child w becomes state w of the next beam
    const int nxt = cur ^ 1;
    const bool mine = lane < npick;
    if (!mine) c_par = 0, c_eng = -1;
    const uint32_t p_fm = __shfl_sync(kFull, st_fm, c_par);
    const int p_nd = __shfl_sync(kFull, st_nd, c_par);
    const int p_lq = __shfl_sync(kFull, st_lq, c_par);
    const int p_ln = __shfl_sync(kFull, st_ln, c_par);
    const bool mknode = c_eng >= 0;
    const uint32_t nb = __ballot_sync(kFull, mknode);
    if (nnodes + __popc(nb) > A.max_nodes) wstatus = AG_ERR_INTERNAL + 300;  // history overflow (uniform)
    const int c_mdl = mknode ? e_model[c_eng] : 0;
    const uint64_t mykey = mknode ? key_base | (uint64_t)(uint32_t)c_mdl : kEnd;
    // occupancy rows of the new states: lane (w, e) takes engine e of the
    // parent of state w, plus one on the adopted engine; p_occ = the parent's
    // occupancy of the adopted engine (for state w's free mask)
    int p_occ = 0;
    if (regocc) {
      p_occ = __shfl_sync(kFull, occ_r, (c_par << lgE) + (mknode ? c_eng : 0));
      const int pw = __shfl_sync(kFull, c_par, ow);
      const int ew = __shfl_sync(kFull, c_eng, ow);
      occ_r = __shfl_sync(kFull, occ_r, (pw << lgE) + oe) + (oe == ew ? 1 : 0);
    } else {
      if (mine && mknode) p_occ = s_occ[cur][c_par][c_eng];
      for (int i0 = 0; i0 < (npick << lgE); i0 += 32) {
        const int i = i0 + lane, w = min(i >> lgE, 31), e = i & ((1 << lgE) - 1);
        const int pw = __shfl_sync(kFull, c_par, w);
        const int ew = __shfl_sync(kFull, c_eng, w);
        if (w < npick && e < E) s_occ[nxt][w][e] = s_occ[cur][pw][e] + (e == ew ? 1 : 0);
      }
    }
    if (mine) {
      st_u = c_u;
      st_fs = c_fs;
      st_fc = c_fc;
      st_sk = c_sk;
      st_ns = c_ns;
      st_fm = p_fm;
      if (mknode) {
        if (p_occ + 1 >= e_slots[c_eng]) st_fm &= ~(1u << c_eng);
        const int id = nnodes + __popc(nb & lt);
        if (!wstatus) {
          Node nd;
          nd.qi = qcur;
          nd.am = (a << 8) | c_mdl;
          nd.prev = p_nd;
          nd.depth = p_ln + 1;
          nd.nsurv = c_ns;
          nd.nvia = cr.nvia;
          nd.slot = slot;
          nd.pad = 0;
          if (id < kSmemNodes) s_nodes[id] = nd;
          else A.gnodes[id - kSmemNodes] = nd;
        }
        st_nd = id;
        st_lq = qcur;
        st_ln = p_ln + 1;
      } else {
        st_nd = p_nd;
        st_lq = p_lq;
        st_ln = p_ln;
      }
    }
    // triples_less relation of the new beam: lane (w1, w2) per ordered pair
    {
      const int lgP = npick <= 1 ? 0 : 32 - __clz(npick - 1);
      for (int i0 = 0; i0 < (1 << (2 * lgP)); i0 += 32) {
        const int i = i0 + lane, w1 = min(i >> lgP, 31), w2 = i & ((1 << lgP) - 1);
        const int p1 = __shfl_sync(kFull, c_par, w1), p2 = __shfl_sync(kFull, c_par, w2);
        const uint64_t k1 = __shfl_sync(kFull, mykey, w1), k2 = __shfl_sync(kFull, mykey, w2);
        if (w1 < npick && w2 < npick && w1 != w2)
          s_rel[nxt][w1][w2] = rel_extend_sel(p1 == p2, R[p1][p2], k1, k2);
      }
    }
    nnodes += __popc(nb);
    __syncwarp();
    cur = nxt;
    nst = npick;
    AG_PHASE_TICK(3);
  }
  if (regocc && ow < nst && oe < E) s_occ[cur][ow][oe] = occ_r;
  __syncwarp();
  // producers stop at their next chunk boundary
  if (lane == 0) *(volatile unsigned*)&s_walk_done = 1u;
  if (lane == 0 && A.timing) {
#pragma unroll
    for (int k = 0; k < 4; ++k) A.timing[5 + k] = (unsigned long long)tw[k];
    A.timing[9] = n_steps;
    A.timing[10] = n_child;
    A.timing[3] = gtimer();
  }
  // RoundContext validation covers every pair: wait for the full scan
  if (check_all) {
    if (lane == 0)
      while (!ld_acquire(&s_prod_done)) {
      }
    __syncwarp();
    if (s_status) wstatus = s_status;
  }
  if (wstatus) {
    if (lane == 0) round_done(A, wstatus, 0);
    return;
  }
  {  // the remaining pairs are skips (all-full exit or no candidate left)
    const long long rem = A.npairs - pi;
    if (rem > 0) {
      if (lane < nst) st_sk += rem;
      explored += (unsigned long long)nst * (unsigned long long)rem;
    }
  }

  // ---- winner and finalize (scheduler.cpp:373-377, 208-220, 248-287)
  const uint64_t(*R)[kMaxBeam] = s_rel[cur];
  double bu = st_u, bf = st_fc > 0 ? st_fs / st_fc : 1.0;
  long long bsk = st_sk;
  int best = lane < nst ? lane : -1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ou = __shfl_xor_sync(kFull, bu, o);
    const double of = __shfl_xor_sync(kFull, bf, o);
    const long long os = __shfl_xor_sync(kFull, bsk, o);
    const int other = __shfl_xor_sync(kFull, best, o);
    if (other < 0) continue;
    bool o_better;  // is `other` strictly better than `best`?
    if (best < 0) o_better = true;
    else if (ou != bu) o_better = ou > bu;
    else if (of != bf) o_better = of > bf;
    else if (os != bsk) o_better = os < bsk;
    else o_better = rel_before(R[other][best]);
    if (o_better) best = other, bu = ou, bf = of, bsk = os;
  }
  const int w_nd = __shfl_sync(kFull, st_nd, best);
  const int D = __shfl_sync(kFull, st_ln, best);
  ag_assignment* res = reinterpret_cast<ag_assignment*>((char*)A.out + kOutHeader);
  int32_t* occ_out = reinterpret_cast<int32_t*>(res + 1);
  ag_triple* triples = reinterpret_cast<ag_triple*>(occ_out + kMaxEng);
  if (D > A.triples_cap) {
    if (lane == 0) round_done(A, AG_ERR_VALIDATION + 400, D);
    return;
  }
  // the path, root first (node ids into the children area, free now)
  int* path = reinterpret_cast<int*>(children);
  const int path_cap = (int)(sizeof(Child) * A.max_children / sizeof(int));
  if (lane == 0) {
    int n = w_nd;
    for (int i = D - 1; i >= 0; --i) {
      if (i < path_cap) path[i] = n;
      n = nv[n].prev;
    }
  }
  __syncwarp();
  double* fr = reinterpret_cast<double*>(s_cnt);  // per-request ratios (<= 512)
  bool ascending = D <= path_cap;
  for (int i0 = 0; i0 < D; i0 += 32) {
    const int i = i0 + lane;
    int n = -1;
    if (i < D) {
      if (i < path_cap) {
        n = path[i];
      } else {  // long path: walk from the winner (rare)
        n = w_nd;
        for (int k = D - 1; k > i; --k) n = nv[n].prev;
      }
      const Node nd = nv[n];
      ag_triple t;
      t.request_index = nd.qi;
      t.agent = nd.am >> 8;
      t.model = nd.am & 0xFF;
      t.slot = nd.slot;
      t.request_id = A.ids[nd.slot];
      triples[i] = t;
    }
    if (ascending) {
      // a request's triples are consecutive on the path; in a session the
      // queue is in FIFO = container order, so requests appear ascending
      const bool viol = i + 1 < D && nv[n].qi > nv[path[i + 1]].qi;
      if (__any_sync(kFull, viol)) ascending = false;
    }
  }
  __syncwarp();
  double flex_sum = 0.0;
  int flex_count = 0;
  if (D > 0 && ascending && D <= (int)(sizeof(s_cnt) / sizeof(double))) {
    // the last triple of each request carries its survivors; fold in order
    for (int i = lane; i < D; i += 32) {
      const Node& nd = nv[path[i]];
      const bool last = i + 1 == D || nv[path[i + 1]].qi != nd.qi;
      fr[i] = last ? (double)nd.nsurv / (double)nd.nvia : -1.0;
    }
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < D; ++i)
        if (fr[i] >= 0.0) {
          flex_sum += fr[i];
          ++flex_count;
        }
  } else if (D > 0 && lane == 0) {
    // general container order: repeatedly take the smallest unseen request
    int prev = -1;
    for (;;) {
      int nq = 0x7fffffff;
      for (int i = 0; i < D; ++i) {
        const int q = triples[i].request_index;
        if (q > prev && q < nq) nq = q;
      }
      if (nq == 0x7fffffff) break;
      for (int nn = w_nd; nn >= 0; nn = nv[nn].prev)
        if (nv[nn].qi == nq) {
          flex_sum += (double)nv[nn].nsurv / (double)nv[nn].nvia;
          ++flex_count;
          break;
        }
      prev = nq;
    }
  }
  if (lane != 0) return;
  // score_assignment: utilization in engine order
  double util = 0.0;
  for (int k = 0; k < E; ++k) {  // the caller's engine order
    const int e = A.eng.inv[k];
    const int o = s_occ[cur][best][e];
    if (o < 0 || o > e_slots[e]) {
      round_done(A, AG_ERR_VALIDATION + 500, 0);
      return;
    }
    util += o * e_weight[e];
    occ_out[k] = o;
  }
  ag_assignment r;
  r.n_triples = D;
  r.pad = 0;
  r.utilization = util;
  r.flexibility = flex_count > 0 ? flex_sum / flex_count : 1.0;
  r.skips = bsk;
  r.states_explored = explored;
  *res = r;
  if (A.timing) A.timing[4] = gtimer();
  round_done(A, 0, 0);
}

// ------------------------------------------------------------ prune kernel
struct PruneArgs {
  int N, M;
  const int32_t* g_slot;   // [G] slot per group
  const int32_t* g_begin;  // [G+1] ranges into g_am
  const int32_t* g_am;     // agent << 8 | model, in apply order
  const uint64_t* g_meta;  // [G*3] (voff, nviable, id) for new requests, or null
  uint32_t* pool;
  uint64_t* voff;
  uint32_t* nviable;
  uint64_t* ids;
  uint32_t* hist;
  uint32_t* cand;
  uint32_t place[kMaxAgents];
  uint64_t place_magic[kMaxAgents];
  uint64_t div_m;
  int32_t* status;
  uint32_t* ever;  // OR of every installed candidate-model mask (round validation)
  // small dispatches: g_slot / g_begin / g_am travel in the parameter block
  // (no staging copy, no wait for the previous one); g_* then point here
  int inl;
  int32_t inl_data[kPruneInline];
};

__device__ __forceinline__ uint32_t digit_p(uint32_t c, int a, const PruneArgs& A) {
  const uint32_t q = A.place[a] == 1 ? c : (uint32_t)__umul64hi(c, A.place_magic[a]);
  return q - divm(q, A.div_m) * (uint32_t)A.M;
}

// Request::mark_dispatched prefix pruning (request.cpp:70-86) for every
// triple of one request, then its histogram / candidate masks from scratch.
// With g_meta it first installs a new request's metadata (Request::make).
__global__ void __launch_bounds__(256) k_sched_prune(const __grid_constant__ PruneArgs A) {
  __shared__ uint32_t s_hist[kMaxAgents * 32];
  __shared__ int s_w[8], s_tot;
  const int g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x;
  const int32_t* g_slot = A.inl ? A.inl_data : A.g_slot;
  const int32_t* g_begin = A.inl ? A.inl_data + G : A.g_begin;
  const int32_t* g_am = A.inl ? A.inl_data + 2 * G + 1 : A.g_am;
  const int s = g_slot[g];
  uint64_t vo;
  uint32_t len;
  if (A.g_meta) {
    vo = A.g_meta[3 * g];
    len = (uint32_t)A.g_meta[3 * g + 1];
    if (tid == 0) {
      A.voff[s] = vo;
      A.nviable[s] = len;
      A.ids[s] = A.g_meta[3 * g + 2];
    }
  } else {
    vo = A.voff[s];
    len = A.nviable[s];
  }
  uint32_t* vl = A.pool + vo;
  for (int t = g_begin[g]; t < g_begin[g + 1]; ++t) {
    const int a = g_am[t] >> 8, mdl = g_am[t] & 0xFF;
    // count survivors first: an empty result leaves the list untouched
    int c = 0;
    for (uint32_t q = tid; q < len; q += blockDim.x) c += (int)digit_p(vl[q], a, A) == mdl;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) s_w[wid] = c;
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int k = 0; k < (int)(blockDim.x / 32); ++k) tot += s_w[k];
      s_tot = tot;
    }
    __syncthreads();
    const int kept = s_tot;
    if (kept == 0) {
      if (tid == 0) atomicExch(A.status, AG_ERR_VALIDATION);  // model is not a viable candidate
      return;
    }
    // stable in-place compaction, one block-wide chunk at a time
    uint32_t wpos = 0;
    for (uint32_t b0 = 0; b0 < len; b0 += blockDim.x) {
      const uint32_t q = b0 + tid;
      const uint32_t v = q < len ? vl[q] : 0u;
      const bool keep = q < len && (int)digit_p(v, a, A) == mdl;
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) s_w[wid] = __popc(bal);
      __syncthreads();
      int pre = 0, tot = 0;
      for (int k = 0; k < (int)(blockDim.x / 32); ++k) {
        if (k < wid) pre += s_w[k];
        tot += s_w[k];
      }
      pre += __popc(bal & ((1u << lane) - 1u));
      __syncthreads();
      if (keep) vl[wpos + pre] = v;
      wpos += tot;
      __syncthreads();
    }
    len = (uint32_t)kept;
  }
  // histogram + candidate masks (candidate_models, request.cpp:60-68)
  for (int i = tid; i < A.N * A.M; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  for (uint32_t q = tid; q < len; q += blockDim.x) {
    const uint32_t v = vl[q];
    for (int a = 0; a < A.N; ++a) atomicAdd(&s_hist[a * A.M + digit_p(v, a, A)], 1u);
  }
  __syncthreads();
  uint32_t* h = A.hist + (size_t)s * A.N * A.M;
  for (int i = tid; i < A.N * A.M; i += blockDim.x) h[i] = s_hist[i];
  if (tid < A.N) {
    uint32_t cm = 0;
    for (int mdl = 0; mdl < A.M; ++mdl)
      if (s_hist[tid * A.M + mdl]) cm |= 1u << mdl;
    A.cand[(size_t)s * A.N + tid] = cm;
    if (A.g_meta) atomicOr(A.ever, cm);
  }
  if (tid == 0) A.nviable[s] = len;
}

// snapshot_load's queued_ahead (simulation.cpp:194-213): per tier, ready
// pairs whose candidate models include it.  Dead slots have ready == 0.
__global__ void __launch_bounds__(256)
    k_queued_ahead(const int32_t* __restrict__ order, int Q, const uint64_t* __restrict__ ready,
                   const uint32_t* __restrict__ cand, int N, int M, int n_upd,
                   const int32_t* __restrict__ upd_slot, const uint64_t* __restrict__ upd_mask,
                   uint32_t* __restrict__ out) {
  __shared__ uint32_t h[32];
  if (threadIdx.x < 32) h[threadIdx.x] = 0;
  __syncthreads();
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < Q; p += gridDim.x * blockDim.x) {
    const int s = order[p];
    uint64_t r = ready[s];
    for (int i = 0; i < n_upd; ++i)  // pending host-side updates win
      if (upd_slot[i] == s) r = upd_mask[i];
    for (uint64_t b = r; b; b &= b - 1) {
      const int a = __ffsll((long long)b) - 1;
      for (uint32_t c = cand[(size_t)s * N + a]; c; c &= c - 1) atomicAdd(&h[__ffs(c) - 1], 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x < M) atomicAdd(out + threadIdx.x, h[threadIdx.x]);
}

// audit_round_fairness (scheduler.cpp:456-480) of an assignment against the
// session's last round queue, one block.  The reference walks the pairs in
// two-level order with a cursor into the triples: a triple counts as assigned
// only while the triples match pairs in increasing pair order (the matched
// prefix, length L); at an unassigned pair the state is initial_state
// extended by the matched triples before it, so its allowed_engines is the
// pair's candidate engines (or, for a request re-touched earlier in the
// round, the models at the agent over the viable configurations consistent
// with its earlier triples) & the free mask after those triples.  A
// non-empty mask is a violation.
struct AuditArgs {
  int N, M, Q, n;
  const int32_t* order;
  const uint64_t* ready;
  const uint32_t* cand;
  const uint64_t* ids;
  const uint64_t* voff;
  const uint32_t* nviable;
  const uint32_t* pool;
  const int4* trip;  // {request_index, agent, model, -}
  int32_t* q_slot;   // scratch [Q]: slot of the q-th request of the queue
  const int32_t* cidx;  // stateless call: container index per FIFO position (else null)
  int32_t* c_rank;      // scratch [Q]: queue rank of each container index
  int8_t prio_rank[64];
  EngDev eng;
  uint32_t place[kMaxAgents];
  uint64_t place_magic[kMaxAgents];
  uint64_t div_m;
  uint64_t* out_ids;
  int32_t* out_agents;
  int cap;
  int32_t* out;  // [0] violations, [1] status, [2] matched triples
};

__device__ __forceinline__ uint32_t digit_a(uint32_t c, int a, const AuditArgs& A) {
  const uint32_t q = A.place[a] == 1 ? c : (uint32_t)__umul64hi(c, A.place_magic[a]);
  return q - divm(q, A.div_m) * (uint32_t)A.M;
}

constexpr int kAuditThreads = 1024, kAuditMaxTrip = 2048;

__global__ void __launch_bounds__(kAuditThreads, 1) k_sched_audit(const __grid_constant__ AuditArgs A) {
  __shared__ int s_wsum[32];
  __shared__ int s_carry, s_L, s_status;
  __shared__ uint32_t s_key[kAuditMaxTrip];  // q << 6 | priority rank of the agent
  __shared__ uint32_t s_fm[kAuditMaxTrip + 1];
  __shared__ int s_model[kAuditMaxTrip];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int per = (A.Q + kAuditThreads - 1) / kAuditThreads;
  const int p0 = tid * per, p1 = min(A.Q, p0 + per);
  // A: queue index of every FIFO position with a ready stage
  int nq = 0;
  for (int p = p0; p < p1; ++p) nq += A.ready[A.order[p]] != 0;
  auto block_scan = [&](int x, int* total) -> int {  // exclusive
    int y = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += t;
    }
    if (lane == 31) s_wsum[w] = y;
    __syncthreads();
    if (w == 0) {
      const int v = s_wsum[lane];
      int z = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += t;
      }
      s_wsum[lane] = z - v;
      if (lane == 31) s_carry = z;
    }
    __syncthreads();
    const int r = s_wsum[w] + y - x;
    *total = s_carry;
    __syncthreads();
    return r;
  };
  int n_queue = 0;
  const int q0 = block_scan(nq, &n_queue);
  if (A.cidx)
    for (int i = tid; i < A.Q; i += kAuditThreads) A.c_rank[i] = -1;
  __syncthreads();
  {
    int q = q0;
    for (int p = p0; p < p1; ++p) {
      const int sl = A.order[p];
      if (!A.ready[sl]) continue;
      if (A.cidx) {
        const int c = A.cidx[p];
        if (c >= 0 && c < A.Q) A.c_rank[c] = q;
      }
      A.q_slot[q++] = sl;
    }
  }
  if (tid == 0) s_status = 0;
  __syncthreads();
  // B: the matched prefix of the triples (valid pairs in strictly increasing
  // pair order) and the free mask after each of its triples
  const int n = min(A.n, kAuditMaxTrip);
  int first_bad = n;
  for (int k = tid; k < n; k += kAuditThreads) {
    const int4 t = A.trip[k];
    // the triple's queue rank (container order -> FIFO rank for a stateless call)
    const int qr = A.cidx ? (t.x >= 0 && t.x < A.Q ? A.c_rank[t.x] : -1) : t.x;
    bool ok = qr >= 0 && qr < n_queue && t.y >= 0 && t.y < A.N;
    uint32_t key = 0;
    if (ok) {
      ok = (A.ready[A.q_slot[qr]] >> t.y) & 1ull;
      key = ((uint32_t)qr << 6) | (uint32_t)A.prio_rank[t.y];
    }
    s_key[k] = key;
    s_model[k] = t.z;
    if (!ok) first_bad = min(first_bad, k);
  }
  __syncthreads();
  for (int k = tid; k < n; k += kAuditThreads)
    if (k > 0 && s_key[k] <= s_key[k - 1]) first_bad = min(first_bad, k);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) first_bad = min(first_bad, __shfl_xor_sync(0xffffffffu, first_bad, o));
  if (tid == 0) s_L = n;
  __syncthreads();
  if (lane == 0) atomicMin(&s_L, first_bad);
  __syncthreads();
  const int L = s_L;
  if (tid == 0) {
    // initial_state (scheduler.cpp:117-128) and extend_state's free mask
    int occ[kMaxEng];
    uint32_t fm = 0;
    for (int e = 0; e < A.eng.E; ++e) {
      occ[e] = A.eng.occ[e];
      if (occ[e] > A.eng.slots[e] || occ[e] < 0) s_status = AG_ERR_VALIDATION + 200;
      if (occ[e] < A.eng.slots[e]) fm |= 1u << e;
    }
    s_fm[0] = fm;
    for (int k = 0; k < L; ++k) {
      const int mdl = s_model[k];
      const int e = mdl >= 0 && mdl < 32 ? A.eng.m2e[mdl] : -1;
      if (e < 0) {
        s_status = AG_ERR_VALIDATION + 300;  // a triple names a model without a pool
        break;
      }
      if (++occ[e] >= A.eng.slots[e]) fm &= ~(1u << e);
      s_fm[k + 1] = fm;
    }
  }
  __syncthreads();
  if (s_status) {
    if (tid == 0) A.out[1] = s_status;
    return;
  }
  // C: every pair in order; violations counted per thread, then written in
  // pair order
  int nv = 0;
  bool bad_tier = false;
  for (int pass = 0; pass < 2; ++pass) {
    int wbase = 0;
    if (pass == 1) {
      int tot = 0;
      wbase = block_scan(nv, &tot);
      if (tid == 0) A.out[0] = tot;
    }
    int q = q0, o = wbase;
    for (int p = p0; p < p1; ++p) {
      const int sl = A.order[p];
      const uint64_t r = A.ready[sl];
      if (!r) continue;
      // ready agents in (depth desc, declaration asc) order = by priority rank
      uint64_t left = r;
      while (left) {
        int a = -1, br = 1 << 30;
        for (uint64_t b = left; b; b &= b - 1) {
          const int ag = __ffsll((long long)b) - 1;
          if (A.prio_rank[ag] < br) br = A.prio_rank[ag], a = ag;
        }
        left &= ~(1ull << a);
        const uint32_t key = ((uint32_t)q << 6) | (uint32_t)br;
        int lo = 0, hi = L;  // lower_bound of key in the matched prefix
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (s_key[mid] < key) lo = mid + 1; else hi = mid;
        }
        if (lo < L && s_key[lo] == key) continue;  // assigned
        const uint32_t cm = A.cand[(size_t)sl * A.N + a];
        bad_tier |= (cm & ~A.eng.mapped) != 0u;
        uint32_t models = cm;
        if (lo > 0 && (s_key[lo - 1] >> 6) == (uint32_t)q) {
          // re-touched request: models at agent a over the viable
          // configurations consistent with its earlier triples this round
          int k0 = lo;
          while (k0 > 0 && (s_key[k0 - 1] >> 6) == (uint32_t)q) --k0;
          models = 0;
          const uint32_t* vl = A.pool + A.voff[sl];
          for (uint32_t j = 0; j < A.nviable[sl]; ++j) {
            const uint32_t c = vl[j];
            bool okc = true;
            for (int k = k0; k < lo && okc; ++k)
              okc = (int)digit_a(c, A.trip[k].y, A) == s_model[k];
            if (okc) models |= 1u << digit_a(c, a, A);
          }
        }
        uint32_t em = 0;
        for (uint32_t b = models; b; b &= b - 1) {
          const int e = A.eng.m2e[__ffs(b) - 1];
          if (e >= 0) em |= 1u << e;
        }
        if (em & s_fm[lo]) {
          if (pass == 0) {
            ++nv;
          } else {
            if (o < A.cap) {
              A.out_ids[o] = A.ids[sl];
              A.out_agents[o] = a;
            }
            ++o;
          }
        }
      }
      ++q;
    }
  }
  if (__syncthreads_or(bad_tier) && tid == 0) A.out[1] = AG_ERR_VALIDATION + 100;
  if (tid == 0) A.out[2] = L;
}

}  // namespace
}  // namespace agb

// ============================================================ host session
struct ag_sched {
  ag_ctx* ctx = nullptr;
  int N = 0, M = 0;
  int cap = 0;
  uint64_t pool_cap = 0, pool_top = 0;
  // host mirror of Request state
  std::vector<uint64_t> ids;
  std::vector<double> arrival;
  std::vector<uint8_t> stages;  // [cap * N]
  std::vector<uint64_t> ready;  // [cap]
  std::vector<char> live;
  std::vector<uint32_t> nviable;
  std::vector<int32_t> free_slots;
  std::vector<int32_t> quarantine;  // freed slots still listed on the device
  // device queue order: live and dead (ready 0) slots in FIFO order; host copy
  std::vector<int32_t> order;
  size_t dirty_from = 0;  // device copy valid before this index
  size_t pinfo_from = 0;  // device pair records (pinfo) valid before this index
  std::vector<int32_t> pos_of;  // slot -> FIFO position (-1: not listed)
  size_t dead = 0;
  std::vector<int32_t> upd_slot;
  std::vector<uint64_t> upd_mask;
  long long npairs = 0;  // ready pairs over live slots (sum of popcount(ready))
  std::vector<uint32_t> seen;  // update dedup stamps
  uint32_t seen_stamp = 0;
  int8_t prio[64];
  uint32_t place[agb::kMaxAgents];
  uint64_t place_magic[agb::kMaxAgents];
  bool attr_set = false;
  int walker = 0;  // AG_SCHED_WALKER: 0 automatic, 1 always the general walker
  uint32_t round_seq = 0;
  double last_round_us = 0.0;
  double host_us[4] = {0, 0, 0, 0};  // last round: prep, launch call, wait, readback (host clock)
  // session changes since creation; the audit needs the last round's queue
  uint64_t epoch = 1, round_epoch = 0;
  uint64_t stateless_fp = 0;  // fingerprint of the queue of the last stateless round
  agb::Scratch d_audit;
  // device
  agb::Scratch d_ready, d_cand, d_hist, d_nv, d_voff, d_pool, d_ids, d_order, d_cidx, d_pinfo;
  agb::Scratch d_cpos, d_det, d_nodes, d_status, d_gam, d_qa, d_upd;  // d_cpos / d_det: candidate overflow
  // pinned host staging
  void* h_res = nullptr;
  size_t h_res_bytes = 0;
  void* h_stage = nullptr;  // dispatch / add uploads
  size_t h_stage_bytes = 0;
  void* h_rstage = nullptr;  // round uploads
  size_t h_rstage_bytes = 0;
  // device views of the mapped buffers (refreshed when reallocated)
  void* h_rstage_mapped = nullptr;
  void* h_res_mapped = nullptr;
  char* h_rstage_dev = nullptr;
  int32_t* h_res_dev = nullptr;
  void* h_vstage = nullptr;  // viable lists of added requests
  size_t h_vstage_bytes = 0;
  void* h_ostage = nullptr;  // FIFO re-uploads after a compaction
  size_t h_ostage_bytes = 0;
  void* h_fstage = nullptr;  // eager refresh records (refresh_records)
  size_t h_fstage_bytes = 0;
  cudaEvent_t fstage_free = nullptr;  // the last copy out of h_fstage
  agb::Scratch d_frec;
  agb::Scratch d_pool2, d_pscan;  // pool compaction: the other pool, live slots + offsets
  size_t dev_q = 0;               // positions holding records on the device
  ~ag_sched() {
    if (h_res) cudaFreeHost(h_res);
    if (h_stage) cudaFreeHost(h_stage);
    if (h_rstage) cudaFreeHost(h_rstage);
    if (h_ostage) cudaFreeHost(h_ostage);
    if (h_fstage) cudaFreeHost(h_fstage);
    if (fstage_free) cudaEventDestroy(fstage_free);
    if (h_vstage) cudaFreeHost(h_vstage);
  }
};

namespace agb {
namespace {

int ensure_pinned(void** p, size_t* have, size_t bytes) {
  if (bytes <= *have) return AG_OK;
  const size_t b = std::max<size_t>(std::max<size_t>(bytes, 4096), *have + *have / 2);
  if (*p) cudaFreeHost(*p);
  *p = nullptr;
  *have = 0;
  AG_CUDA(cudaHostAlloc(p, b, cudaHostAllocMapped));
  *have = b;
  return AG_OK;
}

// device view of mapped pinned memory
template <typename T>
int dev_ptr(void* host, T** out) {
  void* d = nullptr;
  AG_CUDA(cudaHostGetDevicePointer(&d, host, 0));
  *out = reinterpret_cast<T*>(d);
  return AG_OK;
}

// the host mirror of Request::ready_agents and the queue's pair count
void set_ready(ag_sched* s, int slot, uint64_t r) {
  s->npairs += (long long)__builtin_popcountll(r) - (long long)__builtin_popcountll(s->ready[slot]);
  s->ready[slot] = r;
  s->upd_slot.push_back(slot);
  s->upd_mask.push_back(r);
}

uint64_t ready_of(const ag_sched* s, int slot) {
  uint64_t r = 0;
  for (int a = 0; a < s->N; ++a)
    if (s->stages[(size_t)slot * s->N + a] == AG_STAGE_READY) r |= 1ull << a;
  return r;
}

bool fifo_less(const ag_sched* s, int x, int y) {
  if (s->arrival[x] != s->arrival[y]) return s->arrival[x] < s->arrival[y];
  return s->ids[x] < s->ids[y];
}

void compact_order(ag_sched* s) {
  std::vector<int32_t> live_order;
  live_order.reserve(s->order.size());
  for (int slot : s->order) {
    s->pos_of[slot] = -1;
    if (s->live[slot]) live_order.push_back(slot);
  }
  s->order.swap(live_order);
  for (size_t p = 0; p < s->order.size(); ++p) s->pos_of[s->order[p]] = (int32_t)p;
  s->dirty_from = 0;
  s->pinfo_from = 0;
  s->dead = 0;
  s->free_slots.insert(s->free_slots.end(), s->quarantine.begin(), s->quarantine.end());
  s->quarantine.clear();
}

// A long dirty FIFO tail (after a compaction or a large add) is copied now,
// outside the next round's decision latency.
int flush_order(ag_sched* s) {
  const size_t Q = s->order.size();
  if (Q <= s->dirty_from || Q - s->dirty_from < 4096) return AG_OK;
  const size_t n = Q - s->dirty_from;
  // the staging buffer may still be in use by an earlier async copy
  AG_CUDA(cudaStreamSynchronize(s->ctx->stream));
  int rc = ensure_pinned(&s->h_ostage, &s->h_ostage_bytes, n * 4);
  if (rc) return rc;
  std::memcpy(s->h_ostage, s->order.data() + s->dirty_from, n * 4);
  AG_CUDA(cudaMemcpyAsync((int32_t*)s->d_order.p + s->dirty_from, s->h_ostage, n * 4, cudaMemcpyHostToDevice,
                          s->ctx->stream));
  s->dirty_from = Q;
  return AG_OK;
}

int launch_prune_args(ag_sched* s, PruneArgs& A, int G, bool prep);

int launch_prune(ag_sched* s, const std::vector<int32_t>& g_slot, const std::vector<int32_t>& g_begin,
                 const std::vector<int32_t>& g_am, const std::vector<uint64_t>* meta) {
  ag_ctx* ctx = s->ctx;
  const int G = (int)g_slot.size();
  if (G == 0) return AG_OK;
  int rc;
  const size_t n32 = (size_t)G + (G + 1) + g_am.size();
  PruneArgs A;
  if (!meta && n32 <= (size_t)kPruneInline) {
    A.inl = 1;
    std::memcpy(A.inl_data, g_slot.data(), 4 * (size_t)G);
    std::memcpy(A.inl_data + G, g_begin.data(), 4 * (size_t)(G + 1));
    if (!g_am.empty()) std::memcpy(A.inl_data + 2 * G + 1, g_am.data(), 4 * g_am.size());
    A.g_slot = A.g_begin = A.g_am = nullptr;
    A.g_meta = nullptr;
    return launch_prune_args(s, A, G, false);
  }
  A.inl = 0;
  const size_t off_meta = (n32 * 4 + 15) & ~(size_t)15;
  const size_t bytes = off_meta + (meta ? meta->size() * 8 : 0);
  if ((rc = s->d_gam.ensure(bytes))) return rc;
  if ((rc = ensure_pinned(&s->h_stage, &s->h_stage_bytes, bytes))) return rc;
  // the staging buffer may still be in use by an earlier async copy
  AG_CUDA(cudaStreamSynchronize(ctx->stream));
  char* h = (char*)s->h_stage;
  int32_t* h32 = (int32_t*)h;
  std::memcpy(h32, g_slot.data(), 4 * (size_t)G);
  std::memcpy(h32 + G, g_begin.data(), 4 * (size_t)(G + 1));
  if (!g_am.empty()) std::memcpy(h32 + 2 * G + 1, g_am.data(), 4 * g_am.size());
  if (meta) std::memcpy(h + off_meta, meta->data(), meta->size() * 8);
  AG_CUDA(cudaMemcpyAsync(s->d_gam.p, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
  const int32_t* d = (const int32_t*)s->d_gam.p;
  A.g_slot = d;
  A.g_begin = d + G;
  A.g_am = d + 2 * G + 1;
  A.g_meta = meta ? (const uint64_t*)((const char*)s->d_gam.p + off_meta) : nullptr;
  return launch_prune_args(s, A, G, meta != nullptr);
}

// the session's device arrays into A, then the launch (one block per group)
int launch_prune_args(ag_sched* s, PruneArgs& A, int G, bool prep) {
  ag_ctx* ctx = s->ctx;
  A.N = s->N;
  A.M = s->M;
  A.pool = (uint32_t*)s->d_pool.p;
  A.voff = (uint64_t*)s->d_voff.p;
  A.nviable = (uint32_t*)s->d_nv.p;
  A.ids = (uint64_t*)s->d_ids.p;
  A.hist = (uint32_t*)s->d_hist.p;
  A.cand = (uint32_t*)s->d_cand.p;
  std::memcpy(A.place, s->place, sizeof A.place);
  std::memcpy(A.place_magic, s->place_magic, sizeof A.place_magic);
  A.div_m = ctx->space->dev().div_m;
  A.status = (int32_t*)s->d_status.p;
  A.ever = (uint32_t*)((char*)s->d_status.p + 8);
  {
    Launch L(ctx, prep ? K_SCHED_PREP : K_SCHED_APPLY);
    k_sched_prune<<<G, 256, 0, ctx->stream>>>(A);
  }
  AG_CUDA(cudaGetLastError());
  return AG_OK;
}

int engines_dev(const ag_engines* e, EngDev* out, bool* ordered = nullptr) {
  // RoundContext validation (scheduler.cpp:39-52)
  if (!e) return fail(AG_ERR_VALIDATION, "engines is null");
  if (e->n_engines > kMaxEng) return fail(AG_ERR_VALIDATION, "more engine pools than the scheduler supports");
  EngDev d{};
  d.E = e->n_engines;
  for (int i = 0; i < 32; ++i) d.m2e[i] = -1;
  bool nan = false;
  for (int i = 0; i < d.E; ++i) {
    const int mdl = e->model[i];
    if (mdl < 0) return fail(AG_ERR_VALIDATION, "engine with negative model tier");
    for (int k = 0; k < i; ++k)
      if (e->model[k] == mdl) return fail(AG_ERR_VALIDATION, "two engine pools serve the same model tier");
    nan |= std::isnan(e->weight[i]);
  }
  // internal order: weight descending, ties by the caller's index
  std::vector<int> ord(d.E);
  std::iota(ord.begin(), ord.end(), 0);
  if (!nan) std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return e->weight[x] > e->weight[y]; });
  for (int i = 0; i < d.E; ++i) {
    const int k = ord[i];
    const int mdl = e->model[k];
    if (mdl < 32) {
      d.m2e[mdl] = (int8_t)i;
      d.mapped |= 1u << mdl;
    }
    d.model[i] = mdl;
    d.slots[i] = e->slots[k];
    d.occ[i] = e->occupancy[k];
    d.weight[i] = e->weight[k];
    d.inv[k] = (int8_t)i;
  }
  if (ordered) *ordered = !nan;
  *out = d;
  return AG_OK;
}

// Packs the live requests' viable lists into the other pool buffer.
int compact_pool(ag_sched* s) {
  ag_ctx* ctx = s->ctx;
  std::vector<int32_t> live;
  for (int i = 0; i < s->cap; ++i)
    if (s->live[i]) live.push_back(i);
  int rc;
  const size_t nl = live.size();
  if ((rc = s->d_pool2.ensure(s->pool_cap * 4)) || (rc = s->d_pscan.ensure(4 * nl + 8 * nl + 64))) return rc;
  char* d = (char*)s->d_pscan.p;
  int32_t* d_live = (int32_t*)d;
  uint64_t* d_off = (uint64_t*)(d + ((4 * nl + 15) & ~(size_t)15));
  uint64_t* d_tot = d_off + nl;
  uint64_t total = 0;
  if (nl) {
    AG_CUDA(cudaMemcpyAsync(d_live, live.data(), 4 * nl, cudaMemcpyHostToDevice, ctx->stream));
    {
      Launch L(ctx, K_SCHED_APPLY);
      k_pool_scan<<<1, 1024, 0, ctx->stream>>>(d_live, (int)nl, (const uint32_t*)s->d_nv.p, d_off, d_tot);
    }
    {
      Launch L(ctx, K_SCHED_APPLY);
      k_pool_copy<<<(unsigned)nl, 256, 0, ctx->stream>>>(d_live, d_off, (const uint32_t*)s->d_nv.p,
                                                         (uint64_t*)s->d_voff.p, (const uint32_t*)s->d_pool.p,
                                                         (uint32_t*)s->d_pool2.p);
    }
    AG_CUDA(cudaGetLastError());
    AG_CUDA(cudaMemcpyAsync(&total, d_tot, 8, cudaMemcpyDeviceToHost, ctx->stream));
  }
  AG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::swap(s->d_pool.p, s->d_pool2.p);
  std::swap(s->d_pool.bytes, s->d_pool2.bytes);
  s->pool_top = total;
  return AG_OK;
}

// Pending ready updates, deduplicated (the last one per slot wins).
void dedup_updates(ag_sched* s) {
  if (s->upd_slot.size() <= 1) return;
  if (s->seen.size() != (size_t)s->cap) s->seen.assign(s->cap, 0);
  const uint32_t stamp = ++s->seen_stamp;
  size_t w = s->upd_slot.size();
  for (size_t i = s->upd_slot.size(); i-- > 0;) {
    const int slot = s->upd_slot[i];
    if (s->seen[slot] == stamp) continue;
    s->seen[slot] = stamp;
    --w;
    s->upd_slot[w] = slot;
    s->upd_mask[w] = s->upd_mask[i];
  }
  s->upd_slot.erase(s->upd_slot.begin(), s->upd_slot.begin() + w);
  s->upd_mask.erase(s->upd_mask.begin(), s->upd_mask.begin() + w);
}

// Refresh records the next round would apply: every FIFO position from the
// first stale one, then the other slots whose ready mask changed.
size_t build_records(ag_sched* s, int32_t* r) {
  const size_t Q = s->order.size();
  const size_t from = std::min(std::min(s->dirty_from, s->pinfo_from), Q);
  size_t n = 0;
  auto put = [&](int32_t pos, int32_t slot) {
    const uint64_t m = s->ready[slot];
    if (r) {
      r[0] = pos, r[1] = slot, r[2] = (int32_t)(uint32_t)m, r[3] = (int32_t)(uint32_t)(m >> 32);
      r += 4;
    }
    ++n;
  };
  for (size_t p = from; p < Q; ++p) put((int32_t)p, s->order[p]);
  for (size_t i = 0; i < s->upd_slot.size(); ++i) {
    const int32_t p = s->pos_of[s->upd_slot[i]];
    if (!(p >= 0 && (size_t)p >= from)) put(p, s->upd_slot[i]);
  }
  // positions a compaction left behind Q: empty records (their bits clear)
  for (size_t p = Q; p < s->dev_q; ++p) {
    if (r) {
      r[0] = (int32_t)p, r[1] = -1, r[2] = 0, r[3] = 0;
      r += 4;
    }
    ++n;
  }
  if (r) s->dev_q = Q;
  return n;
}

// Applies large pending record batches now (FIFO compaction, arrival
// batches), asynchronously on the stream, so the next round's decision only
// carries the small per-round deltas.
constexpr size_t kEagerRecords = 256;

int refresh_records(ag_sched* s, bool force) {
  const size_t Q = s->order.size();
  const size_t from = std::min(std::min(s->dirty_from, s->pinfo_from), Q);
  if (!force && (Q - from) + s->upd_slot.size() + (s->dev_q > Q ? s->dev_q - Q : 0) <= kEagerRecords) return AG_OK;
  dedup_updates(s);
  const size_t n = build_records(s, nullptr);
  if (n == 0) return AG_OK;
  ag_ctx* ctx = s->ctx;
  int rc;
  if (!s->fstage_free) AG_CUDA(cudaEventCreateWithFlags(&s->fstage_free, cudaEventDisableTiming));
  AG_CUDA(cudaEventSynchronize(s->fstage_free));  // h_fstage's previous copy is done
  if ((rc = ensure_pinned(&s->h_fstage, &s->h_fstage_bytes, n * 16)) || (rc = s->d_frec.ensure(n * 16))) return rc;
  build_records(s, (int32_t*)s->h_fstage);
  AG_CUDA(cudaMemcpyAsync(s->d_frec.p, s->h_fstage, n * 16, cudaMemcpyHostToDevice, ctx->stream));
  AG_CUDA(cudaEventRecord(s->fstage_free, ctx->stream));
  RefreshArgs A;
  A.N = s->N;
  A.ready = (uint64_t*)s->d_ready.p;
  A.cand = (const uint32_t*)s->d_cand.p;
  A.nviable = (const uint32_t*)s->d_nv.p;
  A.order = (int32_t*)s->d_order.p;
  A.pinfo = (uint4*)s->d_pinfo.p;
  for (int i = 0; i < 64; ++i) A.prio_rank[i] = 0;
  for (int t = 0; t < s->N; ++t) A.prio_rank[(int)s->prio[t]] = (int8_t)t;
  {
    Launch L(ctx, K_SCHED_PREP);
    const unsigned blocks = (unsigned)std::min<size_t>(148, (n + 255) / 256);
    k_sched_refresh<<<blocks, 256, 0, ctx->stream>>>((const int4*)s->d_frec.p, (int)n, A);
  }
  AG_CUDA(cudaGetLastError());
  s->dirty_from = Q;
  s->pinfo_from = Q;
  s->upd_slot.clear();
  s->upd_mask.clear();
  return AG_OK;
}

// One round over the session queue (or an explicit FIFO/container mapping).
constexpr size_t kMappedMax = 32 * 1024;  // round deltas read over PCIe by the kernel

int run_round(ag_sched* s, const ag_engines* engines, int B, const int32_t* cidx_host,
              ag_assignment* out, ag_triple* triples, int32_t triples_cap, int32_t* occupancy) {
  const auto t_start = std::chrono::steady_clock::now();
  ag_ctx* ctx = s->ctx;
  if (B < 1) return fail(AG_ERR_VALIDATION, "beam width < 1");
  if (B > kMaxBeam) return fail(AG_ERR_VALIDATION, "GPU scheduler supports beam width <= 32");
  EngDev ed;
  bool ordered = false;
  int rc = engines_dev(engines, &ed, &ordered);
  if (rc) return rc;
  // the fast walker (ag_sched_fast.cuh): B <= 4, <= 8 pools of <= 255 free slots
  bool fast = ordered && B <= 4 && ed.E <= 8;
  for (int i = 0; i < ed.E; ++i) fast &= ed.slots[i] - ed.occ[i] <= 255;
  const int bm = fast && s->walker != 1 ? (B == 1 ? 1 : 4) : 0;
  int total_free = 0;
  for (int i = 0; i < ed.E; ++i) total_free += std::max(0, ed.slots[i] - ed.occ[i]);
  const int Q = (int)s->order.size();
  const int cap_t = total_free + 1;
  const int max_children = B * (ed.E + 1);
  const size_t max_pairs = (size_t)Q * (size_t)s->N + 1;
  const int max_nodes = (int)std::min<size_t>((size_t)B * max_pairs + 16, (size_t)1 << 30);
  // ---- ready updates (deduplicated: the last one per slot wins)
  dedup_updates(s);
  const size_t nu = s->upd_slot.size();
  // refresh records: every FIFO position from the first stale one, then the
  // other slots whose ready mask changed (the host mirror holds the masks)
  (void)nu;
  const size_t n_rec = build_records(s, nullptr);
  const size_t off_cidx = n_rec * 16;
  const size_t up_bytes = off_cidx + (cidx_host ? (size_t)Q * 4 : 0) + 16;
  const size_t res_bytes = kOutHeader + sizeof(ag_assignment) + 4 * kMaxEng + (size_t)cap_t * sizeof(ag_triple);
  if ((rc = ensure_pinned(&s->h_rstage, &s->h_rstage_bytes, up_bytes)) ||
      (rc = ensure_pinned(&s->h_res, &s->h_res_bytes, res_bytes)) || (rc = s->d_status.ensure(192)) ||
      (rc = s->d_cidx.ensure(cidx_host ? (size_t)Q * 4 : 4)))
    return rc;
  // the previous round synchronised after its last use of h_rstage / h_res
  char* h = (char*)s->h_rstage;
  build_records(s, reinterpret_cast<int32_t*>(h));
  if (cidx_host) std::memcpy(h + off_cidx, cidx_host, (size_t)Q * 4);
  if (s->h_rstage != s->h_rstage_mapped) {
    if ((rc = dev_ptr(s->h_rstage, &s->h_rstage_dev))) return rc;
    s->h_rstage_mapped = s->h_rstage;
  }
  if (s->h_res != s->h_res_mapped) {
    if ((rc = dev_ptr(s->h_res, &s->h_res_dev))) return rc;
    s->h_res_mapped = s->h_res;
  }
  char* hd = s->h_rstage_dev;
  int32_t* out_d = s->h_res_dev;
  if (up_bytes > kMappedMax) {
    // large deltas (a fresh session): one DMA copy instead of PCIe reads
    if ((rc = s->d_upd.ensure(up_bytes))) return rc;
    AG_CUDA(cudaMemcpyAsync(s->d_upd.p, h, up_bytes, cudaMemcpyHostToDevice, ctx->stream));
    hd = (char*)s->d_upd.p;
  }
  // ---- shared memory plan: nodes | children | ratio rows | cand records |
  // cand masks | count rows
  const size_t static_bytes = sizeof(int) * 2 * kMaxBeam * kMaxEng + 2 * 8 * kMaxBeam * kMaxBeam +
                              sizeof(RankKey) * 32 + kMaxBeam * 32 * 4 + 4 * 1024 + 4096 +
                              kLookahead * (sizeof(Cand) + 8) + 64;
  const size_t max_dyn = 227 * 1024 - static_bytes;
  const size_t fixed = sizeof(Node) * kSmemNodes + sizeof(Child) * (size_t)max_children;
  if (fixed > max_dyn) return fail(AG_ERR_VALIDATION, "beam too wide for one CTA");
  const int wor_cap = (int)((max_pairs + 31) / 32) + 1;
  if (fixed + 4 * (size_t)wor_cap > max_dyn) return fail(AG_ERR_VALIDATION, "beam too wide for one CTA");
  size_t room = max_dyn - fixed - 4 * (size_t)wor_cap;
  // the walk visits the head of the candidate list (engines fill quickly):
  // histogram rows and ratios are staged for that head only
  const size_t row_bytes = (size_t)s->M * (sizeof(double) + sizeof(uint32_t));
  int hist_cap = bm ? 0 : (int)std::min<size_t>(std::min<size_t>(max_pairs, 512), (48 * 1024) / row_bytes);
  hist_cap &= ~1;  // keeps the records after the ratio rows 16-byte aligned
  // the fast walker's lookahead ring holds its rows in the same area
  const int la_rows = bm ? kLookahead : 0;
  const int rows_alloc = std::max(hist_cap, la_rows);
  room -= (size_t)rows_alloc * row_bytes;
  const int cand_cap = (int)std::min<size_t>(max_pairs, room / (sizeof(Cand) + 4) & ~(size_t)3);
  hist_cap = std::min(hist_cap, cand_cap & ~1);
  const size_t dyn = fixed + (size_t)rows_alloc * row_bytes + (size_t)cand_cap * (sizeof(Cand) + 4) +
                     4 * (size_t)wor_cap;
  const size_t g_over = max_pairs > (size_t)cand_cap ? max_pairs - cand_cap : 1;
  if ((rc = s->d_cpos.ensure(g_over * 4)) || (rc = s->d_det.ensure(g_over * sizeof(Cand))) ||
      (rc = s->d_nodes.ensure((size_t)std::max(1, max_nodes - kSmemNodes) * sizeof(Node))))
    return rc;
  if (!s->attr_set) {
    AG_CUDA(cudaFuncSetAttribute(k_sched_round<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_dyn));
    AG_CUDA(cudaFuncSetAttribute(k_sched_round<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_dyn));
    AG_CUDA(cudaFuncSetAttribute(k_sched_round<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_dyn));
    s->attr_set = true;
  }
  RoundArgs A;
  std::memset(&A, 0, sizeof A);
  A.N = s->N;
  A.M = s->M;
  A.B = B;
  A.Q = Q;
  A.npairs = s->npairs;
  A.order = (int32_t*)s->d_order.p;
  A.cidx = cidx_host ? (int32_t*)s->d_cidx.p : nullptr;
  A.ready = (uint64_t*)s->d_ready.p;
  A.cand = (const uint32_t*)s->d_cand.p;
  A.hist = (const uint32_t*)s->d_hist.p;
  A.voff = (const uint64_t*)s->d_voff.p;
  A.pool = (const uint32_t*)s->d_pool.p;
  A.nviable = (const uint32_t*)s->d_nv.p;
  A.ids = (const uint64_t*)s->d_ids.p;
  A.ever = (const uint32_t*)((char*)s->d_status.p + 8);
  A.h_rec = (const int4*)hd;
  A.n_rec = (int)n_rec;
  if (!cidx_host && n_rec <= (size_t)kInlineRec) {
    std::memcpy(A.inl_rec, h, n_rec * 16);
    A.n_inl = 1;
  }
  A.h_cidx = cidx_host ? (const int32_t*)(hd + off_cidx) : nullptr;
  A.pinfo = (uint4*)s->d_pinfo.p;
  std::memcpy(A.prio, s->prio, sizeof A.prio);
  for (int t = 0; t < s->N; ++t) A.prio_rank[(int)s->prio[t]] = (int8_t)t;
  std::memcpy(A.place, s->place, sizeof A.place);
  std::memcpy(A.place_magic, s->place_magic, sizeof A.place_magic);
  A.div_m = ctx->space->dev().div_m;
  A.eng = ed;
  A.gmask = (uint32_t*)s->d_cpos.p;
  A.grec = (Cand*)s->d_det.p;
  A.cand_cap = cand_cap;
  A.wor_cap = wor_cap;
  A.hist_cap = hist_cap;
  A.rows_alloc = rows_alloc;
  A.la_rows = la_rows;
  A.gnodes = (Node*)s->d_nodes.p;
  A.max_nodes = max_nodes;
  A.max_children = max_children;
  A.out = out_d;
  // the host spins on this number in the mapped header: clear the word first
  // (a fresh or recycled pinned buffer may hold any value) and never use 0
  if (++s->round_seq == 0) s->round_seq = 1;
  A.seq = s->round_seq;
  ((volatile int32_t*)s->h_res)[2] = 0;
  A.triples_cap = cap_t;
  A.timing = (unsigned long long*)((char*)s->d_status.p + 32);
  A.async_status = (int32_t*)s->d_status.p;
  const auto t_prep = std::chrono::steady_clock::now();
  {
    Launch L(ctx, K_SCHED_ROUND);
    if (bm == 1) k_sched_round<1><<<1, RoundShape<1>::threads, dyn, ctx->stream>>>(A);
    else if (bm == 4) k_sched_round<4><<<1, RoundShape<4>::threads, dyn, ctx->stream>>>(A);
    else k_sched_round<0><<<1, RoundShape<0>::threads, dyn, ctx->stream>>>(A);
  }
  AG_CUDA(cudaGetLastError());
  const auto t_launch = std::chrono::steady_clock::now();
  {
    // spin on the round's sequence number in the mapped result header (a
    // stream synchronisation costs several microseconds more); a kernel that
    // ends without writing it (a fault) is caught by the stream query
    volatile const int32_t* flag = (volatile const int32_t*)s->h_res + 2;
    for (unsigned it = 1; *flag != (int32_t)A.seq; ++it)
      if ((it & 1023u) == 0 && cudaStreamQuery(ctx->stream) != cudaErrorNotReady) break;
    if (*flag != (int32_t)A.seq) AG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  const auto t_seen = std::chrono::steady_clock::now();
  s->dirty_from = Q;
  s->pinfo_from = Q;
  s->upd_slot.clear();
  s->upd_mask.clear();
  const char* hr = (const char*)s->h_res;
  const int32_t status = ((const int32_t*)hr)[0];
  if (status) {
    if (status == AG_ERR_VALIDATION + 100)
      return fail(AG_ERR_VALIDATION, "viable model tier without an engine pool");
    if (status == AG_ERR_VALIDATION + 200) return fail(AG_ERR_VALIDATION, "engine over capacity");
    if (status == AG_ERR_VALIDATION + 500)
      return fail(AG_ERR_VALIDATION, "occupancy outside engine capacity");
    if (status == AG_ERR_VALIDATION + 600)
      return fail(AG_ERR_VALIDATION, "dispatched model is not a viable candidate");
    return fail(AG_ERR_INTERNAL, "scheduler round failed (status " + std::to_string(status) + ")");
  }
  const ag_assignment res = *(const ag_assignment*)(hr + kOutHeader);
  if (out) *out = res;
  if (res.n_triples > triples_cap) return fail(AG_ERR_VALIDATION, "triples_cap too small");
  const char* occ = hr + kOutHeader + sizeof(ag_assignment);
  if (occupancy) std::memcpy(occupancy, occ, 4 * (size_t)engines->n_engines);
  if (res.n_triples)
    std::memcpy(triples, occ + 4 * kMaxEng, sizeof(ag_triple) * (size_t)res.n_triples);
  const auto t_end = std::chrono::steady_clock::now();
  auto us = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::micro>(b - a).count();
  };
  s->host_us[0] = us(t_start, t_prep);
  s->host_us[1] = us(t_prep, t_launch);
  s->host_us[2] = us(t_launch, t_seen);
  s->host_us[3] = us(t_seen, t_end);
  s->last_round_us = us(t_start, t_end);
  s->round_epoch = s->epoch;
  return AG_OK;
}

// Empties a session for reuse (stateless beam_schedule): host mirror back to
// its initial state; device arrays are rewritten by the next add before use.
void reset_session(ag_sched* s) {
  for (int slot : s->order) s->pos_of[slot] = -1;
  s->order.clear();
  s->dirty_from = 0;
  s->pinfo_from = 0;
  s->dead = 0;
  s->quarantine.clear();
  s->free_slots.clear();
  for (int i = s->cap - 1; i >= 0; --i) s->free_slots.push_back(i);
  std::fill(s->live.begin(), s->live.end(), 0);
  std::fill(s->ready.begin(), s->ready.end(), 0);
  s->npairs = 0;
  s->upd_slot.clear();
  s->upd_mask.clear();
  s->pool_top = 0;
}

// deferred error of an asynchronous dispatch / add (read at round time)
int check_async_status(ag_sched* s) {
  int32_t st = 0;
  AG_CUDA(cudaMemcpyAsync(&st, s->d_status.p, 4, cudaMemcpyDeviceToHost, s->ctx->stream));
  AG_CUDA(cudaStreamSynchronize(s->ctx->stream));
  if (st) {
    AG_CUDA(cudaMemsetAsync(s->d_status.p, 0, 4, s->ctx->stream));
    return fail(AG_ERR_VALIDATION, "dispatched model is not a viable candidate");
  }
  return AG_OK;
}

}  // namespace
}  // namespace agb

using agb::fail;

extern "C" {

int ag_sched_create(ag_ctx* ctx, int32_t max_requests, uint64_t max_configs, ag_sched** out) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  if (!ctx || !out) return fail(AG_ERR_VALIDATION, "null argument");
  *out = nullptr;
  const ag_space* sp = ctx->space;
  if (!sp->gpu_ok) return fail(AG_ERR_VALIDATION, "GPU path needs M^N <= 2^32 and N <= 32");
  if (sp->m > 32) return fail(AG_ERR_VALIDATION, "GPU scheduler supports at most 32 model tiers");
  if (max_requests < 1) return fail(AG_ERR_VALIDATION, "max_requests < 1");
  if (max_requests >= (1 << 26)) return fail(AG_ERR_VALIDATION, "GPU scheduler supports < 2^26 requests per session");
  ag_sched* s = new ag_sched();
  s->ctx = ctx;
  s->N = sp->n;
  s->M = sp->m;
  s->cap = max_requests;
  s->pool_cap = std::max<uint64_t>(max_configs, 1);
  if (const char* w = std::getenv("AG_SCHED_WALKER")) s->walker = std::strcmp(w, "general") == 0 ? 1 : 0;
  s->ids.assign(max_requests, 0);
  s->arrival.assign(max_requests, 0.0);
  s->stages.assign((size_t)max_requests * sp->n, 0);
  s->ready.assign(max_requests, 0);
  s->live.assign(max_requests, 0);
  s->pos_of.assign(max_requests, -1);
  s->nviable.assign(max_requests, 0);
  for (int i = max_requests - 1; i >= 0; --i) s->free_slots.push_back(i);
  // agent priority: depth descending, declaration ascending (scheduler.cpp:238-242)
  std::vector<int> pr(sp->n);
  std::iota(pr.begin(), pr.end(), 0);
  std::sort(pr.begin(), pr.end(), [&](int x, int y) {
    if (sp->depth[x] != sp->depth[y]) return sp->depth[x] > sp->depth[y];
    return sp->decl[x] < sp->decl[y];
  });
  for (int i = 0; i < 64; ++i) s->prio[i] = i < sp->n ? (int8_t)pr[i] : 0;
  uint64_t pl = 1;
  for (int a = sp->n - 1; a >= 0; --a) {
    s->place[a] = (uint32_t)pl;
    s->place_magic[a] = pl > 1 ? (~0ULL) / pl + 1 : 0;
    pl *= (uint64_t)sp->m;
  }
  int rc;
  const size_t R = (size_t)max_requests;
  if ((rc = s->d_ready.ensure(R * 8)) || (rc = s->d_cand.ensure(R * sp->n * 4)) ||
      (rc = s->d_hist.ensure(R * sp->n * sp->m * 4)) || (rc = s->d_nv.ensure(R * 4)) ||
      (rc = s->d_voff.ensure(R * 8)) || (rc = s->d_ids.ensure(R * 8)) ||
      (rc = s->d_pool.ensure(s->pool_cap * 4)) || (rc = s->d_status.ensure(192)) ||
      (rc = s->d_order.ensure(((size_t)2 * max_requests + 1024) * 4)) ||
      (rc = s->d_pinfo.ensure(((size_t)2 * max_requests + 1024) * 16))) {
    delete s;
    return rc;
  }
  cudaMemsetAsync(s->d_pinfo.p, 0, ((size_t)2 * max_requests + 1024) * 16, ctx->stream);
  cudaMemsetAsync(s->d_ready.p, 0, R * 8, ctx->stream);
  cudaMemsetAsync(s->d_status.p, 0, 128, ctx->stream);
  *out = s;
  return AG_OK;
}

void ag_sched_destroy(ag_sched* s) {
  agb::DeviceGuard device_guard(s ? s->ctx->device : -1);
  delete s;
}

int ag_sched_add(ag_sched* s, const ag_queue* q, int32_t* slots_out) {
  agb::DeviceGuard device_guard(s ? s->ctx->device : -1);
  if (s) ++s->epoch;
  if (!s || !q) return fail(AG_ERR_VALIDATION, "null argument");
  ag_ctx* ctx = s->ctx;
  const int R = q->n_requests;
  if (R <= 0) return R == 0 ? AG_OK : fail(AG_ERR_VALIDATION, "negative request count");
  if ((int)s->free_slots.size() < R && !s->quarantine.empty()) agb::compact_order(s);
  if ((int)s->free_slots.size() < R) return fail(AG_ERR_VALIDATION, "session is full");
  const uint64_t total = (uint64_t)(q->viable_ptr[R] - q->viable_ptr[0]);
  if (s->pool_top + total > s->pool_cap) {
    // removed requests left dead space behind pool_top: pack the live lists
    int rc0 = agb::compact_pool(s);
    if (rc0) return rc0;
  }
  if (s->pool_top + total > s->pool_cap) return fail(AG_ERR_VALIDATION, "session viable pool is full");
  const int N = s->N;
  // Request::make (request.cpp:24-50)
  for (int i = 0; i < R; ++i) {
    const int64_t len = q->viable_ptr[i + 1] - q->viable_ptr[i];
    if (len <= 0) return fail(AG_ERR_VALIDATION, "request needs a nonempty viable set");
    for (int64_t j = q->viable_ptr[i]; j < q->viable_ptr[i + 1]; ++j)
      if ((uint64_t)q->viable[j] >= ctx->space->size)
        return fail(AG_ERR_VALIDATION, "viable configuration length mismatch");
  }
  std::vector<int32_t> slots(R), g_begin(R + 1, 0);
  std::vector<uint64_t> meta(3 * (size_t)R);
  for (int i = 0; i < R; ++i) {
    const int slot = s->free_slots.back();
    s->free_slots.pop_back();
    slots[i] = slot;
    s->ids[slot] = q->ids[i];
    s->arrival[slot] = q->arrival[i];
    for (int a = 0; a < N; ++a)
      s->stages[(size_t)slot * N + a] =
          q->stages ? q->stages[(size_t)i * N + a]
                    : (ctx->space->pred[a] ? AG_STAGE_PENDING : AG_STAGE_READY);
    s->live[slot] = 1;
    s->nviable[slot] = (uint32_t)(q->viable_ptr[i + 1] - q->viable_ptr[i]);
    meta[3 * i] = s->pool_top + (uint64_t)(q->viable_ptr[i] - q->viable_ptr[0]);
    meta[3 * i + 1] = s->nviable[slot];
    meta[3 * i + 2] = q->ids[i];
    agb::set_ready(s, slot, agb::ready_of(s, slot));
    if (slots_out) slots_out[i] = slot;
  }
  {
    // through pinned staging: a pageable source would make the copy synchronous
    AG_CUDA(cudaStreamSynchronize(ctx->stream));  // the staging buffer's previous copy
    int rc0 = agb::ensure_pinned(&s->h_vstage, &s->h_vstage_bytes, total * 4 + 4);
    if (rc0) return rc0;
    std::memcpy(s->h_vstage, q->viable + q->viable_ptr[0], total * 4);
    AG_CUDA(cudaMemcpyAsync((uint32_t*)s->d_pool.p + s->pool_top, s->h_vstage, total * 4,
                            cudaMemcpyHostToDevice, ctx->stream));
  }
  s->pool_top += total;
  // FIFO insertion (Sim::insert_schedulable, simulation.cpp:182-192)
  for (int i = 0; i < R; ++i) {
    const int slot = slots[i];
    if (s->order.size() + 1 > (size_t)2 * s->cap + 1024) agb::compact_order(s);
    size_t pos = s->order.size();
    if (!s->order.empty() && agb::fifo_less(s, slot, s->order.back())) {
      pos = (size_t)(std::lower_bound(s->order.begin(), s->order.end(), slot,
                                      [&](int x, int y) {
                                        // dead entries keep their place; compare live keys
                                        return agb::fifo_less(s, x, y);
                                      }) -
                     s->order.begin());
    }
    s->order.insert(s->order.begin() + pos, slot);
    for (size_t k = pos; k < s->order.size(); ++k) s->pos_of[s->order[k]] = (int32_t)k;
    s->dirty_from = std::min(s->dirty_from, pos);
    s->pinfo_from = std::min(s->pinfo_from, pos);
  }
  // the viable copy must land before the histogram pass reads it (same stream)
  int rc = agb::launch_prune(s, slots, g_begin, {}, &meta);
  if (rc || (rc = agb::flush_order(s))) return rc;
  return agb::refresh_records(s, false);
}

int ag_sched_remove(ag_sched* s, int32_t n, const int32_t* slots) {
  agb::DeviceGuard device_guard(s ? s->ctx->device : -1);
  if (s) ++s->epoch;
  if (!s) return fail(AG_ERR_VALIDATION, "null argument");
  for (int i = 0; i < n; ++i) {
    const int slot = slots[i];
    if (slot < 0 || slot >= s->cap || !s->live[slot]) return fail(AG_ERR_VALIDATION, "bad slot");
    s->live[slot] = 0;
    agb::set_ready(s, slot, 0);
    s->quarantine.push_back(slot);  // still listed on the device until compaction
    ++s->dead;
  }
  if (s->dead > std::max<size_t>(256, s->order.size() / 4)) agb::compact_order(s);
  bool any_live = false;
  for (int slot : s->order) any_live |= s->live[slot] != 0;
  if (!any_live) {
    agb::compact_order(s);
    s->pool_top = 0;  // everything left: reuse the pool
  }
  int rc = agb::flush_order(s);
  return rc ? rc : agb::refresh_records(s, false);
}

int ag_sched_complete(ag_sched* s, int32_t slot, int32_t agent) {
  agb::DeviceGuard device_guard(s ? s->ctx->device : -1);
  if (s) ++s->epoch;
  if (!s || slot < 0 || slot >= s->cap || !s->live[slot]) return fail(AG_ERR_VALIDATION, "bad slot");
  const int N = s->N;
  if (agent < 0 || agent >= N || s->stages[(size_t)slot * N + agent] != AG_STAGE_INFLIGHT)
    return fail(AG_ERR_VALIDATION, "completion of a stage that is not in flight");
  uint8_t* st = &s->stages[(size_t)slot * N];
  st[agent] = AG_STAGE_DONE;
  const ag_space* sp = s->ctx->space;
  for (uint64_t b = sp->succ[agent]; b; b &= b - 1) {
    const int sc = __builtin_ctzll(b);
    if (st[sc] != AG_STAGE_PENDING) continue;
    bool all_done = true;
    for (uint64_t pb = sp->pred[sc]; pb && all_done; pb &= pb - 1)
      all_done = st[__builtin_ctzll(pb)] == AG_STAGE_DONE;
    if (all_done) st[sc] = AG_STAGE_READY;
  }
  const uint64_t r = agb::ready_of(s, slot);
  if (r != s->ready[slot]) agb::set_ready(s, slot, r);
  return AG_OK;
}

int ag_sched_round(ag_sched* s, const ag_engines* engines, int beam_width, ag_assignment* out,
                   ag_triple* triples, int32_t triples_cap, int32_t* occupancy) {
  agb::DeviceGuard device_guard(s ? s->ctx->device : -1);
  if (!s) return fail(AG_ERR_VALIDATION, "null argument");
  return agb::run_round(s, engines, beam_width, nullptr, out, triples, triples_cap, occupancy);
}

int ag_sched_dispatch(ag_sched* s, int32_t n, const ag_triple* applied) {
  agb::DeviceGuard device_guard(s ? s->ctx->device : -1);
  if (s) ++s->epoch;
  if (!s) return fail(AG_ERR_VALIDATION, "null argument");
  const int N = s->N;
  for (int i = 0; i < n; ++i) {
    const ag_triple& t = applied[i];
    if (t.slot < 0 || t.slot >= s->cap || !s->live[t.slot]) return fail(AG_ERR_VALIDATION, "bad slot");
    if (t.agent < 0 || t.agent >= N || s->stages[(size_t)t.slot * N + t.agent] != AG_STAGE_READY)
      return fail(AG_ERR_VALIDATION, "dispatch of a stage that is not ready");
    if (t.model < 0 || t.model >= s->M)
      return fail(AG_ERR_VALIDATION, "dispatched model is not a viable candidate");
  }
  // group by slot, apply order kept inside a group
  std::vector<int32_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return applied[x].slot < applied[y].slot; });
  std::vector<int32_t> g_slot, g_begin{0}, g_am;
  for (int k = 0; k < n; ++k) {
    const ag_triple& t = applied[idx[k]];
    if (g_slot.empty() || g_slot.back() != t.slot) {
      if (!g_slot.empty()) g_begin.push_back((int32_t)g_am.size());
      g_slot.push_back(t.slot);
    }
    g_am.push_back((t.agent << 8) | t.model);
    s->stages[(size_t)t.slot * N + t.agent] = AG_STAGE_INFLIGHT;
  }
  g_begin.push_back((int32_t)g_am.size());
  for (int slot : g_slot) {
    agb::set_ready(s, slot, agb::ready_of(s, slot));
  }
  return agb::launch_prune(s, g_slot, g_begin, g_am, nullptr);
}

// apply_assignment (scheduler.cpp:421-454): triples in order; a triple whose
// engine pool has no free slot left (occupancy + triples applied before it
// on the same pool >= slots) is stale and dropped, the rest are applied:
// Request::mark_dispatched (prefix prune on the device, ag_sched_dispatch).
int ag_sched_apply(ag_sched* s, const ag_engines* engines, int32_t n, const ag_triple* triples,
                   uint8_t* applied, int32_t* n_applied, int32_t* n_stale) {
  agb::DeviceGuard device_guard(s ? s->ctx->device : -1);
  if (!s || !engines || (n > 0 && !triples)) return fail(AG_ERR_VALIDATION, "null argument");
  std::vector<int> left(std::max(engines->n_engines, 1));
  std::vector<int> pool_of(64, -1);
  for (int i = 0; i < engines->n_engines; ++i) {
    const int mdl = engines->model[i];
    if (mdl >= 0 && mdl < 64) pool_of[mdl] = i;
    left[i] = engines->slots[i] - engines->occupancy[i];
  }
  std::vector<ag_triple> keep;
  keep.reserve(n);
  int na = 0, ns = 0;
  for (int k = 0; k < n; ++k) {
    const int mdl = triples[k].model;
    if (mdl < 0 || mdl >= 64 || pool_of[mdl] < 0)
      return fail(AG_ERR_VALIDATION, "assignment names a model without an engine pool");
    const bool ok = left[pool_of[mdl]] > 0;  // EngineState::slots_available (engine.h:47)
    if (ok) {
      --left[pool_of[mdl]];
      keep.push_back(triples[k]);
      ++na;
    } else {
      ++ns;
    }
    if (applied) applied[k] = ok ? 1 : 0;
  }
  if (n_applied) *n_applied = na;
  if (n_stale) *n_stale = ns;
  return keep.empty() ? AG_OK : ag_sched_dispatch(s, (int32_t)keep.size(), keep.data());
}

namespace agb {
namespace {
// the audit kernel over the session's device queue; cidx: container index per
// FIFO position (device) for a stateless queue, else null
int audit_impl(ag_sched* s, const ag_engines* engines, int32_t n, const ag_triple* triples, const int32_t* cidx,
               uint64_t* viol_ids, int32_t* viol_agents, int32_t cap, int32_t* n_viol) {
  if (n > agb::kAuditMaxTrip) return fail(AG_ERR_VALIDATION, "audit supports at most 2048 triples");
  agb::EngDev ed;
  int rc = agb::engines_dev(engines, &ed);
  if (rc) return rc;
  ag_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  const int Q = (int)s->order.size();
  const size_t tb = 16 * (size_t)std::max(n, 1), qb = 4 * (size_t)std::max(Q, 1);
  const size_t ob = 16 + 12 * (size_t)std::max(cap, 0);
  if ((rc = s->d_audit.ensure(tb + 2 * qb + ob + 64)) ||
      (rc = agb::ensure_pinned(&s->h_stage, &s->h_stage_bytes, tb + ob + 64)))
    return rc;
  AG_CUDA(cudaStreamSynchronize(st));  // the staging buffer's previous use
  int4* ht = (int4*)s->h_stage;
  for (int k = 0; k < n; ++k) ht[k] = make_int4(triples[k].request_index, triples[k].agent, triples[k].model, 0);
  char* d = (char*)s->d_audit.p;
  agb::AuditArgs A;
  std::memset(&A, 0, sizeof A);
  A.N = s->N;
  A.M = s->M;
  A.Q = Q;
  A.n = n;
  A.order = (const int32_t*)s->d_order.p;
  A.ready = (const uint64_t*)s->d_ready.p;
  A.cand = (const uint32_t*)s->d_cand.p;
  A.ids = (const uint64_t*)s->d_ids.p;
  A.voff = (const uint64_t*)s->d_voff.p;
  A.nviable = (const uint32_t*)s->d_nv.p;
  A.pool = (const uint32_t*)s->d_pool.p;
  A.trip = (const int4*)d;
  A.q_slot = (int32_t*)(d + tb);
  for (int t = 0; t < s->N; ++t) A.prio_rank[(int)s->prio[t]] = (int8_t)t;
  A.eng = ed;
  std::memcpy(A.place, s->place, sizeof A.place);
  std::memcpy(A.place_magic, s->place_magic, sizeof A.place_magic);
  A.div_m = ctx->space->dev().div_m;
  A.cidx = cidx;
  A.c_rank = (int32_t*)(d + tb + qb);
  A.out = (int32_t*)(d + tb + 2 * qb);
  A.out_ids = (uint64_t*)(d + tb + 2 * qb + 16);
  A.out_agents = (int32_t*)(d + tb + 2 * qb + 16 + 8 * (size_t)std::max(cap, 0));
  A.cap = std::max(cap, 0);
  if (n) AG_CUDA(cudaMemcpyAsync(d, ht, 16 * (size_t)n, cudaMemcpyHostToDevice, st));
  AG_CUDA(cudaMemsetAsync(A.out, 0, 16, st));
  {
    agb::Launch L(ctx, agb::K_SCHED_PREP);
    agb::k_sched_audit<<<1, agb::kAuditThreads, 0, st>>>(A);
  }
  AG_CUDA(cudaGetLastError());
  char* ho = (char*)s->h_stage + tb;
  AG_CUDA(cudaMemcpyAsync(ho, A.out, ob, cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaStreamSynchronize(st));
  const int32_t* hout = (const int32_t*)ho;
  if (hout[1] == AG_ERR_VALIDATION + 100) return fail(AG_ERR_VALIDATION, "viable model tier without an engine pool");
  if (hout[1] == AG_ERR_VALIDATION + 200) return fail(AG_ERR_VALIDATION, "engine over capacity");
  if (hout[1] == AG_ERR_VALIDATION + 300)
    return fail(AG_ERR_VALIDATION, "assignment names a model without an engine pool");
  if (hout[1]) return fail(AG_ERR_INTERNAL, "audit failed");
  *n_viol = hout[0];
  const int k = std::min(hout[0], std::max(cap, 0));
  if (k && viol_ids) std::memcpy(viol_ids, ho + 16, 8 * (size_t)k);
  if (k && viol_agents) std::memcpy(viol_agents, ho + 16 + 8 * (size_t)std::max(cap, 0), 4 * (size_t)k);
  return AG_OK;
}
}  // namespace
}  // namespace agb

// audit_round_fairness (scheduler.cpp:456-480) over the last round's queue:
// must follow ag_sched_round with no session change in between.
int ag_sched_audit(ag_sched* s, const ag_engines* engines, int32_t n, const ag_triple* triples,
                   uint64_t* viol_ids, int32_t* viol_agents, int32_t cap, int32_t* n_viol) {
  agb::DeviceGuard device_guard(s ? s->ctx->device : -1);
  if (!s || !engines || !n_viol || (n > 0 && !triples)) return fail(AG_ERR_VALIDATION, "null argument");
  if (s->round_epoch != s->epoch)
    return fail(AG_ERR_VALIDATION, "audit needs the queue of the last round (session changed since)");
  return agb::audit_impl(s, engines, n, triples, nullptr, viol_ids, viol_agents, cap, n_viol);
}

int ag_sched_queued_ahead(ag_sched* s, int32_t* out) {
  agb::DeviceGuard device_guard(s ? s->ctx->device : -1);
  if (!s || !out) return fail(AG_ERR_VALIDATION, "null argument");
  ag_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  const int Q = (int)s->order.size();
  const size_t nu = s->upd_slot.size();
  int rc;
  if ((rc = s->d_qa.ensure(4 * 32 + nu * 12 + 16))) return rc;
  // the device order must be current; pending ready updates are passed along
  if (Q > (int)s->dirty_from) {
    AG_CUDA(cudaMemcpyAsync((int32_t*)s->d_order.p + s->dirty_from, s->order.data() + s->dirty_from,
                            (Q - s->dirty_from) * 4, cudaMemcpyHostToDevice, st));
    s->dirty_from = Q;
  }
  char* d = (char*)s->d_qa.p;
  AG_CUDA(cudaMemsetAsync(d, 0, 4 * 32, st));
  if (nu) {
    AG_CUDA(cudaMemcpyAsync(d + 128, s->upd_mask.data(), nu * 8, cudaMemcpyHostToDevice, st));
    AG_CUDA(cudaMemcpyAsync(d + 128 + nu * 8, s->upd_slot.data(), nu * 4, cudaMemcpyHostToDevice, st));
  }
  const int blocks = std::max(1, std::min(148, (Q + 255) / 256));
  {
    agb::Launch L(ctx, agb::K_SCHED_PREP);
    agb::k_queued_ahead<<<blocks, 256, 0, st>>>(
        (const int32_t*)s->d_order.p, Q, (const uint64_t*)s->d_ready.p, (const uint32_t*)s->d_cand.p,
        s->N, s->M, (int)nu, (const int32_t*)(d + 128 + nu * 8), (const uint64_t*)(d + 128),
        (uint32_t*)d);
  }
  AG_CUDA(cudaGetLastError());
  AG_CUDA(cudaMemcpyAsync(out, d, 4 * (size_t)s->M, cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaStreamSynchronize(st));
  return AG_OK;
}

int ag_sched_round_timing(ag_sched* s, uint64_t* ns) {
  agb::DeviceGuard device_guard(s ? s->ctx->device : -1);
  if (!s || !ns) return fail(AG_ERR_VALIDATION, "null argument");
  AG_CUDA(cudaMemcpyAsync(ns, (char*)s->d_status.p + 32, 128, cudaMemcpyDeviceToHost, s->ctx->stream));
  AG_CUDA(cudaStreamSynchronize(s->ctx->stream));
  return AG_OK;
}

double ag_sched_last_round_us(const ag_sched* s) { return s ? s->last_round_us : 0.0; }

int ag_sched_round_host_timing(const ag_sched* s, double* out4) {
  if (!s || !out4) return fail(AG_ERR_VALIDATION, "null argument");
  for (int i = 0; i < 4; ++i) out4[i] = s->host_us[i];
  return AG_OK;
}

int ag_sched_viable(ag_sched* s, int32_t slot, uint32_t* out, int64_t cap, int64_t* n) {
  agb::DeviceGuard device_guard(s ? s->ctx->device : -1);
  if (!s || slot < 0 || slot >= s->cap || !s->live[slot]) return fail(AG_ERR_VALIDATION, "bad slot");
  int rc = agb::check_async_status(s);
  if (rc) return rc;
  uint32_t len = 0;
  uint64_t vo = 0;
  AG_CUDA(cudaMemcpyAsync(&len, (uint32_t*)s->d_nv.p + slot, 4, cudaMemcpyDeviceToHost, s->ctx->stream));
  AG_CUDA(cudaMemcpyAsync(&vo, (uint64_t*)s->d_voff.p + slot, 8, cudaMemcpyDeviceToHost, s->ctx->stream));
  AG_CUDA(cudaStreamSynchronize(s->ctx->stream));
  if (n) *n = len;
  if (out && (int64_t)len <= cap && len) {
    AG_CUDA(cudaMemcpyAsync(out, (uint32_t*)s->d_pool.p + vo, (size_t)len * 4,
                            cudaMemcpyDeviceToHost, s->ctx->stream));
    AG_CUDA(cudaStreamSynchronize(s->ctx->stream));
  }
  return AG_OK;
}

// The context's cached session, emptied, holding exactly this queue (grown
// when a call needs more room); cidx: container index per FIFO position.
static int stateless_prepare(ag_ctx* ctx, const ag_queue* q, ag_sched** out, std::vector<int32_t>* cidx) {
  const int R = q->n_requests;
  if (R < 0) return fail(AG_ERR_VALIDATION, "negative request count");
  const uint64_t total = R > 0 ? (uint64_t)(q->viable_ptr[R] - q->viable_ptr[0]) : 0;
  ag_sched* s = ctx->beam_cache;
  if (s && (s->cap < std::max(R, 1) || s->pool_cap < std::max<uint64_t>(total, 1))) {
    const int cap = std::max(std::max(R, 1), 2 * s->cap);
    const uint64_t pcap = std::max<uint64_t>(std::max<uint64_t>(total, 1), 2 * s->pool_cap);
    delete s;
    ctx->beam_cache = s = nullptr;
    int rc = ag_sched_create(ctx, cap, pcap, &s);
    if (rc) return rc;
    ctx->beam_cache = s;
  } else if (!s) {
    int rc = ag_sched_create(ctx, std::max(R, 64), std::max<uint64_t>(total, 1 << 14), &s);
    if (rc) return rc;
    ctx->beam_cache = s;
  } else {
    agb::reset_session(s);
  }
  std::vector<int32_t> slots(std::max(R, 1));
  int rc = ag_sched_add(s, q, slots.data());
  if (rc) {
    agb::reset_session(s);
    return rc;
  }
  // container index per FIFO position; requests without ready stages keep
  // their container index (they simply contribute no pairs)
  std::vector<int32_t> slot_to_ci(s->cap, -1);
  for (int i = 0; i < R; ++i) slot_to_ci[slots[i]] = i;
  cidx->resize(s->order.size());
  for (size_t p = 0; p < s->order.size(); ++p) (*cidx)[p] = slot_to_ci[s->order[p]];
  *out = s;
  return AG_OK;
}

// fingerprint of a stateless queue (ids, arrivals, stages, viable sizes)
static uint64_t queue_fp(const ag_queue* q, int N) {
  uint64_t h = 0x9e3779b97f4a7c15ull ^ (uint64_t)q->n_requests;
  auto mixin = [&](uint64_t x) {
    h ^= x + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  };
  for (int i = 0; i < q->n_requests; ++i) {
    mixin(q->ids[i]);
    uint64_t ab;
    std::memcpy(&ab, &q->arrival[i], 8);
    mixin(ab);
    mixin((uint64_t)(q->viable_ptr[i + 1] - q->viable_ptr[i]));
    for (int a = 0; a < N; ++a) mixin(q->stages ? q->stages[(size_t)i * N + a] : 255u);
  }
  return h | 1ull;
}

// Stateless beam_schedule over the context's cached session.
int ag_beam_schedule(ag_ctx* ctx, const ag_queue* q, const ag_engines* engines, int beam_width,
                     ag_assignment* out, ag_triple* triples, int32_t triples_cap,
                     int32_t* occupancy) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  if (!ctx || !q || !engines) return fail(AG_ERR_VALIDATION, "null argument");
  if (beam_width < 1) return fail(AG_ERR_VALIDATION, "beam width < 1");
  ag_sched* s = nullptr;
  std::vector<int32_t> cidx;
  int rc = stateless_prepare(ctx, q, &s, &cidx);
  if (rc) return rc;
  rc = agb::run_round(s, engines, beam_width, cidx.data(), out, triples, triples_cap, occupancy);
  if (rc == AG_OK && out)
    for (int i = 0; i < out->n_triples; ++i) triples[i].slot = -1;
  s->stateless_fp = rc == AG_OK ? queue_fp(q, s->N) : 0;
  return rc;
}

// Stateless audit_round_fairness(queue, engines, assignment)
// (scheduler.cpp:456-480): the queue is installed in the context's cached
// session (as ag_beam_schedule does) and audited on the device; triples'
// request_index is the container index, as in the reference.
int ag_audit_round_fairness(ag_ctx* ctx, const ag_queue* q, const ag_engines* engines, int32_t n,
                            const ag_triple* triples, uint64_t* viol_ids, int32_t* viol_agents,
                            int32_t cap, int32_t* n_viol) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  if (!ctx || !q || !engines || !n_viol || (n > 0 && !triples)) return fail(AG_ERR_VALIDATION, "null argument");
  // the queue of the last stateless round, untouched since: audit in place
  ag_sched* c = ctx->beam_cache;
  if (c && c->stateless_fp && c->round_epoch == c->epoch && c->stateless_fp == queue_fp(q, c->N))
    return agb::audit_impl(c, engines, n, triples, (const int32_t*)c->d_cidx.p, viol_ids, viol_agents, cap,
                           n_viol);
  ag_sched* s = nullptr;
  std::vector<int32_t> cidx;
  int rc = stateless_prepare(ctx, q, &s, &cidx);
  if (rc) return rc;
  s->stateless_fp = 0;
  // the device queue as the host mirror holds it (no round has applied the
  // pending ready updates / FIFO tail yet): full copies, the next round
  // still refreshes its records from the pending lists
  cudaStream_t st = ctx->stream;
  const size_t Q = s->order.size();
  if ((rc = s->d_cidx.ensure(4 * std::max<size_t>(Q, 1)))) return rc;
  if (Q) {
    AG_CUDA(cudaMemcpyAsync(s->d_order.p, s->order.data(), 4 * Q, cudaMemcpyHostToDevice, st));
    AG_CUDA(cudaMemcpyAsync(s->d_cidx.p, cidx.data(), 4 * Q, cudaMemcpyHostToDevice, st));
  }
  AG_CUDA(cudaMemcpyAsync(s->d_ready.p, s->ready.data(), 8 * (size_t)s->cap, cudaMemcpyHostToDevice, st));
  s->dirty_from = Q;
  return agb::audit_impl(s, engines, n, triples, (const int32_t*)s->d_cidx.p, viol_ids, viol_agents, cap, n_viol);
}

}  // extern "C"
