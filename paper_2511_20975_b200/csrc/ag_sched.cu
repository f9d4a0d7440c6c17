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
// One round = one CTA (k_sched_round):
//   A. block-parallel RoundContext over the FIFO queue (loads batched per
//      thread so the dependent order -> ready -> cand chain costs a few memory
//      latencies, not one per request): pairs in (arrival, id) x (depth desc,
//      declaration asc) order, validation, and the compacted list of
//      "candidate" pairs -- those whose candidate models meet the engines free
//      at round start.  Every other pair is a whole-beam skip in every branch
//      (scheduler.cpp:317-329), so the walk never looks at it.  Candidates get
//      (position, mask) in shared memory and, for the first few thousand,
//      their request details and model histogram row too.
//   B. warp 0 walks the candidates exactly as beam_schedule walks pairs:
//      skipped runs are fast-forwarded with one ballot scan; at a step lanes
//      are children (extend_state); nested retention (scheduler.cpp:351-370)
//      is a warp bitonic sort under the exact state_better order followed by
//      one ballot per beam level; a child's triple list is a node of a history
//      tree (triples_less compares two tree paths).
//   C. finalize: the winner's triples from the tree (written in parallel),
//      score_assignment's utilization and flexibility folded in the
//      reference's order.
// All fp64 arithmetic repeats the reference's operations in the same order
// (the library builds with --fmad=false).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "ag_internal.h"

namespace agb {

namespace {

constexpr int kRoundThreads = 512;  // 128 registers per thread: no local memory in the walk
constexpr int kMaxBeam = 32;
constexpr int kMaxEng = 32;
constexpr int kSmemNodes = 1024;
constexpr int kPer = 8;  // FIFO positions per thread per pass chunk

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

struct Det {  // details of one candidate pair
  int32_t qi;
  int32_t slot;
  uint32_t nvia;
  int32_t agent;
};

struct BState {  // BeamState (scheduler.cpp:80-93)
  double util, flex_sum;
  long long skips;
  int flex_count;
  uint32_t free_mask;
  int node;  // latest history node, -1 = no triple
  int nsurv; // survivors of the request of `node`
  int occ[kMaxEng];
};

struct Child {
  double util, flex_sum, flex;
  long long skips;
  int flex_count, nsurv;
  int16_t parent, eng;  // eng < 0: skip child
};

struct EngDev {
  int E;
  int model[kMaxEng];
  int slots[kMaxEng];
  int occ[kMaxEng];
  double weight[kMaxEng];
  int8_t m2e[32];  // model -> engine, -1 none
  uint32_t mapped;  // models with a pool
};

struct RoundArgs {
  int N, M, B;
  const int32_t* order;  // [Q] slots in FIFO order (dead slots have ready 0)
  const int32_t* cidx;   // [Q] container index per FIFO position, or null
  int Q;
  uint64_t* ready;
  int n_upd;
  const int32_t* upd_slot;
  const uint64_t* upd_mask;
  const uint32_t* cand;
  const uint32_t* hist;
  const uint32_t* nviable;
  const uint64_t* voff;
  const uint32_t* pool;
  const uint64_t* ids;
  int8_t prio[64];
  int8_t prio_rank[64];
  uint32_t place[kMaxAgents];
  uint64_t place_magic[kMaxAgents];
  uint64_t div_m;
  EngDev eng;
  // scratch
  uint32_t* gcpos;  // candidate positions / masks beyond shared memory
  uint32_t* gcmask;
  Det* gdet;  // candidate details beyond shared memory
  int cand_cap, det_cap, hist_cap;
  Node* gnodes;
  int max_nodes;
  int max_children;
  // outputs: one contiguous block copied back in a single transfer
  int32_t* out;  // [0] status [1] queue size | ag_assignment | occ[32] | triples
  int triples_cap;
  unsigned long long* timing;  // [5] globaltimer at phase boundaries (ns)
  int32_t* async_status;       // errors latched by earlier dispatch / add kernels
};

constexpr int kOutHeader = 16;  // bytes before the ag_assignment

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

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

__device__ __forceinline__ int depth_of(const NodeView& nv, int n) {
  return n < 0 ? 0 : nv[n].depth;
}

// Per-step lexicographic structure of the beam states' triple lists, so that
// triples_less (scheduler.cpp:95-105) costs O(1): lcp[i][j] is the length of
// the common prefix of states i and j, nxt[i][j] the key of state i's element
// at that position (kEnd when its list ends there).  Adopting children updates
// it in O(B^2): two children of one parent share its whole list; children of
// different parents keep their parents' common prefix.
constexpr uint64_t kEnd = 0;  // below every triple key

__device__ __forceinline__ uint64_t tkey(int qi, int agent, int model) {
  return ((uint64_t)(uint32_t)(qi + 1) << 32) | ((uint64_t)(uint32_t)agent << 16) |
         (uint64_t)(uint32_t)model;
}

struct Lex {
  int len[kMaxBeam];
  int lcp[kMaxBeam][kMaxBeam];
  uint64_t nxt[kMaxBeam][kMaxBeam];
};

// triples_less between item (parent p1 + extra k1) and (p2 + k2); k = kEnd
// for "no extra".  Items with p1 == p2 differ only in their extras.
__device__ __forceinline__ bool lex_less(const Lex& L, int p1, uint64_t k1, int p2, uint64_t k2) {
  if (p1 == p2) return k1 < k2;
  const int l = L.lcp[p1][p2];
  const uint64_t y1 = l < L.len[p1] ? L.nxt[p1][p2] : k1;
  const uint64_t y2 = l < L.len[p2] ? L.nxt[p2][p1] : k2;
  return y1 < y2;
}

struct WalkCtx {
  const Child* ch;
  const Lex* L;
  uint64_t key_base;  // tkey(qcur, agent, 0)
  const EngDev* eng;
  __device__ __forceinline__ uint64_t key(int c) const {
    return ch[c].eng >= 0 ? key_base | (uint64_t)(uint32_t)eng->model[ch[c].eng] : kEnd;
  }
  // strict total order: state_better (scheduler.cpp:109-115), then the lower
  // child index (retention adopts the first best child, scheduler.cpp:357-362)
  __device__ __forceinline__ bool before(int c1, int c2) const {
    if (c1 < 0) return false;
    if (c2 < 0) return true;
    const Child &x = ch[c1], &y = ch[c2];
    if (x.util != y.util) return x.util > y.util;
    if (x.flex != y.flex) return x.flex > y.flex;
    if (x.skips != y.skips) return x.skips < y.skips;
    const uint64_t k1 = key(c1), k2 = key(c2);
    if (lex_less(*L, x.parent, k1, y.parent, k2)) return true;
    if (lex_less(*L, y.parent, k2, x.parent, k1)) return false;
    return c1 < c2;
  }
};

// ------------------------------------------------------------ round kernel
__global__ void __launch_bounds__(kRoundThreads, 1) k_sched_round(RoundArgs A) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ BState st[2][kMaxBeam];
  __shared__ Lex lex[2];
  __shared__ int s_cnt[kMaxBeam][32];
  __shared__ long long s_scan[kRoundThreads / 32][3];
  __shared__ long long s_carry[3];
  __shared__ int s_status;
  __shared__ int s_picked[kMaxBeam];
  __shared__ int s_cons[kMaxAgents][2];
  __shared__ int s_ncons;
  // dynamic: nodes | children | cand pos | cand mask | details | hist rows
  Node* s_nodes = reinterpret_cast<Node*>(dsm);
  Child* children = reinterpret_cast<Child*>(s_nodes + kSmemNodes);
  uint32_t* c_pos = reinterpret_cast<uint32_t*>(children + A.max_children);
  uint32_t* c_mask = c_pos + A.cand_cap;
  Det* c_det = reinterpret_cast<Det*>(c_mask + A.cand_cap);
  uint32_t* c_hist = reinterpret_cast<uint32_t*>(c_det + A.det_cap);

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int T = blockDim.x;
  const int N = A.N, M = A.M, B = A.B;
  if (tid == 0) {
    s_status = 0;
    s_carry[0] = s_carry[1] = s_carry[2] = 0;
    if (A.timing) A.timing[0] = gtimer();
    if (*A.async_status) {
      s_status = AG_ERR_VALIDATION + 600;  // a dispatch pruned a request to nothing
      *A.async_status = 0;
    }
  }
  for (int i = tid; i < A.n_upd; i += T) A.ready[A.upd_slot[i]] = A.upd_mask[i];
  __syncthreads();
  if (s_status) {
    if (tid == 0) A.out[0] = s_status;
    return;
  }
  // engines / models with a free slot at round start
  uint32_t U0 = 0, U0m = 0;
  for (int e = 0; e < A.eng.E; ++e)
    if (A.eng.slots[e] - A.eng.occ[e] > 0) {
      U0 |= 1u << e;
      if (A.eng.model[e] < 32) U0m |= 1u << A.eng.model[e];
    }

  // ---- A: RoundContext (scheduler.cpp:36-72) in chunks of T*kPer positions.
  // Loads are batched per thread (slot -> ready -> cand/nviable) so the
  // dependent chain costs three memory latencies per chunk.
  long long ta[4] = {0, 0, 0, 0};
  long long tq = clock64();
  for (int base = 0; base < A.Q; base += T * kPer) {
    const int p0 = base + tid * kPer;
    int slot[kPer];
    uint64_t rdy[kPer];
    uint32_t cm1[kPer], nvia[kPer];
    int a1[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) slot[i] = p0 + i < A.Q ? __ldg(A.order + p0 + i) : -1;
#pragma unroll
    for (int i = 0; i < kPer; ++i) rdy[i] = slot[i] >= 0 ? A.ready[slot[i]] : 0ull;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      // first ready agent in (depth desc, declaration asc) order
      int best = -1, br = 1 << 30;
      for (uint64_t b = rdy[i]; b; b &= b - 1) {
        const int a = __ffsll((long long)b) - 1;
        if (A.prio_rank[a] < br) br = A.prio_rank[a], best = a;
      }
      a1[i] = best;
      cm1[i] = best >= 0 ? A.cand[(size_t)slot[i] * N + best] : 0u;
      nvia[i] = best >= 0 ? A.nviable[slot[i]] : 0u;
    }
    { const long long t = clock64(); ta[0] += t - tq; tq = t; }
    // pass 1: counts (pairs, requests, candidates) of this thread's positions
    long long np = 0, nq = 0, nc = 0;
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
    { const long long t = clock64(); ta[1] += t - tq; tq = t; }
    long long x[3] = {np, nq, nc};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1)
#pragma unroll
      #pragma unroll
      for (int k = 0; k < 3; ++k) {
        const long long y = __shfl_up_sync(0xffffffffu, x[k], o);
        if (lane >= o) x[k] += y;
      }
    if (lane == 31)
      #pragma unroll
      for (int k = 0; k < 3; ++k) s_scan[wid][k] = x[k];
    __syncthreads();
    if (wid == 0) {
      long long v[3], z[3];
      #pragma unroll
      for (int k = 0; k < 3; ++k) v[k] = z[k] = lane < T / 32 ? s_scan[lane][k] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1)
        #pragma unroll
        for (int k = 0; k < 3; ++k) {
          const long long y = __shfl_up_sync(0xffffffffu, z[k], o);
          if (lane >= o) z[k] += y;
        }
      if (lane < T / 32)
        #pragma unroll
        for (int k = 0; k < 3; ++k) s_scan[lane][k] = z[k] - v[k] + s_carry[k];
      __syncwarp();
      if (lane == 31)
        #pragma unroll
        for (int k = 0; k < 3; ++k) s_carry[k] += z[k];
    }
    __syncthreads();
    { const long long t = clock64(); ta[2] += t - tq; tq = t; }
    // pass 2: write this thread's candidates (position, engine mask, details,
    // histogram row) in pair order
    int pos = (int)(s_scan[wid][0] + x[0] - np);
    int qr = (int)(s_scan[wid][1] + x[1] - nq);
    int cw = (int)(s_scan[wid][2] + x[2] - nc);
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      if (!rdy[i]) continue;
      const int qi = A.cidx ? A.cidx[p0 + i] : qr;
      ++qr;
      const bool single = (rdy[i] & (rdy[i] - 1)) == 0;
      for (int t = 0; t < N; ++t) {
        const int a = single ? a1[i] : A.prio[t];
        if (!single && !((rdy[i] >> a) & 1ull)) continue;
        const uint32_t cm = single ? cm1[i] : A.cand[(size_t)slot[i] * N + a];
        if (cm & U0m) {
          uint32_t em = 0;  // engine mask of the candidate models
          for (uint32_t b = cm; b; b &= b - 1) em |= 1u << A.eng.m2e[__ffs(b) - 1];
          if (cw < A.cand_cap) {
            c_pos[cw] = (uint32_t)pos;
            c_mask[cw] = em & U0;
          } else {
            A.gcpos[cw - A.cand_cap] = (uint32_t)pos;
            A.gcmask[cw - A.cand_cap] = em & U0;
          }
          const Det d{qi, slot[i], nvia[i], a};
          if (cw < A.det_cap) c_det[cw] = d;
          else A.gdet[cw - A.det_cap] = d;
          if (cw < A.hist_cap) {
            const uint32_t* hr = A.hist + ((size_t)slot[i] * N + a) * M;
            for (int mdl = 0; mdl < M; ++mdl) c_hist[cw * M + mdl] = __ldg(hr + mdl);
          }
          ++cw;
        }
        ++pos;
        if (single) break;
      }
    }
    __syncthreads();
    { const long long t = clock64(); ta[3] += t - tq; tq = t; }
  }
  if (tid == 0 && A.timing)
    #pragma unroll
    for (int k = 0; k < 4; ++k) A.timing[9 + k] = (unsigned long long)ta[k];
  const int npairs = (int)s_carry[0], nreq = (int)s_carry[1], ncand = (int)s_carry[2];
  if (tid == 0 && A.timing) A.timing[1] = gtimer();
  if (s_status) {
    if (tid == 0) A.out[0] = s_status;
    return;
  }
  if (wid != 0) return;
  if (lane == 0 && A.timing) A.timing[2] = gtimer();

  // ---- B: the beam walk (warp 0)
  const NodeView nv{s_nodes, A.gnodes};
  const int E = A.eng.E;
  auto cposf = [&](int j) -> int { return (int)(j < A.cand_cap ? c_pos[j] : A.gcpos[j - A.cand_cap]); };
  auto cmaskf = [&](int j) -> uint32_t { return j < A.cand_cap ? c_mask[j] : A.gcmask[j - A.cand_cap]; };
  auto detf = [&](int j) -> Det { return j < A.det_cap ? c_det[j] : A.gdet[j - A.det_cap]; };
  if (lane == 0) {  // initial_state (scheduler.cpp:117-128)
    BState& s0 = st[0][0];
    s0.util = 0.0;
    s0.flex_sum = 0.0;
    s0.skips = 0;
    s0.flex_count = 0;
    s0.free_mask = 0;
    s0.node = -1;
    s0.nsurv = 0;
    for (int e = 0; e < E; ++e) {
      const int occ = A.eng.occ[e];
      if (occ > A.eng.slots[e]) s_status = AG_ERR_VALIDATION + 200;  // engine over capacity
      s0.occ[e] = occ;
      s0.util += occ * A.eng.weight[e];
      if (A.eng.slots[e] - occ > 0) s0.free_mask |= 1u << e;
    }
    lex[0].len[0] = 0;
  }
  __syncwarp();
  if (s_status) {
    if (lane == 0) A.out[0] = s_status;
    return;
  }
  int cur = 0, nst = 1, nnodes = 0;
  unsigned long long explored = 1;
  int pi = 0;       // next pair position not yet accounted for
  int j = 0;        // next candidate index
  int last_q = -1;  // request of the last visited candidate
  long long tw[4] = {0, 0, 0, 0};
  long long tp = clock64();
  while (true) {
    uint32_t U = lane < nst ? st[cur][lane].free_mask : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) U |= __shfl_xor_sync(0xffffffffu, U, o);
    if (!U) break;  // all-full early exit (scheduler.cpp:303-315)
    // the next candidate of the current request is visited unconditionally
    // (a touched state may still have a constrained mask); otherwise the next
    // candidate whose mask meets a free engine
    int found = ncand;
    if (j < ncand && last_q >= 0 && detf(j).qi == last_q) {
      found = j;
    } else {
      for (int j0 = j; j0 < ncand; j0 += 32) {
        const int jj = j0 + lane;
        const bool ok = jj < ncand && (cmaskf(jj) & U) != 0;
        const uint32_t b = __ballot_sync(0xffffffffu, ok);
        if (b) {
          found = j0 + __ffs(b) - 1;
          break;
        }
      }
    }
    { const long long t = clock64(); tw[0] += t - tp; tp = t; }
    if (found >= ncand) break;
    j = found;
    const int ppos = cposf(j);
    {  // whole-beam skips before this pair
      const long long k = ppos - pi;
      if (k > 0) {
        if (lane < nst) st[cur][lane].skips += k;
        explored += (unsigned long long)nst * (unsigned long long)k;
      }
      pi = ppos + 1;
    }
    const Det d = detf(j);
    const int qcur = d.qi, a = d.agent, slot = d.slot;
    const uint32_t base = cmaskf(j);
    const double initial = (double)d.nvia;
    const bool tch = lane < nst && st[cur][lane].node >= 0 && nv[st[cur][lane].node].qi == qcur;
    // allowed_engines (scheduler.cpp:140-156)
    uint32_t mk = (lane < nst && !tch) ? (base & st[cur][lane].free_mask) : 0u;
    const uint32_t tmask = __ballot_sync(0xffffffffu, tch);
    // re-touch: counts per model of this agent over the request's viable
    // configurations consistent with the state's earlier triples for it
    for (uint32_t tb = tmask; tb; tb &= tb - 1) {
      const int si = __ffs(tb) - 1;
      if (lane == 0) {
        int n = st[cur][si].node, nc = 0;
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
          if (s_cnt[si][mdl] > 0) em |= 1u << A.eng.m2e[mdl];
        mk = em & st[cur][si].free_mask;
      }
      __syncwarp();
    }
    last_q = qcur;
    ++j;
    const bool has = lane < nst && mk != 0;
    if (!__any_sync(0xffffffffu, has)) {  // whole-beam skip (scheduler.cpp:317-329)
      if (lane < nst) st[cur][lane].skips += 1;
      explored += (unsigned long long)nst;
      continue;
    }
    // children in (state, engine ascending) order; a state with no free
    // candidate contributes one skip child (scheduler.cpp:331-349)
    const int my_n = lane < nst ? (mk ? __popc(mk) : 1) : 0;
    int xs = my_n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, xs, o);
      if (lane >= o) xs += y;
    }
    const int nchild = __shfl_sync(0xffffffffu, xs, 31);
    const int hrow = j - 1;  // this candidate's index
    explored += (unsigned long long)nchild;
    const Lex& L = lex[cur];
    const uint64_t key_base = tkey(qcur, a, 0);
    int npick = 0;
    if (nchild <= 32) {
      // lane c builds child c in registers (extend_state, scheduler.cpp:158-206)
      const int c = lane;
      int si = 0, off = 0;
      for (int s2 = 0; s2 < nst; ++s2) {
        const int o2 = __shfl_sync(0xffffffffu, xs - my_n, s2);
        if (c >= o2) si = s2, off = o2;
      }
      const uint32_t pm = __shfl_sync(0xffffffffu, mk, si);
      const bool ptch = __shfl_sync(0xffffffffu, (int)tch, si) != 0;
      double cu = -1.0, cfs = 0.0, cf = 0.0;
      long long csk = 0;
      int cfc = 0, cns = 0, ce = -1;
      uint64_t ck = kEnd;
      const bool valid = c < nchild;
      if (valid) {
        const BState& p = st[cur][si];
        if (!pm) {
          cu = p.util;
          cfs = p.flex_sum;
          cfc = p.flex_count;
          csk = p.skips + 1;
          cns = p.nsurv;
        } else {
          ce = __fns(pm, 0, c - off + 1);
          const int mdl = A.eng.model[ce];
          cu = p.util + A.eng.weight[ce];
          csk = p.skips;
          if (!ptch) {
            const uint32_t surv = hrow < A.hist_cap ? c_hist[hrow * M + mdl]
                                                    : __ldg(A.hist + ((size_t)slot * N + a) * M + mdl);
            cfs = p.flex_sum + (double)surv / initial;
            cfc = p.flex_count + 1;
            cns = (int)surv;
          } else {
            const int surv = s_cnt[si][mdl];
            const double before = (double)p.nsurv / initial;
            cfs = p.flex_sum + ((double)surv / initial - before);
            cfc = p.flex_count;
            cns = surv;
          }
          ck = key_base | (uint64_t)(uint32_t)mdl;
        }
        cf = cfc > 0 ? cfs / cfc : 1.0;
        Child& chd = children[c];
        chd.util = cu;
        chd.flex_sum = cfs;
        chd.flex = cf;
        chd.skips = csk;
        chd.flex_count = cfc;
        chd.nsurv = cns;
        chd.parent = (int16_t)si;
        chd.eng = (int16_t)ce;
      }
      // warp bitonic sort, best first, under state_better (scheduler.cpp:
      // 109-115) then the lower child index; only keys move between lanes
      double ku = cu, kf = cf;
      long long ks = csk;
      int kp = si, ki = valid ? c : -1;
      uint64_t kk = ck;
#pragma unroll 1
      for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll 1
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
          const double ou = __shfl_xor_sync(0xffffffffu, ku, jj);
          const double of = __shfl_xor_sync(0xffffffffu, kf, jj);
          const long long os = __shfl_xor_sync(0xffffffffu, ks, jj);
          const int op = __shfl_xor_sync(0xffffffffu, kp, jj);
          const int oi = __shfl_xor_sync(0xffffffffu, ki, jj);
          const uint64_t ok = __shfl_xor_sync(0xffffffffu, kk, jj);
          bool ob;  // other strictly before mine
          if (oi < 0) ob = false;
          else if (ki < 0) ob = true;
          else if (ou != ku) ob = ou > ku;
          else if (of != kf) ob = of > kf;
          else if (os != ks) ob = os < ks;
          else if (lex_less(L, op, ok, kp, kk)) ob = true;
          else if (lex_less(L, kp, kk, op, ok)) ob = false;
          else ob = oi < ki;
          const bool lo = (lane & jj) == 0, asc = (lane & k) == 0;
          const bool take = (lo == asc) ? ob : (!ob && oi != ki);
          if (take) ku = ou, kf = of, ks = os, kp = op, ki = oi, kk = ok;
        }
      }
      // nested retention (scheduler.cpp:351-370): level w adopts the best
      // unused child of parents < w -- the first eligible in sorted order
      uint32_t used = 0;
      for (int w = 1; w <= B; ++w) {
        const uint32_t el = __ballot_sync(0xffffffffu, ki >= 0 && kp < w) & ~used;
        if (!el) continue;
        const int src = __ffs(el) - 1;
        used |= 1u << src;
        const int pc = __shfl_sync(0xffffffffu, ki, src);
        if (lane == 0) s_picked[npick] = pc;
        ++npick;
      }
    } else {
      // wide beams: children through shared memory, per level a warp arg-max
      if (lane < nst) {
        const BState& p = st[cur][lane];
        int c = xs - my_n;
        if (!mk) {
          Child& chd = children[c];
          chd.parent = (int16_t)lane;
          chd.eng = -1;
          chd.util = p.util;
          chd.flex_sum = p.flex_sum;
          chd.flex_count = p.flex_count;
          chd.skips = p.skips + 1;
          chd.nsurv = p.nsurv;
          chd.flex = chd.flex_count > 0 ? chd.flex_sum / chd.flex_count : 1.0;
        } else {
          for (uint32_t b = mk; b; b &= b - 1, ++c) {
            const int e = __ffs(b) - 1;
            const int mdl = A.eng.model[e];
            Child& chd = children[c];
            chd.parent = (int16_t)lane;
            chd.eng = (int16_t)e;
            chd.util = p.util + A.eng.weight[e];
            chd.skips = p.skips;
            if (!tch) {
              const uint32_t surv = hrow < A.hist_cap ? c_hist[hrow * M + mdl]
                                                      : A.hist[((size_t)slot * N + a) * M + mdl];
              chd.flex_sum = p.flex_sum + (double)surv / initial;
              chd.flex_count = p.flex_count + 1;
              chd.nsurv = (int)surv;
            } else {
              const int surv = s_cnt[lane][mdl];
              const double before = (double)p.nsurv / initial;
              chd.flex_sum = p.flex_sum + ((double)surv / initial - before);
              chd.flex_count = p.flex_count;
              chd.nsurv = surv;
            }
            chd.flex = chd.flex_count > 0 ? chd.flex_sum / chd.flex_count : 1.0;
          }
        }
      }
      __syncwarp();
      const WalkCtx wc{children, &lex[cur], key_base, &A.eng};
      uint32_t used[(kMaxBeam * (kMaxEng + 1) + 31) / 32];
      for (int i = 0; i < (nchild + 31) / 32; ++i) used[i] = 0;
      for (int w = 1; w <= B; ++w) {
        int best = -1;
        for (int c = lane; c < nchild; c += 32) {
          if ((used[c >> 5] >> (c & 31)) & 1u) continue;
          if (children[c].parent >= w) continue;
          if (wc.before(c, best)) best = c;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const int other = __shfl_xor_sync(0xffffffffu, best, o);
          if (wc.before(other, best)) best = other;
        }
        if (best < 0) continue;
        used[best >> 5] |= 1u << (best & 31);
        if (lane == 0) s_picked[npick] = best;
        ++npick;
      }
    }
    __syncwarp();
    { const long long t = clock64(); tw[1] += t - tp; tp = t; }
    // adopt: picked child w becomes state w of the next beam
    const int nxt = cur ^ 1;
    bool mknode = false;
    int pc = -1;
    if (lane < npick) {
      pc = s_picked[lane];
      mknode = children[pc].eng >= 0;
    }
    const uint32_t nb = __ballot_sync(0xffffffffu, mknode);
    if (lane < npick) {
      const Child& chd = children[pc];
      const BState& p = st[cur][chd.parent];
      BState& q = st[nxt][lane];
      for (int e = 0; e < E; ++e) q.occ[e] = p.occ[e];
      q.util = chd.util;
      q.flex_sum = chd.flex_sum;
      q.flex_count = chd.flex_count;
      q.skips = chd.skips;
      q.free_mask = p.free_mask;
      q.node = p.node;
      q.nsurv = chd.nsurv;
      lex[nxt].len[lane] = L.len[chd.parent] + (mknode ? 1 : 0);
      if (mknode) {
        const int e = chd.eng;
        if (++q.occ[e] >= A.eng.slots[e]) q.free_mask &= ~(1u << e);
        const int id = nnodes + __popc(nb & ((1u << lane) - 1u));
        if (id < A.max_nodes) {
          Node nd;
          nd.qi = qcur;
          nd.am = (a << 8) | A.eng.model[e];
          nd.prev = p.node;
          nd.depth = depth_of(nv, p.node) + 1;
          nd.nsurv = chd.nsurv;
          nd.nvia = d.nvia;
          nd.slot = slot;
          nd.pad = 0;
          if (id < kSmemNodes) s_nodes[id] = nd;
          else A.gnodes[id - kSmemNodes] = nd;
        } else {
          s_status = AG_ERR_INTERNAL + 300;  // history overflow
        }
        q.node = id;
      }
    }
    // lexicographic structure of the new beam
    for (int pr = lane; pr < npick * npick; pr += 32) {
      const int w1 = pr / npick, w2 = pr - w1 * npick;
      if (w1 == w2) continue;
      const Child& c1 = children[s_picked[w1]];
      const int p1 = c1.parent, p2 = children[s_picked[w2]].parent;
      const uint64_t k1 = c1.eng >= 0 ? key_base | (uint64_t)(uint32_t)A.eng.model[c1.eng] : kEnd;
      int l;
      uint64_t nx;
      if (p1 == p2) {
        l = L.len[p1];
        nx = k1;
      } else {
        l = L.lcp[p1][p2];
        nx = l < L.len[p1] ? L.nxt[p1][p2] : k1;
      }
      lex[nxt].lcp[w1][w2] = l;
      lex[nxt].nxt[w1][w2] = nx;
    }
    nnodes += __popc(nb);
    { const long long t = clock64(); tw[2] += t - tp; tp = t; }

    __syncwarp();
    if (s_status) {
      if (lane == 0) A.out[0] = s_status;
      return;
    }
    cur = nxt;
    nst = npick;
    { const long long t = clock64(); tw[3] += t - tp; tp = t; }
  }
  if (lane == 0 && A.timing)
    #pragma unroll
    for (int k = 0; k < 4; ++k) A.timing[5 + k] = (unsigned long long)tw[k];
  {  // the remaining pairs are skips (all-full exit or no candidate left)
    const long long rem = npairs - pi;
    if (rem > 0) {
      if (lane < nst) st[cur][lane].skips += rem;
      explored += (unsigned long long)nst * (unsigned long long)rem;
    }
  }
  __syncwarp();
  if (lane == 0 && A.timing) A.timing[3] = gtimer();

  // ---- C: winner and finalize (scheduler.cpp:373-377, 208-220, 248-287)
  int best = lane < nst ? lane : -1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int other = __shfl_xor_sync(0xffffffffu, best, o);
    if (other < 0) continue;
    if (best < 0) {
      best = other;
      continue;
    }
    const BState& s1 = st[cur][best];
    const BState& s2 = st[cur][other];
    const double f1 = s1.flex_count > 0 ? s1.flex_sum / s1.flex_count : 1.0;
    const double f2 = s2.flex_count > 0 ? s2.flex_sum / s2.flex_count : 1.0;
    bool o_better;  // is `other` strictly better than `best`?
    if (s1.util != s2.util) o_better = s2.util > s1.util;
    else if (f1 != f2) o_better = f2 > f1;
    else if (s1.skips != s2.skips) o_better = s2.skips < s1.skips;
    else if (lex_less(lex[cur], other, kEnd, best, kEnd)) o_better = true;
    else if (lex_less(lex[cur], best, kEnd, other, kEnd)) o_better = false;
    else o_better = other < best;
    if (o_better) best = other;
  }
  const BState& w = st[cur][best];
  const int D = depth_of(nv, w.node);
  ag_assignment* res = reinterpret_cast<ag_assignment*>((char*)A.out + kOutHeader);
  int32_t* occ_out = reinterpret_cast<int32_t*>(res + 1);
  ag_triple* triples = reinterpret_cast<ag_triple*>(occ_out + kMaxEng);
  if (D > A.triples_cap) {
    if (lane == 0) {
      A.out[0] = AG_ERR_VALIDATION + 400;
      A.out[1] = D;
    }
    return;
  }
  // the path, root first (node ids into the children area, free now)
  int* path = reinterpret_cast<int*>(children);
  int path_cap = (int)(sizeof(Child) * A.max_children / sizeof(int));
  if (lane == 0) {
    int n = w.node;
    for (int i = D - 1; i >= 0; --i) {
      if (i < path_cap) path[i] = n;
      n = nv[n].prev;
    }
  }
  __syncwarp();
  for (int i = lane; i < D; i += 32) {
    int n = -1;
    if (i < path_cap) {
      n = path[i];
    } else {  // long path: walk from the winner (rare)
      n = w.node;
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
  __syncwarp();
  if (lane != 0) return;
  // score_assignment (scheduler.cpp:248-287): utilization in engine order;
  // flexibility over touched requests in queue (container) order with the
  // survivors consistent with all of a request's triples (its last node)
  double util = 0.0;
  for (int e = 0; e < E; ++e) {
    if (w.occ[e] < 0 || w.occ[e] > A.eng.slots[e]) {
      A.out[0] = AG_ERR_VALIDATION + 500;
      return;
    }
    util += w.occ[e] * A.eng.weight[e];
    occ_out[e] = w.occ[e];
  }
  double flex_sum = 0.0;
  int flex_count = 0;
  if (D > 0) {
    // a request's triples are consecutive on the path; in a session the
    // queue is in FIFO = container order, so requests appear ascending
    bool ascending = D <= path_cap;
    int prevq = -1;
    for (int i = 0; i < D && ascending; ++i) {
      const int q = nv[path[i]].qi;
      if (q != prevq) {
        if (q < prevq) ascending = false;
        prevq = q;
      }
    }
    if (ascending) {
      int n = w.node, lastq = -1;
      // walk back: the first node met per request is its last triple; fold
      // order must be ascending, so accumulate into a stack then fold
      int* stk = path + min(D, path_cap);  // reuse space after the path
      int ns = 0;
      const int stk_cap = path_cap - min(D, path_cap);
      bool spill = false;
      while (n >= 0) {
        const Node& nd = nv[n];
        if (nd.qi != lastq) {
          if (ns < stk_cap) stk[ns] = n;
          else spill = true;
          ++ns;
          lastq = nd.qi;
        }
        n = nd.prev;
      }
      if (!spill) {
        for (int k = ns - 1; k >= 0; --k) {
          const Node& nd = nv[stk[k]];
          flex_sum += (double)nd.nsurv / (double)nd.nvia;
          ++flex_count;
        }
      } else {
        ascending = false;  // fall through to the general fold
      }
    }
    if (!ascending) {
      // general container order: repeatedly take the smallest unseen request
      int prev = -1;
      for (;;) {
        int nq = 0x7fffffff;
        for (int i = 0; i < D; ++i) {
          const int q = triples[i].request_index;
          if (q > prev && q < nq) nq = q;
        }
        if (nq == 0x7fffffff) break;
        for (int nn = w.node; nn >= 0; nn = nv[nn].prev)
          if (nv[nn].qi == nq) {
            flex_sum += (double)nv[nn].nsurv / (double)nv[nn].nvia;
            ++flex_count;
            break;
          }
        prev = nq;
      }
    }
  }
  ag_assignment r;
  r.n_triples = D;
  r.pad = 0;
  r.utilization = util;
  r.flexibility = flex_count > 0 ? flex_sum / flex_count : 1.0;
  r.skips = w.skips;
  r.states_explored = explored;
  *res = r;
  if (A.timing) A.timing[4] = gtimer();
  A.out[0] = 0;
  A.out[1] = nreq;
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
};

__device__ __forceinline__ uint32_t digit_p(uint32_t c, int a, const PruneArgs& A) {
  const uint32_t q = A.place[a] == 1 ? c : (uint32_t)__umul64hi(c, A.place_magic[a]);
  return q - divm(q, A.div_m) * (uint32_t)A.M;
}

// Request::mark_dispatched prefix pruning (request.cpp:70-86) for every
// triple of one request, then its histogram / candidate masks from scratch.
// With g_meta it first installs a new request's metadata (Request::make).
__global__ void __launch_bounds__(256) k_sched_prune(PruneArgs A) {
  __shared__ uint32_t s_hist[kMaxAgents * 32];
  __shared__ int s_w[8], s_tot;
  const int g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int s = A.g_slot[g];
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
  for (int t = A.g_begin[g]; t < A.g_begin[g + 1]; ++t) {
    const int a = A.g_am[t] >> 8, mdl = A.g_am[t] & 0xFF;
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
  size_t dead = 0;
  std::vector<int32_t> upd_slot;
  std::vector<uint64_t> upd_mask;
  int8_t prio[64];
  uint32_t place[agb::kMaxAgents];
  uint64_t place_magic[agb::kMaxAgents];
  bool attr_set = false;
  double last_round_us = 0.0;
  // device
  agb::Scratch d_ready, d_cand, d_hist, d_nv, d_voff, d_pool, d_ids, d_order, d_cidx;
  agb::Scratch d_cpos, d_cmask, d_det, d_nodes, d_out, d_status, d_upd, d_gam, d_qa;
  // pinned host staging
  void* h_res = nullptr;
  size_t h_res_bytes = 0;
  void* h_stage = nullptr;  // dispatch / add uploads
  size_t h_stage_bytes = 0;
  void* h_rstage = nullptr;  // round uploads
  size_t h_rstage_bytes = 0;
  ~ag_sched() {
    if (h_res) cudaFreeHost(h_res);
    if (h_stage) cudaFreeHost(h_stage);
    if (h_rstage) cudaFreeHost(h_rstage);
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
  AG_CUDA(cudaMallocHost(p, b));
  *have = b;
  return AG_OK;
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
  for (int slot : s->order)
    if (s->live[slot]) live_order.push_back(slot);
  s->order.swap(live_order);
  s->dirty_from = 0;
  s->dead = 0;
  s->free_slots.insert(s->free_slots.end(), s->quarantine.begin(), s->quarantine.end());
  s->quarantine.clear();
}

int launch_prune(ag_sched* s, const std::vector<int32_t>& g_slot, const std::vector<int32_t>& g_begin,
                 const std::vector<int32_t>& g_am, const std::vector<uint64_t>* meta) {
  ag_ctx* ctx = s->ctx;
  const int G = (int)g_slot.size();
  if (G == 0) return AG_OK;
  int rc;
  const size_t n32 = (size_t)G + (G + 1) + g_am.size();
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
  PruneArgs A;
  A.N = s->N;
  A.M = s->M;
  const int32_t* d = (const int32_t*)s->d_gam.p;
  A.g_slot = d;
  A.g_begin = d + G;
  A.g_am = d + 2 * G + 1;
  A.g_meta = meta ? (const uint64_t*)((const char*)s->d_gam.p + off_meta) : nullptr;
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
  {
    Launch L(ctx, meta ? K_SCHED_PREP : K_SCHED_APPLY);
    k_sched_prune<<<G, 256, 0, ctx->stream>>>(A);
  }
  AG_CUDA(cudaGetLastError());
  return AG_OK;
}

int engines_dev(const ag_engines* e, EngDev* out) {
  // RoundContext validation (scheduler.cpp:39-52)
  if (!e) return fail(AG_ERR_VALIDATION, "engines is null");
  if (e->n_engines > kMaxEng) return fail(AG_ERR_VALIDATION, "more engine pools than the scheduler supports");
  EngDev d{};
  d.E = e->n_engines;
  for (int i = 0; i < 32; ++i) d.m2e[i] = -1;
  for (int i = 0; i < d.E; ++i) {
    const int mdl = e->model[i];
    if (mdl < 0) return fail(AG_ERR_VALIDATION, "engine with negative model tier");
    for (int k = 0; k < i; ++k)
      if (e->model[k] == mdl) return fail(AG_ERR_VALIDATION, "two engine pools serve the same model tier");
    if (mdl < 32) {
      d.m2e[mdl] = (int8_t)i;
      d.mapped |= 1u << mdl;
    }
    d.model[i] = mdl;
    d.slots[i] = e->slots[i];
    d.occ[i] = e->occupancy[i];
    d.weight[i] = e->weight[i];
  }
  *out = d;
  return AG_OK;
}

// One round over the session queue (or an explicit FIFO/container mapping).
int run_round(ag_sched* s, const ag_engines* engines, int B, const int32_t* cidx_host,
              ag_assignment* out, ag_triple* triples, int32_t triples_cap, int32_t* occupancy) {
  const auto t_start = std::chrono::steady_clock::now();
  ag_ctx* ctx = s->ctx;
  if (B < 1) return fail(AG_ERR_VALIDATION, "beam width < 1");
  if (B > kMaxBeam) return fail(AG_ERR_VALIDATION, "GPU scheduler supports beam width <= 32");
  EngDev ed;
  int rc = engines_dev(engines, &ed);
  if (rc) return rc;
  int total_free = 0;
  for (int i = 0; i < ed.E; ++i) total_free += std::max(0, ed.slots[i] - ed.occ[i]);
  const int Q = (int)s->order.size();
  const int cap_t = total_free + 1;
  const int max_children = B * (ed.E + 1);
  const size_t max_pairs = (size_t)Q * (size_t)s->N + 1;
  const int max_nodes = (int)std::min<size_t>((size_t)B * max_pairs + 16, (size_t)1 << 30);
  // ---- uploads: order tail, ready updates (deduplicated: one entry per slot)
  cudaStream_t st = ctx->stream;
  if (s->upd_slot.size() > 1) {
    std::vector<char> seen(s->cap, 0);
    size_t w = s->upd_slot.size();
    for (size_t i = s->upd_slot.size(); i-- > 0;) {
      const int slot = s->upd_slot[i];
      if (seen[slot]) continue;
      seen[slot] = 1;
      --w;
      s->upd_slot[w] = slot;
      s->upd_mask[w] = s->upd_mask[i];
    }
    s->upd_slot.erase(s->upd_slot.begin(), s->upd_slot.begin() + w);
    s->upd_mask.erase(s->upd_mask.begin(), s->upd_mask.begin() + w);
  }
  const size_t nu = s->upd_slot.size();
  const size_t n_tail = Q > (int)s->dirty_from ? Q - s->dirty_from : 0;
  const size_t up_bytes = nu * 12 + 16 + n_tail * 4 + (cidx_host ? (size_t)Q * 4 : 0);
  const size_t res_bytes = kOutHeader + sizeof(ag_assignment) + 4 * kMaxEng + (size_t)cap_t * sizeof(ag_triple);
  if ((rc = ensure_pinned(&s->h_rstage, &s->h_rstage_bytes, up_bytes)) ||
      (rc = ensure_pinned(&s->h_res, &s->h_res_bytes, res_bytes)) ||
      (rc = s->d_upd.ensure(up_bytes)) ||
      (rc = s->d_out.ensure(res_bytes)) || (rc = s->d_status.ensure(192)))
    return rc;
  // the previous round synchronised after its last use of h_rstage
  char* h = (char*)s->h_rstage;
  std::memcpy(h, s->upd_mask.data(), nu * 8);
  std::memcpy(h + nu * 8, s->upd_slot.data(), nu * 4);
  const size_t off_cidx = (nu * 12 + 15) & ~(size_t)15;
  if (cidx_host) std::memcpy(h + off_cidx, cidx_host, (size_t)Q * 4);
  const size_t up_main = off_cidx + (cidx_host ? (size_t)Q * 4 : 0);
  if (up_main) AG_CUDA(cudaMemcpyAsync(s->d_upd.p, h, up_main, cudaMemcpyHostToDevice, st));
  if (n_tail) {
    std::memcpy(h + up_main, s->order.data() + s->dirty_from, n_tail * 4);
    AG_CUDA(cudaMemcpyAsync((int32_t*)s->d_order.p + s->dirty_from, h + up_main, n_tail * 4,
                            cudaMemcpyHostToDevice, st));
    s->dirty_from = Q;
  }
  // ---- shared memory plan: nodes | children | cand (pos, mask) | details | hist rows
  const size_t static_bytes = 2 * kMaxBeam * sizeof(BState) + 2 * sizeof(Lex) + kMaxBeam * 32 * 4 + 8192;
  const size_t max_dyn = 227 * 1024 - static_bytes;
  const size_t fixed = sizeof(Node) * kSmemNodes + sizeof(Child) * (size_t)max_children;
  if (fixed > max_dyn) return fail(AG_ERR_VALIDATION, "beam too wide for one CTA");
  size_t room = max_dyn - fixed;
  const int cand_cap = (int)std::min<size_t>(max_pairs, room * 5 / 10 / 8);
  room -= (size_t)cand_cap * 8;
  // the walk visits the head of the candidate list (engines fill quickly);
  // details and histogram rows are staged for that head only
  const int det_cap = (int)std::min<size_t>(std::min<size_t>(max_pairs, 2048), room / 2 / sizeof(Det));
  room -= (size_t)det_cap * sizeof(Det);
  const int hist_cap =
      (int)std::min<size_t>(std::min<size_t>((size_t)det_cap, 512), room / (4 * (size_t)s->M));
  const size_t dyn = fixed + (size_t)cand_cap * 8 + (size_t)det_cap * sizeof(Det) +
                     (size_t)hist_cap * 4 * s->M;
  const size_t g_over = max_pairs > (size_t)cand_cap ? max_pairs - cand_cap : 1;
  const size_t g_det = max_pairs > (size_t)det_cap ? max_pairs - det_cap : 1;
  if ((rc = s->d_cpos.ensure(g_over * 4)) || (rc = s->d_cmask.ensure(g_over * 4)) ||
      (rc = s->d_det.ensure(g_det * sizeof(Det))) ||
      (rc = s->d_nodes.ensure((size_t)std::max(1, max_nodes - kSmemNodes) * sizeof(Node))))
    return rc;
  if (!s->attr_set) {
    AG_CUDA(cudaFuncSetAttribute(k_sched_round, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_dyn));
    s->attr_set = true;
  }
  RoundArgs A;
  std::memset(&A, 0, sizeof A);
  A.N = s->N;
  A.M = s->M;
  A.B = B;
  A.order = (const int32_t*)s->d_order.p;
  A.cidx = cidx_host ? (const int32_t*)((char*)s->d_upd.p + off_cidx) : nullptr;
  A.Q = Q;
  A.ready = (uint64_t*)s->d_ready.p;
  A.n_upd = (int)nu;
  A.upd_mask = (const uint64_t*)s->d_upd.p;
  A.upd_slot = (const int32_t*)((char*)s->d_upd.p + nu * 8);
  A.cand = (const uint32_t*)s->d_cand.p;
  A.hist = (const uint32_t*)s->d_hist.p;
  A.nviable = (const uint32_t*)s->d_nv.p;
  A.voff = (const uint64_t*)s->d_voff.p;
  A.pool = (const uint32_t*)s->d_pool.p;
  A.ids = (const uint64_t*)s->d_ids.p;
  std::memcpy(A.prio, s->prio, sizeof A.prio);
  for (int t = 0; t < s->N; ++t) A.prio_rank[(int)s->prio[t]] = (int8_t)t;
  std::memcpy(A.place, s->place, sizeof A.place);
  std::memcpy(A.place_magic, s->place_magic, sizeof A.place_magic);
  A.div_m = ctx->space->dev().div_m;
  A.eng = ed;
  A.gcpos = (uint32_t*)s->d_cpos.p;
  A.gcmask = (uint32_t*)s->d_cmask.p;
  A.gdet = (Det*)s->d_det.p;
  A.cand_cap = cand_cap;
  A.det_cap = det_cap;
  A.hist_cap = hist_cap;
  A.gnodes = (Node*)s->d_nodes.p;
  A.max_nodes = max_nodes;
  A.max_children = max_children;
  A.out = (int32_t*)s->d_out.p;
  A.triples_cap = cap_t;
  A.timing = (unsigned long long*)((char*)s->d_status.p + 32);
  A.async_status = (int32_t*)s->d_status.p;
  {
    Launch L(ctx, K_SCHED_ROUND);
    k_sched_round<<<1, kRoundThreads, dyn, st>>>(A);
  }
  AG_CUDA(cudaGetLastError());
  char* hr = (char*)s->h_res;
  AG_CUDA(cudaMemcpyAsync(hr, s->d_out.p, res_bytes, cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaStreamSynchronize(st));
  s->upd_slot.clear();
  s->upd_mask.clear();
  const int32_t status = ((int32_t*)hr)[0];
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
  s->last_round_us =
      std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_start).count();
  return AG_OK;
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
  if (!ctx || !out) return fail(AG_ERR_VALIDATION, "null argument");
  *out = nullptr;
  const ag_space* sp = ctx->space;
  if (!sp->gpu_ok) return fail(AG_ERR_VALIDATION, "GPU path needs M^N <= 2^32 and N <= 32");
  if (sp->m > 32) return fail(AG_ERR_VALIDATION, "GPU scheduler supports at most 32 model tiers");
  if (max_requests < 1) return fail(AG_ERR_VALIDATION, "max_requests < 1");
  ag_sched* s = new ag_sched();
  s->ctx = ctx;
  s->N = sp->n;
  s->M = sp->m;
  s->cap = max_requests;
  s->pool_cap = std::max<uint64_t>(max_configs, 1);
  s->ids.assign(max_requests, 0);
  s->arrival.assign(max_requests, 0.0);
  s->stages.assign((size_t)max_requests * sp->n, 0);
  s->ready.assign(max_requests, 0);
  s->live.assign(max_requests, 0);
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
      (rc = s->d_order.ensure(((size_t)2 * max_requests + 1024) * 4))) {
    delete s;
    return rc;
  }
  cudaMemsetAsync(s->d_ready.p, 0, R * 8, ctx->stream);
  cudaMemsetAsync(s->d_status.p, 0, 128, ctx->stream);
  *out = s;
  return AG_OK;
}

void ag_sched_destroy(ag_sched* s) { delete s; }

int ag_sched_add(ag_sched* s, const ag_queue* q, int32_t* slots_out) {
  if (!s || !q) return fail(AG_ERR_VALIDATION, "null argument");
  ag_ctx* ctx = s->ctx;
  const int R = q->n_requests;
  if (R <= 0) return R == 0 ? AG_OK : fail(AG_ERR_VALIDATION, "negative request count");
  if ((int)s->free_slots.size() < R && !s->quarantine.empty()) agb::compact_order(s);
  if ((int)s->free_slots.size() < R) return fail(AG_ERR_VALIDATION, "session is full");
  const uint64_t total = (uint64_t)(q->viable_ptr[R] - q->viable_ptr[0]);
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
    s->ready[slot] = agb::ready_of(s, slot);
    s->live[slot] = 1;
    s->nviable[slot] = (uint32_t)(q->viable_ptr[i + 1] - q->viable_ptr[i]);
    meta[3 * i] = s->pool_top + (uint64_t)(q->viable_ptr[i] - q->viable_ptr[0]);
    meta[3 * i + 1] = s->nviable[slot];
    meta[3 * i + 2] = q->ids[i];
    s->upd_slot.push_back(slot);
    s->upd_mask.push_back(s->ready[slot]);
    if (slots_out) slots_out[i] = slot;
  }
  AG_CUDA(cudaMemcpyAsync((uint32_t*)s->d_pool.p + s->pool_top, q->viable + q->viable_ptr[0],
                          total * 4, cudaMemcpyHostToDevice, ctx->stream));
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
    s->dirty_from = std::min(s->dirty_from, pos);
  }
  // the viable copy must land before the histogram pass reads it (same stream)
  return agb::launch_prune(s, slots, g_begin, {}, &meta);
}

int ag_sched_remove(ag_sched* s, int32_t n, const int32_t* slots) {
  if (!s) return fail(AG_ERR_VALIDATION, "null argument");
  for (int i = 0; i < n; ++i) {
    const int slot = slots[i];
    if (slot < 0 || slot >= s->cap || !s->live[slot]) return fail(AG_ERR_VALIDATION, "bad slot");
    s->live[slot] = 0;
    s->ready[slot] = 0;
    s->upd_slot.push_back(slot);
    s->upd_mask.push_back(0);
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
  return AG_OK;
}

int ag_sched_complete(ag_sched* s, int32_t slot, int32_t agent) {
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
  if (r != s->ready[slot]) {
    s->ready[slot] = r;
    s->upd_slot.push_back(slot);
    s->upd_mask.push_back(r);
  }
  return AG_OK;
}

int ag_sched_round(ag_sched* s, const ag_engines* engines, int beam_width, ag_assignment* out,
                   ag_triple* triples, int32_t triples_cap, int32_t* occupancy) {
  if (!s) return fail(AG_ERR_VALIDATION, "null argument");
  return agb::run_round(s, engines, beam_width, nullptr, out, triples, triples_cap, occupancy);
}

int ag_sched_dispatch(ag_sched* s, int32_t n, const ag_triple* applied) {
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
    const uint64_t r = agb::ready_of(s, slot);
    s->ready[slot] = r;
    s->upd_slot.push_back(slot);
    s->upd_mask.push_back(r);
  }
  return agb::launch_prune(s, g_slot, g_begin, g_am, nullptr);
}

int ag_sched_queued_ahead(ag_sched* s, int32_t* out) {
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
  if (!s || !ns) return fail(AG_ERR_VALIDATION, "null argument");
  AG_CUDA(cudaMemcpyAsync(ns, (char*)s->d_status.p + 32, 104, cudaMemcpyDeviceToHost, s->ctx->stream));
  AG_CUDA(cudaStreamSynchronize(s->ctx->stream));
  return AG_OK;
}

double ag_sched_last_round_us(const ag_sched* s) { return s ? s->last_round_us : 0.0; }

int ag_sched_viable(ag_sched* s, int32_t slot, uint32_t* out, int64_t cap, int64_t* n) {
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

// Stateless beam_schedule: a throwaway session holding exactly this queue.
int ag_beam_schedule(ag_ctx* ctx, const ag_queue* q, const ag_engines* engines, int beam_width,
                     ag_assignment* out, ag_triple* triples, int32_t triples_cap,
                     int32_t* occupancy) {
  if (!ctx || !q || !engines) return fail(AG_ERR_VALIDATION, "null argument");
  if (beam_width < 1) return fail(AG_ERR_VALIDATION, "beam width < 1");
  const int R = q->n_requests;
  const uint64_t total = R > 0 ? (uint64_t)(q->viable_ptr[R] - q->viable_ptr[0]) : 0;
  ag_sched* s = nullptr;
  int rc = ag_sched_create(ctx, std::max(R, 1), std::max<uint64_t>(total, 1), &s);
  if (rc) return rc;
  std::vector<int32_t> slots(std::max(R, 1));
  if ((rc = ag_sched_add(s, q, slots.data()))) {
    delete s;
    return rc;
  }
  // container index per FIFO position; requests without ready stages keep
  // their container index (they simply contribute no pairs)
  std::vector<int32_t> slot_to_ci(s->cap, -1);
  for (int i = 0; i < R; ++i) slot_to_ci[slots[i]] = i;
  std::vector<int32_t> cidx(s->order.size());
  for (size_t p = 0; p < s->order.size(); ++p) cidx[p] = slot_to_ci[s->order[p]];
  rc = agb::run_round(s, engines, beam_width, cidx.data(), out, triples, triples_cap, occupancy);
  if (rc == AG_OK && out)
    for (int i = 0; i < out->n_triples; ++i) triples[i].slot = -1;
  delete s;
  return rc;
}

}  // extern "C"
