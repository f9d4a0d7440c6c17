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
//   A. block-parallel RoundContext: FIFO pairs (arrival, id) x ready agents
//      by (depth desc, declaration asc), per-pair engine masks, validation;
//      then the list of pairs that can ever be non-skipped in this round
//      (mask & initial-free != 0) is compacted into shared memory.
//   B. warp 0 walks the pairs exactly as beam_schedule does.  A run of pairs
//      whose masks miss every state's free engines is a run of whole-beam
//      skips (scheduler.cpp:317-329) and is fast-forwarded with one ballot
//      scan over the candidate list; at a non-skip step lanes are children
//      (extend_state), nested retention is a warp arg-max per level with the
//      exact state_better order, and a child's triple list is a node in a
//      history tree (triples_less compares two tree paths).
//   C. finalize: the winner's triples from the tree, score_assignment's
//      utilization and flexibility recomputed in the reference's order.
// All fp64 arithmetic repeats the reference's operations in the same order
// (the library builds with --fmad=false).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "ag_internal.h"

namespace agb {

namespace {

constexpr int kRoundThreads = 1024;
constexpr int kMaxBeam = 32;
constexpr int kMaxEng = 32;
constexpr int kSmemNodes = 2048;

struct Node {  // one AssignmentTriple in the beam history tree
  int32_t qi;
  int32_t am;  // agent << 8 | model
  int32_t prev;
  int32_t depth;
  int32_t nsurv;  // survivors of request qi after this triple
};

struct BState {  // BeamState (scheduler.cpp:80-93)
  double util, flex_sum;
  long long skips;
  int flex_count;
  uint32_t free_mask;
  int node;   // latest history node, -1 = no triple
  int nsurv;  // survivors of the request of `node`
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
};

struct RoundArgs {
  int N, M, B;
  const int32_t* order;  // [Q] slots in FIFO order
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
  uint32_t place[kMaxAgents];
  uint64_t place_magic[kMaxAgents];
  uint64_t div_m;
  EngDev eng;
  // scratch
  int32_t* pair_qi;
  uint8_t* pair_agent;
  uint32_t* pair_mask;
  int32_t* qslot;
  uint32_t* gcand_pos;
  uint32_t* gcand_mask;
  int cand_smem_cap;
  Node* gnodes;
  int max_nodes;
  int max_children;
  // outputs
  ag_triple* triples;
  int triples_cap;
  int32_t* occ_out;
  ag_assignment* result;
  int32_t* status;  // [0] status code, [1] queue size
};

__device__ __forceinline__ uint32_t digit_at(uint32_t c, int a, const RoundArgs& A) {
  const uint32_t q = A.place[a] == 1 ? c : (uint32_t)__umul64hi(c, A.place_magic[a]);
  return q - divm(q, A.div_m) * (uint32_t)A.M;
}

// ------------------------------------------------------------ comparisons
struct NodeView {
  const Node* s;  // shared-memory nodes [0, kSmemNodes)
  const Node* g;  // global overflow
  __device__ const Node& operator[](int i) const { return i < kSmemNodes ? s[i] : g[i - kSmemNodes]; }
};

struct Item {  // a beam state or a child: path(node) [+ extra triple]
  int node;
  bool has_extra;
  int eqi, eam;
};

__device__ __forceinline__ int depth_of(const NodeView& nv, int n) { return n < 0 ? 0 : nv[n].depth; }

// triples_less (scheduler.cpp:95-105): lexicographic (request_index, agent,
// model) over two triple sequences, compared through their tree paths.
__device__ bool triples_less(const NodeView& nv, const Item& a, const Item& b) {
  // ca/cb: the element right after the common prefix; kind 0 none, 1 node, 2 extra
  int ka = a.has_extra ? 2 : 0, kb = b.has_extra ? 2 : 0;
  int na = -1, nb = -1;  // node ids when kind == 1
  int x = a.node, y = b.node;
  while (depth_of(nv, x) > depth_of(nv, y)) {
    ka = 1;
    na = x;
    x = nv[x].prev;
  }
  while (depth_of(nv, y) > depth_of(nv, x)) {
    kb = 1;
    nb = y;
    y = nv[y].prev;
  }
  while (x != y) {
    ka = 1;
    na = x;
    kb = 1;
    nb = y;
    x = nv[x].prev;
    y = nv[y].prev;
  }
  if (ka == 0) return kb != 0;  // a is a prefix of b (or equal)
  if (kb == 0) return false;
  const int qa = ka == 1 ? nv[na].qi : a.eqi, ama = ka == 1 ? nv[na].am : a.eam;
  const int qb = kb == 1 ? nv[nb].qi : b.eqi, amb = kb == 1 ? nv[nb].am : b.eam;
  if (qa != qb) return qa < qb;
  return ama < amb;  // agent in bits 8.., model in bits 0..7
}

// state_better (scheduler.cpp:109-115)
__device__ bool better(const NodeView& nv, double ua, double fa, long long sa, const Item& ia,
                       double ub, double fb, long long sb, const Item& ib) {
  if (ua != ub) return ua > ub;
  if (fa != fb) return fa > fb;
  if (sa != sb) return sa < sb;
  return triples_less(nv, ia, ib);
}

__device__ __forceinline__ Item child_item(const Child& c, const BState* st, int qcur, int am) {
  Item it;
  it.node = st[c.parent].node;
  it.has_extra = c.eng >= 0;
  it.eqi = qcur;
  it.eam = am;
  return it;
}

// ------------------------------------------------------------ round kernel
__global__ void __launch_bounds__(kRoundThreads, 1) k_sched_round(RoundArgs A) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ BState st[2][kMaxBeam];
  __shared__ int s_cnt[kMaxBeam][32];
  __shared__ long long s_scan[kRoundThreads / 32][2];
  __shared__ int s_status, s_npairs, s_nreq, s_ncand;
  __shared__ int s_picked[kMaxBeam];
  __shared__ int s_cons[kMaxAgents][2];
  __shared__ int s_ncons;
  // dynamic shared memory: history nodes | children | candidate pairs
  Node* s_nodes = reinterpret_cast<Node*>(dsm);
  Child* children = reinterpret_cast<Child*>(dsm + sizeof(Node) * kSmemNodes);
  uint32_t* c_pos =
      reinterpret_cast<uint32_t*>(dsm + sizeof(Node) * kSmemNodes + sizeof(Child) * A.max_children);
  uint32_t* c_mask = c_pos + A.cand_smem_cap;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int T = blockDim.x;
  if (tid == 0) s_status = 0;
  for (int i = tid; i < A.n_upd; i += T) A.ready[A.upd_slot[i]] = A.upd_mask[i];
  __syncthreads();

  // ---- A1: count pairs / requests per contiguous FIFO range
  const int per = (A.Q + T - 1) / T;
  const int p0 = min(A.Q, tid * per), p1 = min(A.Q, p0 + per);
  long long npair = 0, nreq = 0;
  for (int p = p0; p < p1; ++p) {
    const uint64_t r = A.ready[A.order[p]];
    npair += __popcll(r);
    nreq += r != 0;
  }
  {
    long long x0 = npair, x1 = nreq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y0 = __shfl_up_sync(0xffffffffu, x0, o);
      const long long y1 = __shfl_up_sync(0xffffffffu, x1, o);
      if (lane >= o) x0 += y0, x1 += y1;
    }
    if (lane == 31) s_scan[wid][0] = x0, s_scan[wid][1] = x1;
    __syncthreads();
    if (wid == 0) {
      long long v0 = lane < T / 32 ? s_scan[lane][0] : 0, v1 = lane < T / 32 ? s_scan[lane][1] : 0;
      long long z0 = v0, z1 = v1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y0 = __shfl_up_sync(0xffffffffu, z0, o);
        const long long y1 = __shfl_up_sync(0xffffffffu, z1, o);
        if (lane >= o) z0 += y0, z1 += y1;
      }
      if (lane < T / 32) s_scan[lane][0] = z0 - v0, s_scan[lane][1] = z1 - v1;
      if (lane == 31) s_npairs = (int)z0, s_nreq = (int)z1;
    }
    __syncthreads();
    npair = s_scan[wid][0] + x0 - npair;  // exclusive offsets of this thread
    nreq = s_scan[wid][1] + x1 - nreq;
  }
  // ---- A2: write pairs with engine masks (RoundContext, scheduler.cpp:36-72)
  {
    int k = (int)npair, qr = (int)nreq;
    for (int p = p0; p < p1; ++p) {
      const int s = A.order[p];
      const uint64_t r = A.ready[s];
      if (!r) continue;
      const int ci = A.cidx ? A.cidx[p] : qr++;
      A.qslot[ci] = s;
      for (int t = 0; t < A.N; ++t) {
        const int a = A.prio[t];
        if (!((r >> a) & 1ull)) continue;
        const uint32_t cm = A.cand[(size_t)s * A.N + a];
        uint32_t em = 0;
        for (uint32_t b = cm; b; b &= b - 1) {
          const int mdl = __ffs(b) - 1;
          const int e = A.eng.m2e[mdl];
          if (e < 0) s_status = AG_ERR_VALIDATION + 100;  // viable tier without a pool
          else em |= 1u << e;
        }
        A.pair_qi[k] = ci;
        A.pair_agent[k] = (uint8_t)a;
        A.pair_mask[k] = em;
        ++k;
      }
    }
  }
  __syncthreads();
  const int npairs = s_npairs;
  if (s_status) {
    if (tid == 0) A.status[0] = s_status;
    return;
  }
  uint32_t U0 = 0;
  for (int e = 0; e < A.eng.E; ++e)
    if (A.eng.slots[e] - A.eng.occ[e] > 0) U0 |= 1u << e;
  // ---- A3: candidate pairs (can be non-skip in this round) -> shared memory
  {
    const int pp = (npairs + T - 1) / T;
    const int q0 = min(npairs, tid * pp), q1 = min(npairs, q0 + pp);
    int c = 0;
    for (int i = q0; i < q1; ++i) c += (A.pair_mask[i] & U0) != 0;
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_scan[wid][0] = x;
    __syncthreads();
    if (wid == 0) {
      long long v = lane < T / 32 ? s_scan[lane][0] : 0, z = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += y;
      }
      if (lane < T / 32) s_scan[lane][0] = z - v;
      if (lane == 31) s_ncand = (int)z;
    }
    __syncthreads();
    int w = (int)s_scan[wid][0] + x - c;
    const bool in_smem = s_ncand <= A.cand_smem_cap;
    uint32_t* dp = in_smem ? c_pos : A.gcand_pos;
    uint32_t* dm = in_smem ? c_mask : A.gcand_mask;
    for (int i = q0; i < q1; ++i) {
      const uint32_t mk = A.pair_mask[i] & U0;
      if (mk) {
        dp[w] = (uint32_t)i;
        dm[w] = mk;
        ++w;
      }
    }
  }
  __syncthreads();
  if (wid != 0) return;

  // ---- B: the beam walk (warp 0)
  const int ncand = s_ncand;
  const uint32_t* cpos = ncand <= A.cand_smem_cap ? c_pos : A.gcand_pos;
  const uint32_t* cmsk = ncand <= A.cand_smem_cap ? c_mask : A.gcand_mask;
  const NodeView nv{s_nodes, A.gnodes};
  const int E = A.eng.E;
  const int N = A.N, M = A.M, B = A.B;
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
  }
  __syncwarp();
  if (s_status) {
    if (lane == 0) A.status[0] = s_status;
    return;
  }
  int cur = 0, nst = 1, nnodes = 0;
  unsigned long long explored = 1;
  int pi = 0, ci = 0;
  while (pi < npairs) {
    uint32_t U = lane < nst ? st[cur][lane].free_mask : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) U |= __shfl_xor_sync(0xffffffffu, U, o);
    if (!U) {  // all-full early exit (scheduler.cpp:303-315)
      const long long rem = npairs - pi;
      if (lane < nst) st[cur][lane].skips += rem;
      explored += (unsigned long long)nst * (unsigned long long)rem;
      break;
    }
    int qcur = A.pair_qi[pi];
    bool tch = lane < nst && st[cur][lane].node >= 0 && nv[st[cur][lane].node].qi == qcur;
    if (!__any_sync(0xffffffffu, tch)) {
      // fast-forward over whole-beam skips to the next pair whose mask meets U
      int found = ncand;
      for (int j0 = ci; j0 < ncand; j0 += 32) {
        const int j = j0 + lane;
        const bool ok = j < ncand && (int)cpos[j] >= pi && (cmsk[j] & U) != 0;
        const uint32_t b = __ballot_sync(0xffffffffu, ok);
        if (b) {
          found = j0 + __ffs(b) - 1;
          break;
        }
      }
      ci = found;
      const int target = found < ncand ? (int)cpos[found] : npairs;
      const long long k = target - pi;
      if (k > 0) {
        if (lane < nst) st[cur][lane].skips += k;
        explored += (unsigned long long)nst * (unsigned long long)k;
        pi = target;
      }
      if (pi >= npairs) break;
      qcur = A.pair_qi[pi];
      tch = false;
    }
    const int a = A.pair_agent[pi];
    const uint32_t base = A.pair_mask[pi];
    const int slot = A.qslot[qcur];
    const uint32_t nvia = A.nviable[slot];
    const double initial = (double)nvia;
    // allowed_engines (scheduler.cpp:140-156)
    uint32_t mk = 0;
    if (lane < nst) mk = tch ? 0u : (base & st[cur][lane].free_mask);
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
      for (uint32_t j = lane; j < nvia; j += 32) {
        const uint32_t c = vl[j];
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
    const bool has = lane < nst && mk != 0;
    if (!__any_sync(0xffffffffu, has)) {  // whole-beam skip (scheduler.cpp:317-329)
      if (lane < nst) st[cur][lane].skips += 1;
      explored += (unsigned long long)nst;
      ++pi;
      continue;
    }
    // children in (state, engine ascending) order; a state with no free
    // candidate contributes one skip child (scheduler.cpp:331-349)
    const int my_n = lane < nst ? (mk ? __popc(mk) : 1) : 0;
    int x = my_n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const int nchild = __shfl_sync(0xffffffffu, x, 31);
    if (lane < nst) {
      const BState& p = st[cur][lane];
      int c = x - my_n;
      if (!mk) {
        Child& ch = children[c];
        ch.parent = (int16_t)lane;
        ch.eng = -1;
        ch.util = p.util;
        ch.flex_sum = p.flex_sum;
        ch.flex_count = p.flex_count;
        ch.skips = p.skips + 1;
        ch.nsurv = p.nsurv;
        ch.flex = ch.flex_count > 0 ? ch.flex_sum / ch.flex_count : 1.0;
      } else {
        for (uint32_t b = mk; b; b &= b - 1, ++c) {  // extend_state (scheduler.cpp:158-206)
          const int e = __ffs(b) - 1;
          const int mdl = A.eng.model[e];
          Child& ch = children[c];
          ch.parent = (int16_t)lane;
          ch.eng = (int16_t)e;
          ch.util = p.util + A.eng.weight[e];
          ch.skips = p.skips;
          if (!tch) {
            const uint32_t surv = A.hist[((size_t)slot * N + a) * M + mdl];
            ch.flex_sum = p.flex_sum + (double)surv / initial;
            ch.flex_count = p.flex_count + 1;
            ch.nsurv = (int)surv;
          } else {
            const int surv = s_cnt[lane][mdl];
            const double before = (double)p.nsurv / initial;
            ch.flex_sum = p.flex_sum + ((double)surv / initial - before);
            ch.flex_count = p.flex_count;
            ch.nsurv = surv;
          }
          ch.flex = ch.flex_count > 0 ? ch.flex_sum / ch.flex_count : 1.0;
        }
      }
    }
    explored += (unsigned long long)nchild;
    __syncwarp();
    // nested retention (scheduler.cpp:351-370): level w adopts the best
    // unused child of parents < w; ties go to the lower child index
    uint32_t used[(kMaxBeam * (kMaxEng + 1) + 31) / 32];
    for (int i = 0; i < (nchild + 31) / 32; ++i) used[i] = 0;
    int npick = 0;
    for (int w = 1; w <= B; ++w) {
      int best = -1;
      for (int c = lane; c < nchild; c += 32) {
        if ((used[c >> 5] >> (c & 31)) & 1u) continue;
        const Child& cc = children[c];
        if (cc.parent >= w) continue;
        if (best < 0) {
          best = c;
        } else {
          const Child& cb = children[best];
          const int amc = (a << 8) | (cc.eng >= 0 ? A.eng.model[cc.eng] : 0);
          const int amb = (a << 8) | (cb.eng >= 0 ? A.eng.model[cb.eng] : 0);
          if (better(nv, cc.util, cc.flex, cc.skips, child_item(cc, st[cur], qcur, amc), cb.util,
                     cb.flex, cb.skips, child_item(cb, st[cur], qcur, amb)))
            best = c;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int other = __shfl_xor_sync(0xffffffffu, best, o);
        if (other < 0) continue;
        if (best < 0) {
          best = other;
          continue;
        }
        const Child& c1 = children[best];
        const Child& c2 = children[other];
        const int am1 = (a << 8) | (c1.eng >= 0 ? A.eng.model[c1.eng] : 0);
        const int am2 = (a << 8) | (c2.eng >= 0 ? A.eng.model[c2.eng] : 0);
        const Item i1 = child_item(c1, st[cur], qcur, am1), i2 = child_item(c2, st[cur], qcur, am2);
        if (better(nv, c2.util, c2.flex, c2.skips, i2, c1.util, c1.flex, c1.skips, i1)) best = other;
        else if (!better(nv, c1.util, c1.flex, c1.skips, i1, c2.util, c2.flex, c2.skips, i2) &&
                 other < best)
          best = other;
      }
      if (best < 0) continue;
      used[best >> 5] |= 1u << (best & 31);
      if (lane == 0) s_picked[npick] = best;
      ++npick;
    }
    __syncwarp();
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
      const Child& ch = children[pc];
      const BState& p = st[cur][ch.parent];
      BState& q = st[nxt][lane];
      for (int e = 0; e < E; ++e) q.occ[e] = p.occ[e];
      q.util = ch.util;
      q.flex_sum = ch.flex_sum;
      q.flex_count = ch.flex_count;
      q.skips = ch.skips;
      q.free_mask = p.free_mask;
      q.node = p.node;
      q.nsurv = ch.nsurv;
      if (mknode) {
        const int e = ch.eng;
        if (++q.occ[e] >= A.eng.slots[e]) q.free_mask &= ~(1u << e);
        const int id = nnodes + __popc(nb & ((1u << lane) - 1u));
        if (id < A.max_nodes) {
          Node nd;
          nd.qi = qcur;
          nd.am = (a << 8) | A.eng.model[e];
          nd.prev = p.node;
          nd.depth = depth_of(nv, p.node) + 1;
          nd.nsurv = ch.nsurv;
          if (id < kSmemNodes) s_nodes[id] = nd;
          else A.gnodes[id - kSmemNodes] = nd;
        } else {
          s_status = AG_ERR_INTERNAL + 300;  // history overflow
        }
        q.node = id;
      }
    }
    nnodes += __popc(nb);
    __syncwarp();
    if (s_status) {
      if (lane == 0) A.status[0] = s_status;
      return;
    }
    cur = nxt;
    nst = npick;
    ++pi;
  }

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
    const Item i1{s1.node, false, 0, 0}, i2{s2.node, false, 0, 0};
    if (better(nv, s2.util, f2, s2.skips, i2, s1.util, f1, s1.skips, i1)) best = other;
    else if (!better(nv, s1.util, f1, s1.skips, i1, s2.util, f2, s2.skips, i2) && other < best)
      best = other;
  }
  if (lane != 0) return;
  const BState& w = st[cur][best];
  const int D = depth_of(nv, w.node);
  if (D > A.triples_cap) {
    A.status[0] = AG_ERR_VALIDATION + 400;
    A.status[1] = D;
    return;
  }
  // triples in decision order; the distinct requests with their final
  // survivor counts (a request's triples are consecutive on the path, the
  // first one met walking back is its last) for score_assignment's fold
  double flex_sum = 0.0;
  int flex_count = 0;
  {
    uint32_t* lq = A.gcand_pos;  // scratch, >= npairs >= D entries
    uint32_t* ls = A.gcand_mask;
    int n = w.node, i = D, nd_req = 0;
    bool desc = true;
    while (n >= 0) {
      const Node nd = nv[n];
      --i;
      ag_triple t;
      t.request_index = nd.qi;
      t.agent = nd.am >> 8;
      t.model = nd.am & 0xFF;
      t.slot = A.qslot[nd.qi];
      t.request_id = A.ids[t.slot];
      A.triples[i] = t;
      if (nd_req == 0 || (int)lq[nd_req - 1] != nd.qi) {
        if (nd_req > 0 && (int)lq[nd_req - 1] < nd.qi) desc = false;
        lq[nd_req] = (uint32_t)nd.qi;
        ls[nd_req] = (uint32_t)nd.nsurv;
        ++nd_req;
      }
      n = nd.prev;
    }
    // score_assignment (scheduler.cpp:262-284) folds in queue (container)
    // order: session queues are FIFO = container order, so the list is
    // descending; an arbitrary container order is sorted first
    if (!desc) {
      for (int x = 1; x < nd_req; ++x) {
        const uint32_t kq = lq[x], ks = ls[x];
        int y = x - 1;
        while (y >= 0 && lq[y] < kq) {
          lq[y + 1] = lq[y];
          ls[y + 1] = ls[y];
          --y;
        }
        lq[y + 1] = kq;
        ls[y + 1] = ks;
      }
    }
    for (int x = nd_req - 1; x >= 0; --x) {
      flex_sum += (double)ls[x] / (double)A.nviable[A.qslot[lq[x]]];
      ++flex_count;
    }
  }
  double util = 0.0;
  for (int e = 0; e < E; ++e) {
    if (w.occ[e] < 0 || w.occ[e] > A.eng.slots[e]) {
      A.status[0] = AG_ERR_VALIDATION + 500;
      return;
    }
    util += w.occ[e] * A.eng.weight[e];
    A.occ_out[e] = w.occ[e];
  }
  ag_assignment res;
  res.n_triples = D;
  res.pad = 0;
  res.utilization = util;
  res.flexibility = flex_count > 0 ? flex_sum / flex_count : 1.0;
  res.skips = w.skips;
  res.states_explored = explored;
  *A.result = res;
  A.status[0] = 0;
  A.status[1] = s_nreq;
}

// ------------------------------------------------------------ prune kernel
struct PruneArgs {
  int N, M;
  const int32_t* g_slot;   // [G] slot per group
  const int32_t* g_begin;  // [G+1] ranges into g_am
  const int32_t* g_am;     // agent << 8 | model, in apply order
  uint32_t* pool;
  const uint64_t* voff;
  uint32_t* nviable;
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
__global__ void __launch_bounds__(256) k_sched_prune(PruneArgs A) {
  __shared__ uint32_t s_hist[kMaxAgents * 32];
  __shared__ int s_w[8], s_tot;
  const int g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int s = A.g_slot[g];
  uint32_t* vl = A.pool + A.voff[s];
  uint32_t len = A.nviable[s];
  for (int t = A.g_begin[g]; t < A.g_begin[g + 1]; ++t) {
    const int a = A.g_am[t] >> 8, mdl = A.g_am[t] & 0xFF;
    // count survivors first: an empty result leaves the list untouched
    int c = 0;
    for (uint32_t j = tid; j < len; j += blockDim.x) c += (int)digit_p(vl[j], a, A) == mdl;
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
      if (tid == 0) A.status[0] = AG_ERR_VALIDATION;  // model is not a viable candidate
      return;
    }
    // stable in-place compaction, one block-wide chunk at a time
    uint32_t wpos = 0;
    for (uint32_t b0 = 0; b0 < len; b0 += blockDim.x) {
      const uint32_t j = b0 + tid;
      const uint32_t v = j < len ? vl[j] : 0u;
      const bool keep = j < len && (int)digit_p(v, a, A) == mdl;
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
  for (uint32_t j = tid; j < len; j += blockDim.x) {
    const uint32_t v = vl[j];
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
  std::vector<uint64_t> voff;
  std::vector<uint32_t> nviable;
  std::vector<int32_t> free_slots;
  std::vector<int32_t> fifo;  // live slots by (arrival, id)
  bool fifo_dirty = true;
  bool attr_set = false;
  std::vector<int32_t> upd_slot;
  std::vector<uint64_t> upd_mask;
  int8_t prio[64];
  uint32_t place[agb::kMaxAgents];
  uint64_t place_magic[agb::kMaxAgents];
  // device
  agb::Scratch d_ready, d_cand, d_hist, d_nv, d_voff, d_pool, d_ids, d_order, d_cidx;
  agb::Scratch d_pair_qi, d_pair_agent, d_pair_mask, d_qslot, d_cpos, d_cmask, d_nodes;
  agb::Scratch d_triples, d_occ, d_result, d_status, d_upd_slot, d_upd_mask, d_gam;
  // pinned host staging for results
  void* h_res = nullptr;
  size_t h_res_bytes = 0;
  ~ag_sched() {
    if (h_res) cudaFreeHost(h_res);
  }
};

namespace agb {
namespace {

int ensure_host(ag_sched* s, size_t bytes) {
  if (bytes <= s->h_res_bytes) return AG_OK;
  if (s->h_res) cudaFreeHost(s->h_res);
  s->h_res = nullptr;
  s->h_res_bytes = 0;
  AG_CUDA(cudaMallocHost(&s->h_res, bytes));
  s->h_res_bytes = bytes;
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

// recompute hist/cand of the given slots with zero constraints
int prep_slots(ag_sched* s, const std::vector<int32_t>& slots);

int run_prune(ag_sched* s, const std::vector<int32_t>& g_slot, const std::vector<int32_t>& g_begin,
              const std::vector<int32_t>& g_am) {
  ag_ctx* ctx = s->ctx;
  const int G = (int)g_slot.size();
  if (G == 0) return AG_OK;
  int rc;
  const size_t bytes = (size_t)4 * (G + (G + 1) + g_am.size() + 1);
  if ((rc = s->d_gam.ensure(bytes))) return rc;
  std::vector<int32_t> buf;
  buf.reserve(bytes / 4);
  buf.insert(buf.end(), g_slot.begin(), g_slot.end());
  buf.insert(buf.end(), g_begin.begin(), g_begin.end());
  buf.insert(buf.end(), g_am.begin(), g_am.end());
  AG_CUDA(cudaMemcpyAsync(s->d_gam.p, buf.data(), buf.size() * 4, cudaMemcpyHostToDevice,
                          ctx->stream));
  if ((rc = s->d_status.ensure(64))) return rc;
  AG_CUDA(cudaMemsetAsync(s->d_status.p, 0, 8, ctx->stream));
  PruneArgs A;
  A.N = s->N;
  A.M = s->M;
  const int32_t* d = (const int32_t*)s->d_gam.p;
  A.g_slot = d;
  A.g_begin = d + G;
  A.g_am = d + G + G + 1;
  A.pool = (uint32_t*)s->d_pool.p;
  A.voff = (const uint64_t*)s->d_voff.p;
  A.nviable = (uint32_t*)s->d_nv.p;
  A.hist = (uint32_t*)s->d_hist.p;
  A.cand = (uint32_t*)s->d_cand.p;
  std::memcpy(A.place, s->place, sizeof A.place);
  std::memcpy(A.place_magic, s->place_magic, sizeof A.place_magic);
  A.div_m = ctx->space->dev().div_m;
  A.status = (int32_t*)s->d_status.p;
  {
    Launch L(ctx, g_am.empty() ? K_SCHED_PREP : K_SCHED_APPLY);
    k_sched_prune<<<G, 256, 0, ctx->stream>>>(A);
  }
  AG_CUDA(cudaGetLastError());
  int32_t st[2];
  AG_CUDA(cudaMemcpyAsync(st, s->d_status.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  AG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (st[0]) return fail(AG_ERR_VALIDATION, "dispatched model is not a viable candidate");
  return AG_OK;
}

int prep_slots(ag_sched* s, const std::vector<int32_t>& slots) {
  std::vector<int32_t> begin(slots.size() + 1, 0);
  return run_prune(s, slots, begin, {});
}

int upload_updates(ag_sched* s, int* n_upd) {
  ag_ctx* ctx = s->ctx;
  int rc;
  if (s->fifo_dirty) {
    if ((rc = s->d_order.ensure(s->fifo.size() * 4 + 4))) return rc;
    if (!s->fifo.empty())
      AG_CUDA(cudaMemcpyAsync(s->d_order.p, s->fifo.data(), s->fifo.size() * 4,
                              cudaMemcpyHostToDevice, ctx->stream));
    s->fifo_dirty = false;
  }
  // keep only the latest mask per slot: the kernel applies updates in
  // parallel, so one slot must appear once
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
  *n_upd = (int)nu;
  if (nu) {
    if ((rc = s->d_upd_slot.ensure(nu * 4)) || (rc = s->d_upd_mask.ensure(nu * 8))) return rc;
    AG_CUDA(cudaMemcpyAsync(s->d_upd_slot.p, s->upd_slot.data(), nu * 4, cudaMemcpyHostToDevice,
                            ctx->stream));
    AG_CUDA(cudaMemcpyAsync(s->d_upd_mask.p, s->upd_mask.data(), nu * 8, cudaMemcpyHostToDevice,
                            ctx->stream));
  }
  return AG_OK;
}

int engines_dev(const ag_sched* s, const ag_engines* e, EngDev* out) {
  // RoundContext validation (scheduler.cpp:39-52)
  if (!e) return fail(AG_ERR_VALIDATION, "engines is null");
  if (e->n_engines > kMaxEng) return fail(AG_ERR_VALIDATION, "more engine pools than the scheduler supports");
  EngDev d{};
  d.E = e->n_engines;
  for (int i = 0; i < 32; ++i) d.m2e[i] = -1;
  int max_model = -1;
  for (int i = 0; i < d.E; ++i) max_model = std::max(max_model, e->model[i]);
  for (int i = 0; i < d.E; ++i) {
    const int mdl = e->model[i];
    if (mdl < 0) return fail(AG_ERR_VALIDATION, "engine with negative model tier");
    if (mdl < 32) {
      if (d.m2e[mdl] != -1) return fail(AG_ERR_VALIDATION, "two engine pools serve the same model tier");
      d.m2e[mdl] = (int8_t)i;
    } else {
      for (int j = 0; j < i; ++j)
        if (e->model[j] == mdl) return fail(AG_ERR_VALIDATION, "two engine pools serve the same model tier");
    }
    d.model[i] = mdl;
    d.slots[i] = e->slots[i];
    d.occ[i] = e->occupancy[i];
    d.weight[i] = e->weight[i];
  }
  (void)s;
  *out = d;
  return AG_OK;
}

// One round over the session queue (or an explicit FIFO/container mapping).
int run_round(ag_sched* s, const ag_engines* engines, int B, const int32_t* cidx_host,
              ag_assignment* out, ag_triple* triples, int32_t triples_cap, int32_t* occupancy) {
  ag_ctx* ctx = s->ctx;
  if (B < 1) return fail(AG_ERR_VALIDATION, "beam width < 1");
  if (B > kMaxBeam) return fail(AG_ERR_VALIDATION, "GPU scheduler supports beam width <= 32");
  EngDev ed;
  int rc = engines_dev(s, engines, &ed);
  if (rc) return rc;
  int n_upd = 0;
  if ((rc = upload_updates(s, &n_upd))) return rc;
  const int Q = (int)s->fifo.size();
  size_t max_pairs = 1;
  for (int slot : s->fifo) max_pairs += (size_t)__builtin_popcountll(s->ready[slot]);
  int total_free = 0;
  for (int i = 0; i < ed.E; ++i) total_free += std::max(0, ed.slots[i] - ed.occ[i]);
  const int max_children = B * (ed.E + 1);
  const int cap_t = std::max(1, (int)std::min<size_t>(max_pairs, (size_t)total_free) + 1);
  const int max_nodes = (int)std::min<size_t>((size_t)B * max_pairs + 16, (size_t)1 << 30);
  if ((rc = s->d_pair_qi.ensure(max_pairs * 4)) || (rc = s->d_pair_agent.ensure(max_pairs)) ||
      (rc = s->d_pair_mask.ensure(max_pairs * 4)) || (rc = s->d_qslot.ensure((size_t)Q * 4 + 4)) ||
      (rc = s->d_cpos.ensure(max_pairs * 4)) || (rc = s->d_cmask.ensure(max_pairs * 4)) ||
      (rc = s->d_nodes.ensure(
           (size_t)std::max(1, max_nodes - kSmemNodes) * sizeof(Node))) ||
      (rc = s->d_triples.ensure((size_t)cap_t * sizeof(ag_triple))) ||
      (rc = s->d_result.ensure(sizeof(ag_assignment) + 4 * kMaxEng + 16)) ||
      (rc = s->d_status.ensure(64)))
    return rc;
  if (cidx_host) {
    if ((rc = s->d_cidx.ensure((size_t)Q * 4 + 4))) return rc;
    AG_CUDA(cudaMemcpyAsync(s->d_cidx.p, cidx_host, (size_t)Q * 4, cudaMemcpyHostToDevice,
                            ctx->stream));
  }
  RoundArgs A;
  std::memset(&A, 0, sizeof A);
  A.N = s->N;
  A.M = s->M;
  A.B = B;
  A.order = (const int32_t*)s->d_order.p;
  A.cidx = cidx_host ? (const int32_t*)s->d_cidx.p : nullptr;
  A.Q = Q;
  A.ready = (uint64_t*)s->d_ready.p;
  A.n_upd = n_upd;
  A.upd_slot = (const int32_t*)s->d_upd_slot.p;
  A.upd_mask = (const uint64_t*)s->d_upd_mask.p;
  A.cand = (const uint32_t*)s->d_cand.p;
  A.hist = (const uint32_t*)s->d_hist.p;
  A.nviable = (const uint32_t*)s->d_nv.p;
  A.voff = (const uint64_t*)s->d_voff.p;
  A.pool = (const uint32_t*)s->d_pool.p;
  A.ids = (const uint64_t*)s->d_ids.p;
  std::memcpy(A.prio, s->prio, sizeof A.prio);
  std::memcpy(A.place, s->place, sizeof A.place);
  std::memcpy(A.place_magic, s->place_magic, sizeof A.place_magic);
  A.div_m = ctx->space->dev().div_m;
  A.eng = ed;
  A.pair_qi = (int32_t*)s->d_pair_qi.p;
  A.pair_agent = (uint8_t*)s->d_pair_agent.p;
  A.pair_mask = (uint32_t*)s->d_pair_mask.p;
  A.qslot = (int32_t*)s->d_qslot.p;
  A.gcand_pos = (uint32_t*)s->d_cpos.p;
  A.gcand_mask = (uint32_t*)s->d_cmask.p;
  A.gnodes = (Node*)s->d_nodes.p;
  A.max_nodes = max_nodes;
  A.max_children = max_children;
  A.triples = (ag_triple*)s->d_triples.p;
  A.triples_cap = cap_t;
  char* rp = (char*)s->d_result.p;
  A.result = (ag_assignment*)rp;
  A.occ_out = (int32_t*)(rp + sizeof(ag_assignment));
  A.status = (int32_t*)s->d_status.p;
  // dynamic shared memory: children, then the candidate list
  const size_t static_bytes = 2 * kMaxBeam * sizeof(BState) + 8192;  // + scans, counters
  const size_t max_dyn = 227 * 1024 - static_bytes;
  const size_t fixed = sizeof(Node) * kSmemNodes + ((sizeof(Child) * (size_t)max_children + 15) & ~(size_t)15);
  if (fixed > max_dyn) return fail(AG_ERR_VALIDATION, "beam too wide for one CTA");
  const int cand_cap = (int)std::min<size_t>(max_pairs, (max_dyn - fixed) / 8);
  A.cand_smem_cap = cand_cap;
  const size_t dyn = fixed + (size_t)cand_cap * 8;
  if (!s->attr_set) {
    AG_CUDA(cudaFuncSetAttribute(k_sched_round, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)max_dyn));
    s->attr_set = true;
  }
  {
    Launch L(ctx, K_SCHED_ROUND);
    k_sched_round<<<1, kRoundThreads, dyn, ctx->stream>>>(A);
  }
  AG_CUDA(cudaGetLastError());
  // results: status | assignment | occupancy | triples in one pinned buffer
  const size_t res_bytes = 16 + sizeof(ag_assignment) + 4 * kMaxEng + (size_t)cap_t * sizeof(ag_triple);
  if ((rc = ensure_host(s, res_bytes))) return rc;
  char* h = (char*)s->h_res;
  AG_CUDA(cudaMemcpyAsync(h, s->d_status.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  AG_CUDA(cudaMemcpyAsync(h + 16, rp, sizeof(ag_assignment) + 4 * kMaxEng, cudaMemcpyDeviceToHost,
                          ctx->stream));
  AG_CUDA(cudaStreamSynchronize(ctx->stream));
  s->upd_slot.clear();
  s->upd_mask.clear();
  const int32_t status = ((int32_t*)h)[0];
  if (status) {
    if (status == AG_ERR_VALIDATION + 100)
      return fail(AG_ERR_VALIDATION, "viable model tier without an engine pool");
    if (status == AG_ERR_VALIDATION + 200) return fail(AG_ERR_VALIDATION, "engine over capacity");
    if (status == AG_ERR_VALIDATION + 500)
      return fail(AG_ERR_VALIDATION, "occupancy outside engine capacity");
    return fail(AG_ERR_INTERNAL, "scheduler round failed (status " + std::to_string(status) + ")");
  }
  const ag_assignment res = *(const ag_assignment*)(h + 16);
  if (res.n_triples > triples_cap) {
    if (out) *out = res;
    return fail(AG_ERR_VALIDATION, "triples_cap too small");
  }
  if (res.n_triples) {
    AG_CUDA(cudaMemcpyAsync(triples, s->d_triples.p, sizeof(ag_triple) * res.n_triples,
                            cudaMemcpyDeviceToHost, ctx->stream));
    AG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  if (occupancy) std::memcpy(occupancy, h + 16 + sizeof(ag_assignment), 4 * (size_t)engines->n_engines);
  if (out) *out = res;
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
  s->voff.assign(max_requests, 0);
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
      (rc = s->d_pool.ensure(s->pool_cap * 4))) {
    delete s;
    return rc;
  }
  cudaMemsetAsync(s->d_ready.p, 0, R * 8, ctx->stream);
  *out = s;
  return AG_OK;
}

void ag_sched_destroy(ag_sched* s) { delete s; }

int ag_sched_add(ag_sched* s, const ag_queue* q, int32_t* slots_out) {
  if (!s || !q) return fail(AG_ERR_VALIDATION, "null argument");
  ag_ctx* ctx = s->ctx;
  const int R = q->n_requests;
  if (R <= 0) return R == 0 ? AG_OK : fail(AG_ERR_VALIDATION, "negative request count");
  if ((int)s->free_slots.size() < R) return fail(AG_ERR_VALIDATION, "session is full");
  const uint64_t total = (uint64_t)(q->viable_ptr[R] - q->viable_ptr[0]);
  if (s->pool_top + total > s->pool_cap) return fail(AG_ERR_VALIDATION, "session viable pool is full");
  const int N = s->N;
  // Request::make (request.cpp:24-50)
  for (int i = 0; i < R; ++i) {
    const int64_t len = q->viable_ptr[i + 1] - q->viable_ptr[i];
    if (len <= 0) return fail(AG_ERR_VALIDATION, "request needs a nonempty viable set");
    for (int64_t j = q->viable_ptr[i]; j < q->viable_ptr[i + 1]; ++j)
      if ((uint64_t)q->viable[j] >= s->ctx->space->size)
        return fail(AG_ERR_VALIDATION, "viable configuration length mismatch");
  }
  std::vector<int32_t> slots(R);
  std::vector<uint64_t> offs(R);
  std::vector<uint32_t> nv(R);
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
    s->voff[slot] = s->pool_top + (uint64_t)(q->viable_ptr[i] - q->viable_ptr[0]);
    s->nviable[slot] = (uint32_t)(q->viable_ptr[i + 1] - q->viable_ptr[i]);
    offs[i] = s->voff[slot];
    nv[i] = s->nviable[slot];
    s->upd_slot.push_back(slot);
    s->upd_mask.push_back(s->ready[slot]);
    if (slots_out) slots_out[i] = slot;
  }
  cudaStream_t st = ctx->stream;
  AG_CUDA(cudaMemcpyAsync((uint32_t*)s->d_pool.p + s->pool_top, q->viable + q->viable_ptr[0],
                          total * 4, cudaMemcpyHostToDevice, st));
  s->pool_top += total;
  // scatter per-slot metadata (slots are arbitrary): stage through a small
  // host-built copy of the whole arrays when the batch is large, else per
  // slot copies
  for (int i = 0; i < R; ++i) {
    const int slot = slots[i];
    AG_CUDA(cudaMemcpyAsync((uint64_t*)s->d_voff.p + slot, &s->voff[slot], 8, cudaMemcpyHostToDevice, st));
    AG_CUDA(cudaMemcpyAsync((uint32_t*)s->d_nv.p + slot, &s->nviable[slot], 4, cudaMemcpyHostToDevice, st));
    AG_CUDA(cudaMemcpyAsync((uint64_t*)s->d_ids.p + slot, &s->ids[slot], 8, cudaMemcpyHostToDevice, st));
  }
  // FIFO insertion (Sim::insert_schedulable, simulation.cpp:182-192)
  for (int i = 0; i < R; ++i) {
    const int slot = slots[i];
    if (s->fifo.empty() || !agb::fifo_less(s, slot, s->fifo.back())) {
      s->fifo.push_back(slot);
    } else {
      auto pos = std::lower_bound(s->fifo.begin(), s->fifo.end(), slot,
                                  [&](int x, int y) { return agb::fifo_less(s, x, y); });
      s->fifo.insert(pos, slot);
    }
  }
  s->fifo_dirty = true;
  return agb::prep_slots(s, slots);
}

int ag_sched_remove(ag_sched* s, int32_t n, const int32_t* slots) {
  if (!s) return fail(AG_ERR_VALIDATION, "null argument");
  std::vector<char> gone(s->cap, 0);
  for (int i = 0; i < n; ++i) {
    const int slot = slots[i];
    if (slot < 0 || slot >= s->cap || !s->live[slot]) return fail(AG_ERR_VALIDATION, "bad slot");
    s->live[slot] = 0;
    s->ready[slot] = 0;
    s->upd_slot.push_back(slot);
    s->upd_mask.push_back(0);
    s->free_slots.push_back(slot);
    gone[slot] = 1;
  }
  s->fifo.erase(std::remove_if(s->fifo.begin(), s->fifo.end(), [&](int x) { return gone[x] != 0; }),
                s->fifo.end());
  s->fifo_dirty = true;
  if (s->fifo.empty()) s->pool_top = 0;  // everything left: reuse the pool
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
  // group by slot, apply order kept inside a group (triples of one request
  // are consecutive in decision order)
  std::vector<int32_t> g_slot, g_begin{0}, g_am;
  for (int i = 0; i < n; ++i) {
    const ag_triple& t = applied[i];
    const int slot = t.slot;
    if (slot < 0 || slot >= s->cap || !s->live[slot]) return fail(AG_ERR_VALIDATION, "bad slot");
    uint8_t& stg = s->stages[(size_t)slot * N + t.agent];
    if (t.agent < 0 || t.agent >= N || stg != AG_STAGE_READY)
      return fail(AG_ERR_VALIDATION, "dispatch of a stage that is not ready");
    if (t.model < 0 || t.model >= s->M)
      return fail(AG_ERR_VALIDATION, "dispatched model is not a viable candidate");
    stg = AG_STAGE_INFLIGHT;
    if (g_slot.empty() || g_slot.back() != slot) {
      if (!g_slot.empty()) g_begin.push_back((int32_t)g_am.size());
      g_slot.push_back(slot);
    }
    g_am.push_back((t.agent << 8) | t.model);
  }
  g_begin.push_back((int32_t)g_am.size());
  for (int slot : g_slot) {
    const uint64_t r = agb::ready_of(s, slot);
    s->ready[slot] = r;
    s->upd_slot.push_back(slot);
    s->upd_mask.push_back(r);
  }
  // g_slot may repeat a slot if its triples were not consecutive; the
  // kernel handles each group independently, which is only correct for
  // distinct slots -- merge repeats
  std::vector<int32_t> order(g_slot.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return g_slot[x] < g_slot[y]; });
  std::vector<int32_t> ms, mb{0}, ma;
  for (size_t k = 0; k < order.size(); ++k) {
    const int gi = order[k];
    if (ms.empty() || ms.back() != g_slot[gi]) {
      if (!ms.empty()) mb.push_back((int32_t)ma.size());
      ms.push_back(g_slot[gi]);
    }
    ma.insert(ma.end(), g_am.begin() + g_begin[gi], g_am.begin() + g_begin[gi + 1]);
  }
  mb.push_back((int32_t)ma.size());
  return agb::run_prune(s, ms, mb, ma);
}

int ag_sched_viable(ag_sched* s, int32_t slot, uint32_t* out, int64_t cap, int64_t* n) {
  if (!s || slot < 0 || slot >= s->cap || !s->live[slot]) return fail(AG_ERR_VALIDATION, "bad slot");
  uint32_t len = 0;
  AG_CUDA(cudaMemcpyAsync(&len, (uint32_t*)s->d_nv.p + slot, 4, cudaMemcpyDeviceToHost, s->ctx->stream));
  AG_CUDA(cudaStreamSynchronize(s->ctx->stream));
  if (n) *n = len;
  if (out && (int64_t)len <= cap && len) {
    AG_CUDA(cudaMemcpyAsync(out, (uint32_t*)s->d_pool.p + s->voff[slot], (size_t)len * 4,
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
  std::vector<int32_t> cidx(s->fifo.size());
  for (size_t p = 0; p < s->fifo.size(); ++p) cidx[p] = slot_to_ci[s->fifo[p]];
  rc = agb::run_round(s, engines, beam_width, cidx.data(), out, triples, triples_cap, occupancy);
  if (rc == AG_OK && out)
    for (int i = 0; i < out->n_triples; ++i) triples[i].slot = -1;
  delete s;
  return rc;
}

}  // extern "C"
