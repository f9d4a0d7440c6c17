// Routing hot path, chain mode: ConfigPredictor::predict replayed on the GPU,
// one warp per request (reference src/predictor.cpp:107-262).
//
// Host side (once per space, like the reference ctor predictor.cpp:158-163):
// build_chains' DFS (predictor.cpp:80-131) produces the chain plan; every
// distinct configuration on a chain gets a uid, and the plan is uploaded as
//   chain_uid[n_chains][len]  uid of each rung
//   uniq_index[U]             canonical index of each uid
//   uid_by_cost[U]            uids sorted by (static_cost, canonical index),
//                             the verification order (predictor.cpp:240-245)
//   uid_by_index[U]           uids sorted by canonical index, the output order
//
// Device side, per request (one warp): the verdict cache of predict() is a
// pair of U-bit sets (known, value) in shared memory -- every evaluated
// configuration lies on a chain, so uids cover it.  Phase 1 narrows each
// chain's bounds with cached verdicts (a warp ballot over the rungs) and
// binary-searches the rest (warp-uniform sequential probes).  Phase 2 walks
// the candidates in cost order 32 at a time: lane 0 replays the budget
// arithmetic (router_time += latency, allowed iff router_time + latency <=
// budget) in order, then the charged lanes evaluate in parallel.  Output is
// the kept set plus top in canonical order, with search/verify counts,
// router_time and truncated exactly as the reference reports them.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "ag_internal.h"

namespace agb {

namespace {

// ------------------------------------------------------------ host: plan
struct ChainBuilder {  // predictor.cpp:28-99
  int n, m;
  uint64_t size;
  bool track;
  size_t cap;
  std::vector<std::vector<uint64_t>> chains;
  std::vector<uint64_t> uncovered;
  std::vector<char> covered;

  void decode(uint64_t idx, uint8_t* d) const {
    for (int i = n - 1; i >= 0; --i) {
      d[i] = (uint8_t)(idx % (uint64_t)m);
      idx /= (uint64_t)m;
    }
  }
  uint64_t encode(const uint8_t* d) const {
    uint64_t idx = 0;
    for (int i = 0; i < n; ++i) idx = idx * (uint64_t)m + d[i];
    return idx;
  }
  bool done() const {
    if (cap != 0 && chains.size() >= cap) return true;
    return track && uncovered.empty();
  }
  bool has_uncovered_above(const uint8_t* c) const {
    uint8_t d[64];
    for (size_t k = uncovered.size(); k-- > 0;) {
      decode(uncovered[k], d);
      bool le = true;
      for (int i = 0; i < n && le; ++i) le = c[i] <= d[i];
      if (le) return true;
    }
    return false;
  }
  bool path_has_fresh(const std::vector<uint64_t>& path) const {
    for (uint64_t c : path)
      if (!covered[c]) return true;
    return false;
  }
  bool cover(const std::vector<uint64_t>& path) {
    bool fresh = false;
    for (uint64_t c : path)
      if (!covered[c]) covered[c] = 1, fresh = true;
    if (fresh)
      uncovered.erase(std::remove_if(uncovered.begin(), uncovered.end(),
                                     [&](uint64_t i) { return covered[i] != 0; }),
                      uncovered.end());
    return fresh;
  }
  void dfs(std::vector<uint64_t>& path) {
    if (done()) return;
    const uint64_t tail = path.back();
    if (tail == size - 1) {  // is_top
      if (!track || cover(path)) chains.push_back(path);
      return;
    }
    uint8_t t[64];
    decode(tail, t);
    for (int i = 0; i < n && !done(); ++i) {
      if (t[i] + 1 >= m) continue;
      uint8_t nx[64];
      std::memcpy(nx, t, (size_t)n);
      ++nx[i];
      if (track && !path_has_fresh(path) && !has_uncovered_above(nx)) continue;
      path.push_back(encode(nx));
      dfs(path);
      path.pop_back();
    }
  }
};

__device__ __forceinline__ bool bit_get(const uint32_t* b, uint32_t i) {
  return (b[i >> 5] >> (i & 31)) & 1u;
}
// the known / value bitsets interleaved word by word: one 8-byte load gives
// both bits of a rung
__device__ __forceinline__ uint2 kv_word(const uint32_t* kv, uint32_t u) {
  return reinterpret_cast<const uint2*>(kv)[u >> 5];
}

struct PredictArgs {
  SpaceDev sp;
  TruthDev t;
  RouterDev rt;
  double latency;
  const uint32_t* chain_uid;
  int n_chains, len;
  const uint32_t* uniq_index;
  int U;
  uint32_t uid_top;
  const uint32_t* uid_by_cost;
  const uint32_t* uid_by_index;
  const double* budgets;  // [R] device, or nullptr with budget_all
  double budget_all;
  int R;
  ag_predict_out out;
  uint32_t* gscratch;  // per-warp bitsets when they do not fit shared memory
  int words;           // 32-bit words per bitset
  int smem_bits;       // bitsets live in shared memory
};

// RouterBackend::evaluate for one configuration (router.cpp:37-57)
__device__ bool verdict(const PredictArgs& a, int r, uint32_t idx, uint64_t P) {
  const int n = a.sp.n;
  const uint32_t m = (uint32_t)a.sp.m;
  uint32_t d[kMaxAgents];
  {
    uint32_t x = idx;
    for (int i = n - 1; i >= 0; --i) {
      const uint32_t q = divm(x, a.sp.div_m);
      d[i] = x - q * m;
      x = q;
    }
  }
  bool truth = false;
  const int r0 = __ldg(a.t.removed_ptr + r), r1 = __ldg(a.t.removed_ptr + r + 1);
  bool removed = false;
  for (int i = r0; i < r1; ++i) removed |= __ldg(a.t.removed + i) == (uint64_t)idx;
  if (!removed) {
    const int s0 = __ldg(a.t.seed_ptr + r), s1 = __ldg(a.t.seed_ptr + r + 1);
    for (int s = s0; s < s1 && !truth; ++s) {
      const uint8_t* sd = a.t.seeds + (size_t)s * n;
      bool le = true;
      for (int i = 0; i < n && le; ++i) le = __ldg(sd + i) <= d[i];
      truth = le;
    }
  }
  if (a.rt.kind != AG_ROUTER_NOISY) return truth;
  uint64_t h = kHashIV;  // hash_config (router.cpp:22-28)
  for (int i = 0; i < n; ++i) h = absorb(absorb(kMixIV, h), d[i]);
  const uint64_t key = absorb(P, h) >> 11;
  return truth ? key >= a.rt.t_fn : key < a.rt.t_fp;
}

constexpr int kPredWarps = 4;

__global__ void __launch_bounds__(kPredWarps * 32) k_predict(PredictArgs a) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int r = blockIdx.x * kPredWarps + wid;
  if (r >= a.R) return;
  uint32_t* base = a.smem_bits ? smem + (size_t)wid * 4 * a.words
                               : a.gscratch + (size_t)r * 4 * a.words;
  uint32_t* kv = base;  // known / value interleaved, 2 * words
  uint32_t* cand = base + 2 * a.words;
  uint32_t* kept = base + 3 * a.words;
  for (int i = lane; i < 4 * a.words; i += 32) base[i] = 0;
  __syncwarp();

  const double budget = a.budgets ? a.budgets[r] : a.budget_all;
  const double lat = a.latency;
  uint64_t P = 0;
  if (a.rt.kind == AG_ROUTER_NOISY)
    P = absorb(absorb(absorb(kMixIV, a.rt.noise_seed), kRouterSalt), __ldg(a.t.request_ids + r));
  double router_time = 0.0;
  int search_evals = 0, verify_evals = 0;
  bool truncated = false;
  const int len = a.len;

  // ---- phase 1: per-chain boundary search (predictor.cpp:198-227)
  for (int ci = 0; ci < a.n_chains; ++ci) {
    if (truncated) break;
    const uint32_t* ch = a.chain_uid + (size_t)ci * len;
    // bounds from cached verdicts: hi = first cached-true rung, lo = last
    // cached-false rung + 1 (top counts as cached true)
    int lo = 0, hi = len;
    for (int b = 0; b < len; b += 32) {
      const int i = b + lane;
      bool ct = false, cf = false;
      if (i < len) {
        const uint32_t u = __ldg(ch + i);
        const uint2 w = kv_word(kv, u);
        const bool k = u == a.uid_top || ((w.x >> (u & 31)) & 1u);
        const bool v = u == a.uid_top || ((w.y >> (u & 31)) & 1u);
        ct = k && v;
        cf = k && !v;
      }
      const uint32_t mt = __ballot_sync(0xffffffffu, ct), mf = __ballot_sync(0xffffffffu, cf);
      if (mt && hi == len) hi = b + __ffs(mt) - 1;
      if (mf) lo = b + 32 - __clz(mf);
    }
    int bound;
    if (lo > hi) {
      bound = hi;  // non-monotone cached verdicts (predictor.cpp:216-222)
    } else {
      // find_chain_boundary (predictor.cpp:133-148): warp-uniform probes
      bool aborted = false;
      while (lo < hi) {
        const int mid = lo + (hi - lo) / 2;
        const uint32_t u = __ldg(ch + mid);
        const uint2 w = kv_word(kv, u);
        bool v;
        if (u == a.uid_top) {
          v = true;
        } else if ((w.x >> (u & 31)) & 1u) {
          v = (w.y >> (u & 31)) & 1u;
        } else if (router_time + lat > budget) {
          truncated = true;
          aborted = true;
          break;
        } else {
          v = verdict(a, r, __ldg(a.uniq_index + u), P);
          router_time += lat;
          ++search_evals;
          if (lane == 0) {
            kv[2 * (u >> 5)] |= 1u << (u & 31);
            if (v) kv[2 * (u >> 5) + 1] |= 1u << (u & 31);
          }
          __syncwarp();
        }
        if (v) hi = mid;
        else lo = mid + 1;
      }
      if (aborted) break;
      bound = lo;
    }
    // candidates: rungs bound.. of a searched chain, top excluded
    for (int i = bound + lane; i < len; i += 32) {
      const uint32_t u = __ldg(ch + i);
      if (u != a.uid_top) atomicOr(cand + (u >> 5), 1u << (u & 31));
    }
    __syncwarp();
  }

  // ---- phase 2: verify candidates cheapest first (predictor.cpp:229-254)
  for (int b = 0; b < a.U; b += 32) {
    const int j = b + lane;
    uint32_t u = 0;
    bool is_cand = false, is_known = false, val = false;
    if (j < a.U) {
      u = __ldg(a.uid_by_cost + j);
      is_cand = bit_get(cand, u);
      const uint2 w = kv_word(kv, u);
      is_known = (w.x >> (u & 31)) & 1u;
      val = (w.y >> (u & 31)) & 1u;
    }
    const uint32_t need = __ballot_sync(0xffffffffu, is_cand && !is_known);
    uint32_t charged = 0;
    if (need) {
      // budget replay in cost order, repeated addition as the reference does
      if (lane == 0) {
        for (uint32_t mk = need; mk; mk &= mk - 1) {
          if (router_time + lat > budget) {
            truncated = true;
            break;
          }
          router_time += lat;
          charged |= mk & (~mk + 1);
        }
      }
      charged = __shfl_sync(0xffffffffu, charged, 0);
      router_time = __shfl_sync(0xffffffffu, router_time, 0);
      truncated = __shfl_sync(0xffffffffu, (int)truncated, 0) != 0;
      verify_evals += __popc(charged);
    }
    bool keep = false;
    if (is_cand) {
      if (is_known) {
        keep = val;
      } else if ((charged >> lane) & 1u) {
        keep = verdict(a, r, __ldg(a.uniq_index + u), P);
        atomicOr(kv + 2 * (u >> 5), 1u << (u & 31));
        if (keep) atomicOr(kv + 2 * (u >> 5) + 1, 1u << (u & 31));
      }
    }
    if (keep) atomicOr(kept + (u >> 5), 1u << (u & 31));
    __syncwarp();
  }

  // ---- output: kept + top in canonical order (predictor.cpp:255-260)
  uint32_t* out = a.out.viable + (size_t)r * a.out.viable_stride;
  int count = 0;
  for (int b = 0; b < a.U; b += 32) {
    const int j = b + lane;
    bool emit = false;
    uint32_t u = 0;
    if (j < a.U) {
      u = __ldg(a.uid_by_index + j);
      emit = u == a.uid_top || bit_get(kept, u);
    }
    const uint32_t mk = __ballot_sync(0xffffffffu, emit);
    if (emit) {
      const int pos = count + __popc(mk & ((1u << lane) - 1u));
      if (pos < a.out.viable_stride) out[pos] = __ldg(a.uniq_index + u);
    }
    count += __popc(mk);
  }
  if (lane == 0) {
    a.out.n_viable[r] = count;
    if (a.out.search_evals) a.out.search_evals[r] = search_evals;
    if (a.out.verify_evals) a.out.verify_evals[r] = verify_evals;
    if (a.out.router_time) a.out.router_time[r] = router_time;
    if (a.out.truncated) a.out.truncated[r] = truncated ? 1 : 0;
  }
}

}  // namespace

}  // namespace agb

struct ag_predictor {
  ag_ctx* ctx = nullptr;
  int n_chains = 0, len = 0, U = 0;
  bool exhaustive = false;
  uint32_t uid_top = 0;
  std::vector<uint64_t> chains_host;  // canonical indices [n_chains * len]
  agb::Scratch d_chain_uid, d_uniq_index, d_by_cost, d_by_index, d_scratch;
  void* h_out = nullptr;  // ag_predict_host outputs, mapped pinned memory
  size_t h_out_bytes = 0;
  char* h_out_dev = nullptr;
  ~ag_predictor() {
    if (h_out) cudaFreeHost(h_out);
  }
};

using agb::fail;

extern "C" {

// ConfigPredictor ctor (predictor.cpp:158-163) -> build_chains (:107-131)
int ag_predictor_create(ag_ctx* ctx, int chain_cap, uint64_t exhaustive_limit,
                        ag_predictor** out) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  if (!ctx || !out) return fail(AG_ERR_VALIDATION, "null argument");
  *out = nullptr;
  const ag_space* sp = ctx->space;
  if (!sp->gpu_ok) return fail(AG_ERR_VALIDATION, "GPU path needs M^N <= 2^32 and N <= 32");
  agb::ChainBuilder b{sp->n, sp->m, sp->size, sp->size <= exhaustive_limit, 0, {}, {}, {}};
  if (b.track) {
    b.covered.assign(b.size, 0);
    b.uncovered.resize(b.size);
    std::iota(b.uncovered.begin(), b.uncovered.end(), 0ULL);
  } else {
    b.cap = (size_t)(chain_cap > 0 ? chain_cap : 64);
  }
  std::vector<uint64_t> path{0};
  b.dfs(path);
  ag_predictor* p = new ag_predictor();
  p->ctx = ctx;
  p->n_chains = (int)b.chains.size();
  p->len = sp->n * (sp->m - 1) + 1;
  p->exhaustive = b.track && b.uncovered.empty();
  // uids over the distinct rungs
  std::vector<uint64_t> uniq;
  for (auto& ch : b.chains) {
    if ((int)ch.size() != p->len) {
      delete p;
      return fail(AG_ERR_INTERNAL, "chain length mismatch");
    }
    uniq.insert(uniq.end(), ch.begin(), ch.end());
    p->chains_host.insert(p->chains_host.end(), ch.begin(), ch.end());
  }
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  p->U = (int)uniq.size();
  std::vector<uint32_t> uniq_index(uniq.begin(), uniq.end());  // sorted: uid == index rank
  std::vector<uint32_t> chain_uid(p->chains_host.size());
  for (size_t i = 0; i < chain_uid.size(); ++i)
    chain_uid[i] = (uint32_t)(std::lower_bound(uniq.begin(), uniq.end(), p->chains_host[i]) -
                              uniq.begin());
  p->uid_top = p->U ? (uint32_t)(p->U - 1) : 0;  // top has the largest index
  std::vector<uint32_t> by_index(p->U), by_cost(p->U);
  std::iota(by_index.begin(), by_index.end(), 0u);
  std::vector<double> cost(p->U);
  for (int u = 0; u < p->U; ++u) {  // static_cost: left fold (workflow.cpp:291-296)
    uint64_t idx = uniq[u];
    uint8_t d[64];
    for (int i = sp->n - 1; i >= 0; --i) {
      d[i] = (uint8_t)(idx % (uint64_t)sp->m);
      idx /= (uint64_t)sp->m;
    }
    double c = 0.0;
    for (int i = 0; i < sp->n; ++i) c += sp->cost[d[i]];
    cost[u] = c;
  }
  std::iota(by_cost.begin(), by_cost.end(), 0u);
  std::stable_sort(by_cost.begin(), by_cost.end(), [&](uint32_t x, uint32_t y) {
    if (cost[x] != cost[y]) return cost[x] < cost[y];
    return uniq[x] < uniq[y];
  });
  int rc;
  auto up = [&](agb::Scratch& s, const std::vector<uint32_t>& v) -> int {
    int e = s.ensure(v.size() * 4 + 4);
    if (e) return e;
    if (!v.empty()) AG_CUDA(cudaMemcpy(s.p, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
    return AG_OK;
  };
  if ((rc = up(p->d_chain_uid, chain_uid)) || (rc = up(p->d_uniq_index, uniq_index)) ||
      (rc = up(p->d_by_cost, by_cost)) || (rc = up(p->d_by_index, by_index))) {
    delete p;
    return rc;
  }
  *out = p;
  return AG_OK;
}

void ag_predictor_destroy(ag_predictor* p) {
  agb::DeviceGuard device_guard(p ? p->ctx->device : -1);
  delete p;
}

int ag_predictor_info(const ag_predictor* p, int32_t* n_chains, int32_t* chain_len,
                      int32_t* exhaustive, int32_t* n_unique, uint64_t* chains) {
  if (!p) return fail(AG_ERR_VALIDATION, "predictor is null");
  if (n_chains) *n_chains = p->n_chains;
  if (chain_len) *chain_len = p->len;
  if (exhaustive) *exhaustive = p->exhaustive ? 1 : 0;
  if (n_unique) *n_unique = p->U;
  if (chains) std::memcpy(chains, p->chains_host.data(), p->chains_host.size() * 8);
  return AG_OK;
}

// ConfigPredictor::predict (predictor.cpp:165-262) for a batch of requests
int ag_predict(ag_predictor* p, const ag_truth* t, const ag_router* router,
               const double* budgets, double budget_all, const ag_predict_out* out) {
  agb::DeviceGuard device_guard(p ? p->ctx->device : -1);
  if (!p || !t || !out || !out->viable || !out->n_viable)
    return fail(AG_ERR_VALIDATION, "null argument");
  ag_ctx* ctx = p->ctx;
  agb::RouterDev rt;
  int rc = agb::make_router(router, &rt);
  if (rc) return rc;
  const int R = t->n_requests;
  if (R <= 0) return R == 0 ? AG_OK : fail(AG_ERR_VALIDATION, "negative request count");
  if (out->viable_stride < 1) return fail(AG_ERR_VALIDATION, "viable_stride < 1");
  agb::PredictArgs a{};
  a.sp = ctx->space->dev();
  a.t = agb::TruthDev{R, t->request_ids, t->seed_ptr, t->seeds, t->removed_ptr, t->removed};
  a.rt = rt;
  a.latency = router->eval_latency;
  a.chain_uid = (const uint32_t*)p->d_chain_uid.p;
  a.n_chains = p->n_chains;
  a.len = p->len;
  a.uniq_index = (const uint32_t*)p->d_uniq_index.p;
  a.U = p->U;
  a.uid_top = p->uid_top;
  a.uid_by_cost = (const uint32_t*)p->d_by_cost.p;
  a.uid_by_index = (const uint32_t*)p->d_by_index.p;
  a.budgets = budgets;
  a.budget_all = budget_all;
  a.R = R;
  a.out = *out;
  a.words = (p->U + 31) / 32;
  const size_t per_warp = (size_t)4 * a.words * 4;
  size_t smem = per_warp * agb::kPredWarps;
  a.smem_bits = smem <= 48 * 1024 ? 1 : 0;
  if (!a.smem_bits) {
    if ((rc = p->d_scratch.ensure(per_warp * (size_t)R))) return rc;
    a.gscratch = (uint32_t*)p->d_scratch.p;
    smem = 0;
  }
  const int blocks = (R + agb::kPredWarps - 1) / agb::kPredWarps;
  {
    agb::Launch L(ctx, agb::K_PREDICT);
    agb::k_predict<<<blocks, agb::kPredWarps * 32, smem, ctx->stream>>>(a);
  }
  AG_CUDA(cudaGetLastError());
  return AG_OK;
}

// The same with host buffers, copies included (the simulator drop-in path):
// viable [R * viable_stride]; the other outputs optional.
int ag_predict_host(ag_predictor* p, const ag_truth* th, const ag_router* router,
                    const double* budgets, double budget_all, uint32_t* viable,
                    int32_t viable_stride, int32_t* n_viable, int32_t* search_evals,
                    int32_t* verify_evals, double* router_time, uint8_t* truncated) {
  agb::DeviceGuard device_guard(p ? p->ctx->device : -1);
  if (!p || !th || !viable || !n_viable || !router) return fail(AG_ERR_VALIDATION, "null argument");
  ag_ctx* ctx = p->ctx;
  const int R = th->n_requests;
  if (R <= 0) return R == 0 ? AG_OK : fail(AG_ERR_VALIDATION, "negative request count");
  if (viable_stride < 1) return fail(AG_ERR_VALIDATION, "viable_stride < 1");
  ag_truth td;
  int rc = agb::upload_truth(ctx, th, &td);
  if (rc) return rc;
  // device outputs: viable | n_viable | search | verify | router_time | budgets | truncated
  const size_t o_v = 0;
  const size_t o_n = o_v + 4 * (size_t)R * viable_stride;
  const size_t o_s = o_n + 4 * (size_t)R, o_f = o_s + 4 * (size_t)R;
  const size_t o_t = (o_f + 4 * (size_t)R + 7) & ~(size_t)7;
  const size_t o_b = o_t + 8 * (size_t)R, o_u = o_b + 8 * (size_t)R;
  const size_t bytes = o_u + (size_t)R;
  // outputs (and budgets) in mapped pinned memory: the kernel writes the
  // host's copy directly, one launch + one synchronisation per call
  if (bytes > p->h_out_bytes) {
    if (p->h_out) cudaFreeHost(p->h_out);
    p->h_out = nullptr;
    p->h_out_bytes = 0;
    AG_CUDA(cudaHostAlloc(&p->h_out, std::max<size_t>(bytes, 4096), cudaHostAllocMapped));
    p->h_out_bytes = std::max<size_t>(bytes, 4096);
    void* dv = nullptr;
    AG_CUDA(cudaHostGetDevicePointer(&dv, p->h_out, 0));
    p->h_out_dev = (char*)dv;
  }
  char* hbuf = (char*)p->h_out;
  char* d = p->h_out_dev;
  cudaStream_t s = ctx->stream;
  if (budgets) std::memcpy(hbuf + o_b, budgets, 8 * (size_t)R);
  ag_predict_out o{(uint32_t*)(d + o_v), viable_stride, (int32_t*)(d + o_n), (int32_t*)(d + o_s),
                   (int32_t*)(d + o_f), (double*)(d + o_t), (uint8_t*)(d + o_u)};
  if ((rc = ag_predict(p, &td, router, budgets ? (const double*)(d + o_b) : nullptr, budget_all, &o)))
    return rc;
  AG_CUDA(cudaStreamSynchronize(s));
  std::memcpy(n_viable, hbuf + o_n, 4 * (size_t)R);
  for (int r = 0; r < R; ++r) {  // only each request's viable prefix is meaningful
    const int32_t nv = ((const int32_t*)(hbuf + o_n))[r];
    std::memcpy(viable + (size_t)r * viable_stride, hbuf + o_v + 4 * (size_t)r * viable_stride,
                4 * (size_t)std::max(0, std::min(nv, viable_stride)));
  }
  if (search_evals) std::memcpy(search_evals, hbuf + o_s, 4 * (size_t)R);
  if (verify_evals) std::memcpy(verify_evals, hbuf + o_f, 4 * (size_t)R);
  if (router_time) std::memcpy(router_time, hbuf + o_t, 8 * (size_t)R);
  if (truncated) std::memcpy(truncated, hbuf + o_u, (size_t)R);
  return AG_OK;
}

}  // extern "C"
