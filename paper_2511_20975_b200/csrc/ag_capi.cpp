// C ABI entry points: spaces, contexts, memory helpers, routing wrappers and
// the host-side input generator.  Host C++ only; kernels live in *.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "ag_internal.h"

namespace agb {

static thread_local std::string g_error;

void set_error(const std::string& msg) { g_error = msg; }

int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

int Scratch::ensure(size_t want) {
  if (want <= bytes) return AG_OK;
  if (p) cudaFree(p);
  p = nullptr;
  // geometric growth: per-round buffers must not reallocate round after round
  // (cudaFree synchronises the device)
  size_t b = std::max<size_t>(std::max<size_t>(want, 256), bytes + bytes / 2);
  bytes = 0;
  cudaError_t e = cudaMalloc(&p, b);
  if (e != cudaSuccess) {
    p = nullptr;
    return fail(AG_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  bytes = b;
  return AG_OK;
}

Scratch::~Scratch() {
  if (p) cudaFree(p);
}

const char* const kKernelNames[K_NUM_KERNELS] = {
    "k_route_score", "k_chunk_scan", "k_request_scan", "k_route_compact", "k_predict",
    "k_sched_round", "k_sched_apply", "k_sched_prep", "k_cost_argmin", "k_linear_score",
    "k_route_noise"};

static_assert(K_NUM_KERNELS == AG_NUM_KERNELS, "kernel id table out of sync with the header");

static cudaEvent_t take_event(ag_ctx* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

Launch::Launch(ag_ctx* ctx, int kernel) : c(ctx), k(kernel) {
  c->launches++;
  if (c->profiling) {
    e0 = take_event(c);
    cudaEventRecord(e0, c->stream);
  }
}

Launch::~Launch() {
  if (c->profiling && e0) {
    cudaEvent_t e1 = take_event(c);
    cudaEventRecord(e1, c->stream);
    c->prof.push_back({k, e0, e1});
  }
}

}  // namespace agb

using agb::fail;

namespace agb {
// Errors latched on the device by asynchronous entry points (bit 0: a member
// uses a tier the estimator context lacks, workload.cpp:140-142; bit 1: an
// empty accurate set, workload.cpp:151-156); the stream is synchronised.
int take_async_status(ag_ctx* c) {
  if (!c->async_status.p) return AG_OK;
  int32_t st = 0;
  AG_CUDA(cudaMemcpy(&st, c->async_status.p, 4, cudaMemcpyDeviceToHost));
  if (!st) return AG_OK;
  AG_CUDA(cudaMemset(c->async_status.p, 0, 4));
  if (st & 2) return fail(AG_ERR_VALIDATION, "accurate set is empty");
  return fail(AG_ERR_VALIDATION, "estimator context missing a model tier");
}
}  // namespace agb

extern "C" {

const char* ag_last_error(void) { return agb::g_error.c_str(); }
int ag_abi_version(void) { return 1; }

// WorkflowGraph::build (workflow.cpp:69-173), ModelCatalog (workflow.cpp:38-60),
// ConfigSpace (workflow.cpp:209-224).
int ag_space_create(int n, int n_edges, const int32_t* edges, int m, const double* cost,
                    const double* weight, ag_space** out) {
  if (!out) return fail(AG_ERR_VALIDATION, "out is null");
  *out = nullptr;
  if (n < 1) return fail(AG_ERR_VALIDATION, "workflow needs at least 1 agent");
  if (n > 64) return fail(AG_ERR_VALIDATION, "at most 64 agents supported");
  if (m < 2) return fail(AG_ERR_VALIDATION, "model catalog needs at least 2 tiers");
  if (m > agb::kMaxModels) return fail(AG_ERR_VALIDATION, "at most 255 model tiers supported");
  for (int i = 0; i < m; ++i) {
    if (!(cost[i] > 0.0) || !(weight[i] > 0.0))
      return fail(AG_ERR_VALIDATION, "model needs positive cost and slot_throughput");
    if (i > 0) {
      if (cost[i] <= cost[i - 1])
        return fail(AG_ERR_VALIDATION, "model costs must strictly increase with tier");
      if (weight[i] >= weight[i - 1])
        return fail(AG_ERR_VALIDATION, "model slot_throughput must strictly decrease with tier");
    }
  }
  std::vector<uint64_t> outm(n, 0), inm(n, 0);
  for (int e = 0; e < n_edges; ++e) {
    int f = edges[2 * e], t = edges[2 * e + 1];
    if (f < 0 || f >= n) return fail(AG_ERR_VALIDATION, "edge from unknown agent");
    if (t < 0 || t >= n) return fail(AG_ERR_VALIDATION, "edge to unknown agent");
    if (f == t) return fail(AG_ERR_VALIDATION, "self loop on agent");
    outm[f] |= 1ULL << t;
    inm[t] |= 1ULL << f;
  }
  // Kahn releasing the smallest declaration index first (min-heap semantics)
  std::vector<int> indeg(n), order;
  uint64_t ready = 0;
  for (int i = 0; i < n; ++i) {
    indeg[i] = __builtin_popcountll(inm[i]);
    if (!indeg[i]) ready |= 1ULL << i;
  }
  while (ready) {
    int u = __builtin_ctzll(ready);
    ready &= ready - 1;
    order.push_back(u);
    for (uint64_t o = outm[u]; o; o &= o - 1) {
      int v = __builtin_ctzll(o);
      if (--indeg[v] == 0) ready |= 1ULL << v;
    }
  }
  if ((int)order.size() != n) return fail(AG_ERR_VALIDATION, "workflow has a cycle");
  ag_space* s = new ag_space();
  s->n = n;
  s->m = m;
  s->decl.assign(order.begin(), order.end());
  std::vector<int> pos_of(n);
  for (int p = 0; p < n; ++p) pos_of[order[p]] = p;
  s->pred.assign(n, 0);
  s->succ.assign(n, 0);
  for (int p = 0; p < n; ++p) {
    int d = order[p];
    for (uint64_t o = outm[d]; o; o &= o - 1) s->succ[p] |= 1ULL << pos_of[__builtin_ctzll(o)];
    for (uint64_t o = inm[d]; o; o &= o - 1) s->pred[p] |= 1ULL << pos_of[__builtin_ctzll(o)];
  }
  s->depth.assign(n, 0);
  for (int p = n - 1; p >= 0; --p)
    for (uint64_t o = s->succ[p]; o; o &= o - 1)
      s->depth[p] = std::max(s->depth[p], s->depth[__builtin_ctzll(o)] + 1);
  s->cost.assign(cost, cost + m);
  s->weight.assign(weight, weight + m);
  // size = M^N when it fits u64 (ConfigSpace::indexable, workflow.cpp:209-224)
  uint64_t size = 1;
  bool fits = true;
  for (int i = 0; i < n; ++i) {
    if (size > UINT64_MAX / (uint64_t)m) {
      fits = false;
      break;
    }
    size *= (uint64_t)m;
  }
  s->size = fits ? size : 0;
  s->gpu_ok = fits && size <= (1ULL << 32) && n <= agb::kMaxAgents;
  *out = s;
  return AG_OK;
}

void ag_space_destroy(ag_space* s) { delete s; }

int ag_space_info(const ag_space* s, int32_t* n, int32_t* m, int32_t* decl, int32_t* depth,
                  uint64_t* size) {
  if (!s) return fail(AG_ERR_VALIDATION, "space is null");
  if (n) *n = s->n;
  if (m) *m = s->m;
  if (decl) std::memcpy(decl, s->decl.data(), sizeof(int32_t) * s->n);
  if (depth) std::memcpy(depth, s->depth.data(), sizeof(int32_t) * s->n);
  if (size) *size = s->size;
  return AG_OK;
}

int ag_ctx_create(const ag_space* space, int device, ag_ctx** out) {
  if (!space || !out) return fail(AG_ERR_VALIDATION, "null argument");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(AG_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0 || device >= count) return fail(AG_ERR_VALIDATION, "device out of range");
  agb::DeviceGuard device_guard(device);
  ag_ctx* c = new ag_ctx();
  c->space = space;
  c->device = device;
  *out = c;
  return AG_OK;
}

void ag_ctx_destroy(ag_ctx* c) {
  agb::DeviceGuard device_guard(c ? c->device : -1);
  if (!c) return;
  for (auto& r : c->prof) {
    cudaEventDestroy(r.start);
    cudaEventDestroy(r.stop);
  }
  for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  ag_sched_destroy(c->beam_cache);
  delete c;
}

int ag_ctx_set_stream(ag_ctx* c, void* stream) {
  if (!c) return fail(AG_ERR_VALIDATION, "ctx is null");
  c->stream = (cudaStream_t)stream;
  return AG_OK;
}

int ag_ctx_synchronize(ag_ctx* c) {
  agb::DeviceGuard device_guard(c ? c->device : -1);
  if (!c) return fail(AG_ERR_VALIDATION, "ctx is null");
  AG_CUDA(cudaStreamSynchronize(c->stream));
  return agb::take_async_status(c);
}

uint64_t ag_ctx_launch_count(const ag_ctx* c) { return c ? c->launches : 0; }

int ag_ctx_profile_begin(ag_ctx* c) {
  agb::DeviceGuard device_guard(c ? c->device : -1);
  if (!c) return fail(AG_ERR_VALIDATION, "ctx is null");
  for (auto& r : c->prof) {
    c->event_pool.push_back(r.start);
    c->event_pool.push_back(r.stop);
  }
  c->prof.clear();
  c->profiling = true;
  return AG_OK;
}

int ag_ctx_profile_end(ag_ctx* c, double* ms, uint64_t* launches) {
  agb::DeviceGuard device_guard(c ? c->device : -1);
  if (!c) return fail(AG_ERR_VALIDATION, "ctx is null");
  c->profiling = false;
  AG_CUDA(cudaStreamSynchronize(c->stream));
  for (int k = 0; k < agb::K_NUM_KERNELS; ++k) {
    if (ms) ms[k] = 0.0;
    if (launches) launches[k] = 0;
  }
  for (auto& r : c->prof) {
    float t = 0.f;
    AG_CUDA(cudaEventElapsedTime(&t, r.start, r.stop));
    if (ms) ms[r.kernel] += t;
    if (launches) launches[r.kernel] += 1;
    c->event_pool.push_back(r.start);
    c->event_pool.push_back(r.stop);
  }
  c->prof.clear();
  return AG_OK;
}

const char* ag_kernel_name(int k) {
  return (k >= 0 && k < agb::K_NUM_KERNELS) ? agb::kKernelNames[k] : "";
}

int ag_host_alloc(size_t bytes, void** out) {
  AG_CUDA(cudaMallocHost(out, bytes ? bytes : 1));
  return AG_OK;
}
int ag_host_free(void* p) {
  AG_CUDA(cudaFreeHost(p));
  return AG_OK;
}
int ag_device_alloc(size_t bytes, void** out) {
  AG_CUDA(cudaMalloc(out, bytes ? bytes : 1));
  return AG_OK;
}
int ag_device_free(void* p) {
  AG_CUDA(cudaFree(p));
  return AG_OK;
}

int ag_route_enumerate(ag_ctx* ctx, const ag_truth* truth, const ag_router* router,
                       uint64_t begin, uint64_t end, uint32_t flags, const ag_route_out* out) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  if (!ctx) return fail(AG_ERR_VALIDATION, "ctx is null");
  return agb::route_enumerate(ctx, truth, router, begin, end, flags, out);
}

}  // extern "C"

namespace agb {
// pinned staging for small host-path uploads (synchronised before reuse)
int ensure_host_stage(ag_ctx* ctx, size_t bytes) {
  AG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->h_stage && ctx->h_stage_bytes >= bytes) return AG_OK;
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  ctx->h_stage = nullptr;
  ctx->h_stage_bytes = 0;
  const size_t b = std::max<size_t>(bytes, (size_t)1 << 16);
  AG_CUDA(cudaMallocHost(&ctx->h_stage, b));
  ctx->h_stage_bytes = b;
  return AG_OK;
}

// Copies a host ag_truth batch into the context's device staging buffer in
// one transfer (ids | seed_ptr | removed_ptr | removed | seeds) and returns
// its device view.
int upload_truth(ag_ctx* ctx, const ag_truth* th, ag_truth* td) {
  const int R = th->n_requests;
  const int n = ctx->space->n;
  const size_t rows = (size_t)th->seed_ptr[R];
  const size_t nrem = (size_t)th->removed_ptr[R];
  const size_t o_ids = 0, o_sp = o_ids + 8 * (size_t)R, o_rp = o_sp + 4 * ((size_t)R + 1);
  const size_t o_rem = (o_rp + 4 * ((size_t)R + 1) + 7) & ~(size_t)7;
  const size_t o_seeds = o_rem + 8 * nrem;
  const size_t bytes = o_seeds + rows * (size_t)n;
  int rc;
  if ((rc = ctx->h_truth.ensure(bytes))) return rc;
  if ((rc = ensure_host_stage(ctx, bytes))) return rc;
  char* h = (char*)ctx->h_stage;
  std::memcpy(h + o_ids, th->request_ids, 8 * (size_t)R);
  std::memcpy(h + o_sp, th->seed_ptr, 4 * ((size_t)R + 1));
  std::memcpy(h + o_rp, th->removed_ptr, 4 * ((size_t)R + 1));
  if (nrem) std::memcpy(h + o_rem, th->removed, 8 * nrem);
  if (rows) std::memcpy(h + o_seeds, th->seeds, rows * (size_t)n);
  char* d = (char*)ctx->h_truth.p;
  AG_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
  *td = ag_truth{R, (const uint64_t*)(d + o_ids), (const int32_t*)(d + o_sp),
                 (const uint8_t*)(d + o_seeds), (const int32_t*)(d + o_rp),
                 (const uint64_t*)(d + o_rem)};
  return AG_OK;
}
}  // namespace agb

extern "C" {

// select_per_input_config for a batch of host AccurateSets: each set's
// verdict bitmap over the whole space (oracle verdicts, canonical order) is
// built on the device and the re-cost + arg-min runs straight from it
// (accuracy.cpp:227-238 + workload.cpp:149-176; ag_select_bitmap: no member
// list, no host round trip in between); only the choice comes back.
int ag_select_per_input_host(ag_ctx* ctx, const ag_truth* th, int32_t kind, const ag_load* load,
                             uint32_t* chosen, double* est) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  if (!ctx || !th || !chosen) return fail(AG_ERR_VALIDATION, "null argument");
  const int R = th->n_requests;
  if (R < 0) return fail(AG_ERR_VALIDATION, "negative request count");
  if (R == 0) return AG_OK;
  const ag_space* sp = ctx->space;
  if (!sp->gpu_ok) return fail(AG_ERR_VALIDATION, "GPU path needs M^N <= 2^32 and N <= 32");
  ag_truth td;
  int rc = agb::upload_truth(ctx, th, &td);
  if (rc) return rc;
  const uint64_t S = sp->size;
  const size_t W = (size_t)((S + 31) / 32);
  if ((rc = ctx->counts.ensure(8 * (size_t)R)) || (rc = ctx->offsets.ensure(8 * ((size_t)R + 1))) ||
      (rc = ctx->bitmap.ensure((size_t)R * W * 4 + 4)) || (rc = ctx->d_sel.ensure(16 * (size_t)R + 16)))
    return rc;
  const ag_router oracle{AG_ROUTER_ORACLE, 0.0, 0.0, 0, 0.0};
  ag_route_out o1{(uint32_t*)ctx->bitmap.p, (uint64_t*)ctx->counts.p, (uint64_t*)ctx->offsets.p,
                  nullptr, 0, nullptr};
  if ((rc = agb::route_enumerate(ctx, &td, &oracle, 0, S, 0, &o1))) return rc;
  uint32_t* d_chosen = (uint32_t*)ctx->d_sel.p;
  double* d_est = (double*)((char*)ctx->d_sel.p + ((4 * (size_t)R + 15) & ~(size_t)15));
  if ((rc = ag_select_bitmap(ctx, (const uint32_t*)ctx->bitmap.p, (const uint64_t*)ctx->counts.p, 0, S, R, kind,
                             load, d_chosen, d_est, nullptr)))
    return rc;
  AG_CUDA(cudaMemcpyAsync(chosen, d_chosen, 4 * (size_t)R, cudaMemcpyDeviceToHost, ctx->stream));
  if (est) AG_CUDA(cudaMemcpyAsync(est, d_est, 8 * (size_t)R, cudaMemcpyDeviceToHost, ctx->stream));
  AG_CUDA(cudaStreamSynchronize(ctx->stream));
  return agb::take_async_status(ctx);
}

int ag_route_enumerate_host(ag_ctx* ctx, const ag_truth* th, const ag_router* router,
                            uint64_t begin, uint64_t end, uint32_t flags, uint64_t* counts,
                            uint64_t* offsets, uint32_t* indices, uint64_t capacity,
                            uint64_t* total) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  if (!ctx || !th || !offsets || (th->n_requests > 0 && !counts))
    return fail(AG_ERR_VALIDATION, "null argument");
  const int R = th->n_requests;
  if (R < 0) return fail(AG_ERR_VALIDATION, "negative request count");
  if (R == 0) {
    offsets[0] = 0;
    if (total) *total = 0;
    return AG_OK;
  }
  ag_truth td;
  int rc = agb::upload_truth(ctx, th, &td);
  if (rc) return rc;
  cudaStream_t s = ctx->stream;
  if ((rc = ctx->counts.ensure(8 * (size_t)R))) return rc;
  if ((rc = ctx->offsets.ensure(8 * ((size_t)R + 1)))) return rc;
  const uint64_t range = end > begin ? end - begin : 0;
  const size_t W = (size_t)((range + 31) / 32);
  if ((rc = ctx->bitmap.ensure((size_t)R * W * 4 + 4))) return rc;
  // phase 1: score + scan (bitmap kept for the compaction pass)
  ag_route_out o1{(uint32_t*)ctx->bitmap.p, (uint64_t*)ctx->counts.p, (uint64_t*)ctx->offsets.p,
                  nullptr, 0, nullptr};
  if ((rc = agb::route_enumerate(ctx, &td, router, begin, end, flags, &o1))) return rc;
  AG_CUDA(cudaMemcpyAsync(offsets, ctx->offsets.p, 8 * ((size_t)R + 1), cudaMemcpyDeviceToHost, s));
  AG_CUDA(cudaMemcpyAsync(counts, ctx->counts.p, 8 * (size_t)R, cudaMemcpyDeviceToHost, s));
  AG_CUDA(cudaStreamSynchronize(s));
  const uint64_t tot = offsets[R];
  if (total) *total = tot;
  if (!indices) return AG_OK;
  if (tot > capacity) return fail(AG_ERR_VALIDATION, "indices capacity too small");
  if ((rc = ctx->d_out_idx.ensure(4 * (size_t)tot + 4))) return rc;
  // phase 2: compaction from the resident bitmap, then copy out
  if ((rc = agb::route_compact(ctx, R, begin, end, (const uint32_t*)ctx->bitmap.p,
                               (const uint64_t*)ctx->offsets.p, (uint32_t*)ctx->d_out_idx.p,
                               tot)))
    return rc;
  if (tot)
    AG_CUDA(cudaMemcpyAsync(indices, ctx->d_out_idx.p, 4 * (size_t)tot, cudaMemcpyDeviceToHost, s));
  AG_CUDA(cudaStreamSynchronize(s));
  return AG_OK;
}

}  // extern "C"
