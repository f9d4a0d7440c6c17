// Internal (C++) definitions behind the opaque C handles.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "ag_common.cuh"

struct ag_space {
  int n = 0, m = 0;
  std::vector<int32_t> decl;     // canonical pos -> declaration index
  std::vector<int32_t> depth;    // by canonical pos
  std::vector<uint64_t> pred;    // predecessor bitmask by canonical pos
  std::vector<uint64_t> succ;    // successor bitmask by canonical pos
  std::vector<double> cost;      // ModelSpec::cost by tier
  std::vector<double> weight;    // ModelSpec::slot_throughput by tier
  uint64_t size = 0;             // M^N (0 when > 2^64)
  bool gpu_ok = false;           // M^N <= 2^32 and N <= 32

  agb::SpaceDev dev() const {
    agb::SpaceDev s;
    s.n = n;
    s.m = m;
    s.size = size;
    // ceil(2^64 / m) for m >= 2
    s.div_m = (~0ULL) / (uint64_t)m + 1;
    return s;
  }
};

namespace agb {

// grow-only device scratch buffer
struct Scratch {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t want);
  ~Scratch();
};

}  // namespace agb

namespace agb {

// kernel ids for the live per-kernel CUDA-event profile (bench.py roofline)
enum KernelId {
  K_ROUTE_SCORE = 0,
  K_CHUNK_SCAN,
  K_REQUEST_SCAN,
  K_ROUTE_COMPACT,
  K_PREDICT,
  K_SCHED_ROUND,
  K_SCHED_APPLY,
  K_SCHED_PREP,
  K_COST_ARGMIN,
  K_LINEAR_SCORE,
  K_ROUTE_NOISE,
  K_NUM_KERNELS
};
extern const char* const kKernelNames[K_NUM_KERNELS];

struct ProfRecord {
  int kernel;
  cudaEvent_t start, stop;
};

}  // namespace agb

struct ag_ctx {
  const ag_space* space = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t launches = 0;
  // live profile: CUDA events around every launch while enabled
  bool profiling = false;
  std::vector<agb::ProfRecord> prof;
  std::vector<cudaEvent_t> event_pool;
  // routing scratch
  agb::Scratch chunk_counts, chunk_off, chunk_part, bitmap, counts, offsets, overflow;
  agb::Scratch colmask;  // per-space last-digit masks (route 2-D path)
  agb::Scratch hc;       // hash_config(c) per canonical index (noisy router)
  bool hc_ready = false;
  agb::Scratch cost_status, cost_tasks, cost_prefix;  // runtime-cost argmin: plan, task bests, prefix folds
  agb::Scratch cost_bm;                                // bitmap argmin: prefix lower bounds + thresholds
  agb::Scratch bm_stats;                               // bitmap argmin diagnostics: words evaluated
  bool bm_stats_on = false;
  int cost_grid[5] = {0, 0, 0, 0, 0};                 // k_cost_tasks<sfx> blocks resident on the device
  bool cost_plan_attr = false;                        // k_cost_plan's dynamic shared memory raised
  int colmask_m = 0;
  // host-path staging
  agb::Scratch h_truth;
  agb::Scratch d_out_idx;
  agb::Scratch d_sel;        // select_per_input host path: chosen / estimate
  agb::Scratch wf_hits, wf_best;  // select_per_workflow: hit counts, block minima
  ag_sched* beam_cache = nullptr;  // session reused by stateless beam_schedule
  // per-device launch configuration (cudaFuncSetAttribute and occupancy are
  // per device, so they are cached per context, never per process)
  bool scan_attr = false;    // k_request_scan<12>/<24> dynamic shared memory
  int compact_resident = 0;  // k_route_compact blocks resident on the device
  int linear_sms = 0;        // SM count; k_linear_score attributes set
  // errors latched by asynchronous kernels (ag_select_per_input), reported
  // by the next synchronising call on the context
  agb::Scratch async_status;
  void* h_stage = nullptr;   // pinned staging for host-path uploads
  size_t h_stage_bytes = 0;
};

namespace agb {

// Every entry point runs on its context's device and leaves the caller's
// current device as it found it.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int cur = 0;
    if (dev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Brackets one kernel launch with CUDA events on the context stream when the
// live profile is enabled, and counts the launch.
struct Launch {
  ag_ctx* c;
  int k;
  cudaEvent_t e0 = nullptr;
  Launch(ag_ctx* ctx, int kernel);
  ~Launch();
};

int route_enumerate(ag_ctx* ctx, const ag_truth* t, const ag_router* r,
                    uint64_t begin, uint64_t end, uint32_t flags,
                    const ag_route_out* out);
int finish_enumerate(ag_ctx* ctx, int R, uint32_t W, uint32_t C, uint64_t begin, uint32_t* bitmap,
                     uint64_t* offsets, const ag_route_out* out, bool scanned = false);
int route_compact(ag_ctx* ctx, int R, uint64_t begin, uint64_t end, const uint32_t* bitmap,
                  const uint64_t* offsets, uint32_t* indices, uint64_t capacity);
int make_router(const ag_router* r, RouterDev* out);
// host ag_truth -> device view in the context's staging buffer
int upload_truth(ag_ctx* ctx, const ag_truth* host, ag_truth* dev);
int ensure_host_stage(ag_ctx* ctx, size_t bytes);
int take_async_status(ag_ctx* ctx);

}  // namespace agb
