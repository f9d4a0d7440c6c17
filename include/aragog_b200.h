/*
 * aragog_b200.h -- C ABI of the B200-native (sm_100a) implementation of
 * Aragog's two data-parallel hot paths (arXiv 2511.20975):
 *
 *   1. one-time routing: enumerate the mixed-radix configuration space of a
 *      batch of requests, score every configuration with the binary accuracy
 *      router, stream-compact the accuracy-preserving set (enumerate mode),
 *      or replay the chain/binary-search predictor (chain mode);
 *   2. per-stage just-in-time scheduling: beam-search round decisions,
 *      prefix pruning, and the runtime-cost re-cost + argmin.
 *
 * Plain C types only (no torch, no C++).  Device-pointer entry points are
 * asynchronous on the context's stream; *_host entry points take host buffers
 * and include the host<->device copies.
 *
 * Every entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj).  Status codes mirror the
 * reference's exception taxonomy (include/aragog/errors.h:22-34,
 * tools/main.cpp:290-303): ValidationError -> AG_ERR_VALIDATION,
 * IoError -> AG_ERR_IO, std::logic_error -> AG_ERR_INTERNAL.
 */
#ifndef ARAGOG_B200_H
#define ARAGOG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AG_OK 0
#define AG_ERR_INTERNAL 1
#define AG_ERR_VALIDATION 2
#define AG_ERR_IO 3
#define AG_ERR_CUDA 4

#define AG_ROUTER_ORACLE 0 /* OracleRouter, include/aragog/router.h:43-53 */
#define AG_ROUTER_NOISY 1  /* NoisyRouter over an oracle, router.h:57-70 */

#define AG_FORCE_TOP 1u /* top is always a member (predictor.cpp:177,255) */

/* Message of the last failing call on this thread. */
const char* ag_last_error(void);
int ag_abi_version(void);

/* ======================================================================== *
 * Configuration space                                                       *
 * ======================================================================== */
typedef struct ag_space ag_space;

/* WorkflowGraph::build + ModelCatalog + ConfigSpace
 * (include/aragog/workflow.h:34-152; src/workflow.cpp:38-173,209-224).
 * edges: n_edges (from, to) pairs of declaration indices.  cost strictly
 * increasing, slot_throughput strictly decreasing (workflow.cpp:38-60).
 * The GPU path additionally requires M^N <= 2^32 and N <= 32. */
int ag_space_create(int n_agents, int n_edges, const int32_t* edges,
                    int n_models, const double* cost,
                    const double* slot_throughput, ag_space** out);
void ag_space_destroy(ag_space* space);
/* decl[pos] = declaration index at canonical position, depth[pos]
 * (WorkflowGraph::declaration_index/depth, workflow.h:68-77); size = M^N. */
int ag_space_info(const ag_space* space, int32_t* n_agents, int32_t* n_models,
                  int32_t* decl, int32_t* depth, uint64_t* size);

/* ======================================================================== *
 * Device context                                                            *
 * ======================================================================== */
typedef struct ag_ctx ag_ctx;

int ag_ctx_create(const ag_space* space, int device, ag_ctx** out);
void ag_ctx_destroy(ag_ctx* ctx);
/* cudaStream_t as void*; NULL = the legacy default stream */
int ag_ctx_set_stream(ag_ctx* ctx, void* stream);
int ag_ctx_synchronize(ag_ctx* ctx);
/* number of kernels this context launched since creation */
uint64_t ag_ctx_launch_count(const ag_ctx* ctx);

/* Live per-kernel profile: while enabled every launch is bracketed by CUDA
 * events on the context stream.  ag_ctx_profile_end synchronises the stream
 * and returns, per kernel id (0 .. AG_NUM_KERNELS-1), the summed device
 * milliseconds and launch counts since ag_ctx_profile_begin. */
#define AG_NUM_KERNELS 11
int ag_ctx_profile_begin(ag_ctx* ctx);
int ag_ctx_profile_end(ag_ctx* ctx, double* ms, uint64_t* launches);
const char* ag_kernel_name(int kernel_id);

/* pinned host / device memory helpers */
int ag_host_alloc(size_t bytes, void** out);
int ag_host_free(void* p);
int ag_device_alloc(size_t bytes, void** out);
int ag_device_free(void* p);

/* ======================================================================== *
 * Routing (hot path 1)                                                      *
 * ======================================================================== */

/* RouterBackend (router.h:33-41) as data.  kind ORACLE: verdict =
 * AccurateSet::contains (accuracy.cpp:116-124).  kind NOISY: NoisyRouter over
 * the oracle (router.cpp:50-57) with fp, fn in [0,1] and noise_seed. */
typedef struct {
  int32_t kind;
  double fp, fn;
  uint64_t noise_seed;
  double eval_latency; /* seconds charged per evaluation (predict only) */
} ag_router;

/* A batch of AccurateSets (accuracy.h:34-40), one row per request, CSR.
 * seeds: rows of N digits in canonical agent order; removed: canonical
 * indices.  request_ids: the RequestId each row answers to (router noise is
 * keyed on it, router.cpp:53-54).  All pointers device-resident for the
 * device entry points, host-resident for *_host. */
typedef struct {
  int32_t n_requests;
  const uint64_t* request_ids; /* [R] */
  const int32_t* seed_ptr;     /* [R+1] */
  const uint8_t* seeds;        /* [seed_ptr[R] * N] */
  const int32_t* removed_ptr;  /* [R+1] */
  const uint64_t* removed;     /* [removed_ptr[R]] */
} ag_truth;

/* Outputs of enumerate mode (device pointers).
 *   bitmap  [R * W] (W = ceil((end-begin)/32)): bit j of word w of request r
 *           <-> canonical index begin + 32w + j.  May be NULL.
 *   counts  [R]   members per request (required).
 *   offsets [R+1] exclusive scan of counts; may be NULL unless indices set.
 *   indices [capacity] the members of every request in canonical order,
 *           request r at [offsets[r], offsets[r+1]).  NULL = bitmap only.
 *   overflow (device uint32) set to 1 when offsets[R] > capacity; members
 *           past capacity are not written. May be NULL. */
typedef struct {
  uint32_t* bitmap;
  uint64_t* counts;
  uint64_t* offsets;
  uint32_t* indices;
  uint64_t capacity;
  uint32_t* overflow;
} ag_route_out;

/* Enumerate mode over the index range [begin, end) of every request:
 * verdict = router.evaluate(request_ids[r], at_index(i)) for each i, members
 * compacted in canonical order.  Replaces enumerate_members
 * (include/aragog/accuracy.h:81-82, src/accuracy.cpp:227-238) and the
 * exhaustive oracle set (tests/acceptance/criteria.cpp:93-101) without the
 * 4096-config guard; [begin, end) sub-ranges shard a deep space across GPUs
 * (ranks concatenate in rank order = canonical order). */
int ag_route_enumerate(ag_ctx* ctx, const ag_truth* truth_dev,
                       const ag_router* router, uint64_t begin, uint64_t end,
                       uint32_t flags, const ag_route_out* out_dev);

/* Same call with host buffers, copies included (the e2e path).  counts [R],
 * offsets [R+1], indices [capacity] are host arrays (pinned recommended);
 * total receives offsets[R].  Returns AG_ERR_VALIDATION if capacity is too
 * small (total is still reported). */
int ag_route_enumerate_host(ag_ctx* ctx, const ag_truth* truth_host,
                            const ag_router* router, uint64_t begin,
                            uint64_t end, uint32_t flags, uint64_t* counts,
                            uint64_t* offsets, uint32_t* indices,
                            uint64_t capacity, uint64_t* total);

/* ---- learned router ----------------------------- */
/* The paper's fused classifier heads as a RouterBackend: one linear head per
 * canonical configuration, verdict(r, c) = emb[r] . heads[c] + bias[c] > 0.
 * Not in the reference: parity is against the numpy restatement in oracle/
 * within fp32 accumulation tolerance.  Device pointers; heads / emb rows of
 * `dim` bf16 (dim a multiple of 16, <= 128, rows 16-byte aligned), indexed by
 * canonical configuration index / request row; bias fp32 [size]. */
typedef struct {
  int32_t dim;
  const void* heads; /* bf16 [space size][dim] */
  const float* bias; /* [space size] */
} ag_linear_heads;

/* Enumerate mode with the learned router: scores every configuration in
 * [begin, end) of every request as the tcgen05 contraction emb . heads^T
 * with a fused threshold epilogue into the verdict bitmap, then the same
 * scans and compaction as ag_route_enumerate (out as there). */
int ag_route_linear(ag_ctx* ctx, const void* emb, int32_t n_requests,
                    const ag_linear_heads* heads, uint64_t begin, uint64_t end,
                    uint32_t flags, const ag_route_out* out_dev);

/* ---- chain mode ---------------------------------------------------------- */
typedef struct ag_predictor ag_predictor;

/* ConfigPredictor(space, router, PredictorParams{chain_cap, exhaustive_limit})
 * (include/aragog/predictor.h:70-103; src/predictor.cpp:107-131,158-163):
 * builds the chain plan on the host once and uploads it.  chain_cap <= 0
 * means 64; the plan covers the lattice when M^N <= exhaustive_limit. */
int ag_predictor_create(ag_ctx* ctx, int chain_cap, uint64_t exhaustive_limit,
                        ag_predictor** out);
void ag_predictor_destroy(ag_predictor* p);
/* ChainPlan (predictor.h:41-46): chains (host, optional) receives
 * n_chains * chain_len canonical indices. */
int ag_predictor_info(const ag_predictor* p, int32_t* n_chains,
                      int32_t* chain_len, int32_t* exhaustive,
                      int32_t* n_unique, uint64_t* chains);

/* PredictionResult (predictor.h:75-83) for a batch, device pointers.
 * viable: [R * viable_stride] canonical indices in canonical order (the
 * ViableSet, always containing top); n_viable [R]; the rest optional. */
typedef struct {
  uint32_t* viable;
  int32_t viable_stride; /* >= ag_predictor_info n_unique suffices */
  int32_t* n_viable;
  int32_t* search_evals;
  int32_t* verify_evals;
  double* router_time;
  uint8_t* truncated;
} ag_predict_out;

/* ConfigPredictor::predict(request, budget) (predictor.cpp:165-262) for every
 * request of the batch; budgets [R] device (seconds, may be +inf) or NULL to
 * use budget_all.  router.eval_latency is the per-evaluation charge. */
int ag_predict(ag_predictor* p, const ag_truth* truth_dev,
               const ag_router* router, const double* budgets,
               double budget_all, const ag_predict_out* out_dev);

/* ag_predict with host buffers, copies included (the path a drop-in
 * ConfigPredictor::predict takes): truth and budgets [R] host; viable
 * [R * viable_stride], n_viable [R] required; search_evals, verify_evals,
 * router_time, truncated [R] optional. */
int ag_predict_host(ag_predictor* p, const ag_truth* truth_host,
                    const ag_router* router, const double* budgets,
                    double budget_all, uint32_t* viable, int32_t viable_stride,
                    int32_t* n_viable, int32_t* search_evals,
                    int32_t* verify_evals, double* router_time,
                    uint8_t* truncated);

/* ======================================================================== *
 * Per-stage scheduling (hot path 2)                                         *
 * ======================================================================== */

/* Engine pools, EngineState (include/aragog/engine.h:38-53), host arrays. */
typedef struct {
  int32_t n_engines;
  const int32_t* model;     /* [E] tier each pool serves */
  const int32_t* slots;     /* [E] */
  const int32_t* occupancy; /* [E] stages in flight */
  const double* weight;     /* [E] utilization weight of one busy slot */
} ag_engines;

/* AssignmentTriple (scheduler.h:50-55) plus the session slot. */
typedef struct {
  int32_t request_index; /* index into the round's queue (container order) */
  int32_t agent;         /* canonical position */
  int32_t model;
  int32_t slot;          /* session slot (ag_sched_*), -1 for ag_beam_schedule */
  uint64_t request_id;
} ag_triple;

/* Assignment (scheduler.h:76-83); triples/occupancy returned separately. */
typedef struct {
  int32_t n_triples;
  int32_t pad;
  double utilization;
  double flexibility;
  int64_t skips;
  uint64_t states_explored;
} ag_assignment;

/* StageState (request.h:24) */
#define AG_STAGE_PENDING 0
#define AG_STAGE_READY 1
#define AG_STAGE_INFLIGHT 2
#define AG_STAGE_DONE 3

/* The round's vector<const Request*> (request.h:30-47) as host arrays:
 * stages [R*N] by canonical position, viable CSR of canonical indices. */
typedef struct {
  int32_t n_requests;
  const uint64_t* ids;       /* [R] */
  const double* arrival;     /* [R] */
  const uint8_t* stages;     /* [R*N] */
  const int64_t* viable_ptr; /* [R+1] */
  const uint32_t* viable;    /* [viable_ptr[R]] */
} ag_queue;

/* beam_schedule(queue, engines, {beam_width}) (scheduler.h:85-87,
 * scheduler.cpp:289-378), stateless: uploads the queue, runs one round on
 * the GPU, returns the Assignment.  triples [triples_cap], occupancy [E].
 * Validation mirrors the reference (beam width < 1, > 32 pools, duplicate
 * or negative tiers, a viable tier without a pool, an over-capacity pool);
 * the GPU path additionally needs beam_width <= 32 and M <= 32. */
int ag_beam_schedule(ag_ctx* ctx, const ag_queue* queue,
                     const ag_engines* engines, int beam_width,
                     ag_assignment* out, ag_triple* triples,
                     int32_t triples_cap, int32_t* occupancy);

/* Resident scheduling session: the in-flight Request objects live in HBM
 * (viable lists, per-agent candidate masks and model histograms, ready
 * masks); rounds read them in place and dispatch prunes them in place. */
typedef struct ag_sched ag_sched;

/* max_requests: requests resident at once; max_configs: the viable-list pool
 * (u32 canonical indices) the resident requests share -- a capacity: when an
 * add does not fit, the live (pruned) lists are packed on the device first. */
int ag_sched_create(ag_ctx* ctx, int32_t max_requests, uint64_t max_configs,
                    ag_sched** out);
void ag_sched_destroy(ag_sched* s);
/* Request::make for each row (request.cpp:24-50); the requests join the FIFO
 * queue ordered by (arrival, id).  slots_out [R] receives their slots. */
int ag_sched_add(ag_sched* s, const ag_queue* requests, int32_t* slots_out);
/* the request leaves the session (finished); its slot is recycled */
int ag_sched_remove(ag_sched* s, int32_t n, const int32_t* slots);
/* Request::mark_complete(agent) (request.cpp:88-107): done, successors whose
 * predecessors are all done become ready. */
int ag_sched_complete(ag_sched* s, int32_t slot, int32_t agent);
/* One scheduling round over every session request with a ready stage, in
 * FIFO order (Sim::on_round, simulation.cpp:300-318 -> beam_schedule). */
int ag_sched_round(ag_sched* s, const ag_engines* engines, int beam_width,
                   ag_assignment* out, ag_triple* triples, int32_t triples_cap,
                   int32_t* occupancy);
/* Request::mark_dispatched for applied triples (request.cpp:70-86): prefix
 * prune of the viable list in HBM, stage -> in flight. */
int ag_sched_dispatch(ag_sched* s, int32_t n, const ag_triple* applied);
/* apply_assignment(assignment, queue, engines, now, service) (scheduler.cpp:
 * 421-454): the triples in order; one whose pool has no free slot left
 * (occupancy + triples applied before it on the pool >= slots, engine.h:47)
 * is stale and dropped, every other one is applied -- Request::
 * mark_dispatched, the prefix prune of ag_sched_dispatch.  engines as passed
 * to the round; applied [n] (optional) receives 1 / 0 per triple. */
int ag_sched_apply(ag_sched* s, const ag_engines* engines, int32_t n,
                   const ag_triple* triples, uint8_t* applied, int32_t* n_applied,
                   int32_t* n_stale);
/* audit_round_fairness(queue, engines, assignment) (scheduler.cpp:456-480)
 * against the last round's queue (call it right after ag_sched_round, before
 * any dispatch / complete / add / remove): an unassigned ready pair whose
 * allowed engines at its point of the walk are non-empty is a violation.
 * One kernel over every pair; n <= 2048 triples.  viol_ids / viol_agents
 * [cap] receive the violations in pair order (RequestId, agent), n_viol
 * their number. */
int ag_sched_audit(ag_sched* s, const ag_engines* engines, int32_t n,
                   const ag_triple* triples, uint64_t* viol_ids, int32_t* viol_agents,
                   int32_t cap, int32_t* n_viol);
/* Stateless audit_round_fairness(queue, engines, assignment): the queue as
 * for ag_beam_schedule, triples' request_index = container index. */
int ag_audit_round_fairness(ag_ctx* ctx, const ag_queue* queue, const ag_engines* engines,
                            int32_t n, const ag_triple* triples, uint64_t* viol_ids,
                            int32_t* viol_agents, int32_t cap, int32_t* n_viol);
/* diagnostics of the last round, 16 u64: [0..4] device timestamps (ns):
 * start, deltas applied, first candidates published, walk done, finalized;
 * [5..8] walk cycles (find, build, rank, adopt); [9..10] walk steps and
 * children; [11..14] timestamps of the first producer chunk (loads, scan,
 * records, histogram rows) */
int ag_sched_round_timing(ag_sched* s, uint64_t* out16);
/* host wall time (us) of the last ag_sched_round call, entry to return */
double ag_sched_last_round_us(const ag_sched* s);
/* the same call split on the host clock (us): record preparation, the launch
 * call, waiting for the round's completion flag, reading the result back */
int ag_sched_round_host_timing(const ag_sched* s, double* out4);
/* read back one request's current viable list (host buffer) */
int ag_sched_viable(ag_sched* s, int32_t slot, uint32_t* out, int64_t cap,
                    int64_t* n);

/* ---- runtime-cost re-cost + argmin -------------------------------------- */
#define AG_POLICY_PER_INPUT_STATIC 2       /* PolicyKind::kPerInputStatic */
#define AG_POLICY_PER_INPUT_RUNTIME_COST 3 /* PolicyKind::kPerInputRuntimeCost */

/* RuntimeCostContext (include/aragog/workload.h:64-69), host arrays over
 * n_tiers model tiers; mean[m] = ServiceTimeModel::mean(m) (engine.cpp:62-65),
 * computed by the caller's libm exactly as the reference does. */
typedef struct {
  int32_t n_tiers;
  const int32_t* occupancy;
  const int32_t* queued_ahead;
  const int32_t* slots;
  const double* mean;
} ag_load;

/* select_per_input_config(set, space, kind, &load) (workload.cpp:149-176) for
 * a batch: members / offsets are the device CSR of each request's accurate
 * set (e.g. ag_route_enumerate's indices); chosen [R] (device) receives the
 * canonical index, est [R] (device, optional) its estimate_completion.
 * Static: minimum (static cost, index).  Runtime: minimum (estimate, static
 * cost, index), the reference's strict '<' scan over the cost-sorted list.
 * Fully asynchronous on the context stream (the task plan is built on the
 * device); the reference's ValidationErrors -- an empty set, a member tier
 * missing from the load context -- are latched on the device and returned by
 * the next ag_ctx_synchronize. */
int ag_select_per_input(ag_ctx* ctx, const uint32_t* members,
                        const uint64_t* offsets, int32_t n_requests,
                        int32_t kind, const ag_load* load, uint32_t* chosen,
                        double* est);

/* The same selection straight from enumerate mode's verdict bitmap
 * (ag_route_out.bitmap over [begin, end), counts [R]) -- no member list:
 * prefix lower bounds of the key's primary term (estimate; static cost for
 * the static kind) prune the words that cannot hold the minimum, the rest
 * are re-costed exactly, so chosen / est equal ag_select_per_input's on the
 * same set (indices are canonical: begin + position).  records [R][4]
 * optional, as ag_shard_records (an empty shard is not an error there);
 * chosen may be NULL when records is set.  Asynchronous; errors latch as
 * ag_select_per_input's.  Replaces the same call sites. */
int ag_select_bitmap(ag_ctx* ctx, const uint32_t* bitmap, const uint64_t* counts,
                     uint64_t begin, uint64_t end, int32_t n_requests, int32_t kind,
                     const ag_load* load, uint32_t* chosen, double* est,
                     uint64_t* records);
/* Diagnostics: enable = 1 starts counting the words ag_select_bitmap's
 * exact pass evaluates on this context; enable = 0 stops and returns the
 * count (synchronises the context stream). */
int ag_select_bitmap_stats(ag_ctx* ctx, int32_t enable, uint64_t* words_evaluated);

/* ---- configuration-space sharding (config 4) ---------- */
/* Per-shard record of select_per_input_config over this rank's canonical
 * index range: records [R][4] u64 (device) = {member count, estimate (f64
 * bits), static cost (f64 bits), canonical index} of the shard's minimum
 * (estimate, static cost, index); an empty shard gives {0, +inf, +inf, ~0}.
 * Asynchronous on the context stream (no host round trip), so the records
 * can feed one NCCL all-gather directly. */
int ag_shard_records(ag_ctx* ctx, const uint32_t* members, const uint64_t* offsets,
                     int32_t n_requests, int32_t kind, const ag_load* load,
                     uint64_t* records);
/* Merge of the all-gathered records gathered [world][R][4] (device): per
 * request the global member count total[R], the members of shards before
 * `rank` before[R] (this rank's offset into the request's global list), and
 * the whole-space choice best_index / best_est / best_cost [R] = the minimum
 * of the shard minima.  Every output may be NULL.  Asynchronous. */
int ag_merge_records(ag_ctx* ctx, const uint64_t* gathered, int32_t world, int32_t rank,
                     int32_t n_requests, uint64_t* total, uint64_t* before,
                     uint64_t* best_index, double* best_est, double* best_cost);

/* select_per_input_config(accurate, space, kind, load) (workload.cpp:149-176)
 * for a batch of host AccurateSets, end to end on the device: every set's
 * members are enumerated (enumerate_members, accuracy.cpp:227-238, without its
 * 4096-config guard) and compacted, then re-costed and arg-minned as
 * ag_select_per_input.  chosen [R] host canonical indices, est [R] optional. */
int ag_select_per_input_host(ag_ctx* ctx, const ag_truth* truth_host,
                             int32_t kind, const ag_load* load,
                             uint32_t* chosen, double* est);

/* select_per_workflow_config(sample, space, tolerance) (workload.cpp:99-127)
 * without the reference's 4096-configuration guard: sample = a batch of host
 * AccurateSets; chosen receives the canonical index of the first
 * configuration in (static cost, index) order that is accurate on at least
 * (1 - tolerance) * |sample| sets, hits (optional) its count.  Every set is
 * scored over the whole space on the device, counts are column popcounts of
 * the verdict bitmap, the choice a (cost, index) min-reduction. */
int ag_select_per_workflow_host(ag_ctx* ctx, const ag_truth* sample_host,
                                double tolerance, uint64_t* chosen,
                                uint64_t* hits);

/* snapshot_load's queued_ahead (simulation.cpp:194-213): per model tier, the
 * number of ready (request, agent) pairs of the session whose candidate set
 * contains the tier.  out [M] host. */
int ag_sched_queued_ahead(ag_sched* s, int32_t* out);

/* ======================================================================== *
 * Trace I/O of accurate sets         *
 * ======================================================================== */
/* Writes one JSON line per request of the host batch: id, arrival (seconds;
 * arrival may be NULL for 0), and the accurate set enumerated on the device
 * -- {"encoding": "bitmap", "size": S, "bits": hex} over the canonical
 * enumeration when S = M^N <= 4096 (byte k = indices 8k..8k+7, bit 0 first),
 * {"encoding": "list", "size": S, "members": [...]} otherwise.  The reference
 * has no writer for this clause: the format is this library's reading of it.
 * AG_ERR_IO when the file cannot be written. */
int ag_trace_write(ag_ctx* ctx, const ag_truth* truth_host, const double* arrival,
                   const char* path, uint64_t* bytes_written);

/* ======================================================================== *
 * Host-side input synthesis (reference generators; not on the hot path)     *
 * ======================================================================== */
typedef struct {
  double p_easy, p_medium, p_hard, easy_base_prob, violation_rate;
} ag_gen_params;

/* generate_accurate_set for request ids first_id .. first_id+count-1
 * (src/accuracy.cpp:144-198; AccuracyGenParams accuracy.h:42-52).
 * Writes seed_ptr[count+1], seeds (cap seeds_cap rows), removed_ptr[count+1],
 * removed (cap removed_cap). */
int ag_generate_truth(const ag_space* space, const ag_gen_params* params,
                      uint64_t seed, uint64_t salt, uint64_t first_id,
                      int32_t count, int32_t* seed_ptr, uint8_t* seeds,
                      int32_t seeds_cap, int32_t* removed_ptr,
                      uint64_t* removed, int32_t removed_cap);

#ifdef __cplusplus
}
#endif
#endif
