/*
 * aragog_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference's two hot paths (routing and
 * per-stage scheduling), used as the parity checker for the CUDA product in
 * paper_2511_20975_b200/.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  The product path never links it.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  Pinning: tests/test_oracle_pinning.py checks this
 * restatement against golden vectors written by oracle/ref_dump.cpp, which
 * links the reference sources compiled unmodified (oracle/Makefile).
 *
 * Configurations are carried as canonical indices (position 0 = most
 * significant digit, include/aragog/workflow.h:18-21, src/workflow.cpp:250-275)
 * or as digit rows of N uint8 values in canonical agent order.
 */
#ifndef ARAGOG_ORACLE_H
#define ARAGOG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the reference's exception taxonomy
 * (include/aragog/errors.h:22-34, tools/main.cpp:290-303) */
#define AGO_OK 0
#define AGO_INTERNAL 1
#define AGO_VALIDATION 2

const char* ago_last_error(void);

/* ---- rng (include/aragog/rng.h:34-51) ---------------------------------- */
uint64_t ago_splitmix64(uint64_t* state);
uint64_t ago_mix(const uint64_t* words, int n);

/* ---- workflow (src/workflow.cpp:69-173) -------------------------------- */
/* edges are (from, to) pairs of declaration indices.  Outputs (arrays sized
 * n_agents): order[pos] = declaration index, depth[pos].  pred/succ adjacency
 * is returned as bitmasks over canonical positions (n_agents <= 64). */
int ago_graph_build(int n_agents, int n_edges, const int32_t* edges,
                    int32_t* order, int32_t* depth, uint64_t* pred_mask,
                    uint64_t* succ_mask);

/* ---- accuracy ground truth (src/accuracy.cpp:144-198) ------------------ */
typedef struct {
  double p_easy, p_medium, p_hard, easy_base_prob, violation_rate;
} ago_gen_params;

/* seeds_out: up to seeds_cap rows of N digits; removed_out: canonical indices
 * in generation order. */
int ago_gen_truth(int n, int m, const ago_gen_params* p, uint64_t seed,
                  uint64_t request_id, uint64_t salt, uint8_t* seeds_out,
                  int seeds_cap, int* n_seeds, uint64_t* removed_out,
                  int removed_cap, int* n_removed, int* tier);

/* AccurateSet::contains (src/accuracy.cpp:116-124) on a canonical index */
int ago_contains(int n, int m, const uint8_t* seeds, int n_seeds,
                 const uint64_t* removed, int n_removed, uint64_t index);

/* ---- routers (src/router.cpp:22-57) ------------------------------------ */
#define AGO_ROUTER_ORACLE 0
#define AGO_ROUTER_NOISY 1
typedef struct {
  int kind;
  double fp, fn;
  uint64_t noise_seed;
  double eval_latency;
} ago_router;

typedef struct {
  int n, m;
  int n_requests;
  const uint64_t* request_ids;  /* [n_requests] router-visible ids */
  const int32_t* seed_ptr;      /* [n_requests+1] rows into seeds */
  const uint8_t* seeds;         /* [rows * n] */
  const int32_t* removed_ptr;   /* [n_requests+1] */
  const uint64_t* removed;      /* canonical indices */
} ago_truth;

int ago_router_eval(const ago_truth* t, const ago_router* r, int req,
                    uint64_t index);

/* Enumerate mode: evaluate every index in [begin, end) for request `req`,
 * write a bitmap (bit j of word w <-> index begin + 32w + j) and return the
 * member count.  force_top: top is always a member (predictor.cpp:177,255). */
uint64_t ago_enumerate(const ago_truth* t, const ago_router* r, int req,
                       uint64_t begin, uint64_t end, int force_top,
                       uint32_t* bitmap);

/* ---- chain predictor (src/predictor.cpp:107-262) ----------------------- */
/* Chains are written as canonical indices, len = n*(m-1)+1 each. Returns the
 * number of chains (or -1 when chains_cap is too small). */
int ago_build_chains(int n, int m, int chain_cap, uint64_t exhaustive_limit,
                     uint64_t* chains, int chains_cap, int* exhaustive);

typedef struct {
  int search_evals, verify_evals, truncated;
  double router_time;
  int n_viable;
} ago_prediction;

int ago_predict(const ago_truth* t, const ago_router* r, const double* cost,
                const uint64_t* chains, int n_chains, int req, double budget,
                uint64_t* viable_out, int viable_cap, ago_prediction* out);

/* ---- runtime-cost selection (src/workload.cpp:129-176) ----------------- */
typedef struct {
  int n_tiers;
  const int32_t* occupancy;
  const int32_t* queued_ahead;
  const int32_t* slots;
  const double* mean;  /* ServiceTimeModel::mean per tier (engine.cpp:62-65) */
} ago_load;

int ago_estimate_completion(const ago_load* ld, int n, const uint8_t* digits,
                            double* out);
/* argmin over `members` (canonical indices) sorted by (static cost, index);
 * kind 0 = per-input-static, 1 = per-input-runtime-cost */
int ago_select_per_input(int n, int m, const double* cost, const ago_load* ld,
                         int kind, const uint64_t* members, int n_members,
                         uint64_t* chosen, double* est);

/* ---- scheduler (src/scheduler.cpp:29-378, request.cpp:60-86) ----------- */
#define AGO_STAGE_PENDING 0
#define AGO_STAGE_READY 1
#define AGO_STAGE_INFLIGHT 2
#define AGO_STAGE_DONE 3

typedef struct {
  int n, m;                 /* agents, models */
  const int32_t* depth;     /* [n] */
  const int32_t* decl;      /* [n] */
  int n_requests;
  const uint64_t* ids;      /* [R] */
  const double* arrival;    /* [R] */
  const uint8_t* stages;    /* [R*n] */
  const int64_t* viable_ptr;/* [R+1] */
  const uint64_t* viable;   /* canonical indices */
} ago_queue;

typedef struct {
  int n_engines;
  const int32_t* model;
  const int32_t* slots;
  const int32_t* occupancy;
  const double* weight;
} ago_engines;

typedef struct {
  int32_t request_index, agent, model, pad;
  uint64_t request_id;
} ago_triple;

typedef struct {
  int n_triples;
  double utilization, flexibility;
  int64_t skips;
  uint64_t states_explored;
} ago_assignment;

int ago_two_level_order(const ago_queue* q, int32_t* pair_req,
                        int32_t* pair_agent, int pairs_cap, int* n_pairs);

int ago_beam_schedule(const ago_queue* q, const ago_engines* e, int width,
                      ago_triple* triples, int triples_cap,
                      int32_t* occupancy_out, ago_assignment* out);

/* audit_round_fairness (scheduler.cpp:456-480): violations written as
 * (RequestId, agent) in pair order, *n_viol their number. */
int ago_audit_round_fairness(const ago_queue* q, const ago_engines* e,
                             const ago_triple* triples, int n_triples,
                             uint64_t* viol_ids, int32_t* viol_agents, int cap,
                             int* n_viol);

/* Request::mark_dispatched prefix prune (request.cpp:70-86) on one request's
 * list; returns new length (or -1 when nothing survives). */
int64_t ago_prefix_prune(int n, int m, uint64_t* viable, int64_t len, int agent,
                         int model);

/* ---- snapshots (src/snapshots.cpp:60-123) ------------------------------ */
/* Writes a generated snapshot into caller arrays (caps: n<=4, m<=4,
 * requests<=8, viable<=4096 total).  Returns AGO_OK. */
typedef struct {
  int n, m, n_requests, n_engines;
  int32_t depth[8], decl[8];
  double cost[4], weight[4];
  int32_t eng_model[4], eng_slots[4], eng_occ[4];
  double eng_weight[4];
  uint64_t ids[8];
  double arrival[8];
  uint8_t stages[8 * 8];   /* [n_requests * n] */
  int64_t viable_ptr[9];
  uint64_t viable[8 * 256];
} ago_snapshot;

int ago_generate_snapshot(uint64_t seed, uint64_t index, ago_snapshot* out);

#ifdef __cplusplus
}
#endif
#endif
