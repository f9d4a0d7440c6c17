/*
 * aragog_oracle.c -- TEST INFRASTRUCTURE ONLY (see aragog_oracle.h).
 *
 * Plain-C restatement of the reference hot paths, used solely as the parity
 * checker for the CUDA product.  Compiled with -ffp-contract=off so every
 * double expression rounds exactly like the reference built without -march
 * (proj/CMakeLists.txt:12).
 */
#include "aragog_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* ago_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ rng */
#define GAMMA 0x9e3779b97f4a7c15ULL

/* rng.h:34-39 */
uint64_t ago_splitmix64(uint64_t* state) {
  uint64_t z = (*state += GAMMA);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.h:43-51 */
uint64_t ago_mix(const uint64_t* words, int n) {
  uint64_t state = 0x6a09e667f3bcc909ULL;
  for (int i = 0; i < n; ++i) {
    state ^= words[i] + GAMMA + (state << 6) + (state >> 2);
    uint64_t s = state;
    state = ago_splitmix64(&s);
  }
  return state;
}

static uint64_t mix2(uint64_t a, uint64_t b) {
  uint64_t w[2] = {a, b};
  return ago_mix(w, 2);
}

static uint64_t mix3(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t w[3] = {a, b, c};
  return ago_mix(w, 3);
}

/* rng::Stream (rng.h:64-96), only the draws the hot-path generators use */
typedef struct {
  uint64_t s;
} stream_t;
static uint64_t st_u64(stream_t* st) { return ago_splitmix64(&st->s); }
static double st_unit(stream_t* st) {
  return (double)(st_u64(st) >> 11) * 0x1.0p-53;
}
static uint64_t st_below(stream_t* st, uint64_t n) { return st_u64(st) % n; }
static int st_bernoulli(stream_t* st, double p) { return st_unit(st) < p; }

/* ---------------------------------------------------------- config index */
static uint64_t space_size(int n, int m) {
  uint64_t s = 1;
  for (int i = 0; i < n; ++i) s *= (uint64_t)m;
  return s;
}

/* ConfigSpace::at_index (workflow.cpp:263-275) */
static void decode(int n, int m, uint64_t idx, uint8_t* d) {
  for (int i = n - 1; i >= 0; --i) {
    d[i] = (uint8_t)(idx % (uint64_t)m);
    idx /= (uint64_t)m;
  }
}

/* ConfigSpace::index_of (workflow.cpp:250-261) */
static uint64_t encode(int n, int m, const uint8_t* d) {
  uint64_t idx = 0;
  for (int i = 0; i < n; ++i) idx = idx * (uint64_t)m + d[i];
  return idx;
}

/* config_leq (workflow.cpp:189-207): x <= y pointwise */
static int leq(int n, const uint8_t* x, const uint8_t* y) {
  for (int i = 0; i < n; ++i)
    if (x[i] > y[i]) return 0;
  return 1;
}

/* compare_configs: 0 equal, 1 below, 2 above, 3 incomparable */
static int compare_cfg(int n, const uint8_t* x, const uint8_t* y) {
  int le = 1, ge = 1;
  for (int i = 0; i < n; ++i) {
    if (x[i] > y[i]) le = 0;
    if (x[i] < y[i]) ge = 0;
  }
  if (le && ge) return 0;
  if (le) return 1;
  if (ge) return 2;
  return 3;
}

/* ConfigSpace::static_cost (workflow.cpp:291-296): left fold */
static double static_cost_idx(int n, int m, const double* cost, uint64_t idx) {
  uint8_t d[64];
  decode(n, m, idx, d);
  double c = 0.0;
  for (int i = 0; i < n; ++i) c += cost[d[i]];
  return c;
}

/* ---------------------------------------------------------------- graph */
/* WorkflowGraph::build (workflow.cpp:69-173): Kahn's algorithm releasing the
 * smallest declaration index first, then a reverse depth sweep. */
int ago_graph_build(int n, int n_edges, const int32_t* edges, int32_t* order,
                    int32_t* depth, uint64_t* pred_mask, uint64_t* succ_mask) {
  if (n < 1) return fail(AGO_VALIDATION, "workflow needs at least 1 agent");
  if (n > 64) return fail(AGO_VALIDATION, "oracle supports <= 64 agents");
  uint64_t out[64] = {0}, in[64] = {0};
  for (int e = 0; e < n_edges; ++e) {
    int f = edges[2 * e], t = edges[2 * e + 1];
    if (f < 0 || f >= n) return fail(AGO_VALIDATION, "edge from unknown agent");
    if (t < 0 || t >= n) return fail(AGO_VALIDATION, "edge to unknown agent");
    if (f == t) return fail(AGO_VALIDATION, "self loop on agent");
    out[f] |= 1ULL << t;
    in[t] |= 1ULL << f;
  }
  int indeg[64];
  for (int i = 0; i < n; ++i) indeg[i] = __builtin_popcountll(in[i]);
  uint64_t ready = 0;
  for (int i = 0; i < n; ++i)
    if (indeg[i] == 0) ready |= 1ULL << i;
  int cnt = 0;
  while (ready) {
    int u = __builtin_ctzll(ready); /* min-heap on declaration index */
    ready &= ready - 1;
    order[cnt++] = u;
    for (int v = 0; v < n; ++v)
      if ((out[u] >> v) & 1)
        if (--indeg[v] == 0) ready |= 1ULL << v;
  }
  if (cnt != n) return fail(AGO_VALIDATION, "workflow has a cycle");
  int pos_of[64];
  for (int p = 0; p < n; ++p) pos_of[order[p]] = p;
  for (int p = 0; p < n; ++p) {
    pred_mask[p] = succ_mask[p] = 0;
    int d = order[p];
    for (int v = 0; v < n; ++v) {
      if ((out[d] >> v) & 1) succ_mask[p] |= 1ULL << pos_of[v];
      if ((in[d] >> v) & 1) pred_mask[p] |= 1ULL << pos_of[v];
    }
  }
  for (int p = n - 1; p >= 0; --p) {
    depth[p] = 0;
    for (int s = 0; s < n; ++s)
      if ((succ_mask[p] >> s) & 1)
        if (depth[s] + 1 > depth[p]) depth[p] = depth[s] + 1;
  }
  return AGO_OK;
}

/* ------------------------------------------------------------- accuracy */
/* AccurateSet::contains (accuracy.cpp:116-124) */
static int contains_digits(int n, int m, const uint8_t* seeds, int ns,
                           const uint64_t* removed, int nr, const uint8_t* c) {
  if (nr) {
    uint64_t idx = encode(n, m, c);
    for (int i = 0; i < nr; ++i)
      if (removed[i] == idx) return 0;
  }
  for (int s = 0; s < ns; ++s)
    if (leq(n, seeds + (size_t)s * n, c)) return 1;
  return 0;
}

int ago_contains(int n, int m, const uint8_t* seeds, int ns,
                 const uint64_t* removed, int nr, uint64_t index) {
  uint8_t d[64];
  decode(n, m, index, d);
  return contains_digits(n, m, seeds, ns, removed, nr, d);
}

/* minimalize (accuracy.cpp:28-42) */
static int minimalize(int n, uint8_t* seeds, int k) {
  uint8_t kept[16 * 64];
  int nk = 0;
  for (int i = 0; i < k; ++i) {
    int dominated = 0;
    for (int j = 0; j < k && !dominated; ++j) {
      if (i == j) continue;
      int o = compare_cfg(n, seeds + j * n, seeds + i * n);
      if (o == 1) dominated = 1;
      if (o == 0 && j < i) dominated = 1;
    }
    if (!dominated) memcpy(kept + (nk++) * n, seeds + i * n, (size_t)n);
  }
  memcpy(seeds, kept, (size_t)nk * n);
  return nk;
}

/* removal_delta (accuracy.cpp:65-82) */
static long long removal_delta(int n, int m, const char* member, uint8_t* c) {
  long long delta = 0;
  for (int i = 0; i < n; ++i) {
    if (c[i] > 0) {
      --c[i];
      if (member[encode(n, m, c)]) ++delta;
      ++c[i];
    }
    if (c[i] + 1 < m) {
      ++c[i];
      if (!member[encode(n, m, c)]) --delta;
      --c[i];
    }
  }
  return delta;
}

/* generate_accurate_set (accuracy.cpp:144-198) incl. inject_violations
 * (accuracy.cpp:84-112) */
int ago_gen_truth(int n, int m, const ago_gen_params* p, uint64_t seed,
                  uint64_t request_id, uint64_t salt, uint8_t* seeds_out,
                  int seeds_cap, int* n_seeds, uint64_t* removed_out,
                  int removed_cap, int* n_removed, int* tier) {
  if (p->p_easy < 0 || p->p_medium < 0 || p->p_hard < 0 ||
      p->p_easy + p->p_medium + p->p_hard <= 0)
    return fail(AGO_VALIDATION, "difficulty mix needs nonnegative weights, sum > 0");
  if (p->easy_base_prob < 0 || p->easy_base_prob > 1)
    return fail(AGO_VALIDATION, "easy_base_prob outside [0, 1]");
  if (p->violation_rate < 0 || p->violation_rate >= 1)
    return fail(AGO_VALIDATION, "violation_rate outside [0, 1)");
  if (n > 64) return fail(AGO_VALIDATION, "oracle supports <= 64 agents");
  double logsz = (double)n * log2((double)m);
  uint64_t size = logsz < 64 ? space_size(n, m) : 0;
  if (p->violation_rate > 0 && (logsz >= 64 || size > 4096))
    return fail(AGO_VALIDATION, "violation injection needs an enumerable configuration space");

  stream_t st = {mix3(seed, salt, request_id)};
  const double total = p->p_easy + p->p_medium + p->p_hard;
  const double u = st_unit(&st) * total;
  uint8_t seeds[16 * 64];
  int k = 0;
  if (u < p->p_easy) {
    *tier = 0;
    if (st_bernoulli(&st, p->easy_base_prob)) {
      memset(seeds, 0, (size_t)n);
      k = 1;
    } else {
      int cnt = 1 + (int)st_below(&st, 2);
      for (int s = 0; s < cnt; ++s) {
        uint8_t* c = seeds + k * n;
        int is_base = 1;
        for (int i = 0; i < n; ++i) {
          double v = st_unit(&st);
          int d = (int)(v * v * m);
          c[i] = (uint8_t)(d < m - 1 ? d : m - 1);
          if (c[i]) is_base = 0;
        }
        if (is_base) c[st_below(&st, (uint64_t)n)] = 1;
        ++k;
      }
    }
  } else if (u < p->p_easy + p->p_medium) {
    *tier = 1;
    int cnt = 1 + (int)st_below(&st, 2);
    for (int s = 0; s < cnt; ++s) {
      uint8_t* c = seeds + k * n;
      for (int i = 0; i < n; ++i) c[i] = (uint8_t)st_below(&st, (uint64_t)m);
      ++k;
    }
  } else {
    *tier = 2;
    memset(seeds, m - 1, (size_t)n);
    k = 1;
  }
  k = minimalize(n, seeds, k);
  if (k > seeds_cap) return fail(AGO_VALIDATION, "seeds_cap too small");
  memcpy(seeds_out, seeds, (size_t)k * n);
  *n_seeds = k;
  *n_removed = 0;

  if (p->violation_rate > 0) {
    uint64_t edges = (uint64_t)(m - 1) * (size / (uint64_t)m) * (uint64_t)n;
    double expectation = p->violation_rate * (double)edges;
    uint64_t target = (uint64_t)floor(expectation);
    if (st_bernoulli(&st, expectation - floor(expectation))) ++target;
    if (target == 0) return AGO_OK;
    char* member = (char*)malloc(size);
    uint64_t* cand = (uint64_t*)malloc(size * sizeof(uint64_t));
    uint8_t c[64];
    for (uint64_t i = 0; i < size; ++i) {
      decode(n, m, i, c);
      member[i] = (char)contains_digits(n, m, seeds, k, NULL, 0, c);
    }
    const uint64_t top_idx = size - 1;
    uint64_t violated = 0;
    int nr = 0;
    while (violated < target) {
      uint64_t remaining = target - violated;
      uint64_t nc = 0;
      for (uint64_t i = 0; i < size; ++i) {
        if (!member[i] || i == top_idx) continue;
        decode(n, m, i, c);
        long long d = removal_delta(n, m, member, c);
        if (d >= 1 && (uint64_t)d <= remaining) cand[nc++] = i;
      }
      if (nc == 0) break;
      uint64_t pick = cand[st_below(&st, nc)];
      decode(n, m, pick, c);
      violated += (uint64_t)removal_delta(n, m, member, c);
      member[pick] = 0;
      if (nr >= removed_cap) {
        free(member);
        free(cand);
        return fail(AGO_VALIDATION, "removed_cap too small");
      }
      removed_out[nr++] = pick;
    }
    *n_removed = nr;
    free(member);
    free(cand);
  }
  return AGO_OK;
}

/* --------------------------------------------------------------- router */
/* hash_config (router.cpp:22-28) */
static uint64_t hash_config(int n, const uint8_t* d) {
  uint64_t h = 0x2545f4914f6cdd1dULL;
  for (int i = 0; i < n; ++i) h = mix2(h, (uint64_t)d[i]);
  return h;
}

static int truth_eval(const ago_truth* t, int req, const uint8_t* d) {
  int s0 = t->seed_ptr[req], s1 = t->seed_ptr[req + 1];
  int r0 = t->removed_ptr[req], r1 = t->removed_ptr[req + 1];
  return contains_digits(t->n, t->m, t->seeds + (size_t)s0 * t->n, s1 - s0,
                         t->removed + r0, r1 - r0, d);
}

/* OracleRouter::evaluate (router.cpp:37-39), NoisyRouter::evaluate
 * (router.cpp:50-57) */
static int router_eval_digits(const ago_truth* t, const ago_router* r, int req,
                              const uint8_t* d) {
  int truth = truth_eval(t, req, d);
  if (r->kind == AGO_ROUTER_ORACLE) return truth;
  uint64_t w[4] = {r->noise_seed, 0xA3, t->request_ids[req],
                   hash_config(t->n, d)};
  uint64_t key = ago_mix(w, 4);
  double u = (double)(key >> 11) * 0x1.0p-53;
  return truth ? (u >= r->fn) : (u < r->fp);
}

int ago_router_eval(const ago_truth* t, const ago_router* r, int req,
                    uint64_t index) {
  uint8_t d[64];
  decode(t->n, t->m, index, d);
  return router_eval_digits(t, r, req, d);
}

/* enumerate_members (accuracy.cpp:227-238) / oracle_accurate_set
 * (tests/acceptance/criteria.cpp:93-101) generalised to any router */
uint64_t ago_enumerate(const ago_truth* t, const ago_router* r, int req,
                       uint64_t begin, uint64_t end, int force_top,
                       uint32_t* bitmap) {
  const uint64_t top = space_size(t->n, t->m) - 1;
  uint64_t count = 0;
  uint8_t d[64];
  uint64_t nwords = (end - begin + 31) / 32;
  if (bitmap) memset(bitmap, 0, nwords * 4);
  for (uint64_t i = begin; i < end; ++i) {
    decode(t->n, t->m, i, d);
    int v = router_eval_digits(t, r, req, d);
    if (force_top && i == top) v = 1;
    if (v) {
      ++count;
      if (bitmap) bitmap[(i - begin) >> 5] |= 1u << ((i - begin) & 31);
    }
  }
  return count;
}

/* ------------------------------------------------------------ predictor */
typedef struct {
  int n, m;
  uint64_t size;
  int track;
  size_t cap;
  uint64_t* out;
  int out_cap;
  int n_chains;
  int overflow;
  uint64_t* uncovered;
  uint64_t n_uncovered;
  char* covered;
  int len; /* chain length n*(m-1)+1 */
} chain_builder;

static int cb_done(const chain_builder* b) {
  if (b->cap != 0 && (size_t)b->n_chains >= b->cap) return 1;
  return b->track && b->n_uncovered == 0;
}

/* ChainBuilder::has_uncovered_above (predictor.cpp:40-45) */
static int cb_has_uncovered_above(const chain_builder* b, const uint8_t* c) {
  uint8_t d[64];
  for (uint64_t k = b->n_uncovered; k-- > 0;) {
    decode(b->n, b->m, b->uncovered[k], d);
    if (leq(b->n, c, d)) return 1;
  }
  return 0;
}

/* ChainBuilder::path_has_fresh (predictor.cpp:50-55) */
static int cb_path_has_fresh(const chain_builder* b, const uint64_t* path,
                             int plen) {
  for (int i = 0; i < plen; ++i)
    if (!b->covered[path[i]]) return 1;
  return 0;
}

/* ChainBuilder::cover (predictor.cpp:58-73) */
static int cb_cover(chain_builder* b, const uint64_t* path, int plen) {
  int fresh = 0;
  for (int i = 0; i < plen; ++i) {
    if (!b->covered[path[i]]) {
      b->covered[path[i]] = 1;
      fresh = 1;
    }
  }
  if (fresh) {
    uint64_t w = 0;
    for (uint64_t k = 0; k < b->n_uncovered; ++k)
      if (!b->covered[b->uncovered[k]]) b->uncovered[w++] = b->uncovered[k];
    b->n_uncovered = w;
  }
  return fresh;
}

/* ChainBuilder::dfs (predictor.cpp:80-98) */
static void cb_dfs(chain_builder* b, uint64_t* path, int plen) {
  if (cb_done(b)) return;
  uint8_t tail[64];
  decode(b->n, b->m, path[plen - 1], tail);
  if (path[plen - 1] == b->size - 1) { /* is_top */
    if (!b->track || cb_cover(b, path, plen)) {
      if (b->n_chains < b->out_cap)
        memcpy(b->out + (size_t)b->n_chains * b->len, path,
               sizeof(uint64_t) * (size_t)plen);
      else
        b->overflow = 1;
      b->n_chains++;
    }
    return;
  }
  for (int i = 0; i < b->n && !cb_done(b); ++i) {
    if (tail[i] + 1 >= b->m) continue;
    uint8_t next[64];
    memcpy(next, tail, (size_t)b->n);
    ++next[i];
    if (b->track && !cb_path_has_fresh(b, path, plen) &&
        !cb_has_uncovered_above(b, next))
      continue;
    path[plen] = encode(b->n, b->m, next);
    cb_dfs(b, path, plen + 1);
  }
}

/* build_chains (predictor.cpp:107-131) */
int ago_build_chains(int n, int m, int chain_cap, uint64_t exhaustive_limit,
                     uint64_t* chains, int chains_cap, int* exhaustive) {
  chain_builder b;
  memset(&b, 0, sizeof b);
  b.n = n;
  b.m = m;
  b.size = space_size(n, m);
  b.len = n * (m - 1) + 1;
  b.track = b.size <= exhaustive_limit;
  b.out = chains;
  b.out_cap = chains_cap;
  if (b.track) {
    b.covered = (char*)calloc(b.size, 1);
    b.uncovered = (uint64_t*)malloc(b.size * sizeof(uint64_t));
    for (uint64_t i = 0; i < b.size; ++i) b.uncovered[i] = i;
    b.n_uncovered = b.size;
  } else {
    b.cap = (size_t)(chain_cap > 0 ? chain_cap : 64);
  }
  uint64_t* path = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)b.len);
  path[0] = 0;
  cb_dfs(&b, path, 1);
  *exhaustive = b.track && b.n_uncovered == 0;
  free(path);
  free(b.covered);
  free(b.uncovered);
  return b.overflow ? -1 : b.n_chains;
}

/* per-request verdict cache keyed by canonical index */
typedef struct {
  uint64_t* key;
  char* val;
  int n, cap;
} vcache;

static int vc_find(const vcache* c, uint64_t k) {
  for (int i = 0; i < c->n; ++i)
    if (c->key[i] == k) return i;
  return -1;
}

static void vc_put(vcache* c, uint64_t k, int v) {
  if (c->n == c->cap) {
    c->cap = c->cap ? 2 * c->cap : 64;
    c->key = (uint64_t*)realloc(c->key, sizeof(uint64_t) * (size_t)c->cap);
    c->val = (char*)realloc(c->val, (size_t)c->cap);
  }
  c->key[c->n] = k;
  c->val[c->n] = (char)v;
  c->n++;
}

typedef struct {
  const ago_truth* t;
  const ago_router* r;
  int req;
  uint64_t top;
  double latency, budget;
  vcache cache;
  ago_prediction* res;
  int* charging;
} pctx;

/* the eval lambda (predictor.cpp:176-189): -1 = refused by the budget */
static int p_eval(pctx* p, uint64_t c) {
  if (c == p->top) return 1;
  int i = vc_find(&p->cache, c);
  if (i >= 0) return p->cache.val[i];
  if (p->res->router_time + p->latency > p->budget) {
    p->res->truncated = 1;
    return -1;
  }
  int v = ago_router_eval(p->t, p->r, p->req, c);
  p->res->router_time += p->latency;
  ++*p->charging;
  vc_put(&p->cache, c, v);
  return v;
}

/* the cached lambda (predictor.cpp:191-196) */
static int p_cached(pctx* p, uint64_t c) {
  if (c == p->top) return 1;
  int i = vc_find(&p->cache, c);
  return i >= 0 ? p->cache.val[i] : -1;
}

static const double* g_sort_cost;
static int g_sort_n, g_sort_m;

static int cmp_cost_lex(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  double cx = static_cost_idx(g_sort_n, g_sort_m, g_sort_cost, x);
  double cy = static_cost_idx(g_sort_n, g_sort_m, g_sort_cost, y);
  if (cx != cy) return cx < cy ? -1 : 1;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* ConfigPredictor::predict (predictor.cpp:165-262) */
int ago_predict(const ago_truth* t, const ago_router* r, const double* cost,
                const uint64_t* chains, int n_chains, int req, double budget,
                uint64_t* viable_out, int viable_cap, ago_prediction* out) {
  memset(out, 0, sizeof *out);
  pctx p;
  memset(&p, 0, sizeof p);
  p.t = t;
  p.r = r;
  p.req = req;
  p.top = space_size(t->n, t->m) - 1;
  p.latency = r->eval_latency;
  p.budget = budget;
  p.res = out;
  p.charging = &out->search_evals;
  const int len = t->n * (t->m - 1) + 1;

  size_t* bound = (size_t*)calloc((size_t)n_chains + 1, sizeof(size_t));
  char* searched = (char*)calloc((size_t)n_chains + 1, 1);
  for (int ci = 0; ci < n_chains; ++ci) {
    if (out->truncated) break;
    const uint64_t* chain = chains + (size_t)ci * len;
    size_t lo = 0, hi = (size_t)len;
    for (size_t i = 0; i < (size_t)len; ++i) {
      int v = p_cached(&p, chain[i]);
      if (v < 0) continue;
      if (v) {
        if (i < hi) hi = i;
      } else {
        if (i + 1 > lo) lo = i + 1;
      }
    }
    if (lo > hi) {
      bound[ci] = hi;
      searched[ci] = 1;
      continue;
    }
    /* find_chain_boundary (predictor.cpp:133-148) */
    int aborted = 0;
    while (lo < hi) {
      size_t mid = lo + (hi - lo) / 2;
      int v = p_eval(&p, chain[mid]);
      if (v < 0) {
        aborted = 1;
        break;
      }
      if (v)
        hi = mid;
      else
        lo = mid + 1;
    }
    if (aborted) break;
    bound[ci] = lo;
    searched[ci] = 1;
  }

  p.charging = &out->verify_evals;
  size_t ncand = 0, cap = 64;
  uint64_t* cand = (uint64_t*)malloc(sizeof(uint64_t) * cap);
  for (int ci = 0; ci < n_chains; ++ci) {
    if (!searched[ci]) continue;
    const uint64_t* chain = chains + (size_t)ci * len;
    for (size_t i = bound[ci]; i < (size_t)len; ++i) {
      if (chain[i] == p.top) continue;
      if (ncand == cap) {
        cap *= 2;
        cand = (uint64_t*)realloc(cand, sizeof(uint64_t) * cap);
      }
      cand[ncand++] = chain[i];
    }
  }
  g_sort_cost = cost;
  g_sort_n = t->n;
  g_sort_m = t->m;
  qsort(cand, ncand, sizeof(uint64_t), cmp_cost_lex);
  size_t u = 0;
  for (size_t i = 0; i < ncand; ++i)
    if (u == 0 || cand[u - 1] != cand[i]) cand[u++] = cand[i];
  ncand = u;

  int nk = 0;
  int rc = AGO_OK;
  for (size_t i = 0; i < ncand; ++i) {
    int v = p_eval(&p, cand[i]);
    if (v < 0) continue;
    if (v) {
      if (nk >= viable_cap) {
        rc = fail(AGO_VALIDATION, "viable_cap too small");
        break;
      }
      viable_out[nk++] = cand[i];
    }
  }
  if (rc == AGO_OK) {
    if (nk >= viable_cap) {
      rc = fail(AGO_VALIDATION, "viable_cap too small");
    } else {
      viable_out[nk++] = p.top;
      qsort(viable_out, (size_t)nk, sizeof(uint64_t), cmp_u64);
      out->n_viable = nk;
    }
  }
  free(cand);
  free(bound);
  free(searched);
  free(p.cache.key);
  free(p.cache.val);
  return rc;
}

/* ---------------------------------------------------------- runtime cost */
/* estimate_completion (workload.cpp:129-147) */
int ago_estimate_completion(const ago_load* ld, int n, const uint8_t* d,
                            double* out) {
  double total = 0.0;
  for (int a = 0; a < n; ++a) {
    int mi = d[a];
    if (mi >= ld->n_tiers || ld->slots[mi] <= 0)
      return fail(AGO_VALIDATION, "estimator context missing a model tier");
    double load = (double)(ld->occupancy[mi] + ld->queued_ahead[mi]);
    double mean = ld->mean[mi];
    total += (load / (double)ld->slots[mi]) * mean + mean;
  }
  *out = total;
  return AGO_OK;
}

/* select_per_input_config (workload.cpp:149-176) with members_by_cost
 * (workload.cpp:32-42) */
int ago_select_per_input(int n, int m, const double* cost, const ago_load* ld,
                         int kind, const uint64_t* members, int n_members,
                         uint64_t* chosen, double* est) {
  if (n_members <= 0) return fail(AGO_VALIDATION, "accurate set is empty");
  uint64_t* sorted = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n_members);
  memcpy(sorted, members, sizeof(uint64_t) * (size_t)n_members);
  g_sort_cost = cost;
  g_sort_n = n;
  g_sort_m = m;
  qsort(sorted, (size_t)n_members, sizeof(uint64_t), cmp_cost_lex);
  if (kind == 0) {
    *chosen = sorted[0];
    *est = 0.0;
    free(sorted);
    return AGO_OK;
  }
  uint8_t d[64];
  size_t best = 0;
  double best_est;
  decode(n, m, sorted[0], d);
  int rc = ago_estimate_completion(ld, n, d, &best_est);
  for (int i = 1; rc == AGO_OK && i < n_members; ++i) {
    double e;
    decode(n, m, sorted[i], d);
    rc = ago_estimate_completion(ld, n, d, &e);
    if (rc == AGO_OK && e < best_est) {
      best = (size_t)i;
      best_est = e;
    }
  }
  *chosen = sorted[best];
  *est = best_est;
  free(sorted);
  return rc;
}

/* ------------------------------------------------------------ scheduler */
typedef struct {
  const ago_queue* q;
  const ago_engines* e;
  int n_pairs;
  int32_t* pair_req;
  int32_t* pair_agent;
  uint32_t* base_mask;
  int model_to_engine[64];
  int n_m2e;
} round_ctx;

static const ago_queue* g_sort_q;

static int cmp_fifo(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  double ax = g_sort_q->arrival[x], ay = g_sort_q->arrival[y];
  if (ax != ay) return ax < ay ? -1 : 1;
  uint64_t ix = g_sort_q->ids[x], iy = g_sort_q->ids[y];
  return ix < iy ? -1 : (ix > iy ? 1 : 0);
}

/* two_level_order (scheduler.cpp:224-246) */
int ago_two_level_order(const ago_queue* q, int32_t* pair_req,
                        int32_t* pair_agent, int pairs_cap, int* n_pairs) {
  int R = q->n_requests, n = q->n;
  int* order = (int*)malloc(sizeof(int) * (size_t)(R ? R : 1));
  for (int i = 0; i < R; ++i) order[i] = i;
  g_sort_q = q;
  qsort(order, (size_t)R, sizeof(int), cmp_fifo);
  int np = 0;
  for (int k = 0; k < R; ++k) {
    int qi = order[k];
    int ready[64], nr = 0;
    for (int a = 0; a < n; ++a)
      if (q->stages[(size_t)qi * n + a] == AGO_STAGE_READY) ready[nr++] = a;
    /* insertion sort on (depth desc, declaration asc) */
    for (int i = 1; i < nr; ++i) {
      int x = ready[i], j = i - 1;
      while (j >= 0) {
        int y = ready[j];
        int before = q->depth[x] != q->depth[y] ? q->depth[x] > q->depth[y]
                                                : q->decl[x] < q->decl[y];
        if (!before) break;
        ready[j + 1] = y;
        --j;
      }
      ready[j + 1] = x;
    }
    for (int i = 0; i < nr; ++i) {
      if (np >= pairs_cap) {
        free(order);
        return fail(AGO_VALIDATION, "pairs_cap too small");
      }
      pair_req[np] = qi;
      pair_agent[np] = ready[i];
      ++np;
    }
  }
  *n_pairs = np;
  free(order);
  return AGO_OK;
}

static int digit_of(int n, int m, uint64_t idx, int agent) {
  for (int i = n - 1; i > agent; --i) idx /= (uint64_t)m;
  return (int)(idx % (uint64_t)m);
}

/* RoundContext (scheduler.cpp:29-73) */
static int ctx_build(round_ctx* c, const ago_queue* q, const ago_engines* e) {
  memset(c, 0, sizeof *c);
  c->q = q;
  c->e = e;
  if (e->n_engines > 32)
    return fail(AGO_VALIDATION, "more engine pools than the scheduler supports");
  int max_model = -1;
  for (int i = 0; i < e->n_engines; ++i)
    if (e->model[i] > max_model) max_model = e->model[i];
  if (max_model >= 64) return fail(AGO_VALIDATION, "oracle supports < 64 tiers");
  c->n_m2e = max_model + 1;
  for (int i = 0; i < c->n_m2e; ++i) c->model_to_engine[i] = -1;
  for (int i = 0; i < e->n_engines; ++i) {
    int m = e->model[i];
    if (m < 0) return fail(AGO_VALIDATION, "engine with negative model tier");
    if (c->model_to_engine[m] != -1)
      return fail(AGO_VALIDATION, "two engine pools serve the same model tier");
    c->model_to_engine[m] = i;
  }
  int cap = 0;
  for (int r = 0; r < q->n_requests; ++r)
    for (int a = 0; a < q->n; ++a)
      cap += q->stages[(size_t)r * q->n + a] == AGO_STAGE_READY;
  c->pair_req = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap + 1));
  c->pair_agent = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap + 1));
  c->base_mask = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(cap + 1));
  int rc = ago_two_level_order(q, c->pair_req, c->pair_agent, cap, &c->n_pairs);
  if (rc) return rc;
  for (int p = 0; p < c->n_pairs; ++p) {
    int r = c->pair_req[p], a = c->pair_agent[p];
    uint32_t mask = 0;
    for (int64_t j = q->viable_ptr[r]; j < q->viable_ptr[r + 1]; ++j) {
      int mdl = digit_of(q->n, q->m, q->viable[j], a);
      if (mdl >= c->n_m2e || c->model_to_engine[mdl] < 0)
        return fail(AGO_VALIDATION, "viable model tier without an engine pool");
      mask |= 1u << c->model_to_engine[mdl];
    }
    c->base_mask[p] = mask;
  }
  return AGO_OK;
}

static void ctx_free(round_ctx* c) {
  free(c->pair_req);
  free(c->pair_agent);
  free(c->base_mask);
}

typedef struct {
  int req;
  int n_surv;
  int32_t* surv; /* indices into the request's viable list */
} touched_t;

/* BeamState (scheduler.cpp:80-93) */
typedef struct {
  int n_triples, cap_triples;
  ago_triple* triples;
  int32_t occ[32];
  uint32_t free_mask;
  double util, flex_sum;
  int flex_count;
  int64_t skips;
  int n_touched, cap_touched;
  touched_t* touched;
} bstate;

static void bs_free(bstate* s) {
  for (int i = 0; i < s->n_touched; ++i) free(s->touched[i].surv);
  free(s->touched);
  free(s->triples);
  memset(s, 0, sizeof *s);
}

static void bs_copy(bstate* dst, const bstate* src) {
  *dst = *src;
  dst->triples = (ago_triple*)malloc(sizeof(ago_triple) * (size_t)(src->cap_triples + 1));
  memcpy(dst->triples, src->triples, sizeof(ago_triple) * (size_t)src->n_triples);
  dst->touched = (touched_t*)malloc(sizeof(touched_t) * (size_t)(src->cap_touched + 1));
  for (int i = 0; i < src->n_touched; ++i) {
    dst->touched[i] = src->touched[i];
    dst->touched[i].surv = (int32_t*)malloc(sizeof(int32_t) * (size_t)(src->touched[i].n_surv + 1));
    memcpy(dst->touched[i].surv, src->touched[i].surv,
           sizeof(int32_t) * (size_t)src->touched[i].n_surv);
  }
}

static double bs_flex(const bstate* s) {
  return s->flex_count > 0 ? s->flex_sum / s->flex_count : 1.0;
}

/* triples_less (scheduler.cpp:95-105) */
static int triples_less(const bstate* a, const bstate* b) {
  int n = a->n_triples < b->n_triples ? a->n_triples : b->n_triples;
  for (int i = 0; i < n; ++i) {
    const ago_triple *x = &a->triples[i], *y = &b->triples[i];
    if (x->request_index != y->request_index) return x->request_index < y->request_index;
    if (x->agent != y->agent) return x->agent < y->agent;
    if (x->model != y->model) return x->model < y->model;
  }
  return a->n_triples < b->n_triples;
}

/* state_better (scheduler.cpp:109-115) */
static int state_better(const bstate* a, const bstate* b) {
  if (a->util != b->util) return a->util > b->util;
  double fa = bs_flex(a), fb = bs_flex(b);
  if (fa != fb) return fa > fb;
  if (a->skips != b->skips) return a->skips < b->skips;
  return triples_less(a, b);
}

/* initial_state (scheduler.cpp:117-128) */
static int initial_state(const round_ctx* c, bstate* s, int cap_triples) {
  memset(s, 0, sizeof *s);
  s->cap_triples = cap_triples;
  s->triples = (ago_triple*)malloc(sizeof(ago_triple) * (size_t)(cap_triples + 1));
  s->cap_touched = c->q->n_requests;
  s->touched = (touched_t*)malloc(sizeof(touched_t) * (size_t)(s->cap_touched + 1));
  for (int i = 0; i < c->e->n_engines; ++i) {
    int occ = c->e->occupancy[i];
    if (occ > c->e->slots[i]) return fail(AGO_VALIDATION, "engine over capacity");
    s->occ[i] = occ;
    s->util += occ * c->e->weight[i];
    if (c->e->slots[i] - occ > 0) s->free_mask |= 1u << i;
  }
  return AGO_OK;
}

static const touched_t* find_touched(const bstate* s, int req) {
  for (int i = 0; i < s->n_touched; ++i)
    if (s->touched[i].req == req) return &s->touched[i];
  return NULL;
}

/* allowed_engines (scheduler.cpp:140-156) */
static uint32_t allowed_engines(const round_ctx* c, const bstate* s, int pi) {
  int r = c->pair_req[pi], a = c->pair_agent[pi];
  const touched_t* t = find_touched(s, r);
  uint32_t mask;
  if (!t) {
    mask = c->base_mask[pi];
  } else {
    mask = 0;
    const uint64_t* v = c->q->viable + c->q->viable_ptr[r];
    for (int k = 0; k < t->n_surv; ++k) {
      int mdl = digit_of(c->q->n, c->q->m, v[t->surv[k]], a);
      mask |= 1u << c->model_to_engine[mdl];
    }
  }
  return mask & s->free_mask;
}

/* extend_state (scheduler.cpp:158-206) */
static void extend_state(const round_ctx* c, const bstate* s, int pi,
                         int engine, bstate* next) {
  int r = c->pair_req[pi], a = c->pair_agent[pi];
  const int model = c->e->model[engine];
  const ago_queue* q = c->q;
  bs_copy(next, s);
  ago_triple t;
  t.request_index = r;
  t.request_id = q->ids[r];
  t.agent = a;
  t.model = model;
  t.pad = 0;
  next->triples[next->n_triples++] = t;
  int occ = ++next->occ[engine];
  if (occ >= c->e->slots[engine]) next->free_mask &= ~(1u << engine);
  next->util += c->e->weight[engine];

  const int64_t v0 = q->viable_ptr[r];
  const int64_t nv = q->viable_ptr[r + 1] - v0;
  const double initial = (double)nv;
  touched_t* entry = NULL;
  for (int i = 0; i < next->n_touched; ++i)
    if (next->touched[i].req == r) entry = &next->touched[i];
  if (!entry) {
    touched_t tt;
    tt.req = r;
    tt.surv = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nv + 1));
    tt.n_surv = 0;
    for (int64_t j = 0; j < nv; ++j)
      if (digit_of(q->n, q->m, q->viable[v0 + j], a) == model)
        tt.surv[tt.n_surv++] = (int32_t)j;
    next->flex_sum += (double)tt.n_surv / initial;
    ++next->flex_count;
    next->touched[next->n_touched++] = tt;
  } else {
    double before = (double)entry->n_surv / initial;
    int w = 0;
    for (int k = 0; k < entry->n_surv; ++k)
      if (digit_of(q->n, q->m, q->viable[v0 + entry->surv[k]], a) == model)
        entry->surv[w++] = entry->surv[k];
    entry->n_surv = w;
    next->flex_sum += (double)entry->n_surv / initial - before;
  }
}

/* score_assignment (scheduler.cpp:248-287) */
static int score_assignment(const round_ctx* c, const bstate* s, double* util,
                            double* flex) {
  const ago_queue* q = c->q;
  double u = 0.0;
  for (int i = 0; i < c->e->n_engines; ++i) {
    if (s->occ[i] < 0 || s->occ[i] > c->e->slots[i])
      return fail(AGO_VALIDATION, "occupancy outside engine capacity");
    u += s->occ[i] * c->e->weight[i];
  }
  double flex_sum = 0.0;
  int flex_count = 0;
  for (int qi = 0; qi < q->n_requests; ++qi) {
    int touched = 0, consistent = 0;
    for (int64_t j = q->viable_ptr[qi]; j < q->viable_ptr[qi + 1]; ++j) {
      int ok = 1;
      for (int k = 0; k < s->n_triples; ++k) {
        const ago_triple* t = &s->triples[k];
        if (t->request_index != qi) continue;
        touched = 1;
        if (digit_of(q->n, q->m, q->viable[j], t->agent) != t->model) {
          ok = 0;
          break;
        }
      }
      if (ok) ++consistent;
    }
    if (touched) {
      flex_sum += (double)consistent /
                  (double)(q->viable_ptr[qi + 1] - q->viable_ptr[qi]);
      ++flex_count;
    }
  }
  *util = u;
  *flex = flex_count > 0 ? flex_sum / flex_count : 1.0;
  return AGO_OK;
}

/* audit_round_fairness (scheduler.cpp:456-480): replay the assignment's
 * triples in pair order (a cursor that advances only on a match) from
 * initial_state; an unassigned pair with allowed engines is a violation. */
int ago_audit_round_fairness(const ago_queue* q, const ago_engines* e,
                             const ago_triple* triples, int n_triples,
                             uint64_t* viol_ids, int32_t* viol_agents, int cap,
                             int* n_viol) {
  round_ctx c;
  int rc = ctx_build(&c, q, e);
  if (rc) {
    ctx_free(&c);
    return rc;
  }
  bstate st;
  rc = initial_state(&c, &st, n_triples + 1);
  if (rc) {
    bs_free(&st);
    ctx_free(&c);
    return rc;
  }
  int pos = 0, nv = 0;
  for (int pi = 0; pi < c.n_pairs; ++pi) {
    int assigned = pos < n_triples && triples[pos].request_index == c.pair_req[pi] &&
                   triples[pos].agent == c.pair_agent[pi];
    if (assigned) {
      int mdl = triples[pos].model;
      int eng = mdl >= 0 && mdl < c.n_m2e ? c.model_to_engine[mdl] : -1;
      if (eng < 0) {
        bs_free(&st);
        ctx_free(&c);
        return fail(AGO_VALIDATION, "assignment names a model without an engine pool");
      }
      bstate next;
      extend_state(&c, &st, pi, eng, &next);
      bs_free(&st);
      st = next;
      ++pos;
    } else if (allowed_engines(&c, &st, pi) != 0) {
      if (nv < cap) {
        viol_ids[nv] = q->ids[c.pair_req[pi]];
        viol_agents[nv] = c.pair_agent[pi];
      }
      ++nv;
    }
  }
  *n_viol = nv;
  bs_free(&st);
  ctx_free(&c);
  return AGO_OK;
}

/* beam_schedule (scheduler.cpp:289-378) */
int ago_beam_schedule(const ago_queue* q, const ago_engines* e, int width,
                      ago_triple* triples, int triples_cap,
                      int32_t* occupancy_out, ago_assignment* out) {
  if (width < 1) return fail(AGO_VALIDATION, "beam width < 1");
  round_ctx c;
  int rc = ctx_build(&c, q, e);
  if (rc) {
    ctx_free(&c);
    return rc;
  }
  const int W = width;
  const int E = e->n_engines;
  int n_states = 1;
  bstate* states = (bstate*)calloc((size_t)W + 1, sizeof(bstate));
  rc = initial_state(&c, &states[0], c.n_pairs);
  if (rc) {
    bs_free(&states[0]);
    free(states);
    ctx_free(&c);
    return rc;
  }
  uint64_t explored = 1;
  bstate* children = (bstate*)calloc((size_t)W * (E + 1) + 1, sizeof(bstate));
  int* parent_of = (int*)malloc(sizeof(int) * ((size_t)W * (E + 1) + 1));
  char* used = (char*)malloc((size_t)W * (E + 1) + 1);
  uint32_t masks[64];

  for (int pi = 0; pi < c.n_pairs; ++pi) {
    int any_free = 0;
    for (int si = 0; si < n_states; ++si)
      if (states[si].free_mask) {
        any_free = 1;
        break;
      }
    if (!any_free) {
      int64_t remaining = (int64_t)(c.n_pairs - pi);
      for (int si = 0; si < n_states; ++si) states[si].skips += remaining;
      explored += (uint64_t)n_states * (uint64_t)remaining;
      break;
    }
    int any_cand = 0;
    for (int si = 0; si < n_states; ++si) {
      masks[si] = allowed_engines(&c, &states[si], pi);
      if (masks[si]) any_cand = 1;
    }
    if (!any_cand) {
      for (int si = 0; si < n_states; ++si) ++states[si].skips;
      explored += (uint64_t)n_states;
      continue;
    }
    int nc = 0;
    for (int si = 0; si < n_states; ++si) {
      if (masks[si] == 0) {
        bs_copy(&children[nc], &states[si]);
        ++children[nc].skips;
        parent_of[nc++] = si;
        continue;
      }
      for (int eng = 0; eng < E; ++eng) {
        if ((masks[si] >> eng) & 1u) {
          extend_state(&c, &states[si], pi, eng, &children[nc]);
          parent_of[nc++] = si;
        }
      }
    }
    explored += (uint64_t)nc;
    int picked[64], np = 0;
    memset(used, 0, (size_t)nc);
    for (int w = 1; w <= W; ++w) {
      int best = nc;
      for (int j = 0; j < nc; ++j) {
        if (used[j] || parent_of[j] >= w) continue;
        if (best == nc || state_better(&children[j], &children[best])) best = j;
      }
      if (best == nc) continue;
      used[best] = 1;
      picked[np++] = best;
    }
    for (int si = 0; si < n_states; ++si) bs_free(&states[si]);
    for (int k = 0; k < np; ++k) {
      states[k] = children[picked[k]];
      memset(&children[picked[k]], 0, sizeof(bstate));
    }
    for (int j = 0; j < nc; ++j) bs_free(&children[j]);
    n_states = np;
  }

  int best = 0;
  for (int si = 1; si < n_states; ++si)
    if (state_better(&states[si], &states[best])) best = si;
  const bstate* w = &states[best];
  /* finalize (scheduler.cpp:208-220) */
  out->n_triples = w->n_triples;
  out->skips = w->skips;
  out->states_explored = explored;
  rc = score_assignment(&c, w, &out->utilization, &out->flexibility);
  if (rc == AGO_OK) {
    if (w->n_triples > triples_cap) {
      rc = fail(AGO_VALIDATION, "triples_cap too small");
    } else {
      memcpy(triples, w->triples, sizeof(ago_triple) * (size_t)w->n_triples);
      for (int i = 0; i < E; ++i) occupancy_out[i] = w->occ[i];
    }
  }
  for (int si = 0; si < n_states; ++si) bs_free(&states[si]);
  free(states);
  free(children);
  free(parent_of);
  free(used);
  ctx_free(&c);
  return rc;
}

/* Request::mark_dispatched prefix pruning (request.cpp:70-86) */
int64_t ago_prefix_prune(int n, int m, uint64_t* viable, int64_t len, int agent,
                         int model) {
  int64_t w = 0;
  for (int64_t j = 0; j < len; ++j)
    if (digit_of(n, m, viable[j], agent) == model) viable[w++] = viable[j];
  return w ? w : -1;
}

/* ------------------------------------------------------------ snapshots */
/* generate_snapshot (snapshots.cpp:60-123) */
int ago_generate_snapshot(uint64_t seed, uint64_t index, ago_snapshot* s) {
  static const double kCosts[] = {1.0, 2.1, 4.4, 9.0};
  static const double kWeights[] = {3.0, 1.7, 0.9, 0.5};
  memset(s, 0, sizeof *s);
  stream_t st = {mix3(seed, 0xA6, index)};
  const int tiers = 3 + (int)st_below(&st, 2);
  s->m = tiers;
  for (int m = 0; m < tiers; ++m) {
    s->cost[m] = kCosts[m];
    s->weight[m] = kWeights[m];
  }
  /* make_graph (snapshots.cpp:31-49) */
  int32_t edges[16];
  int ne, n;
  if (st_bernoulli(&st, 0.6)) {
    n = 4;
    int32_t e[8] = {0, 1, 0, 2, 1, 3, 2, 3};
    memcpy(edges, e, sizeof e);
    ne = 4;
  } else {
    n = 1 + (int)st_below(&st, 3);
    ne = 0;
    for (int i = 1; i < n; ++i) {
      edges[2 * ne] = i - 1;
      edges[2 * ne + 1] = i;
      ++ne;
    }
  }
  s->n = n;
  uint64_t pred[64], succ[64];
  int rc = ago_graph_build(n, ne, edges, s->decl, s->depth, pred, succ);
  if (rc) return rc;
  s->n_engines = tiers;
  for (int m = 0; m < tiers; ++m) {
    s->eng_model[m] = m;
    s->eng_slots[m] = 2 + (int)st_below(&st, 3);
    s->eng_weight[m] = kWeights[m];
    s->eng_occ[m] = (int)st_below(&st, (uint64_t)(s->eng_slots[m] / 2) + 1);
  }
  ago_gen_params gp = {0.2, 0.55, 0.25, 0.5, 0.0};
  int count = tiers == 4 ? 2 + (int)st_below(&st, 2) : 2 + (int)st_below(&st, 4);
  s->n_requests = count;
  const uint64_t size = space_size(n, tiers);
  int64_t vp = 0;
  for (int i = 0; i < count; ++i) {
    uint8_t seeds[16 * 64];
    uint64_t removed[8];
    int ns, nr, tier;
    rc = ago_gen_truth(n, tiers, &gp, seed, index * 64 + (uint64_t)i, 0xA6,
                       seeds, 16, &ns, removed, 8, &nr, &tier);
    if (rc) return rc;
    s->ids[i] = (uint64_t)i;
    s->arrival[i] = (double)i;
    s->viable_ptr[i] = vp;
    uint64_t* v = s->viable + vp;
    int64_t len = 0;
    for (uint64_t k = 0; k < size; ++k)
      if (ago_contains(n, tiers, seeds, ns, removed, nr, k)) v[len++] = k;
    uint8_t* stg = s->stages + i * n;
    for (int p = 0; p < n; ++p) stg[p] = pred[p] ? AGO_STAGE_PENDING : AGO_STAGE_READY;
    double advance = n == 4 ? 0.7 : 0.45;
    int progressed = 0;
    while (progressed + 1 < n) {
      int ready[8], nrd = 0;
      for (int p = 0; p < n; ++p)
        if (stg[p] == AGO_STAGE_READY) ready[nrd++] = p;
      if (nrd == 0 || !st_bernoulli(&st, advance)) break;
      int agent = ready[st_below(&st, (uint64_t)nrd)];
      int cands[8], ncd = 0;
      uint32_t seen = 0;
      for (int64_t j = 0; j < len; ++j) seen |= 1u << digit_of(n, tiers, v[j], agent);
      for (int mm = 0; mm < tiers; ++mm)
        if ((seen >> mm) & 1) cands[ncd++] = mm;
      int model = cands[st_below(&st, (uint64_t)ncd)];
      len = ago_prefix_prune(n, tiers, v, len, agent, model);
      stg[agent] = AGO_STAGE_DONE; /* mark_dispatched + mark_complete */
      for (int sc = 0; sc < n; ++sc) {
        if (!((succ[agent] >> sc) & 1) || stg[sc] != AGO_STAGE_PENDING) continue;
        int all_done = 1;
        for (int pp = 0; pp < n; ++pp)
          if (((pred[sc] >> pp) & 1) && stg[pp] != AGO_STAGE_DONE) all_done = 0;
        if (all_done) stg[sc] = AGO_STAGE_READY;
      }
      ++progressed;
      advance *= 0.35;
    }
    vp += len;
  }
  s->viable_ptr[count] = vp;
  return AGO_OK;
}
