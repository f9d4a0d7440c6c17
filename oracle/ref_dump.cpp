// TEST INFRASTRUCTURE ONLY.
//
// ref_dump: links the UNMODIFIED reference library (oracle/Makefile builds
// /root/reference/proj/src/*.cpp into oracle/_ref/libaragog_ref.a) and writes
// golden vectors for the two hot paths as JSON into the directory given on
// the command line (tests/golden/ by default via oracle/make_golden.sh).
//
// Everything here calls the reference's own public API; nothing is
// re-implemented.  The fixtures pin the C restatement (oracle/aragog_oracle.c)
// and are the first parity gate for the CUDA path.

#include <cmath>
#include <cstdio>
#include <fstream>
#include <limits>
#include <string>
#include <vector>

#include <json.hpp>

#include "aragog/accuracy.h"
#include "aragog/engine.h"
#include "aragog/predictor.h"
#include "aragog/request.h"
#include "aragog/rng.h"
#include "aragog/router.h"
#include "aragog/scheduler.h"
#include "aragog/snapshots.h"
#include "aragog/workflow.h"
#include "aragog/workload.h"

using json = nlohmann::json;
using namespace aragog;

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

WorkflowGraph chain_graph(int n) {
  std::vector<std::string> agents;
  std::vector<std::pair<std::string, std::string>> edges;
  for (int i = 0; i < n; ++i) {
    agents.push_back("a" + std::to_string(i));
    if (i > 0) edges.emplace_back(agents[i - 1], agents[i]);
  }
  return WorkflowGraph::build(agents, edges);
}

WorkflowGraph diamond_graph() {
  return WorkflowGraph::build({"a", "b", "c", "d"},
                              {{"a", "b"}, {"a", "c"}, {"b", "d"}, {"c", "d"}});
}

// cost x1.5 and weight /1.5 per tier
ModelCatalog geometric_catalog(int m) {
  std::vector<ModelSpec> models;
  double cost = 1.0, w = 8.0;
  for (int i = 0; i < m; ++i) {
    models.push_back({"m" + std::to_string(i), cost, w});
    cost *= 1.5;
    w /= 1.5;
  }
  return ModelCatalog(models);
}

json digits(const Configuration& c) { return c.models; }

std::string hex_bitmap(const std::vector<std::uint32_t>& words) {
  static const char* hx = "0123456789abcdef";
  std::string s;
  s.reserve(words.size() * 8);
  for (std::uint32_t w : words)
    for (int k = 7; k >= 0; --k) s.push_back(hx[(w >> (4 * k)) & 15]);
  return s;
}

json graph_json(const WorkflowGraph& g) {
  json j;
  std::vector<int> decl, depth;
  for (int p = 0; p < g.num_agents(); ++p) {
    decl.push_back(g.declaration_index(p));
    depth.push_back(g.depth(p));
  }
  j["decl"] = decl;
  j["depth"] = depth;
  return j;
}

void write(const std::string& dir, const std::string& name, const json& j) {
  std::ofstream f(dir + "/" + name);
  f << j.dump() << "\n";
  std::fprintf(stderr, "wrote %s/%s\n", dir.c_str(), name.c_str());
}

// ---------------------------------------------------------------- rng
json dump_rng() {
  json out = json::array();
  rng::Stream st(12345);
  for (int i = 0; i < 16; ++i) {
    std::uint64_t a = st.next_u64(), b = st.next_u64(), c = st.next_u64();
    out.push_back({{"words", {a, b, c}},
                   {"mix1", rng::mix({a})},
                   {"mix2", rng::mix({a, b})},
                   {"mix3", rng::mix({a, b, c})}});
  }
  return out;
}

// -------------------------------------------------------------- graph
json dump_graphs() {
  json out = json::array();
  auto add = [&](std::vector<std::string> agents,
                 std::vector<std::pair<std::string, std::string>> edges) {
    WorkflowGraph g = WorkflowGraph::build(agents, edges);
    std::vector<std::pair<int, int>> e;
    for (auto& [f, t] : edges) {
      int fi = -1, ti = -1;
      for (std::size_t i = 0; i < agents.size(); ++i) {
        if (agents[i] == f) fi = static_cast<int>(i);
        if (agents[i] == t) ti = static_cast<int>(i);
      }
      e.emplace_back(fi, ti);
    }
    json j = graph_json(g);
    j["n"] = agents.size();
    j["edges"] = e;
    out.push_back(j);
  };
  add({"x", "y", "z"}, {{"z", "x"}});
  add({"a", "b", "c", "d"}, {{"a", "b"}, {"a", "c"}, {"b", "d"}, {"c", "d"}});
  add({"plan", "s1", "s2", "s3", "s4", "agg"},
      {{"plan", "s1"}, {"plan", "s2"}, {"plan", "s3"}, {"plan", "s4"},
       {"s1", "agg"}, {"s2", "agg"}, {"s3", "agg"}, {"s4", "agg"}});
  rng::Stream st(99);
  for (int t = 0; t < 20; ++t) {
    int n = 2 + static_cast<int>(st.next_below(7));
    std::vector<std::string> agents;
    for (int i = 0; i < n; ++i) agents.push_back("v" + std::to_string(i));
    // random DAG over a random permutation so declaration order != topo order
    std::vector<int> perm(n);
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int i = n - 1; i > 0; --i) std::swap(perm[i], perm[st.next_below(i + 1)]);
    std::vector<std::pair<std::string, std::string>> edges;
    for (int i = 0; i < n; ++i)
      for (int k = i + 1; k < n; ++k)
        if (st.next_bernoulli(0.3)) edges.emplace_back(agents[perm[i]], agents[perm[k]]);
    add(agents, edges);
  }
  return out;
}

// -------------------------------------------------------------- truth
json dump_truth() {
  json out = json::array();
  struct P {
    double e, m, h, base, viol;
  };
  const P params[] = {{0.6, 0.3, 0.1, 0.5, 0.0},
                      {0.95, 0.0, 0.05, 0.8, 0.0},
                      {0.2, 0.55, 0.25, 0.5, 0.0},
                      {0.6, 0.3, 0.1, 0.5, 0.05},
                      {1.0, 0.0, 0.0, 0.5, 0.0}};
  const int shapes[][2] = {{1, 2}, {1, 3}, {2, 2}, {2, 3}, {3, 3}, {3, 4},
                           {4, 3}, {5, 8}, {8, 12}, {6, 4}};
  for (auto& sh : shapes) {
    WorkflowGraph g = chain_graph(sh[0]);
    ModelCatalog cat = geometric_catalog(sh[1]);
    ConfigSpace space(g, cat);
    for (int pi = 0; pi < 5; ++pi) {
      AccuracyGenParams ap;
      ap.p_easy = params[pi].e;
      ap.p_medium = params[pi].m;
      ap.p_hard = params[pi].h;
      ap.easy_base_prob = params[pi].base;
      ap.violation_rate = params[pi].viol;
      if (ap.violation_rate > 0 && space.size() > kEnumerableLimit) continue;
      for (std::uint64_t seed : {1ULL, 23ULL}) {
        for (RequestId id = 0; id < 24; ++id) {
          AccurateSet s = generate_accurate_set(space, ap, seed, id);
          json seeds = json::array(), removed = json::array();
          for (auto& c : s.seeds) seeds.push_back(digits(c));
          for (auto& c : s.removed) removed.push_back(space.index_of(c));
          out.push_back({{"n", sh[0]}, {"m", sh[1]}, {"params", {ap.p_easy, ap.p_medium, ap.p_hard, ap.easy_base_prob, ap.violation_rate}},
                         {"seed", seed}, {"id", id}, {"salt", rng::kTableSalt},
                         {"tier", static_cast<int>(s.tier)}, {"seeds", seeds},
                         {"removed", removed}});
        }
      }
    }
  }
  return out;
}

// ------------------------------------------------------------- router
// Full-space verdict bitmaps via RouterBackend::evaluate (the enumerate-mode
// oracle, tests/acceptance/criteria.cpp:93-101 pattern).
json dump_router() {
  json out = json::array();
  struct Case {
    int n, m, count;
    double fp, fn;
    std::uint64_t nseed;
    double viol;
  };
  const Case cases[] = {{2, 3, 40, 0.1, 0.3, 77, 0.0},  {3, 3, 40, 0.0, 0.3, 91, 0.0},
                        {3, 4, 30, 0.05, 0.2, 5, 0.05}, {4, 3, 30, 0.0, 0.0, 5, 0.0},
                        {5, 8, 12, 0.0, 0.3, 7, 0.0},   {5, 8, 6, 0.1, 0.3, 11, 0.0},
                        {1, 2, 8, 0.5, 0.5, 3, 0.0},    {6, 4, 8, 0.02, 0.4, 13, 0.0}};
  for (const Case& cs : cases) {
    WorkflowGraph g = chain_graph(cs.n);
    ModelCatalog cat = geometric_catalog(cs.m);
    ConfigSpace space(g, cat);
    AccuracyGenParams ap;
    ap.violation_rate = cs.viol;
    AccuracyTable table = generate_accuracy_table(space, ap, cs.count, 1);
    OracleRouter oracle(table, 0.002);
    NoisyRouter noisy(oracle, cs.fp, cs.fn, cs.nseed);
    for (RequestId id = 0; id < static_cast<RequestId>(cs.count); ++id) {
      const std::uint64_t S = space.size();
      std::vector<std::uint32_t> wo((S + 31) / 32, 0), wn((S + 31) / 32, 0);
      std::uint64_t co = 0, cn = 0;
      for (std::uint64_t i = 0; i < S; ++i) {
        Configuration c = space.at_index(i);
        if (oracle.evaluate(id, c)) {
          wo[i >> 5] |= 1u << (i & 31);
          ++co;
        }
        if (noisy.evaluate(id, c)) {
          wn[i >> 5] |= 1u << (i & 31);
          ++cn;
        }
      }
      const AccurateSet& s = table.at(id);
      json seeds = json::array(), removed = json::array();
      for (auto& c : s.seeds) seeds.push_back(digits(c));
      for (auto& c : s.removed) removed.push_back(space.index_of(c));
      out.push_back({{"n", cs.n}, {"m", cs.m}, {"id", id}, {"fp", cs.fp},
                     {"fn", cs.fn}, {"noise_seed", cs.nseed}, {"seeds", seeds},
                     {"removed", removed}, {"oracle_count", co},
                     {"noisy_count", cn}, {"oracle_bitmap", hex_bitmap(wo)},
                     {"noisy_bitmap", hex_bitmap(wn)}});
    }
  }
  return out;
}

// ------------------------------------------------------------- chains
json dump_chains() {
  json out = json::array();
  struct Case {
    int n, m, cap;
    std::uint64_t limit;
  };
  const Case cases[] = {{1, 2, 0, 4096}, {2, 2, 0, 4096}, {2, 3, 0, 4096},
                        {3, 3, 0, 4096}, {3, 4, 0, 4096}, {4, 3, 0, 4096},
                        {2, 3, 3, 0},    {5, 8, 0, 4096}, {8, 12, 0, 4096},
                        {6, 4, 0, 4096}, {5, 5, 16, 4096}};
  for (const Case& cs : cases) {
    WorkflowGraph g = chain_graph(cs.n);
    ModelCatalog cat = geometric_catalog(cs.m);
    ConfigSpace space(g, cat);
    ChainPlan plan = build_chains(space, cs.cap, cs.limit);
    json chains = json::array();
    for (auto& ch : plan.chains) {
      std::vector<std::uint64_t> idx;
      for (auto& c : ch) idx.push_back(space.index_of(c));
      chains.push_back(idx);
    }
    out.push_back({{"n", cs.n}, {"m", cs.m}, {"cap", cs.cap}, {"limit", cs.limit},
                   {"exhaustive", plan.exhaustive}, {"chains", chains}});
  }
  return out;
}

// ------------------------------------------------------------ predict
json dump_predict() {
  json out = json::array();
  struct Case {
    int n, m, count;
    int noisy;
    double fp, fn;
    double latency;
    double budget;
    double p_easy, p_medium, p_hard, base, viol;
  };
  const Case cases[] = {
      {3, 3, 60, 0, 0, 0, 0.002, kInf, 0.95, 0.0, 0.05, 0.8, 0.0},
      {3, 3, 60, 0, 0, 0, 0.002, 0.012, 0.95, 0.0, 0.05, 0.8, 0.0},
      {4, 3, 60, 0, 0, 0, 0.002, 0.15, 0.9, 0.0, 0.1, 0.6, 0.0},
      {3, 4, 60, 1, 0.0, 0.3, 0.002, kInf, 0.6, 0.3, 0.1, 0.5, 0.0},
      {3, 4, 60, 1, 0.1, 0.3, 0.001, 0.01, 0.6, 0.3, 0.1, 0.5, 0.05},
      {2, 3, 60, 0, 0, 0, 1.0, 3.0, 1.0, 0.0, 0.0, 0.5, 0.0},
      {3, 3, 40, 0, 0, 0, 0.002, 0.0, 0.6, 0.3, 0.1, 0.5, 0.0},
      {5, 8, 120, 0, 0, 0, 0.002, kInf, 0.6, 0.3, 0.1, 0.5, 0.0},
      {5, 8, 60, 1, 0.0, 0.3, 0.002, kInf, 0.6, 0.3, 0.1, 0.5, 0.0},
      {5, 8, 60, 0, 0, 0, 0.002, 0.03, 0.6, 0.3, 0.1, 0.5, 0.0},
      {8, 12, 30, 1, 0.05, 0.3, 0.002, kInf, 0.6, 0.3, 0.1, 0.5, 0.0},
      {6, 4, 40, 0, 0, 0, 0.001, kInf, 0.6, 0.3, 0.1, 0.5, 0.0},
  };
  int case_id = 0;
  for (const Case& cs : cases) {
    WorkflowGraph g = chain_graph(cs.n);
    ModelCatalog cat = geometric_catalog(cs.m);
    ConfigSpace space(g, cat);
    AccuracyGenParams ap;
    ap.p_easy = cs.p_easy;
    ap.p_medium = cs.p_medium;
    ap.p_hard = cs.p_hard;
    ap.easy_base_prob = cs.base;
    ap.violation_rate = cs.viol;
    AccuracyTable table = generate_accuracy_table(space, ap, cs.count, 5 + case_id);
    OracleRouter oracle(table, cs.latency);
    NoisyRouter noisy(oracle, cs.fp, cs.fn, 1000 + case_id);
    const RouterBackend& router =
        cs.noisy ? static_cast<const RouterBackend&>(noisy) : oracle;
    ConfigPredictor predictor(space, router);
    json reqs = json::array();
    for (RequestId id = 0; id < static_cast<RequestId>(cs.count); ++id) {
      PredictionResult r = predictor.predict(id, cs.budget);
      std::vector<std::uint64_t> v;
      for (auto& c : r.viable.configs) v.push_back(space.index_of(c));
      const AccurateSet& s = table.at(id);
      json seeds = json::array(), removed = json::array();
      for (auto& c : s.seeds) seeds.push_back(digits(c));
      for (auto& c : s.removed) removed.push_back(space.index_of(c));
      reqs.push_back({{"id", id}, {"seeds", seeds}, {"removed", removed},
                      {"viable", v}, {"search_evals", r.search_evals},
                      {"verify_evals", r.verify_evals},
                      {"router_time", r.router_time}, {"truncated", r.truncated}});
    }
    json costs = json::array();
    for (int i = 0; i < cs.m; ++i) costs.push_back(cat.at(i).cost);
    out.push_back({{"n", cs.n}, {"m", cs.m}, {"noisy", cs.noisy}, {"fp", cs.fp},
                   {"fn", cs.fn}, {"noise_seed", 1000 + case_id},
                   {"latency", cs.latency},
                   {"budget", std::isinf(cs.budget) ? -1.0 : cs.budget},
                   {"cost", costs}, {"requests", reqs}});
    ++case_id;
  }
  return out;
}

// --------------------------------------------------------------- beam
json queue_json(const std::vector<const Request*>& queue,
                const std::vector<EngineState>& engines, const ConfigSpace& space) {
  json reqs = json::array();
  for (const Request* r : queue) {
    std::vector<std::uint64_t> v;
    for (auto& c : r->viable) v.push_back(space.index_of(c));
    std::vector<int> stages;
    for (auto s : r->stages) stages.push_back(static_cast<int>(s));
    reqs.push_back({{"id", r->id}, {"arrival", r->arrival}, {"stages", stages},
                    {"viable", v}});
  }
  json eng = json::array();
  for (auto& e : engines)
    eng.push_back({{"model", e.model}, {"slots", e.slots}, {"weight", e.weight},
                   {"occupancy", e.occupancy()}});
  return {{"requests", reqs}, {"engines", eng}};
}

json assignment_json(const Assignment& a) {
  json tr = json::array();
  for (auto& t : a.triples) tr.push_back({t.request_index, t.request, t.agent, t.model});
  return {{"triples", tr},           {"occupancy", a.occupancy},
          {"utilization", a.utilization}, {"flexibility", a.flexibility},
          {"skips", a.skips},        {"states_explored", a.states_explored}};
}

json dump_snapshots(std::uint64_t seed, int count) {
  json out = json::array();
  for (int i = 0; i < count; ++i) {
    auto snap = generate_snapshot(seed, static_cast<std::uint64_t>(i));
    ConfigSpace space(snap->graph, snap->catalog);
    auto queue = snap->queue();
    json j = queue_json(queue, snap->engines, space);
    j["seed"] = seed;
    j["index"] = i;
    j["n"] = snap->graph.num_agents();
    j["m"] = snap->catalog.size();
    j["graph"] = graph_json(snap->graph);
    json res = json::object();
    for (int w : {1, 2, 4, 8})
      res[std::to_string(w)] =
          assignment_json(beam_schedule(queue, snap->engines, SchedulerParams{w}));
    j["beam"] = res;
    out.push_back(j);
  }
  return out;
}

// Larger synthetic rounds: requests with predictor or exhaustive viable sets,
// random progress, partially busy pools, shuffled container order.
json dump_rounds() {
  json out = json::array();
  struct Case {
    int kind;  // 0 chain, 1 diamond
    int n, m, requests;
    int exhaustive;
    std::uint64_t seed;
  };
  const Case cases[] = {{0, 3, 3, 40, 1, 1},  {0, 3, 4, 60, 1, 2}, {1, 4, 3, 30, 1, 3},
                        {1, 4, 4, 25, 0, 4},  {0, 5, 8, 80, 0, 5}, {0, 3, 3, 120, 0, 6},
                        {1, 4, 3, 60, 1, 7},  {0, 2, 4, 50, 1, 8}, {1, 4, 4, 40, 1, 9},
                        {0, 4, 3, 200, 1, 10}};
  for (const Case& cs : cases) {
    WorkflowGraph g = cs.kind ? diamond_graph() : chain_graph(cs.n);
    ModelCatalog cat = geometric_catalog(cs.m);
    ConfigSpace space(g, cat);
    AccuracyGenParams ap;
    AccuracyTable table = generate_accuracy_table(space, ap, cs.requests, cs.seed);
    OracleRouter oracle(table, 0.001);
    ConfigPredictor predictor(space, oracle);
    rng::Stream st(rng::mix({cs.seed, 0xBEEF}));
    std::vector<Request> reqs;
    reqs.reserve(cs.requests);
    for (int i = 0; i < cs.requests; ++i) {
      std::vector<Configuration> viable;
      if (cs.exhaustive) {
        for (std::uint64_t k = 0; k < space.size(); ++k) {
          Configuration c = space.at_index(k);
          if (table.accurate(i, c)) viable.push_back(c);
        }
      } else {
        viable = predictor.predict(i, kInf).viable.configs;
      }
      // equal arrivals in groups of three exercise the id tie-break
      Request r = Request::make(static_cast<RequestId>(1000 - i),
                                static_cast<double>(i / 3) * 0.25, g, viable);
      int steps = static_cast<int>(st.next_below(static_cast<std::uint64_t>(cs.n)));
      for (int s = 0; s < steps; ++s) {
        std::vector<int> ready = r.ready_agents();
        if (ready.empty()) break;
        int agent = ready[st.next_below(ready.size())];
        std::vector<int> cands = r.candidate_models(agent);
        int model = cands[st.next_below(cands.size())];
        r.mark_dispatched(agent, model, 0.0);
        if (st.next_bernoulli(0.8)) r.mark_complete(agent, 0.0);
      }
      reqs.push_back(std::move(r));
    }
    std::vector<const Request*> queue;
    for (auto& r : reqs)
      if (!r.ready_agents().empty()) queue.push_back(&r);
    for (std::size_t i = queue.size(); i > 1; --i)
      std::swap(queue[i - 1], queue[st.next_below(i)]);
    for (int variant = 0; variant < 3; ++variant) {
      std::vector<EngineState> engines;
      for (int mm = 0; mm < cs.m; ++mm) {
        EngineState e;
        e.model = mm;
        e.slots = 1 + static_cast<int>(st.next_below(variant == 2 ? 16 : 4));
        e.weight = cat.at(mm).slot_throughput;
        int busy = static_cast<int>(st.next_below(static_cast<std::uint64_t>(e.slots) + 1));
        for (int b = 0; b < busy; ++b) e.in_flight.push_back({999999, 0, 1e18});
        engines.push_back(std::move(e));
      }
      json j = queue_json(queue, engines, space);
      j["n"] = g.num_agents();
      j["m"] = cs.m;
      j["graph"] = graph_json(g);
      j["case"] = {cs.kind, cs.n, cs.m, cs.requests, cs.exhaustive, cs.seed, variant};
      json res = json::object();
      for (int w : {1, 2, 4, 8}) {
        Assignment a = beam_schedule(queue, engines, SchedulerParams{w});
        json aj = assignment_json(a);
        aj["fairness_violations"] = audit_round_fairness(queue, engines, a).size();
        res[std::to_string(w)] = aj;
      }
      j["beam"] = res;
      // audit_round_fairness of doctored width-4 assignments (the
      // scheduler_test.cpp:211-229 pattern): dropped, truncated, reordered
      {
        Assignment a = beam_schedule(queue, engines, SchedulerParams{4});
        const std::size_t T = a.triples.size();
        std::vector<std::vector<AssignmentTriple>> docs;
        if (T >= 1) {
          docs.push_back(std::vector<AssignmentTriple>(a.triples.begin() + 1, a.triples.end()));
          auto mid = a.triples;
          mid.erase(mid.begin() + (long)(T / 2));
          docs.push_back(mid);
        }
        docs.push_back(std::vector<AssignmentTriple>(a.triples.begin(), a.triples.begin() + (long)(T / 2)));
        if (T >= 2) {
          auto sw = a.triples;
          std::swap(sw[0], sw[1]);
          docs.push_back(sw);
        }
        docs.push_back({});
        json aud = json::array();
        for (const auto& d : docs) {
          Assignment x = a;
          x.triples = d;
          json tj = json::array();
          for (const auto& t : d)
            tj.push_back({t.request_index, t.request, t.agent, t.model});
          json vj = json::array();
          for (const FairnessViolation& v : audit_round_fairness(queue, engines, x))
            vj.push_back({v.request, v.agent});
          aud.push_back({{"triples", tj}, {"violations", vj}});
        }
        j["audit"] = aud;
      }
      out.push_back(j);
    }
  }
  return out;
}

// ----------------------------------------------------------- workload
json dump_workload() {
  json out = json::array();
  rng::Stream st(4242);
  const int shapes[][2] = {{1, 2}, {2, 2}, {2, 3}, {3, 3}, {3, 4}, {4, 3}, {5, 5}};
  for (auto& sh : shapes) {
    WorkflowGraph g = chain_graph(sh[0]);
    ModelCatalog cat = geometric_catalog(sh[1]);
    ConfigSpace space(g, cat);
    std::vector<ServiceTimeModel::Params> sp;
    for (int mm = 0; mm < sh[1]; ++mm)
      sp.push_back({-0.5 + 0.4 * mm, 0.25, 0.05});
    ServiceTimeModel service(sp);
    AccuracyGenParams ap;
    AccuracyTable table = generate_accuracy_table(space, ap, 20, 17);
    for (RequestId id = 0; id < 20; ++id) {
      RuntimeCostContext ctx;
      ctx.service = &service;
      for (int mm = 0; mm < sh[1]; ++mm) {
        ctx.slots.push_back(1 + static_cast<int>(st.next_below(8)));
        ctx.occupancy.push_back(static_cast<int>(st.next_below(ctx.slots.back() + 1)));
        // small loads so estimate ties happen and exercise the cost tie-break
        ctx.queued_ahead.push_back(static_cast<int>(st.next_below(id % 2 ? 3 : 40)));
      }
      Configuration pick_s = select_per_input_config(table.at(id), space,
                                                     PolicyKind::kPerInputStatic);
      Configuration pick_r = select_per_input_config(
          table.at(id), space, PolicyKind::kPerInputRuntimeCost, &ctx);
      std::vector<std::uint64_t> members;
      for (auto& c : enumerate_members(table.at(id), space))
        members.push_back(space.index_of(c));
      std::vector<double> means;
      for (int mm = 0; mm < sh[1]; ++mm) means.push_back(service.mean(mm));
      json costs = json::array();
      for (int i = 0; i < sh[1]; ++i) costs.push_back(cat.at(i).cost);
      out.push_back({{"n", sh[0]}, {"m", sh[1]}, {"cost", costs},
                     {"members", members}, {"occupancy", ctx.occupancy},
                     {"queued_ahead", ctx.queued_ahead}, {"slots", ctx.slots},
                     {"mean", means}, {"static_pick", space.index_of(pick_s)},
                     {"runtime_pick", space.index_of(pick_r)},
                     {"runtime_est", estimate_completion(ctx, pick_r)}});
    }
  }
  return out;
}

// ----------------------------------------------------------- per-workflow
// select_per_workflow_config (workload.cpp:99-127) over generated samples,
// including violation-injected (removed-list) sets on small spaces.
json dump_workflow() {
  json out = json::array();
  const int shapes[][2] = {{1, 2}, {2, 3}, {3, 3}, {3, 4}, {4, 3}, {5, 4}, {6, 4}};
  const std::size_t counts[] = {1, 7, 40};
  const double tols[] = {0.0, 0.1, 0.35};
  const double viols[] = {0.0, 0.05};
  std::uint64_t seed = 900;
  for (auto& sh : shapes) {
    WorkflowGraph g = chain_graph(sh[0]);
    ModelCatalog cat = geometric_catalog(sh[1]);
    ConfigSpace space(g, cat);
    json costs = json::array();
    for (int i = 0; i < sh[1]; ++i) costs.push_back(cat.at(i).cost);
    for (double v : viols)
      for (std::size_t cnt : counts) {
        AccuracyGenParams ap;
        ap.violation_rate = v;
        ++seed;
        AccuracyTable table = generate_accuracy_table(space, ap, cnt, seed);
        std::vector<AccurateSet> sample;
        for (RequestId id = 0; id < cnt; ++id) sample.push_back(table.at(id));
        for (double tol : tols) {
          Configuration pick = select_per_workflow_config(sample, space, tol);
          out.push_back({{"n", sh[0]}, {"m", sh[1]}, {"cost", costs}, {"seed", seed},
                         {"count", cnt}, {"violation_rate", v}, {"tolerance", tol},
                         {"pick", space.index_of(pick)}});
        }
      }
  }
  return out;
}

}  // namespace

int main(int argc, char** argv) {
  std::string dir = argc > 1 ? argv[1] : ".";
  if (argc > 2 && std::string(argv[2]) == "workflow") {
    write(dir, "workflow.json", dump_workflow());
    return 0;
  }
  write(dir, "workflow.json", dump_workflow());
  write(dir, "rng.json", dump_rng());
  write(dir, "graph.json", dump_graphs());
  write(dir, "truth.json", dump_truth());
  write(dir, "router.json", dump_router());
  write(dir, "chains.json", dump_chains());
  write(dir, "predict.json", dump_predict());
  json snaps = json::object();
  snaps["7"] = dump_snapshots(7, 200);
  snaps["42"] = dump_snapshots(42, 300);
  write(dir, "snapshots.json", snaps);
  write(dir, "rounds.json", dump_rounds());
  write(dir, "workload.json", dump_workload());
  return 0;
}
