// TEST / BASELINE INFRASTRUCTURE ONLY.
//
// ref_bench: times the UNMODIFIED reference CPU implementation of the hot
// paths (linked from oracle/_ref/libaragog_ref.a) on the host's cores.  It is
// the `bench.py --impl reference` arm and the `cpu_baseline` leg; it prints
// one JSON object on stdout.
//
//   ref_bench route  <n> <m> <requests> <router:oracle|noisy> <threads> <seed>
//       enumerate-mode routing: for each request, every canonical index is
//       decoded with ConfigSpace::at_index and scored with
//       RouterBackend::evaluate; members are appended in canonical order
//       (the enumerate_members pattern, accuracy.cpp:227-238, without the
//       4096 guard; criteria.cpp:93-101).  Requests are spread over threads
//       with the reference's own parallel_for (metrics.cpp:393-423).
//   ref_bench predict <n> <m> <requests> <router> <threads> <seed>
//       chain-mode routing via ConfigPredictor::predict(id, inf).
//   ref_bench sched <requests> <beam> <rounds> <seed> <exhaustive:0|1>
//       config-3 rounds: beam_schedule p50/p99 on one core (the scheduler is
//       serial per round).
//   ref_bench select <n> <m> <requests> <threads> <seed> <sets:exhaustive|viable>
//       the per-stage re-cost + argmin: select_per_input_config(set, space,
//       kPerInputRuntimeCost, &ctx) (workload.cpp:149-176) for every request,
//       spread over threads with parallel_for.  The member lists are built
//       before the timed region (the accurate set through at_index +
//       AccurateSet::contains, or the predictor's ViableSet); timed per
//       request: the sort by (static_cost, models) of members_by_cost
//       (workload.cpp:32-42, restated: it is in an anonymous namespace) and
//       the strict '<' scan over estimate_completion (workload.cpp:129-147,
//       165-175, called as is).  Load context: occupancy 4, queued_ahead
//       i % 3, 8 slots, ServiceTimeModel{mu -0.3 + 0.35 i, sigma 0.25,
//       floor 0.05} per tier i.  Prints the digest of (chosen index, estimate
//       bits) in request order.

#include <algorithm>
#include <array>
#include <numeric>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "aragog/accuracy.h"
#include "aragog/engine.h"
#include "aragog/metrics.h"
#include "aragog/predictor.h"
#include "aragog/request.h"
#include "aragog/rng.h"
#include "aragog/router.h"
#include "aragog/scheduler.h"
#include "aragog/workflow.h"

using namespace aragog;
using Clock = std::chrono::steady_clock;

namespace {

WorkflowGraph chain_graph(int n) {
  std::vector<std::string> agents;
  std::vector<std::pair<std::string, std::string>> edges;
  for (int i = 0; i < n; ++i) {
    agents.push_back("a" + std::to_string(i));
    if (i > 0) edges.emplace_back(agents[i - 1], agents[i]);
  }
  return WorkflowGraph::build(agents, edges);
}

// config 2 catalog: cost x1.5, weight /1.5 per tier
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

double secs(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

int run_route(int n, int m, std::size_t requests, bool noisy, int threads,
              std::uint64_t seed, bool chain_mode) {
  WorkflowGraph g = chain_graph(n);
  ModelCatalog cat = geometric_catalog(m);
  ConfigSpace space(g, cat);
  AccuracyGenParams ap;  // 0.6 / 0.3 / 0.1, base 0.5, no violations
  AccuracyTable table = generate_accuracy_table(space, ap, requests, seed);
  OracleRouter oracle(table, 0.002);
  NoisyRouter nr(oracle, 0.0, 0.3, 7);
  const RouterBackend& router = noisy ? static_cast<const RouterBackend&>(nr) : oracle;
  std::vector<std::uint64_t> counts(requests, 0);
  // per request: sum and sum of squares of the member indices (the digest)
  std::vector<std::uint64_t> isum(requests, 0), isq(requests, 0);
  std::atomic<std::uint64_t> evals{0};
  const std::uint64_t S = space.size();

  auto t0 = Clock::now();
  if (!chain_mode) {
    parallel_for(requests, threads, [&](std::size_t id) {
      std::vector<Configuration> members;
      std::uint64_t sm = 0, sq = 0;
      for (std::uint64_t i = 0; i < S; ++i) {
        Configuration c = space.at_index(i);
        if (router.evaluate(id, c)) {
          members.push_back(std::move(c));
          sm += i;
          sq += i * i;
        }
      }
      counts[id] = members.size();
      isum[id] = sm;
      isq[id] = sq;
    });
  } else {
    ConfigPredictor predictor(space, router);
    parallel_for(requests, threads, [&](std::size_t id) {
      PredictionResult r =
          predictor.predict(id, std::numeric_limits<double>::infinity());
      counts[id] = r.viable.configs.size();
      evals += static_cast<std::uint64_t>(r.router_eval_count());
    });
  }
  auto t1 = Clock::now();
  double dt = secs(t0, t1);
  std::uint64_t members = 0;
  for (auto c : counts) members += c;
  if (!chain_mode) {
    // checksum of per-request checksums, in request order:
    // D = mix({D, count, sum, sum of squares}) (rng.h mix)
    std::uint64_t digest = 0x5eed;
    for (std::size_t r = 0; r < requests; ++r) digest = rng::mix({digest, counts[r], isum[r], isq[r]});
    double configs = static_cast<double>(S) * static_cast<double>(requests);
    std::printf(
        "{\"mode\":\"route\",\"n\":%d,\"m\":%d,\"requests\":%zu,\"router\":\"%s\","
        "\"threads\":%d,\"seconds\":%.6f,\"configs\":%.0f,\"configs_per_s\":%.6e,"
        "\"members\":%llu,\"digest\":\"%016llx\"}\n",
        n, m, requests, noisy ? "noisy" : "oracle", threads, dt, configs,
        configs / dt, static_cast<unsigned long long>(members),
        static_cast<unsigned long long>(digest));
  } else {
    std::printf(
        "{\"mode\":\"predict\",\"n\":%d,\"m\":%d,\"requests\":%zu,\"router\":\"%s\","
        "\"threads\":%d,\"seconds\":%.6f,\"requests_per_s\":%.6e,\"evals\":%llu,"
        "\"members\":%llu}\n",
        n, m, requests, noisy ? "noisy" : "oracle", threads, dt,
        static_cast<double>(requests) / dt,
        static_cast<unsigned long long>(evals.load()),
        static_cast<unsigned long long>(members));
  }
  return 0;
}

// ---------------------------------------------------------------- config 3
// The per-stage scheduling workload, identical to
// paper_2511_20975_b200/workloads.py:
//   * requests id = 0.. from generate_accurate_set(chain 5 x 8, defaults,
//     seed, id); viable = ConfigPredictor::predict(id, inf) (oracle router)
//     or, with exhaustive=1, the full accurate set;
//   * request id arrives at id * 0.01 and is advanced k = mix({12345, id}) % 5
//     stages, stage a choosing candidate_models(a)[mix({12345, id, a}) % #];
//   * 8 pools x 32 slots; round r frees F = {1, 8, 64}[mix({seed, r}) % 3]
//     slots: all pools full, then F draws e = mix({seed, r, j}) % 8 decrement
//     a pool that is not empty;
//   * every assigned stage dispatches (prefix prune) and completes at once;
//     a finished request is replaced by the next id (steady in-flight count).
// Times beam_schedule per round on one core (p50/p99) and hashes decisions.
int run_sched(std::size_t inflight, int beam, int rounds, std::uint64_t seed, bool exhaustive) {
  const int n = 5, m = 8;
  WorkflowGraph g = chain_graph(n);
  ModelCatalog cat = geometric_catalog(m);
  ConfigSpace space(g, cat);
  AccuracyGenParams ap;
  OracleRouter* router = nullptr;
  std::vector<AccurateSet> sets;
  const std::size_t reserve = inflight + (std::size_t)rounds * 64 + 16;
  sets.reserve(reserve);
  for (std::size_t i = 0; i < reserve; ++i) sets.push_back(generate_accurate_set(space, ap, seed, i));
  AccuracyTable table(space, sets);
  router = new OracleRouter(table, 0.002);
  ConfigPredictor predictor(space, *router);
  auto make_request = [&](std::size_t id) {
    std::vector<Configuration> viable;
    if (exhaustive) {
      for (std::uint64_t k = 0; k < space.size(); ++k) {
        Configuration c = space.at_index(k);
        if (table.accurate(id, c)) viable.push_back(std::move(c));
      }
    } else {
      viable = predictor.predict(id, std::numeric_limits<double>::infinity()).viable.configs;
    }
    Request r = Request::make(id, (double)id * 0.01, g, std::move(viable));
    const int k = (int)(rng::mix({12345ULL, (std::uint64_t)id}) % (std::uint64_t)n);
    for (int a = 0; a < k; ++a) {
      std::vector<int> cands = r.candidate_models(a);
      const int mdl = cands[rng::mix({12345ULL, (std::uint64_t)id, (std::uint64_t)a}) % cands.size()];
      r.mark_dispatched(a, mdl, 0.0);
      r.mark_complete(a, 0.0);
    }
    return r;
  };
  std::vector<Request> live;  // FIFO order (ids increase with arrival)
  live.reserve(inflight);
  std::size_t next_id = 0;
  while (live.size() < inflight) {
    Request r = make_request(next_id++);
    if (!r.finished()) live.push_back(std::move(r));
  }
  std::vector<double> lat_us;
  std::uint64_t hash = 0x9e3779b97f4a7c15ULL;
  std::uint64_t assigned = 0;
  for (int rd = 0; rd < rounds; ++rd) {
    const int F = std::array<int, 3>{1, 8, 64}[rng::mix({seed, (std::uint64_t)rd}) % 3];
    std::vector<EngineState> engines(8);
    for (int e = 0; e < 8; ++e) {
      engines[e].model = e;
      engines[e].slots = 32;
      engines[e].weight = cat.at(e).slot_throughput;
    }
    std::vector<int> occ(8, 32);
    for (int j = 0; j < F; ++j) {
      const int e = (int)(rng::mix({seed, (std::uint64_t)rd, (std::uint64_t)j}) % 8);
      if (occ[e] > 0) --occ[e];
    }
    for (int e = 0; e < 8; ++e)
      for (int b = 0; b < occ[e]; ++b) engines[e].in_flight.push_back({999999, 0, 1e18});
    std::vector<const Request*> queue;
    std::vector<Request*> mut;
    for (Request& r : live)
      if (!r.ready_agents().empty()) {
        queue.push_back(&r);
        mut.push_back(&r);
      }
    auto t0 = Clock::now();
    Assignment a = beam_schedule(queue, engines, SchedulerParams{beam});
    auto t1 = Clock::now();
    lat_us.push_back(secs(t0, t1) * 1e6);
    for (const AssignmentTriple& t : a.triples) {
      hash = rng::mix({hash, (std::uint64_t)t.request_index, t.request, (std::uint64_t)t.agent,
                       (std::uint64_t)t.model});
      ++assigned;
    }
    hash = rng::mix({hash, (std::uint64_t)(a.utilization * 1e6), a.states_explored,
                     (std::uint64_t)a.skips});
    ApplyOutcome out = apply_assignment(a, mut, engines, 0.0,
                                        [](RequestId, int, int) { return 1.0; });
    for (const AssignmentTriple& t : out.applied) mut[t.request_index]->mark_complete(t.agent, 0.0);
    // replace finished requests, keeping FIFO order (new ids arrive last)
    std::vector<Request> keep;
    keep.reserve(live.size());
    for (Request& r : live)
      if (!r.finished()) keep.push_back(std::move(r));
    live = std::move(keep);
    while (live.size() < inflight) {
      Request r = make_request(next_id++);
      if (!r.finished()) live.push_back(std::move(r));
    }
  }
  std::vector<double> s = lat_us;
  std::sort(s.begin(), s.end());
  auto pct = [&](double p) { return s[std::min(s.size() - 1, (std::size_t)(p * (double)s.size()))]; };
  std::printf(
      "{\"mode\":\"sched\",\"inflight\":%zu,\"beam\":%d,\"rounds\":%d,\"exhaustive\":%d,"
      "\"p50_us\":%.3f,\"p99_us\":%.3f,\"mean_us\":%.3f,\"assigned\":%llu,\"hash\":\"%016llx\"}\n",
      inflight, beam, rounds, exhaustive ? 1 : 0, pct(0.5), pct(0.99),
      std::accumulate(s.begin(), s.end(), 0.0) / (double)s.size(),
      (unsigned long long)assigned, (unsigned long long)hash);
  delete router;
  return 0;
}

int run_select(int n, int m, std::size_t requests, int threads, std::uint64_t seed,
               bool exhaustive) {
  WorkflowGraph g = chain_graph(n);
  ModelCatalog cat = geometric_catalog(m);
  ConfigSpace space(g, cat);
  AccuracyGenParams ap;
  AccuracyTable table = generate_accuracy_table(space, ap, requests, seed);
  OracleRouter oracle(table, 0.002);
  ConfigPredictor predictor(space, oracle);
  std::vector<ServiceTimeModel::Params> sp(m);
  for (int i = 0; i < m; ++i) sp[i] = {-0.3 + 0.35 * i, 0.25, 0.05};
  ServiceTimeModel service(sp);
  RuntimeCostContext ctx;
  ctx.service = &service;
  for (int i = 0; i < m; ++i) {
    ctx.occupancy.push_back(4);
    ctx.queued_ahead.push_back(i % 3);
    ctx.slots.push_back(8);
  }
  std::vector<std::vector<Configuration>> sets(requests);
  parallel_for(requests, threads, [&](std::size_t id) {
    if (exhaustive) {
      for (std::uint64_t i = 0; i < space.size(); ++i) {
        Configuration c = space.at_index(i);
        if (table.accurate(id, c)) sets[id].push_back(std::move(c));
      }
    } else {
      sets[id] = predictor.predict(id, std::numeric_limits<double>::infinity()).viable.configs;
    }
  });
  std::uint64_t costed = 0;
  for (const auto& v : sets) costed += v.size();
  std::vector<std::uint64_t> chosen(requests, 0);
  std::vector<double> est(requests, 0.0);
  auto t0 = Clock::now();
  parallel_for(requests, threads, [&](std::size_t id) {
    std::vector<Configuration> members = sets[id];  // members_by_cost copies its input
    std::sort(members.begin(), members.end(), [&](const Configuration& a, const Configuration& b) {
      double ca = space.static_cost(a), cb = space.static_cost(b);
      if (ca != cb) return ca < cb;
      return a.models < b.models;
    });
    std::size_t best = 0;
    double best_est = estimate_completion(ctx, members[0]);
    for (std::size_t i = 1; i < members.size(); ++i) {
      double e = estimate_completion(ctx, members[i]);
      if (e < best_est) {
        best = i;
        best_est = e;
      }
    }
    chosen[id] = space.index_of(members[best]);
    est[id] = best_est;
  });
  auto t1 = Clock::now();
  double dt = secs(t0, t1);
  std::uint64_t digest = 0x5eed;
  for (std::size_t r = 0; r < requests; ++r) {
    std::uint64_t bits;
    std::memcpy(&bits, &est[r], 8);
    digest = rng::mix({digest, chosen[r], bits});
  }
  std::printf(
      "{\"mode\":\"select\",\"n\":%d,\"m\":%d,\"requests\":%zu,\"sets\":\"%s\","
      "\"threads\":%d,\"seconds\":%.6f,\"configs_costed\":%llu,\"configs_costed_per_s\":%.6e,"
      "\"us_per_request\":%.6f,\"digest\":\"%016llx\"}\n",
      n, m, requests, exhaustive ? "exhaustive" : "viable", threads, dt,
      (unsigned long long)costed, (double)costed / dt, dt * 1e6 / (double)requests,
      (unsigned long long)digest);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_bench route|predict|sched|select ...\n");
    return 2;
  }
  std::string mode = argv[1];
  try {
    if (mode == "sched" && argc >= 7) {
      return run_sched(static_cast<std::size_t>(std::atoll(argv[2])), std::atoi(argv[3]),
                       std::atoi(argv[4]), static_cast<std::uint64_t>(std::atoll(argv[5])),
                       std::atoi(argv[6]) != 0);
    }
    if (mode == "select" && argc >= 8) {
      return run_select(std::atoi(argv[2]), std::atoi(argv[3]),
                        static_cast<std::size_t>(std::atoll(argv[4])), std::atoi(argv[5]),
                        static_cast<std::uint64_t>(std::atoll(argv[6])),
                        std::strcmp(argv[7], "exhaustive") == 0);
    }
    if ((mode == "route" || mode == "predict") && argc >= 8) {
      return run_route(std::atoi(argv[2]), std::atoi(argv[3]),
                       static_cast<std::size_t>(std::atoll(argv[4])),
                       std::strcmp(argv[5], "noisy") == 0, std::atoi(argv[6]),
                       static_cast<std::uint64_t>(std::atoll(argv[7])),
                       mode == "predict");
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_bench: %s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "ref_bench: bad arguments\n");
  return 2;
}
