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

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "aragog/accuracy.h"
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
  std::atomic<std::uint64_t> evals{0};
  const std::uint64_t S = space.size();

  auto t0 = Clock::now();
  if (!chain_mode) {
    parallel_for(requests, threads, [&](std::size_t id) {
      std::vector<Configuration> members;
      for (std::uint64_t i = 0; i < S; ++i) {
        Configuration c = space.at_index(i);
        if (router.evaluate(id, c)) members.push_back(std::move(c));
      }
      counts[id] = members.size();
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
    double configs = static_cast<double>(S) * static_cast<double>(requests);
    std::printf(
        "{\"mode\":\"route\",\"n\":%d,\"m\":%d,\"requests\":%zu,\"router\":\"%s\","
        "\"threads\":%d,\"seconds\":%.6f,\"configs\":%.0f,\"configs_per_s\":%.6e,"
        "\"members\":%llu}\n",
        n, m, requests, noisy ? "noisy" : "oracle", threads, dt, configs,
        configs / dt, static_cast<unsigned long long>(members));
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

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_bench route|predict|sched ...\n");
    return 2;
  }
  std::string mode = argv[1];
  try {
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
