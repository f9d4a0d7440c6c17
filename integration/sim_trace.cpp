// Config 5 driver: one reference simulation (run_simulation, src/simulation.cpp)
// of a shipped scenario, its JSONL trace written to a file, and a one-line
// JSON summary on stdout (wall time of a second, warm run; rounds,
// predictions, decisions/s).
// Linked twice by integration/Makefile: against the unmodified reference
// objects (sim_trace_ref) and with the GPU adapter (sim_trace_gpu); the two
// traces must be byte-identical.
//
//   sim_trace <scenario.json> <policy> <trace.jsonl> [--requests N | --horizon S]
//             [--rate R] [--seed S] [--beam B]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>

#include "aragog/metrics.h"
#include "aragog/scenario.h"
#include "aragog/simulation.h"
#include "aragog/workload.h"

// defined by the GPU adapter only (weak: null in the reference build)
extern "C" unsigned long long aragog_gpu_launches() __attribute__((weak));

int main(int argc, char** argv) {
  using namespace aragog;
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s scenario.json policy trace.jsonl [opts]\n", argv[0]);
    return 2;
  }
  try {
    const Scenario sc = Scenario::load(argv[1]);
    RunOptions o;
    o.policy = parse_policy(argv[2]);
    for (int i = 4; i + 1 < argc; i += 2) {
      const std::string k = argv[i];
      if (k == "--requests") o.num_requests = std::strtoull(argv[i + 1], nullptr, 10);
      else if (k == "--horizon") {
        o.mode = RunMode::kHorizon;
        o.horizon = std::strtod(argv[i + 1], nullptr);
      } else if (k == "--rate") o.arrival_rate = std::strtod(argv[i + 1], nullptr);
      else if (k == "--seed") o.seed = std::strtoull(argv[i + 1], nullptr, 10);
      else if (k == "--beam") o.beam_width = std::atoi(argv[i + 1]);
      else {
        std::fprintf(stderr, "unknown option %s\n", k.c_str());
        return 2;
      }
    }
    // warm run first (CUDA context creation, module load and scratch
    // allocation are one-time costs of the GPU build), then the timed run
    run_simulation(sc, o);
    const unsigned long long l0 = aragog_gpu_launches ? aragog_gpu_launches() : 0ULL;
    const auto t0 = std::chrono::steady_clock::now();
    const RunTrace tr = run_simulation(sc, o);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::ofstream f(argv[3]);
    tr.write_jsonl(f);
    const RunReport rep = summarize_run(tr);
    std::size_t pairs = 0, assigned = 0;
    for (const RoundRecord& r : tr.rounds) {
      pairs += r.pairs;
      assigned += r.assigned;
    }
    std::printf(
        "{\"scenario\": \"%s\", \"policy\": \"%s\", \"requests\": %zu, \"rounds\": %zu, "
        "\"pairs\": %zu, \"assigned\": %zu, \"completed\": %zu, \"wall_s\": %.6f, "
        "\"rounds_per_s\": %.3f, \"requests_per_s\": %.3f, \"gpu_launches\": %llu}\n",
        tr.scenario_name.c_str(), tr.policy.c_str(), tr.requests.size(), tr.rounds.size(), pairs,
        assigned, rep.completed, secs, tr.rounds.size() / secs, tr.requests.size() / secs,
        aragog_gpu_launches ? aragog_gpu_launches() - l0 : 0ULL);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
