// tools/bench_trials.cpp — trial batching throughput:
// N independent d4orm solves of a BASELINE config, one at a time vs batched
// on the persistent worker pool (one GPU context + stream per worker).
//   g++ -std=c++17 -O2 -Iinclude -I<json.hpp dir> tools/bench_trials.cpp \
//       -Lpaper_2503_12204_b200 -ld4orm_b200 -Wl,-rpath,$PWD/paper_2503_12204_b200 -o /tmp/bt
//   /tmp/bt <config 1..4> <trials> <workers...>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "d4orm/bench.hpp"

using namespace d4orm;

int main(int argc, char** argv) {
  const int cfg = argc > 1 ? std::atoi(argv[1]) : 2;
  const int n = argc > 2 ? std::atoi(argv[2]) : 16;
  BaselineConfig bc = baseline_config(cfg);
  bc.scenario.id = "C" + std::to_string(cfg);
  std::vector<TrialSpec> batch;
  for (int s = 0; s < n; ++s) {
    TrialSpec t;
    t.spec.d4orm.max_iterations = bc.iterations;
    t.spec.d4orm.horizon = bc.horizon;
    t.spec.d4orm.denoiser.steps = bc.steps;
    t.spec.d4orm.denoiser.batch = bc.samples;
    t.spec.d4orm.stop_on_success = false;
    t.scenario = bc.scenario;
    t.seed = (std::uint64_t)s;
    batch.push_back(t);
  }
  const double evals_per_trial = (double)bc.samples * bc.steps * bc.iterations;
  for (int a = 3; a < argc || a == 3; ++a) {
    const int w = argc > a ? std::atoi(argv[a]) : 1;
    run_trials(batch, w);  // warm: contexts, buffers, graphs of every worker
    const auto t0 = std::chrono::steady_clock::now();
    const auto recs = run_trials(batch, w);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    int err = 0;
    for (const auto& r : recs) err += !r.error.empty();
    std::printf("{\"config\": \"C%d\", \"trials\": %d, \"workers\": %d, \"wall_s\": %.4f, \"trials_per_s\": %.2f, "
                "\"evals_per_s\": %.4g, \"errors\": %d}\n",
                cfg, n, w, s, n / s, n * evals_per_trial / s, err);
    if (argc <= 3) break;
  }
  return 0;
}
