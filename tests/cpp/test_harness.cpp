// tests/cpp/test_harness.cpp — the drop-in's trial harness and I/O
// (include/d4orm/{bench,io,scenario}.hpp).  Mode "host": CSV / aggregate /
// scenario JSON only (no GPU); mode "gpu": run_trials batching, solve outputs.
// Prints JSON that tests/test_harness.py checks against the reference.
#include <cstdio>
#include <cstring>
#include <string>

#include "d4orm/bench.hpp"
#include "d4orm/gpu.hpp"
#include "d4orm/io.hpp"

using namespace d4orm;

static TrialRecord synth(const std::string& solver, const std::string& sc, std::uint64_t seed, int n, int succ_at) {
  TrialRecord r;
  r.solver_id = solver;
  r.scenario_id = sc;
  r.seed = seed;
  double best = -1e300;
  for (int i = 1; i <= n; ++i) {
    const double rew = 0.1 * i + 0.013 * (double)(seed % 7) - 0.05 * (i % 3);
    best = rew > best ? rew : best;
    const bool ok = succ_at > 0 && i >= succ_at;
    r.iterations.push_back({i, 100LL * i, 100LL * i * 256, rew, best, 0.01 * i + 0.001 * (double)seed, ok,
                            0.25 * i + 0.01 * (double)seed});
  }
  return r;
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "host";
  const std::string dir = argc > 2 ? argv[2] : "/tmp";
  nlohmann::json out;
  if (mode == "host") {
    std::vector<TrialRecord> recs = {synth("d4orm", "circle4", 3, 5, 3), synth("d4orm", "circle4", 1, 4, 0),
                                     synth("mppi", "circle4", 2, 6, 5),  synth("d4orm", "square8", 9, 3, 1),
                                     synth("d4orm", "circle4", 2, 5, 2), synth("cem", "square8", 4, 2, 0)};
    std::vector<std::string> paths;
    for (size_t i = 0; i < recs.size(); ++i) {
      paths.push_back(dir + "/trial_" + std::to_string(i) + ".csv");
      write_trial_csv(recs[i], paths.back());
    }
    std::vector<TrialRecord> back;
    for (const auto& p : paths) back.push_back(read_trial_csv(p));
    out["csv_paths"] = paths;
    out["aggregate"] = aggregate_to_json(aggregate(back));
    // scenario JSON v1: the reference's native generator shape, and an extension kind
    out["circle_json"] = scenario_to_json(antipodal_circle(4, 6.0, ModelKind::Holo2D)).dump();
    const Scenario c3 = baseline_config(3).scenario;
    const nlohmann::json j3 = scenario_to_json(c3);
    out["c3_roundtrip_equal"] = scenario_to_json(scenario_from_json(j3)) == j3;
    out["c5_roundtrip_equal"] = scenario_to_json(scenario_from_json(scenario_to_json(baseline_config(5).scenario))) ==
                                scenario_to_json(baseline_config(5).scenario);
    try {
      nlohmann::json bad = j3;
      bad["schema_version"] = 2;
      scenario_from_json(bad);
      out["bad_schema"] = "accepted";
    } catch (const std::invalid_argument& e) {
      out["bad_schema"] = e.what();
    }
  } else {
    // run_trials: a batch of independent solves, concurrently vs one at a time
    BaselineConfig bc = baseline_config(1);
    bc.scenario.id = "c1";
    std::vector<TrialSpec> batch;
    for (std::uint64_t seed = 0; seed < 8; ++seed) {
      TrialSpec t;
      t.spec.name = seed % 4 == 3 ? "mppi" : (seed % 4 == 2 ? "cem" : "d4orm");
      t.spec.d4orm.max_iterations = 3;
      t.spec.d4orm.horizon = bc.horizon;
      t.spec.d4orm.denoiser.steps = 20;
      t.spec.d4orm.denoiser.batch = 512;
      t.spec.d4orm.stop_on_success = false;
      t.spec.mppi.batch = 512;
      t.spec.mppi.iterations = 4;
      t.spec.mppi.horizon = bc.horizon;
      t.spec.mppi.stop_on_success = false;
      t.spec.cem.batch = 512;
      t.spec.cem.iterations = 4;
      t.spec.cem.horizon = bc.horizon;
      t.spec.cem.stop_on_success = false;
      t.scenario = bc.scenario;
      t.seed = seed;
      batch.push_back(t);
    }
    run_trials(batch, 1);  // warm-up: module load, this thread's context and graphs
    run_trials(batch, 8);  // warm-up: the pool workers' contexts
    auto t0 = std::chrono::steady_clock::now();
    const auto seq = run_trials(batch, 1);
    auto t1 = std::chrono::steady_clock::now();
    const auto par = run_trials(batch, 8);
    auto t2 = std::chrono::steady_clock::now();
    bool same = seq.size() == par.size();
    for (size_t i = 0; same && i < seq.size(); ++i) {
      same = seq[i].error.empty() && par[i].error.empty() && seq[i].iterations.size() == par[i].iterations.size();
      for (size_t k = 0; same && k < seq[i].iterations.size(); ++k)
        same = seq[i].iterations[k].reward == par[i].iterations[k].reward &&
               seq[i].iterations[k].objective == par[i].iterations[k].objective &&
               seq[i].iterations[k].success == par[i].iterations[k].success;
    }
    out["batch_identical"] = same;
    out["batch_errors"] = seq[0].error;
    out["seq_s"] = std::chrono::duration<double>(t1 - t0).count();
    out["par_s"] = std::chrono::duration<double>(t2 - t1).count();
    out["iterations"] = (int)seq[0].iterations.size();
    // solve outputs: export, read back, replay the outcome
    OptimizerConfig oc;
    oc.max_iterations = 2;
    oc.stop_on_success = false;
    oc.horizon = bc.horizon;
    oc.denoiser.steps = 10;
    oc.denoiser.batch = 256;
    const SolveResult r = solve(bc.scenario, bc.model, oc);
    write_solve_outputs(dir, bc.scenario, r, "d4orm", nlohmann::json{{"seed", 0}});
    const LoadedTrajectory lt = read_trajectory_json(dir + "/trajectory.json");
    out["replay_success"] = check_success(lt.trajectory, lt.scenario).success == r.success;
    out["replay_objective"] = objective(lt.trajectory, lt.scenario) == lt.result.at("objective").get<double>();
    out["replay_reward"] = total_reward(lt.trajectory, lt.scenario) == r.best_reward;
    out["out_dir"] = dir;
  }
  std::printf("%s\n", out.dump().c_str());
  return 0;
}
