// tests/cpp/test_dropin.cpp — exercises the C++ drop-in (include/d4orm/*.hpp,
// the reference planner interface) on the GPU and prints JSON that
// tests/test_dropin_cpp.py checks against the CPU oracle.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "d4orm/baselines.hpp"
#include "d4orm/denoiser.hpp"
#include "d4orm/gpu.hpp"
#include "d4orm/optimizer.hpp"
#include "d4orm/scenario.hpp"

using namespace d4orm;

static void print_matrix(const char* name, const Matrix& m) {
  std::printf("\"%s\": [", name);
  for (Index j = 0; j < m.size(); ++j) std::printf("%s%.17g", j ? "," : "", m.data()[j]);
  std::printf("],\n");
}

int main() {
  std::printf("{\n");
  // 1. generators: BASELINE C2 and C5 (checked against the Python mirror)
  for (int c : {2, 5}) {
    BaselineConfig bc = baseline_config(c);
    print_matrix(c == 2 ? "c2_starts" : "c5_starts", bc.scenario.starts);
    Matrix oc(bc.scenario.position_dim(), (Index)bc.scenario.obstacles.size());
    Vector orad((Index)bc.scenario.obstacles.size());
    for (std::size_t o = 0; o < bc.scenario.obstacles.size(); ++o) {
      oc.col((Index)o) = bc.scenario.obstacles.obstacles[o].center;
      orad[(Index)o] = bc.scenario.obstacles.obstacles[o].radius;
    }
    print_matrix(c == 2 ? "c2_obs" : "c5_obs", oc);
    print_matrix(c == 2 ? "c2_rad" : "c5_rad", orad);
  }
  // 2. rollout KAT through the GPU fp64 path
  {
    DynamicsModel m = DynamicsModel::make(ModelKind::Holo2D);
    Matrix starts = Matrix::Zero(4, 1);
    JointControls u = JointControls::zeros(1, 2, 10);
    for (int t = 0; t < 10; ++t) u.u(0, t) = 1.0;
    JointTrajectory tr = rollout(m, starts, u, 0.1);
    std::printf("\"kat_px\": %.17g, \"kat_vx\": %.17g,\n", tr.states(0, 10), tr.states(2, 10));
  }
  // 3. run_denoising in correctness mode (fp64 + the reference's NormalStream noise)
  BaselineConfig bc = baseline_config(2);
  const int H = 16;
  GpuOptions o;
  o.precision = D4ORM_PREC_F64;
  o.host_noise = true;
  set_gpu_options(o);
  DenoiserConfig dc;
  dc.steps = 6;
  dc.batch = 256;
  dc.seed = 7;
  const NoiseSchedule sch = make_schedule(dc.steps, dc.alpha_bar_final);
  JointControls base = JointControls::zeros(bc.scenario.robots, bc.model.control_dim, H);
  for (Index j = 0; j < base.u.size(); ++j) base.u.data()[j] = 0.3 * std::sin(0.7 * j);
  DenoiseResult r = run_denoising(base, bc.scenario, bc.model, sch, dc, 0.1);
  print_matrix("rd_variable", r.variable.u);
  std::printf("\"rd_trace\": [");
  for (std::size_t s = 0; s < r.trace.steps.size(); ++s)
    std::printf("%s[%d, %.17g, %.17g, %.17g]", s ? "," : "", r.trace.steps[s].step, r.trace.steps[s].best_reward,
                r.trace.steps[s].mean_reward, r.trace.steps[s].weight_entropy);
  std::printf("],\n");
  // 4. solve (anytime loop) in correctness mode
  OptimizerConfig oc;
  oc.max_iterations = 2;
  oc.stop_on_success = false;
  oc.horizon = H;
  oc.denoiser = dc;
  SolveResult sr = solve(bc.scenario, bc.model, oc);
  std::printf("\"solve_best\": %.17g, \"solve_iters\": %d, \"solve_success\": %d,\n", sr.best_reward, sr.iterations_used,
              sr.success ? 1 : 0);
  print_matrix("solve_states", sr.best_trajectory.states);
  // 4b. MPPI / CEM baselines in correctness mode
  {
    MppiConfig mc;
    mc.batch = 200;
    mc.sigma = 0.6;
    mc.iterations = 3;
    mc.seed = 4;
    mc.horizon = H;
    mc.stop_on_success = false;
    SolveResult mr = mppi_solve(bc.scenario, bc.model, mc);
    std::printf("\"mppi_best\": %.17g, \"mppi_iters\": %d,\n", mr.best_reward, mr.iterations_used);
    print_matrix("mppi_states", mr.best_trajectory.states);
    CemConfig cc;
    cc.batch = 200;
    cc.elite_fraction = 0.1;
    cc.initial_std = 0.7;
    cc.iterations = 3;
    cc.seed = 4;
    cc.horizon = H;
    cc.stop_on_success = false;
    SolveResult cr = cem_solve(bc.scenario, bc.model, cc);
    std::printf("\"cem_best\": %.17g, \"cem_iters\": %d,\n", cr.best_reward, cr.iterations_used);
    print_matrix("cem_states", cr.best_trajectory.states);
    Vector rw(7);
    const double vals[7] = {0.5, 0.9, 0.5, -1.0, 0.9, 0.2, 0.9};
    for (int j = 0; j < 7; ++j) rw[j] = vals[j];
    const std::vector<int> el = select_elites(rw, 3);
    std::printf("\"elites\": [%d, %d, %d],\n", el[0], el[1], el[2]);
  }
  // 4c. mc_average (denoiser.cpp:92-108) through the device K5 (fp64)
  {
    std::vector<JointControls> smp;
    const int M = 600;
    for (int m = 0; m < M; ++m) {
      JointControls c = JointControls::zeros(3, 2, 5);
      for (Index j = 0; j < c.u.size(); ++j) c.u.data()[j] = std::sin(0.37 * m + 1.3 * j) * (1.0 + 0.01 * m);
      smp.push_back(c);
    }
    Vector w(M);
    double tot = 0.0;
    for (int m = 0; m < M; ++m) tot += (w[m] = std::exp(-0.01 * m));
    for (int m = 0; m < M; ++m) w[m] /= tot;
    print_matrix("mc_avg", mc_average(smp, w).u);
    std::string e;
    try {
      w[0] += 0.5;
      mc_average(smp, w);
    } catch (const std::invalid_argument& x) {
      e = x.what();
    }
    std::printf("\"mc_err\": \"%s\",\n", e.c_str());
  }
  // 5. throughput mode (fp32 + Philox) runs and is deterministic
  o.precision = D4ORM_PREC_F32;
  o.host_noise = false;
  set_gpu_options(o);
  DenoiseResult a = run_denoising(base, bc.scenario, bc.model, sch, dc, 0.1);
  DenoiseResult b = run_denoising(base, bc.scenario, bc.model, sch, dc, 0.1);
  double diff = 0.0;
  for (Index j = 0; j < a.variable.u.size(); ++j) diff = std::max(diff, std::abs(a.variable.u.data()[j] - b.variable.u.data()[j]));
  std::printf("\"f32_repeat_maxdiff\": %.17g,\n", diff);
  // 6. the reference's error behaviour
  std::string err;
  try {
    DenoiserConfig bad = dc;
    bad.batch = 1;
    run_denoising(base, bc.scenario, bc.model, sch, bad, 0.1);
  } catch (const std::invalid_argument& e) {
    err = e.what();
  }
  std::printf("\"err_batch\": \"%s\"\n}\n", err.c_str());
  return 0;
}
