// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// C entry points over the *reference's own* C++ library (proj/src/*.cpp from
// /root/reference, compiled unchanged by oracle/Makefile against
// oracle/eigen_shim) so tests can pin the plain-C oracle bitwise against the
// real reference code, and bench.py --impl reference can time it.
//
// Native model kinds (DiffDrive/Holo2D/Holo3D) go through d4orm::rollout /
// d4orm::run_denoising / d4orm::solve untouched.  The three BASELINE
// extensions (velocity-input holonomic 2D/3D, unicycle) use the reference's
// documented extension point: a derivative functor driven by
// d4orm::detail::rk4_with (dynamics.hpp:121-130) inside a loop that mirrors
// rollout_robot<DX,DU> (dynamics.cpp:65-87); every other stage (noise,
// sample_batch, total_reward, score_weights, mc_average, denoise_step,
// make_schedule) is the reference's own function.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../oracle/d4orm_oracle.h"
#include "d4orm/baselines.hpp"
#include "d4orm/bench.hpp"
#include "d4orm/denoiser.hpp"
#include "d4orm/dynamics.hpp"
#include "d4orm/optimizer.hpp"
#include "d4orm/parallel.hpp"
#include "d4orm/reward.hpp"
#include "d4orm/rng.hpp"
#include "d4orm/scenario.hpp"
#include "d4orm/schedule.hpp"

using namespace d4orm;

namespace {

thread_local std::string g_ref_err;

struct VelDerivative {  // xdot = u (2D or 3D single integrator)
  template <class Vec, class UVec>
  Vec operator()(const Vec& x, const UVec& u) const {
    Vec dx(x.size());
    for (Eigen::Index j = 0; j < x.size(); ++j) dx[j] = u[j];
    return dx;
  }
};

struct UnicycleDerivative {  // [x,y,theta], u = [v, omega]
  template <class Vec, class UVec>
  Vec operator()(const Vec& x, const UVec& u) const {
    Vec dx(x.size());
    const double theta = x[2];
    dx[0] = u[0] * std::cos(theta);
    dx[1] = u[0] * std::sin(theta);
    dx[2] = u[1];
    return dx;
  }
};

bool native(int kind) { return kind >= 0 && kind <= 2; }

DynamicsModel make_model(const or_problem* p) {
  DynamicsModel m;
  m.kind = p->kind == OR_DIFFDRIVE ? ModelKind::DiffDrive
           : (p->pdim == 3 ? ModelKind::Holo3D : ModelKind::Holo2D);
  m.state_dim = p->dx;
  m.control_dim = p->du;
  m.control_lower = Vector(p->du);
  m.control_upper = Vector(p->du);
  for (int d = 0; d < p->du; ++d) {
    m.control_lower[d] = p->lower[d];
    m.control_upper[d] = p->upper[d];
  }
  return m;
}

Scenario make_scenario(const or_problem* p) {
  Scenario s;
  s.id = "capi";
  s.model_kind = p->kind == OR_DIFFDRIVE ? ModelKind::DiffDrive
                 : (p->pdim == 3 ? ModelKind::Holo3D : ModelKind::Holo2D);
  s.robots = p->robots;
  s.starts.resize(p->dx, p->robots);
  for (int k = 0; k < p->robots; ++k)
    for (int j = 0; j < p->dx; ++j) s.starts(j, k) = p->starts[k * p->dx + j];
  s.goals.resize(p->pdim, p->robots);
  for (int k = 0; k < p->robots; ++k)
    for (int j = 0; j < p->pdim; ++j) s.goals(j, k) = p->goals[k * p->pdim + j];
  for (int o = 0; o < p->n_obstacles; ++o) {
    Obstacle ob;
    ob.center = Vector(p->pdim);
    for (int j = 0; j < p->pdim; ++j) ob.center[j] = p->obs_centers[o * p->pdim + j];
    ob.radius = p->obs_radii[o];
    s.obstacles.obstacles.push_back(ob);
  }
  s.reward.w_t = p->w_t;
  s.reward.epsilon = p->epsilon;
  s.reward.robot_radius = p->robot_radius;
  s.reward.goal_tolerance = p->goal_tolerance;
  s.reward.obstacle_weight = p->obstacle_weight;
  return s;
}

JointControls to_controls(const or_problem* p, const double* u) {
  JointControls c{p->robots, p->du, Matrix(p->robots * p->du, p->horizon)};
  std::memcpy(c.u.data(), u, sizeof(double) * c.u.size());
  return c;
}

// Mirror of rollout_robot<DX,DU> (dynamics.cpp:65-87) for an extension functor.
template <class Fn>
JointTrajectory ext_rollout(const Fn& f, const DynamicsModel& model, const Matrix& starts,
                            const JointControls& controls, double dt) {
  const int n = controls.robots, horizon = controls.horizon();
  JointTrajectory out;
  out.robots = n;
  out.state_dim = model.state_dim;
  out.control_dim = model.control_dim;
  out.dt = dt;
  out.states.resize(n * model.state_dim, horizon + 1);
  out.controls = Matrix::Zero(n * model.control_dim, horizon + 1);
  const int DX = model.state_dim, DU = model.control_dim;
  for (int k = 0; k < n; ++k) {
    Vector x = starts.col(k);
    out.states.col(0).segment(k * DX, DX) = x;
    for (int t = 0; t < horizon; ++t) {
      const Vector raw = controls.u.col(t).segment(k * DU, DU);
      const Vector u = raw.cwiseMax(model.control_lower).cwiseMin(model.control_upper);
      out.controls.col(t).segment(k * DU, DU) = u;
      x = detail::rk4_with(f, x, u, dt);
      if (!x.allFinite()) {
        throw std::runtime_error("rollout: non-finite state for robot " + std::to_string(k) +
                                 " at step " + std::to_string(t + 1));
      }
      out.states.col(t + 1).segment(k * DX, DX) = x;
    }
  }
  return out;
}

JointTrajectory any_rollout(const or_problem* p, const DynamicsModel& model, const Scenario& sc,
                            const JointControls& c) {
  if (native(p->kind)) return rollout(model, sc.starts, c, p->dt);
  if (p->kind == OR_UNICYCLE) return ext_rollout(UnicycleDerivative{}, model, sc.starts, c, p->dt);
  return ext_rollout(VelDerivative{}, model, sc.starts, c, p->dt);
}

// run_denoising (denoiser.cpp:119-184) with the rollout swapped for the
// extension kinds; identical statement order otherwise.
DenoiseResult ext_run_denoising(const or_problem* p, const JointControls& base, const Scenario& scenario,
                                const DynamicsModel& model, const NoiseSchedule& schedule,
                                const DenoiserConfig& config) {
  const bool deform = config.mode == DenoiseMode::Deformation;
  JointControls variable;
  if (deform) {
    variable = JointControls::zeros(base.robots, base.control_dim, base.horizon());
  } else {
    Matrix z(base.u.rows(), base.u.cols());
    NormalStream stream(mix_seed(config.seed, 0, 0));
    stream.fill(z.data(), z.size());
    variable = {base.robots, base.control_dim, z};
  }
  DenoiseResult result;
  Vector rewards(config.batch);
  for (int i = schedule.steps(); i >= 1; --i) {
    const std::vector<JointControls> samples =
        sample_batch(variable, schedule, i, config.batch, config.seed, config.workers);
    parallel_for(config.batch, config.workers, [&](int m) {
      try {
        JointControls candidate{base.robots, base.control_dim,
                                deform ? Matrix(base.u + samples[m].u) : samples[m].u};
        const JointTrajectory traj = any_rollout(p, model, scenario, candidate);
        rewards[m] = total_reward(traj, scenario, scenario.reward);
      } catch (const std::exception& e) {
        throw std::runtime_error("run_denoising: sample " + std::to_string(m) + " at step " +
                                 std::to_string(i) + ": " + e.what());
      }
    });
    const Vector weights = score_weights(rewards, config.lambda);
    const JointControls averaged = mc_average(samples, weights);
    variable = denoise_step(averaged, schedule, i);
    double best = rewards[0];
    double mean = 0.0;
    for (Eigen::Index m = 0; m < rewards.size(); ++m) {
      best = std::max(best, rewards[m]);
      mean += rewards[m];
    }
    mean /= static_cast<double>(rewards.size());
    double h = 0.0;
    for (Eigen::Index m = 0; m < weights.size(); ++m)
      if (weights[m] > 0.0) h -= weights[m] * std::log(weights[m]);
    result.trace.steps.push_back({i, best, mean, h});
  }
  result.variable = std::move(variable);
  return result;
}

DenoiserConfig to_dcfg(const or_denoiser_config* c) {
  DenoiserConfig d;
  d.steps = c->steps;
  d.batch = static_cast<int>(c->batch);
  d.lambda = c->lambda;
  d.alpha_bar_final = c->alpha_bar_final;
  d.seed = c->seed;
  d.mode = c->mode == 1 ? DenoiseMode::Deformation : DenoiseMode::FromScratch;
  d.workers = c->workers;
  return d;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_ref_err.c_str(); }

uint64_t ref_mix_seed(uint64_t a, uint64_t b) { return mix_seed(a, b); }
uint64_t ref_mix_seed3(uint64_t a, uint64_t b, uint64_t c) { return mix_seed(a, b, c); }

void ref_normal_fill(uint64_t seed, double* out, int64_t n) {
  NormalStream s(seed);
  s.fill(out, n);
}

// sample_batch (denoiser.cpp:34-48) around current=0 with mean_scale/std from
// the schedule: returns the raw z (= (sample - ms*0)/std) is not recoverable,
// so tests compare samples directly.
int ref_sample_batch(const or_problem* p, const double* current, int steps, double abf, int i,
                     int batch, uint64_t seed, double* out /* batch x elems */) {
  try {
    const NoiseSchedule sch = make_schedule(steps, abf);
    const JointControls cur = to_controls(p, current);
    const auto samples = sample_batch(cur, sch, i, batch, seed, 0);
    const size_t e = static_cast<size_t>(cur.u.size());
    for (int m = 0; m < batch; ++m) std::memcpy(out + m * e, samples[m].u.data(), e * sizeof(double));
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 1;
  }
}

int ref_make_schedule(int steps, double abf, double* alpha_bar, double* alpha) {
  try {
    const NoiseSchedule s = make_schedule(steps, abf);
    for (int i = 0; i <= steps; ++i) alpha_bar[i] = s.alpha_bar[i];
    if (alpha)
      for (int i = 0; i < steps; ++i) alpha[i] = s.alpha[i];
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 1;
  }
}

int ref_sampling_spread(int steps, double abf, int i, double* ms, double* sd) {
  try {
    const SamplingSpread s = sampling_spread(make_schedule(steps, abf), i);
    *ms = s.mean_scale;
    *sd = s.std;
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 1;
  }
}

int ref_rk4_step(int kind, const double* x, const double* u, double dt, double* out) {
  try {
    int dx, du, pd;
    or_model_dims(kind, &dx, &du, &pd);
    Vector xv(dx), uv(du), r;
    for (int j = 0; j < dx; ++j) xv[j] = x[j];
    for (int j = 0; j < du; ++j) uv[j] = u[j];
    if (native(kind)) {
      DynamicsModel m = DynamicsModel::make(kind == 0 ? ModelKind::DiffDrive
                                            : kind == 1 ? ModelKind::Holo2D : ModelKind::Holo3D);
      r = rk4_step(m, xv, uv, dt);
    } else if (kind == OR_UNICYCLE) {
      r = detail::rk4_with(UnicycleDerivative{}, xv, uv, dt);
    } else {
      r = detail::rk4_with(VelDerivative{}, xv, uv, dt);
    }
    for (int j = 0; j < dx; ++j) out[j] = r[j];
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 1;
  }
}

int ref_rollout(const or_problem* p, const double* u, double* states, double* controls) {
  try {
    const DynamicsModel model = make_model(p);
    const Scenario sc = make_scenario(p);
    const JointTrajectory tr = any_rollout(p, model, sc, to_controls(p, u));
    std::memcpy(states, tr.states.data(), sizeof(double) * tr.states.size());
    if (controls) std::memcpy(controls, tr.controls.data(), sizeof(double) * tr.controls.size());
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 1;
  }
}

static JointTrajectory traj_from(const or_problem* p, const double* states) {
  JointTrajectory tr;
  tr.robots = p->robots;
  tr.state_dim = p->dx;
  tr.control_dim = p->du;
  tr.dt = p->dt;
  tr.states.resize(p->robots * p->dx, p->horizon + 1);
  std::memcpy(tr.states.data(), states, sizeof(double) * tr.states.size());
  tr.controls = Matrix::Zero(p->robots * p->du, p->horizon + 1);
  return tr;
}

int ref_total_reward(const or_problem* p, const double* states, double* reward) {
  try {
    const Scenario sc = make_scenario(p);
    *reward = total_reward(traj_from(p, states), sc, sc.reward);
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 1;
  }
}

double ref_objective(const or_problem* p, const double* states) {
  const Scenario sc = make_scenario(p);
  return objective(traj_from(p, states), sc, sc.reward);
}

int ref_check_success(const or_problem* p, const double* states, char* msg, int msg_len) {
  const Scenario sc = make_scenario(p);
  const SuccessReport r = check_success(traj_from(p, states), sc, sc.reward);
  if (msg && msg_len > 0) std::snprintf(msg, msg_len, "%s", r.first_violation.c_str());
  return r.success ? 1 : 0;
}

int ref_score_weights(const double* rewards, int64_t m, double lambda, double* w) {
  try {
    Vector r(static_cast<Eigen::Index>(m));
    for (int64_t j = 0; j < m; ++j) r[j] = rewards[j];
    const Vector out = score_weights(r, lambda);
    for (int64_t j = 0; j < m; ++j) w[j] = out[j];
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 1;
  }
}

int ref_mc_average(const double* samples, const double* weights, int64_t m, int rows, int cols,
                   double* out) {
  try {
    std::vector<JointControls> s(static_cast<size_t>(m));
    const size_t e = static_cast<size_t>(rows) * cols;
    for (int64_t j = 0; j < m; ++j) {
      s[j] = {1, rows, Matrix(rows, cols)};
      std::memcpy(s[j].u.data(), samples + j * e, e * sizeof(double));
    }
    Vector w(static_cast<Eigen::Index>(m));
    for (int64_t j = 0; j < m; ++j) w[j] = weights[j];
    const JointControls r = mc_average(s, w);
    std::memcpy(out, r.u.data(), e * sizeof(double));
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 1;
  }
}

int ref_run_denoising(const or_problem* p, const double* base, const or_denoiser_config* c,
                      double* variable, or_trace_rec* trace) {
  try {
    const DynamicsModel model = make_model(p);
    const Scenario sc = make_scenario(p);
    const NoiseSchedule sch = make_schedule(c->steps, c->alpha_bar_final);
    const DenoiserConfig cfg = to_dcfg(c);
    const JointControls b = to_controls(p, base);
    const DenoiseResult r = native(p->kind) ? run_denoising(b, sc, model, sch, cfg, p->dt)
                                            : ext_run_denoising(p, b, sc, model, sch, cfg);
    std::memcpy(variable, r.variable.u.data(), sizeof(double) * r.variable.u.size());
    if (trace) {
      for (size_t s = 0; s < r.trace.steps.size(); ++s) {
        const auto& t = r.trace.steps[s];
        trace[s] = {t.step, t.best_reward, t.mean_reward, t.weight_entropy};
      }
    }
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 1;
  }
}

// solve (optimizer.cpp:48-102).  Native kinds call d4orm::solve; extensions
// replay the same loop around ext_run_denoising.
int ref_solve(const or_problem* p, const or_denoiser_config* dc, const or_optimizer_config* oc,
              double* best_states, double* best_reward, int* success, or_iteration_stats* per_it) {
  try {
    const DynamicsModel model = make_model(p);
    Scenario sc = make_scenario(p);
    OptimizerConfig cfg;
    cfg.max_iterations = oc->max_iterations;
    cfg.stop_on_success = oc->stop_on_success != 0;
    if (oc->deadline_seconds > 0) cfg.deadline_seconds = oc->deadline_seconds;
    cfg.denoiser = to_dcfg(dc);
    cfg.horizon = p->horizon;
    cfg.dt = p->dt;
    if (native(p->kind)) {
      const SolveResult r = solve(sc, model, cfg);
      std::memcpy(best_states, r.best_trajectory.states.data(),
                  sizeof(double) * r.best_trajectory.states.size());
      *best_reward = r.best_reward;
      *success = r.success ? 1 : 0;
      if (per_it)
        for (size_t i = 0; i < r.per_iteration.size(); ++i)
          per_it[i] = {r.per_iteration[i].reward, r.per_iteration[i].objective,
                       r.per_iteration[i].success ? 1 : 0, r.per_iteration[i].wall_seconds};
      return r.iterations_used;
    }
    const NoiseSchedule sch = make_schedule(cfg.denoiser.steps, cfg.denoiser.alpha_bar_final);
    JointTrajectory current =
        any_rollout(p, model, sc, JointControls::zeros(p->robots, p->du, p->horizon));
    JointTrajectory best;
    int best_it = -1, used = 0;
    for (int it = 1; it <= cfg.max_iterations; ++it) {
      DenoiserConfig d = cfg.denoiser;
      d.seed = mix_seed(cfg.denoiser.seed, static_cast<std::uint64_t>(it));
      d.mode = DenoiseMode::Deformation;
      const JointControls base_controls = current.executed_controls();
      const DenoiseResult den = ext_run_denoising(p, base_controls, sc, model, sch, d);
      const JointControls updated{base_controls.robots, base_controls.control_dim,
                                  base_controls.u + den.variable.u};
      current = any_rollout(p, model, sc, updated);
      const double reward = total_reward(current, sc);
      const double quality = objective(current, sc);
      const bool ok = check_success(current, sc).success;
      if (per_it) per_it[it - 1] = {reward, quality, ok ? 1 : 0, 0.0};
      used = it;
      if (best_it < 0 || reward > *best_reward) {
        *best_reward = reward;
        best = current;
        best_it = it;
      }
      if (cfg.stop_on_success && ok) break;
    }
    std::memcpy(best_states, best.states.data(), sizeof(double) * best.states.size());
    *success = check_success(best, sc).success ? 1 : 0;
    return used;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return -1;
  }
}

// ------------------------------------------------------------- baselines
// mppi_solve / cem_solve (baselines.cpp:99-173): native kinds call the
// reference functions; the extension kinds run the same statements with the
// rollout swapped (any_rollout), every other piece the reference's own.
int ref_select_elites(const double* r, int64_t m, int count, int* out) {
  try {
    Vector rw(m);
    for (int64_t i = 0; i < m; ++i) rw[i] = r[i];
    const std::vector<int> e = select_elites(rw, count);
    std::memcpy(out, e.data(), sizeof(int) * e.size());
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 1;
  }
}

}  // extern "C"

namespace {
template <class Update>
int ext_anytime(const or_problem* p, const DynamicsModel& model, const Scenario& sc, int iterations,
                bool stop_on_success, double* best_states, double* best_reward, int* success,
                or_iteration_stats* per_it, Update&& update) {
  JointTrajectory best;
  int best_it = -1, used = 0;
  for (int it = 1; it <= iterations; ++it) {
    const JointControls& mean = update(it);
    const JointTrajectory traj = any_rollout(p, model, sc, mean);
    const double reward = total_reward(traj, sc);
    const double quality = objective(traj, sc);
    const bool ok = check_success(traj, sc).success;
    if (per_it) per_it[it - 1] = {reward, quality, ok ? 1 : 0, 0.0};
    used = it;
    if (best_it < 0 || reward > *best_reward) {
      *best_reward = reward;
      best = traj;
      best_it = it;
    }
    if (stop_on_success && ok) break;
  }
  std::memcpy(best_states, best.states.data(), sizeof(double) * best.states.size());
  *success = check_success(best, sc).success ? 1 : 0;
  return used;
}

Vector ext_evaluate(const or_problem* p, const DynamicsModel& model, const Scenario& sc,
                    const std::vector<JointControls>& samples, int workers) {
  Vector rewards(static_cast<Eigen::Index>(samples.size()));
  parallel_for(static_cast<int>(samples.size()), workers, [&](int m) {
    const JointTrajectory traj = any_rollout(p, model, sc, samples[m]);
    rewards[m] = total_reward(traj, sc, sc.reward);
  });
  return rewards;
}

Matrix ext_normal_matrix(Eigen::Index rows, Eigen::Index cols, std::uint64_t stream_seed) {
  Matrix z(rows, cols);
  NormalStream stream(stream_seed);
  stream.fill(z.data(), z.size());
  return z;
}
}  // namespace

extern "C" {

int ref_mppi_solve(const or_problem* p, const or_mppi_config* c, double* best_states, double* best_reward,
                   int* success, or_iteration_stats* per_it) {
  try {
    const DynamicsModel model = make_model(p);
    Scenario sc = make_scenario(p);
    MppiConfig cfg;
    cfg.batch = static_cast<int>(c->batch);
    cfg.lambda = c->lambda;
    cfg.sigma = c->sigma;
    cfg.iterations = c->iterations;
    cfg.seed = c->seed;
    cfg.horizon = p->horizon;
    cfg.dt = p->dt;
    cfg.stop_on_success = c->stop_on_success != 0;
    cfg.workers = c->workers;
    if (native(p->kind)) {
      const SolveResult r = mppi_solve(sc, model, cfg);
      std::memcpy(best_states, r.best_trajectory.states.data(), sizeof(double) * r.best_trajectory.states.size());
      *best_reward = r.best_reward;
      *success = r.success ? 1 : 0;
      if (per_it)
        for (size_t i = 0; i < r.per_iteration.size(); ++i)
          per_it[i] = {r.per_iteration[i].reward, r.per_iteration[i].objective,
                       r.per_iteration[i].success ? 1 : 0, r.per_iteration[i].wall_seconds};
      return r.iterations_used;
    }
    JointControls mean = JointControls::zeros(p->robots, p->du, p->horizon);
    std::vector<JointControls> samples(static_cast<std::size_t>(cfg.batch));
    return ext_anytime(p, model, sc, cfg.iterations, cfg.stop_on_success, best_states, best_reward, success, per_it,
                       [&](int iteration) -> const JointControls& {
                         parallel_for(cfg.batch, cfg.workers, [&](int m) {
                           const Matrix z = ext_normal_matrix(mean.u.rows(), mean.u.cols(),
                                                              mix_seed(cfg.seed, static_cast<std::uint64_t>(iteration),
                                                                       static_cast<std::uint64_t>(m)));
                           samples[m] = {mean.robots, mean.control_dim, mean.u + cfg.sigma * z};
                         });
                         const Vector rewards = ext_evaluate(p, model, sc, samples, cfg.workers);
                         const Vector weights = score_weights(rewards, cfg.lambda);
                         mean = mc_average(samples, weights);
                         return mean;
                       });
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return -1;
  }
}

int ref_cem_solve(const or_problem* p, const or_cem_config* c, double* best_states, double* best_reward,
                  int* success, or_iteration_stats* per_it) {
  try {
    const DynamicsModel model = make_model(p);
    Scenario sc = make_scenario(p);
    CemConfig cfg;
    cfg.batch = static_cast<int>(c->batch);
    cfg.elite_fraction = c->elite_fraction;
    cfg.initial_std = c->initial_std;
    cfg.min_std = c->min_std;
    cfg.iterations = c->iterations;
    cfg.seed = c->seed;
    cfg.horizon = p->horizon;
    cfg.dt = p->dt;
    cfg.stop_on_success = c->stop_on_success != 0;
    cfg.workers = c->workers;
    if (native(p->kind)) {
      const SolveResult r = cem_solve(sc, model, cfg);
      std::memcpy(best_states, r.best_trajectory.states.data(), sizeof(double) * r.best_trajectory.states.size());
      *best_reward = r.best_reward;
      *success = r.success ? 1 : 0;
      if (per_it)
        for (size_t i = 0; i < r.per_iteration.size(); ++i)
          per_it[i] = {r.per_iteration[i].reward, r.per_iteration[i].objective,
                       r.per_iteration[i].success ? 1 : 0, r.per_iteration[i].wall_seconds};
      return r.iterations_used;
    }
    const int elite_count = static_cast<int>(cfg.elite_fraction * cfg.batch);
    JointControls mean = JointControls::zeros(p->robots, p->du, p->horizon);
    Matrix std_dev = Matrix::Constant(mean.u.rows(), mean.u.cols(), cfg.initial_std);
    std::vector<JointControls> samples(static_cast<std::size_t>(cfg.batch));
    return ext_anytime(p, model, sc, cfg.iterations, cfg.stop_on_success, best_states, best_reward, success, per_it,
                       [&](int iteration) -> const JointControls& {
                         parallel_for(cfg.batch, cfg.workers, [&](int m) {
                           const Matrix z = ext_normal_matrix(mean.u.rows(), mean.u.cols(),
                                                              mix_seed(cfg.seed, static_cast<std::uint64_t>(iteration),
                                                                       static_cast<std::uint64_t>(m)));
                           samples[m] = {mean.robots, mean.control_dim, mean.u + std_dev.cwiseProduct(z)};
                         });
                         const Vector rewards = ext_evaluate(p, model, sc, samples, cfg.workers);
                         const std::vector<int> elites = select_elites(rewards, elite_count);
                         Matrix new_mean = Matrix::Zero(mean.u.rows(), mean.u.cols());
                         for (const int m : elites) new_mean += samples[static_cast<std::size_t>(m)].u;
                         new_mean /= static_cast<double>(elite_count);
                         Matrix variance = Matrix::Zero(mean.u.rows(), mean.u.cols());
                         for (const int m : elites) {
                           const Matrix d = samples[static_cast<std::size_t>(m)].u - new_mean;
                           variance += d.cwiseProduct(d);
                         }
                         variance /= static_cast<double>(elite_count);
                         std_dev = variance.cwiseSqrt().cwiseMax(cfg.min_std);
                         mean.u = new_mean;
                         return mean;
                       });
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return -1;
  }
}

// ------------------------------------------------- trial harness / scenario I/O
// (bench.cpp:46-260, scenario.cpp:296-378) for pinning the drop-in's host logic.
static int copy_out(const std::string& v, char* out, int cap) {
  if (static_cast<int>(v.size()) + 1 > cap) {
    g_ref_err = "output buffer too small";
    return 1;
  }
  std::memcpy(out, v.c_str(), v.size() + 1);
  return 0;
}

/* read_trial_csv on each path, aggregate, aggregate_to_json().dump() */
int ref_aggregate_csv(const char** paths, int n, char* out, int cap) {
  try {
    std::vector<TrialRecord> recs;
    for (int i = 0; i < n; ++i) recs.push_back(read_trial_csv(paths[i]));
    return copy_out(aggregate_to_json(aggregate(recs)).dump(), out, cap);
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 2;
  }
}

/* read_trial_csv then write_trial_csv (the reference's own CSV text) */
int ref_csv_roundtrip(const char* in_path, const char* out_path) {
  try {
    write_trial_csv(read_trial_csv(in_path), out_path);
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 2;
  }
}

/* scenario_to_json(scenario_from_json(text)).dump(): the reference's parser
 * and writer (native model kinds only) */
int ref_scenario_json_roundtrip(const char* text, char* out, int cap) {
  try {
    return copy_out(scenario_to_json(scenario_from_json(nlohmann::json::parse(text))).dump(), out, cap);
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 2;
  }
}

/* scenario_to_json(antipodal_circle(robots, diameter, kind)).dump() */
int ref_antipodal_circle_json(int robots, double diameter, int kind, char* out, int cap) {
  try {
    return copy_out(
        scenario_to_json(antipodal_circle(robots, diameter, kind == 0 ? ModelKind::DiffDrive : ModelKind::Holo2D))
            .dump(),
        out, cap);
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 2;
  }
}

// Scenario generators (scenario.cpp:110-255), for pinning the product's.
static void export_scenario(const Scenario& s, double* starts, double* goals) {
  std::memcpy(starts, s.starts.data(), sizeof(double) * s.starts.size());
  std::memcpy(goals, s.goals.data(), sizeof(double) * s.goals.size());
}

int ref_antipodal_circle(int robots, double diameter, int kind, double robot_radius,
                         double* starts, double* goals) {
  try {
    RewardConfig rc;
    rc.robot_radius = robot_radius;
    export_scenario(antipodal_circle(robots, diameter,
                                     kind == 0 ? ModelKind::DiffDrive : ModelKind::Holo2D, rc),
                    starts, goals);
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 1;
  }
}

int ref_antipodal_sphere(int robots, double diameter, double robot_radius, double* starts,
                         double* goals) {
  try {
    RewardConfig rc;
    rc.robot_radius = robot_radius;
    export_scenario(antipodal_sphere(robots, diameter, rc), starts, goals);
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 1;
  }
}

int ref_random_square(int robots, double diameter, uint64_t seed, int kind, double robot_radius,
                      double* starts, double* goals) {
  try {
    RewardConfig rc;
    rc.robot_radius = robot_radius;
    export_scenario(random_square(robots, diameter, seed,
                                  kind == 0 ? ModelKind::DiffDrive : ModelKind::Holo2D, rc),
                    starts, goals);
    return 0;
  } catch (const std::exception& ex) {
    g_ref_err = ex.what();
    return 1;
  }
}

}  // extern "C"
