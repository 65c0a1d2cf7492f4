// planner.cpp — the C++ drop-in of the reference planner interface
// (proj/include/d4orm/{dynamics,reward,schedule,denoiser,optimizer,scenario,baselines}.hpp)
// over the B200 C-ABI (include/d4orm_cuda.h).
//
//   run_denoising   → d4orm_cuda_run_denoising (the hot path, GPU only)
//   rollout / batch_rollout → d4orm_cuda_rollout_fitness (GPU, fp64 parity
//                     instantiation: the reference's arithmetic)
//   score_weights   → d4orm_cuda_score_weights (GPU K4)
//   mc_average      → d4orm_cuda_weighted_mean (GPU K5a + K5b, fp64)
//   iterate / solve → the anytime loop (optimizer.cpp:19-102) driving the above
//
// Single-trajectory utilities (total_reward/objective/check_success on a given
// trajectory, derivative/rk4_step on one state, sample_batch on host matrices,
// the scenario generators) run on the host exactly as the reference
// defines them; none of them is on the per-step path.  Errors come back as the
// reference's exception types with its messages.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/d4orm/baselines.hpp"
#include "../../include/d4orm/denoiser.hpp"
#include "../../include/d4orm/dynamics.hpp"
#include "../../include/d4orm/gpu.hpp"
#include "../../include/d4orm/optimizer.hpp"
#include "../../include/d4orm/result.hpp"
#include "../../include/d4orm/reward.hpp"
#include "../../include/d4orm/rng.hpp"
#include "../../include/d4orm/scenario.hpp"
#include "../../include/d4orm/schedule.hpp"
#include "../../include/d4orm_cuda.h"

namespace d4orm {

// ================================================================ GPU context
namespace {

// Defaults from the environment, so a caller compiled unchanged against the
// reference headers (which has no set_gpu_options call — e.g. the reference's
// own tools/main.cpp, INTEGRATION.md Option A) can still pick the mode:
//   D4ORM_DEVICE=<n>, D4ORM_PRECISION=f32|f64, D4ORM_NOISE=philox|host,
//   D4ORM_GRAPHS=0|1.  Unset: device 0, fp32, Philox, graphs.
GpuOptions env_defaults() {
  GpuOptions o;
  if (const char* e = std::getenv("D4ORM_DEVICE")) o.device = std::atoi(e);
  if (const char* e = std::getenv("D4ORM_PRECISION")) o.precision = std::strcmp(e, "f64") == 0 ? D4ORM_PREC_F64 : D4ORM_PREC_F32;
  if (const char* e = std::getenv("D4ORM_NOISE")) o.host_noise = std::strcmp(e, "host") == 0;
  if (const char* e = std::getenv("D4ORM_GRAPHS")) o.graphs = std::atoi(e) != 0;
  return o;
}

thread_local GpuOptions g_opts = env_defaults();

struct CtxDeleter {
  void operator()(d4orm_cuda_ctx* c) const { d4orm_cuda_destroy(c); }
};

// One context per (host thread, device, precision); the problem is re-uploaded
// only when it changes, so the per-step CUDA graphs are reused across calls.
struct GpuSlot {
  std::unique_ptr<d4orm_cuda_ctx, CtxDeleter> ctx;
  int device = -1;
  std::vector<double> problem_key;
  int precision = -1, noise = -1, graphs = -1;
};
thread_local GpuSlot g_slot[2];  // [0] = drop-in precision, [1] = fp64 rollouts

void throw_for(int code, const std::string& msg) {
  if (code == D4ORM_OK) return;
  if (code == D4ORM_E_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// The status of a C-ABI call on context c, as the reference's exception.  The
// message is read only after the call returned (a `throw_for(call(c), last_error(c))`
// may evaluate last_error first and report the previous error).
void check_rc(d4orm_cuda_ctx* c, int code) {
  if (code != D4ORM_OK) throw_for(code, d4orm_cuda_last_error(c));
}

int kind_dims(ModelKind kind, int* dx, int* du, int* pd) {
  static const int DX[6] = {4, 4, 6, 2, 3, 3}, DU[6] = {2, 2, 3, 2, 3, 2}, PD[6] = {2, 2, 3, 2, 3, 2};
  const int k = static_cast<int>(kind);
  if (k < 0 || k > 5) return 1;
  *dx = DX[k];
  *du = DU[k];
  *pd = PD[k];
  return 0;
}

struct ProblemArrays {
  d4orm_problem p{};
  std::vector<double> starts, goals, oc, orad, key;
};

ProblemArrays make_problem(const Scenario& sc, const DynamicsModel& model, int horizon, double dt) {
  ProblemArrays a;
  int dx, du, pd;
  if (kind_dims(model.kind, &dx, &du, &pd)) throw std::invalid_argument("unknown model kind");
  a.p.kind = static_cast<int>(model.kind);
  a.p.dx = dx;
  a.p.du = du;
  a.p.pdim = pd;
  a.p.robots = sc.robots;
  a.p.horizon = horizon;
  a.p.dt = dt;
  for (int d = 0; d < du; ++d) {
    a.p.lower[d] = model.control_lower.size() > d ? model.control_lower[d] : -2.0;
    a.p.upper[d] = model.control_upper.size() > d ? model.control_upper[d] : 2.0;
  }
  a.starts.assign(sc.starts.data(), sc.starts.data() + sc.starts.size());
  a.goals.assign(sc.goals.data(), sc.goals.data() + sc.goals.size());
  for (const Obstacle& o : sc.obstacles.obstacles) {
    for (int j = 0; j < pd; ++j) a.oc.push_back(o.center[j]);
    a.orad.push_back(o.radius);
  }
  a.oc.push_back(0.0);
  a.orad.push_back(0.0);
  a.p.starts = a.starts.data();
  a.p.goals = a.goals.data();
  a.p.n_obstacles = static_cast<int>(sc.obstacles.size());
  a.p.obs_centers = a.oc.data();
  a.p.obs_radii = a.orad.data();
  a.p.w_t = sc.reward.w_t;
  a.p.epsilon = sc.reward.epsilon;
  a.p.robot_radius = sc.reward.robot_radius;
  a.p.goal_tolerance = sc.reward.goal_tolerance;
  a.p.obstacle_weight = sc.reward.obstacle_weight;
  a.p.effort_weight = sc.reward.effort_weight;
  a.key = {double(a.p.kind), double(horizon), dt, double(sc.robots)};
  for (int d = 0; d < du; ++d) {
    a.key.push_back(a.p.lower[d]);
    a.key.push_back(a.p.upper[d]);
  }
  a.key.insert(a.key.end(), a.starts.begin(), a.starts.end());
  a.key.insert(a.key.end(), a.goals.begin(), a.goals.end());
  a.key.insert(a.key.end(), a.oc.begin(), a.oc.end());
  a.key.insert(a.key.end(), a.orad.begin(), a.orad.end());
  for (double v : {a.p.w_t, a.p.epsilon, a.p.robot_radius, a.p.goal_tolerance, a.p.obstacle_weight, a.p.effort_weight})
    a.key.push_back(v);
  return a;
}

// Host "correctness mode" noise: exactly the reference's sample_batch draws
// (NormalStream(mix_seed(seed, i, m)), denoiser.cpp:41-43) and the
// FromScratch initial draw (mix_seed(seed, 0, 0), :145).
struct HostNoise {
  std::uint64_t seed;
  int workers;
};
thread_local HostNoise g_noise{0, 0};

int host_noise_fn(void* user, int step, int64_t m0, int64_t count, int64_t elems, double* dst) {
  const HostNoise* hn = static_cast<const HostNoise*>(user);
  const int workers = hn->workers > 0 ? hn->workers : std::max(1u, std::thread::hardware_concurrency());
  auto work = [&](int w) {
    for (int64_t j = w; j < count; j += workers) {
      const std::uint64_t ss = step == 0 ? mix_seed(hn->seed, 0, 0)
                                         : mix_seed(hn->seed, static_cast<std::uint64_t>(step),
                                                    static_cast<std::uint64_t>(m0 + j));
      NormalStream(ss).fill(dst + j * elems, elems);
    }
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < workers; ++w) pool.emplace_back(work, w);
  work(0);
  for (auto& t : pool) t.join();
  return 0;
}

// The slot's context with the given options (created on first use).
d4orm_cuda_ctx* gpu_ctx(int which, int precision, int noise, bool graphs) {
  GpuSlot& s = g_slot[which];
  const GpuOptions& o = g_opts;
  if (!s.ctx || s.device != o.device) {
    d4orm_cuda_ctx* c = nullptr;
    const int rc = d4orm_cuda_create(o.device, 0, 1, nullptr, &c);
    if (rc != D4ORM_OK)
      throw std::runtime_error("d4orm: cannot create a CUDA context on device " + std::to_string(o.device) +
                               " (the B200 library has no CPU fallback)");
    s.ctx.reset(c);
    s.device = o.device;
    s.problem_key.clear();
    s.precision = s.noise = s.graphs = -1;
  }
  d4orm_cuda_ctx* c = s.ctx.get();
  if (s.precision != precision || s.noise != noise || s.graphs != (graphs ? 1 : 0)) {
    check_rc(c, d4orm_cuda_set_options(c, precision, noise, graphs ? 1 : 0));
    s.precision = precision;
    s.noise = noise;
    s.graphs = graphs ? 1 : 0;
  }
  return c;
}

// ... and the problem uploaded (only when it changed).
d4orm_cuda_ctx* gpu(int which, const ProblemArrays& pa, int precision, int noise, bool graphs) {
  GpuSlot& s = g_slot[which];
  d4orm_cuda_ctx* c = gpu_ctx(which, precision, noise, graphs);
  if (s.problem_key != pa.key) {
    check_rc(c, d4orm_cuda_set_problem(c, &pa.p));
    s.problem_key = pa.key;
  }
  return c;
}

// A Scenario-less problem for plain rollouts (dynamics.cpp:122): positions only
// matter; goals are placed one metre off so the reward part stays defined.
Scenario rollout_scenario(const DynamicsModel& model, const Matrix& starts, int robots) {
  Scenario sc;
  sc.model_kind = model.kind;
  sc.robots = robots;
  sc.starts = starts;
  const int pd = model.position_dim();
  sc.goals = Matrix(pd, robots);
  for (int k = 0; k < robots; ++k)
    for (int j = 0; j < pd; ++j) sc.goals(j, k) = starts(j, k) + (j == 0 ? 1.0 : 0.0);
  return sc;
}

}  // namespace

void set_gpu_options(const GpuOptions& options) { g_opts = options; }
GpuOptions gpu_options() { return g_opts; }

// ================================================================== schedule
// schedule.cpp:9-36
NoiseSchedule make_schedule(int steps, double alpha_bar_final) {
  if (steps < 1) throw std::invalid_argument("make_schedule: steps must be >= 1, got " + std::to_string(steps));
  if (!(alpha_bar_final > 0.0) || !(alpha_bar_final < 1.0))
    throw std::invalid_argument("make_schedule: alpha_bar_final must lie in (0, 1), got " +
                                std::to_string(alpha_bar_final));
  NoiseSchedule s;
  s.alpha_bar = Vector(steps + 1);
  s.alpha = Vector(steps);
  s.alpha_bar[0] = 1.0;
  for (int i = 1; i <= steps; ++i) {
    s.alpha_bar[i] = std::pow(alpha_bar_final, static_cast<double>(i) / steps);
    s.alpha[i - 1] = s.alpha_bar[i] / s.alpha_bar[i - 1];
  }
  return s;
}

SamplingSpread sampling_spread(const NoiseSchedule& schedule, int i) {
  if (i < 1 || i > schedule.steps())
    throw std::invalid_argument("sampling_spread: step index " + std::to_string(i) + " outside 1.." +
                                std::to_string(schedule.steps()));
  const double ab = schedule.alpha_bar[i];
  return {1.0 / std::sqrt(ab), std::sqrt(1.0 / ab - 1.0)};
}

// ================================================================== dynamics
const char* to_string(ModelKind kind) {
  switch (kind) {
    case ModelKind::DiffDrive: return "diffdrive";
    case ModelKind::Holo2D: return "holo2d";
    case ModelKind::Holo3D: return "holo3d";
    case ModelKind::Holo2DVel: return "holo2d_vel";
    case ModelKind::Holo3DVel: return "holo3d_vel";
    case ModelKind::Unicycle: return "unicycle";
  }
  return "unknown";
}

ModelKind model_kind_from_string(const std::string& name) {
  for (int k = 0; k < 6; ++k)
    if (name == to_string(static_cast<ModelKind>(k))) return static_cast<ModelKind>(k);
  throw std::invalid_argument("unknown model kind: " + name +
                              " (expected diffdrive, holo2d, holo3d, holo2d_vel, holo3d_vel or unicycle)");
}

DynamicsModel DynamicsModel::make(ModelKind kind, double control_limit) {
  if (!(control_limit > 0.0)) throw std::invalid_argument("control_limit must be positive");
  int dx, du, pd;
  if (kind_dims(kind, &dx, &du, &pd)) throw std::invalid_argument("unknown model kind");
  DynamicsModel m;
  m.kind = kind;
  m.state_dim = dx;
  m.control_dim = du;
  m.control_lower = Vector::Constant(du, -control_limit);
  m.control_upper = Vector::Constant(du, control_limit);
  return m;
}

JointControls JointControls::zeros(int robots, int control_dim, int horizon) {
  if (robots < 1 || control_dim < 1 || horizon < 1)
    throw std::invalid_argument("JointControls::zeros: dimensions must be positive");
  return {robots, control_dim, Matrix::Zero(robots * control_dim, horizon)};
}

JointControls JointTrajectory::executed_controls() const { return {robots, control_dim, controls.leftCols(horizon())}; }

namespace {
void check_dims(const DynamicsModel& model, const Vector& x, const Vector& u, const char* what) {
  if (x.size() != model.state_dim)
    throw std::invalid_argument(std::string(what) + ": state has dimension " + std::to_string(x.size()) +
                                ", model expects " + std::to_string(model.state_dim));
  if (u.size() != model.control_dim)
    throw std::invalid_argument(std::string(what) + ": control has dimension " + std::to_string(u.size()) +
                                ", model expects " + std::to_string(model.control_dim));
}

// xdot = f(x, u) for one robot (dynamics.hpp:81-119 + the extensions).
void deriv(ModelKind kind, const double* x, const double* u, double* f) {
  switch (kind) {
    case ModelKind::DiffDrive:
      f[0] = x[3] * std::cos(x[2]); f[1] = x[3] * std::sin(x[2]); f[2] = u[0]; f[3] = u[1];
      break;
    case ModelKind::Holo2D: f[0] = x[2]; f[1] = x[3]; f[2] = u[0]; f[3] = u[1]; break;
    case ModelKind::Holo3D: f[0] = x[3]; f[1] = x[4]; f[2] = x[5]; f[3] = u[0]; f[4] = u[1]; f[5] = u[2]; break;
    case ModelKind::Holo2DVel: f[0] = u[0]; f[1] = u[1]; break;
    case ModelKind::Holo3DVel: f[0] = u[0]; f[1] = u[1]; f[2] = u[2]; break;
    case ModelKind::Unicycle: f[0] = u[0] * std::cos(x[2]); f[1] = u[0] * std::sin(x[2]); f[2] = u[1]; break;
  }
}
}  // namespace

Vector derivative(const DynamicsModel& model, const Vector& x, const Vector& u) {
  check_dims(model, x, u, "derivative");
  Vector f(model.state_dim);
  deriv(model.kind, x.data(), u.data(), f.data());
  return f;
}

// rk4_with (dynamics.hpp:123-130) in Eigen's per-element expression order.
Vector rk4_step(const DynamicsModel& model, const Vector& x, const Vector& u, double dt) {
  check_dims(model, x, u, "rk4_step");
  if (!(dt > 0.0)) throw std::invalid_argument("rk4_step: dt must be positive");
  const int n = model.state_dim;
  double k1[6], k2[6], k3[6], k4[6], tmp[6];
  deriv(model.kind, x.data(), u.data(), k1);
  for (int j = 0; j < n; ++j) tmp[j] = x[j] + (0.5 * dt) * k1[j];
  deriv(model.kind, tmp, u.data(), k2);
  for (int j = 0; j < n; ++j) tmp[j] = x[j] + (0.5 * dt) * k2[j];
  deriv(model.kind, tmp, u.data(), k3);
  for (int j = 0; j < n; ++j) tmp[j] = x[j] + dt * k3[j];
  deriv(model.kind, tmp, u.data(), k4);
  Vector out(n);
  for (int j = 0; j < n; ++j) out[j] = x[j] + (dt / 6.0) * (((k1[j] + 2.0 * k2[j]) + 2.0 * k3[j]) + k4[j]);
  for (int j = 0; j < n; ++j)
    if (!std::isfinite(out[j])) throw std::runtime_error("rk4_step: non-finite state after step");
  return out;
}

namespace {
void check_rollout_args(const DynamicsModel& model, const Matrix& starts, const JointControls& c, double dt) {
  if (!(dt > 0.0)) throw std::invalid_argument("rollout: dt must be positive");
  if (starts.rows() != model.state_dim)
    throw std::invalid_argument("rollout: starts have " + std::to_string(starts.rows()) +
                                " state entries, model expects " + std::to_string(model.state_dim));
  if (static_cast<int>(starts.cols()) != c.robots)
    throw std::invalid_argument("rollout: " + std::to_string(starts.cols()) + " start states for " +
                                std::to_string(c.robots) + " robots");
  if (c.control_dim != model.control_dim) throw std::invalid_argument("rollout: control dimension mismatch");
  if (c.robots < 1 || c.horizon() < 1) throw std::invalid_argument("rollout: empty control trajectory");
  if (!starts.allFinite()) throw std::invalid_argument("rollout: non-finite start state");
}

std::vector<JointTrajectory> gpu_rollouts(const DynamicsModel& model, const Matrix& starts,
                                          const std::vector<const JointControls*>& batch, double dt, bool batch_msg) {
  const int R = batch[0]->robots, T = batch[0]->horizon();
  const Scenario sc = rollout_scenario(model, starts, R);
  const ProblemArrays pa = make_problem(sc, model, T, dt);
  d4orm_cuda_ctx* c = gpu(1, pa, D4ORM_PREC_F64, D4ORM_NOISE_HOST, false);
  const int64_t E = static_cast<int64_t>(R) * model.control_dim * T, n = static_cast<int64_t>(batch.size());
  std::vector<double> u(static_cast<size_t>(n * E));
  for (int64_t m = 0; m < n; ++m) std::memcpy(u.data() + m * E, batch[m]->u.data(), sizeof(double) * E);
  const int64_t NS = static_cast<int64_t>(R) * model.state_dim * (T + 1), NC = static_cast<int64_t>(R) * model.control_dim * (T + 1);
  std::vector<double> st(static_cast<size_t>(n * NS)), ct(static_cast<size_t>(n * NC));
  const int rc = d4orm_cuda_rollout_fitness(c, u.data(), n, st.data(), ct.data(), nullptr, nullptr);
  if (rc != D4ORM_OK) {
    std::string msg = d4orm_cuda_last_error(c);
    if (!batch_msg) {  // single rollout: the reference's own message, without the batch prefix
      const auto p = msg.find("rollout: ");
      if (p != std::string::npos) msg = msg.substr(p);
    }
    throw_for(rc, msg);
  }
  std::vector<JointTrajectory> out(static_cast<size_t>(n));
  for (int64_t m = 0; m < n; ++m) {
    JointTrajectory& tr = out[m];
    tr.robots = R;
    tr.state_dim = model.state_dim;
    tr.control_dim = model.control_dim;
    tr.dt = dt;
    tr.states = Matrix(R * model.state_dim, T + 1);
    tr.controls = Matrix(R * model.control_dim, T + 1);
    std::memcpy(tr.states.data(), st.data() + m * NS, sizeof(double) * NS);
    std::memcpy(tr.controls.data(), ct.data() + m * NC, sizeof(double) * NC);
  }
  return out;
}
}  // namespace

JointTrajectory rollout(const DynamicsModel& model, const Matrix& starts, const JointControls& controls, double dt) {
  check_rollout_args(model, starts, controls, dt);
  return gpu_rollouts(model, starts, {&controls}, dt, false)[0];
}

std::vector<JointTrajectory> batch_rollout(const DynamicsModel& model, const Matrix& starts,
                                           const std::vector<JointControls>& batch, double dt, int) {
  if (batch.empty()) return {};
  std::vector<const JointControls*> ptrs;
  for (const auto& b : batch) {
    check_rollout_args(model, starts, b, dt);
    if (b.horizon() != batch[0].horizon()) throw std::invalid_argument("batch_rollout: members differ in horizon");
    ptrs.push_back(&b);
  }
  return gpu_rollouts(model, starts, ptrs, dt, true);
}

// ==================================================================== reward
// reward.cpp:35-200, evaluated on one given trajectory.
double goal_reward(const Matrix& states, int t, const Vector& start_position, const Vector& goal_position) {
  const int pd = static_cast<int>(goal_position.size());
  const double sd = (start_position - goal_position).norm();
  if (!(sd > 0.0)) throw std::invalid_argument("goal_reward: start coincides with goal");
  return 1.0 - (states.col(t).head(pd) - goal_position).norm() / sd;
}

double safety_reward(const Matrix& positions, int k, const RewardConfig& config) {
  const int n = static_cast<int>(positions.cols()), pd = static_cast<int>(positions.rows());
  const double m = 2.0 * config.robot_radius + config.epsilon, m2 = m * m;
  for (int l = 0; l < n; ++l) {
    if (l == k) continue;
    double s = 0.0;
    for (int j = 0; j < pd; ++j) {
      const double d = positions(j, k) - positions(j, l);
      s += d * d;
    }
    if (s <= m2) return -1.0;
  }
  return 0.0;
}

double obstacle_penalty(const Vector& position, double robot_radius, const ObstacleSet& obstacles) {
  for (const Obstacle& o : obstacles.obstacles) {
    const double lim = o.radius + robot_radius;
    if ((position - o.center).squaredNorm() <= lim * lim) return -1.0;
  }
  return 0.0;
}

namespace {
void check_consistent(const JointTrajectory& tr, const Scenario& sc, const char* what) {
  if (tr.robots != sc.robots)
    throw std::invalid_argument(std::string(what) + ": trajectory has " + std::to_string(tr.robots) +
                                " robots, scenario " + std::to_string(sc.robots));
  if (tr.state_dim != static_cast<int>(sc.starts.rows()))
    throw std::invalid_argument(std::string(what) + ": state dimension mismatch");
}
}  // namespace

double total_reward(const JointTrajectory& tr, const Scenario& sc, const RewardConfig& cfg) {
  check_consistent(tr, sc, "total_reward");
  const int n = tr.robots, H = tr.horizon(), pd = sc.position_dim(), dx = tr.state_dim;
  const double m = 2.0 * cfg.robot_radius + cfg.epsilon, m2 = m * m;
  std::vector<double> sd(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) {
    sd[k] = (sc.start_position(k) - sc.goals.col(k)).norm();
    if (!(sd[k] > 0.0))
      throw std::invalid_argument("total_reward: robot " + std::to_string(k) + " starts on its goal (degenerate scenario)");
  }
  double sum = 0.0;
  for (int t = 1; t <= H; ++t) {
    const double* col = tr.states.data() + static_cast<size_t>(t) * tr.states.rows();
    for (int k = 0; k < n; ++k) {
      double g = 0.0;
      for (int j = 0; j < pd; ++j) {
        const double d = col[k * dx + j] - sc.goals(j, k);
        g += d * d;
      }
      double v = 1.0 - std::sqrt(g) / sd[k];
      for (int l = 0; l < n; ++l) {
        if (l == k) continue;
        double s = 0.0;
        for (int j = 0; j < pd; ++j) {
          const double d = col[k * dx + j] - col[l * dx + j];
          s += d * d;
        }
        if (s <= m2) {
          v -= cfg.w_t;
          break;
        }
      }
      for (const Obstacle& o : sc.obstacles.obstacles) {
        double s = 0.0;
        for (int j = 0; j < pd; ++j) {
          const double d = col[k * dx + j] - o.center[j];
          s += d * d;
        }
        const double lim = o.radius + cfg.robot_radius;
        if (s <= lim * lim) {
          v -= cfg.obstacle_weight;
          break;
        }
      }
      sum += v;
    }
  }
  if (cfg.effort_weight != 0.0) {
    double e = 0.0;
    for (int t = 0; t < H; ++t)
      for (int r = 0; r < tr.controls.rows(); ++r) e += tr.controls(r, t) * tr.controls(r, t);
    sum -= cfg.effort_weight * e;
  }
  return sum / (static_cast<double>(n) * H);
}

double total_reward(const JointTrajectory& tr, const Scenario& sc) { return total_reward(tr, sc, sc.reward); }

double objective(const JointTrajectory& tr, const Scenario& sc, const RewardConfig& cfg) {
  check_consistent(tr, sc, "objective");
  const int n = tr.robots, H = tr.horizon(), pd = sc.position_dim();
  const double tol2 = cfg.goal_tolerance * cfg.goal_tolerance;
  long hits = 0;
  for (int t = 1; t <= H; ++t)
    for (int k = 0; k < n; ++k) {
      double g = 0.0;
      for (int j = 0; j < pd; ++j) {
        const double d = tr.states(k * tr.state_dim + j, t) - sc.goals(j, k);
        g += d * d;
      }
      if (g <= tol2) ++hits;
    }
  return static_cast<double>(hits) / (static_cast<double>(n) * H);
}

double objective(const JointTrajectory& tr, const Scenario& sc) { return objective(tr, sc, sc.reward); }

SuccessReport check_success(const JointTrajectory& tr, const Scenario& sc, const RewardConfig& cfg) {
  check_consistent(tr, sc, "check_success");
  const int n = tr.robots, H = tr.horizon(), pd = sc.position_dim();
  const double s2 = 4.0 * cfg.robot_radius * cfg.robot_radius;
  for (int t = 0; t <= H; ++t)
    for (int k = 0; k < n; ++k) {
      const Vector pk = tr.position(k, t, pd);
      for (int l = k + 1; l < n; ++l)
        if ((pk - tr.position(l, t, pd)).squaredNorm() <= s2)
          return {false, "safety: robots " + std::to_string(k) + " and " + std::to_string(l) + " within 2*R_a at step " +
                             std::to_string(t)};
      for (std::size_t o = 0; o < sc.obstacles.size(); ++o) {
        const Obstacle& ob = sc.obstacles.obstacles[o];
        const double lim = ob.radius + cfg.robot_radius;
        if ((pk - ob.center).squaredNorm() <= lim * lim)
          return {false, "obstacle: robot " + std::to_string(k) + " hits obstacle " + std::to_string(o) + " at step " +
                             std::to_string(t)};
      }
    }
  for (int k = 0; k < n; ++k) {
    const double e = (tr.position(k, H, pd) - sc.goals.col(k)).norm();
    if (e > cfg.goal_tolerance)
      return {false, "terminal: robot " + std::to_string(k) + " ends " + std::to_string(e) + " m from its goal (tolerance " +
                         std::to_string(cfg.goal_tolerance) + ")"};
  }
  return {true, ""};
}

SuccessReport check_success(const JointTrajectory& tr, const Scenario& sc) { return check_success(tr, sc, sc.reward); }

// ================================================================== denoiser
std::vector<JointControls> sample_batch(const JointControls& current, const NoiseSchedule& schedule, int i, int batch,
                                        std::uint64_t seed, int workers) {
  if (batch < 1) throw std::invalid_argument("sample_batch: batch must be >= 1");
  const SamplingSpread sp = sampling_spread(schedule, i);
  std::vector<JointControls> out(static_cast<size_t>(batch));
  const int W = workers > 0 ? workers : std::max(1u, std::thread::hardware_concurrency());
  auto work = [&](int w) {
    for (int m = w; m < batch; m += W) {
      Matrix z(current.u.rows(), current.u.cols());
      NormalStream(mix_seed(seed, static_cast<std::uint64_t>(i), static_cast<std::uint64_t>(m))).fill(z.data(), z.size());
      out[m] = {current.robots, current.control_dim, sp.mean_scale * current.u + sp.std * z};
    }
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < std::min(W, batch); ++w) pool.emplace_back(work, w);
  work(0);
  for (auto& t : pool) t.join();
  return out;
}

Vector score_weights(const Vector& rewards, double lambda) {
  const int64_t m = rewards.size();
  if (m < 2) throw std::invalid_argument("score_weights: need at least 2 rewards");
  if (!(lambda > 0.0)) throw std::invalid_argument("score_weights: lambda must be positive");
  for (int64_t j = 0; j < m; ++j)
    if (!std::isfinite(rewards[j])) throw std::runtime_error("score_weights: non-finite reward for sample " + std::to_string(j));
  d4orm_cuda_ctx* c = nullptr;
  {
    GpuSlot& s = g_slot[0];
    if (!s.ctx || s.device != g_opts.device) {
      const int rc = d4orm_cuda_create(g_opts.device, 0, 1, nullptr, &c);
      if (rc != D4ORM_OK) throw std::runtime_error("d4orm: cannot create a CUDA context");
      s.ctx.reset(c);
      s.device = g_opts.device;
      s.problem_key.clear();
      s.precision = s.noise = s.graphs = -1;
    }
    c = s.ctx.get();
  }
  Vector w(m);
  check_rc(c, d4orm_cuda_score_weights(c, rewards.data(), m, lambda, w.data(), nullptr));
  return w;
}

// mc_average (denoiser.cpp:92-108) on the GPU (d4orm_cuda_weighted_mean, K5a +
// K5b) in the reference's fp64 arithmetic: each 256-sample chunk in ascending
// m, the chunks by a fixed pairwise tree.
JointControls mc_average(const std::vector<JointControls>& samples, const Vector& weights) {
  if (samples.empty()) throw std::invalid_argument("mc_average: empty sample set");
  if (static_cast<Index>(samples.size()) != weights.size())
    throw std::invalid_argument("mc_average: weight count does not match sample count");
  const Index rows = samples[0].u.rows(), cols = samples[0].u.cols();
  for (const auto& smp : samples)
    if (smp.u.rows() != rows || smp.u.cols() != cols)
      throw std::invalid_argument("mc_average: samples differ in shape");
  const int64_t m = static_cast<int64_t>(samples.size()), E = static_cast<int64_t>(rows) * cols;
  JointControls out{samples[0].robots, samples[0].control_dim, Matrix::Zero(rows, cols)};
  if (E == 0) return out;
  std::vector<double> flat(static_cast<size_t>(m * E));
  for (int64_t j = 0; j < m; ++j) std::memcpy(flat.data() + j * E, samples[j].u.data(), sizeof(double) * E);
  d4orm_cuda_ctx* c = gpu_ctx(1, D4ORM_PREC_F64, D4ORM_NOISE_HOST, false);
  check_rc(c, d4orm_cuda_weighted_mean(c, flat.data(), weights.data(), m, E, out.u.data()));
  return out;
}

JointControls denoise_step(const JointControls& averaged, const NoiseSchedule& schedule, int i) {
  if (i < 1 || i > schedule.steps())
    throw std::invalid_argument("denoise_step: step index " + std::to_string(i) + " outside 1.." +
                                std::to_string(schedule.steps()));
  return {averaged.robots, averaged.control_dim, std::sqrt(schedule.alpha_bar[i - 1]) * averaged.u};
}

DenoiseResult run_denoising(const JointControls& base, const Scenario& scenario, const DynamicsModel& model,
                            const NoiseSchedule& schedule, const DenoiserConfig& config, double dt) {
  // denoiser.cpp:122-135
  if (config.batch < 2) throw std::invalid_argument("run_denoising: batch must be >= 2");
  if (!(config.lambda > 0.0)) throw std::invalid_argument("run_denoising: lambda must be > 0");
  if (config.steps != schedule.steps())
    throw std::invalid_argument("run_denoising: config.steps (" + std::to_string(config.steps) +
                                ") does not match the schedule (" + std::to_string(schedule.steps()) + ")");
  if (base.robots != scenario.robots)
    throw std::invalid_argument("run_denoising: base has " + std::to_string(base.robots) + " robots, scenario " +
                                std::to_string(scenario.robots));
  if (base.control_dim != model.control_dim) throw std::invalid_argument("run_denoising: control dimension mismatch");
  const ProblemArrays pa = make_problem(scenario, model, base.horizon(), dt);
  const bool host = g_opts.host_noise;
  d4orm_cuda_ctx* c = gpu(0, pa, g_opts.precision, host ? D4ORM_NOISE_HOST : D4ORM_NOISE_PHILOX, g_opts.graphs);
  if (host) {
    g_noise = {config.seed, config.workers};
    check_rc(c, d4orm_cuda_set_noise_fn(c, host_noise_fn, &g_noise));
  }
  d4orm_denoiser_config dc{};
  dc.steps = config.steps;
  dc.batch = config.batch;
  dc.lambda = config.lambda;
  dc.alpha_bar_final = config.alpha_bar_final;
  dc.seed = config.seed;
  dc.mode = config.mode == DenoiseMode::Deformation ? D4ORM_DEFORMATION : D4ORM_FROM_SCRATCH;
  dc.alpha_bar = schedule.alpha_bar.data();
  DenoiseResult res;
  res.variable = {base.robots, base.control_dim, Matrix(base.u.rows(), base.u.cols())};
  std::vector<d4orm_trace_rec> tr(static_cast<size_t>(config.steps));
  check_rc(c, d4orm_cuda_run_denoising(c, base.u.data(), &dc, res.variable.u.data(), tr.data()));
  res.trace.steps.reserve(tr.size());
  for (const auto& t : tr) res.trace.steps.push_back({t.step, t.best_reward, t.mean_reward, t.weight_entropy});
  return res;
}

// ================================================================= optimizer
namespace {
struct IterateOutcome {
  JointTrajectory trajectory;
  DenoiseTrace trace;
};

IterateOutcome iterate_impl(const JointTrajectory& base, const Scenario& scenario, const DynamicsModel& model,
                            const NoiseSchedule& schedule, const DenoiserConfig& dcfg, double dt) {
  DenoiserConfig cfg = dcfg;
  cfg.mode = DenoiseMode::Deformation;
  const JointControls base_controls = base.executed_controls();
  DenoiseResult den = run_denoising(base_controls, scenario, model, schedule, cfg, dt);
  const JointControls updated{base_controls.robots, base_controls.control_dim, base_controls.u + den.variable.u};
  return {rollout(model, scenario.starts, updated, dt), std::move(den.trace)};
}

void check_model(const Scenario& scenario, const DynamicsModel& model) {
  if (scenario.model_kind != model.kind)
    throw std::invalid_argument("solve: scenario model kind does not match the dynamics model");
  if (scenario.starts.rows() != model.state_dim)
    throw std::invalid_argument("solve: scenario state dimension does not match the model");
}
}  // namespace

JointTrajectory iterate(const JointTrajectory& base, const Scenario& scenario, const DynamicsModel& model,
                        const NoiseSchedule& schedule, const OptimizerConfig& config) {
  return iterate_impl(base, scenario, model, schedule, config.denoiser, base.dt).trajectory;
}

namespace {
int reseed_host_noise(void* user, int, std::uint64_t seed_it) {  // seed of iteration it (optimizer.cpp:76)
  static_cast<HostNoise*>(user)->seed = seed_it;
  return 0;
}
}  // namespace

// The anytime loop on the device (d4orm_cuda_solve): every iteration's
// denoising, final rollout, total_reward / objective / check_success and best
// tracking run in one CUDA graph; the host reads one record per iteration and
// decides stop_on_success / the deadline exactly where optimizer.cpp:91-92 does.
SolveResult solve(const Scenario& scenario, const DynamicsModel& model, const OptimizerConfig& config) {
  if (config.max_iterations < 1) throw std::invalid_argument("solve: max_iterations must be >= 1");
  if (config.horizon < 2) throw std::invalid_argument("solve: horizon must be >= 2");
  if (!(config.dt > 0.0)) throw std::invalid_argument("solve: dt must be positive");
  validate_scenario(scenario);
  check_model(scenario, model);
  const NoiseSchedule schedule = make_schedule(config.denoiser.steps, config.denoiser.alpha_bar_final);
  const auto t0 = std::chrono::steady_clock::now();
  const DenoiserConfig& dcfg = config.denoiser;
  if (dcfg.batch < 2) throw std::invalid_argument("run_denoising: batch must be >= 2");
  if (!(dcfg.lambda > 0.0)) throw std::invalid_argument("run_denoising: lambda must be > 0");
  const ProblemArrays pa = make_problem(scenario, model, config.horizon, config.dt);
  const bool host = g_opts.host_noise;
  d4orm_cuda_ctx* c = gpu(0, pa, g_opts.precision, host ? D4ORM_NOISE_HOST : D4ORM_NOISE_PHILOX, g_opts.graphs);
  if (host) {
    g_noise = {dcfg.seed, dcfg.workers};
    check_rc(c, d4orm_cuda_set_noise_fn(c, host_noise_fn, &g_noise));
  }
  d4orm_solve_config sc{};
  sc.max_iterations = config.max_iterations;
  sc.stop_on_success = config.stop_on_success ? 1 : 0;
  sc.deadline_seconds = config.deadline_seconds ? *config.deadline_seconds : 0.0;
  sc.denoiser.steps = dcfg.steps;
  sc.denoiser.batch = dcfg.batch;
  sc.denoiser.lambda = dcfg.lambda;
  sc.denoiser.alpha_bar_final = dcfg.alpha_bar_final;
  sc.denoiser.seed = dcfg.seed;
  sc.denoiser.mode = D4ORM_DEFORMATION;
  sc.denoiser.alpha_bar = schedule.alpha_bar.data();
  sc.on_iteration = host ? reseed_host_noise : nullptr;
  sc.on_iteration_user = &g_noise;
  const int R = scenario.robots, H = config.horizon;
  SolveResult result;
  result.best_trajectory = {R, model.state_dim, model.control_dim, config.dt,
                            Matrix(static_cast<Index>(R) * model.state_dim, H + 1),
                            Matrix(static_cast<Index>(R) * model.control_dim, H + 1)};
  std::vector<d4orm_iteration_rec> recs(static_cast<size_t>(config.max_iterations));
  std::vector<d4orm_trace_rec> tr(static_cast<size_t>(config.max_iterations) * dcfg.steps);
  int used = 0, ok = 0;
  double best = 0.0;
  check_rc(c, d4orm_cuda_solve(c, &sc, result.best_trajectory.states.data(), result.best_trajectory.controls.data(),
                             recs.data(), tr.data(), &used, &best, &ok));
  for (int it = 0; it < used; ++it) {
    result.per_iteration.push_back({recs[it].reward, recs[it].objective, recs[it].success != 0, recs[it].elapsed});
    DenoiseTrace t;
    for (int s = 0; s < dcfg.steps; ++s) {
      const d4orm_trace_rec& r = tr[static_cast<size_t>(it) * dcfg.steps + s];
      t.steps.push_back({r.step, r.best_reward, r.mean_reward, r.weight_entropy});
    }
    result.traces.push_back(std::move(t));
  }
  result.best_reward = best;
  result.success = ok != 0;
  result.iterations_used = used;
  result.total_denoise_steps = static_cast<long long>(used) * dcfg.steps;
  result.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return result;
}

// ================================================================= baselines
std::vector<int> select_elites(const Vector& rewards, int count) {
  if (count < 1 || count > rewards.size()) throw std::invalid_argument("select_elites: elite count out of range");
  std::vector<int> order(static_cast<std::size_t>(rewards.size()));
  for (std::size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
  std::stable_sort(order.begin(), order.end(), [&rewards](int a, int b) { return rewards[a] > rewards[b]; });
  order.resize(static_cast<std::size_t>(count));
  std::sort(order.begin(), order.end());
  return order;
}

namespace {
template <class Fn>
SolveResult baseline_result(const Scenario& scenario, const DynamicsModel& model, int horizon, double dt, int iterations,
                            std::uint64_t seed, int workers, const char* what, Fn&& call) {
  validate_scenario(scenario);
  if (scenario.model_kind != model.kind)
    throw std::invalid_argument(std::string(what) + ": scenario model kind mismatch");
  const ProblemArrays pa = make_problem(scenario, model, horizon, dt);
  const bool host = g_opts.host_noise;
  d4orm_cuda_ctx* c = gpu(0, pa, g_opts.precision, host ? D4ORM_NOISE_HOST : D4ORM_NOISE_PHILOX, g_opts.graphs);
  if (host) {  // the provider's step is the iteration: NormalStream(mix_seed(seed, it, m))
    g_noise = {seed, workers};
    check_rc(c, d4orm_cuda_set_noise_fn(c, host_noise_fn, &g_noise));
  }
  const auto t0 = std::chrono::steady_clock::now();
  const int R = scenario.robots;
  SolveResult result;
  result.best_trajectory = {R, model.state_dim, model.control_dim, dt,
                            Matrix(static_cast<Index>(R) * model.state_dim, horizon + 1),
                            Matrix(static_cast<Index>(R) * model.control_dim, horizon + 1)};
  std::vector<d4orm_iteration_rec> recs(static_cast<size_t>(std::max(iterations, 1)));
  int used = 0, ok = 0;
  double best = 0.0;
  check_rc(c, call(c, result.best_trajectory.states.data(), result.best_trajectory.controls.data(), recs.data(), &used,
                   &best, &ok));
  for (int it = 0; it < used; ++it)
    result.per_iteration.push_back({recs[it].reward, recs[it].objective, recs[it].success != 0, recs[it].elapsed});
  result.best_reward = best;
  result.success = ok != 0;
  result.iterations_used = used;
  result.total_denoise_steps = used;
  result.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return result;
}
}  // namespace

SolveResult mppi_solve(const Scenario& scenario, const DynamicsModel& model, const MppiConfig& config) {
  d4orm_mppi_config mc{};
  mc.batch = config.batch;
  mc.lambda = config.lambda;
  mc.sigma = config.sigma;
  mc.iterations = config.iterations;
  mc.seed = config.seed;
  mc.stop_on_success = config.stop_on_success ? 1 : 0;
  mc.deadline_seconds = config.deadline_seconds ? *config.deadline_seconds : 0.0;
  return baseline_result(scenario, model, config.horizon, config.dt, config.iterations, config.seed, config.workers,
                         "mppi_solve", [&](d4orm_cuda_ctx* c, double* st, double* ct, d4orm_iteration_rec* r, int* u,
                                           double* b, int* ok) {
                           return d4orm_cuda_mppi_solve(c, &mc, st, ct, r, u, b, ok);
                         });
}

SolveResult cem_solve(const Scenario& scenario, const DynamicsModel& model, const CemConfig& config) {
  d4orm_cem_config cc{};
  cc.batch = config.batch;
  cc.elite_fraction = config.elite_fraction;
  cc.initial_std = config.initial_std;
  cc.min_std = config.min_std;
  cc.iterations = config.iterations;
  cc.seed = config.seed;
  cc.stop_on_success = config.stop_on_success ? 1 : 0;
  cc.deadline_seconds = config.deadline_seconds ? *config.deadline_seconds : 0.0;
  return baseline_result(scenario, model, config.horizon, config.dt, config.iterations, config.seed, config.workers,
                         "cem_solve", [&](d4orm_cuda_ctx* c, double* st, double* ct, d4orm_iteration_rec* r, int* u,
                                          double* b, int* ok) {
                           return d4orm_cuda_cem_solve(c, &cc, st, ct, r, u, b, ok);
                         });
}

}  // namespace d4orm
