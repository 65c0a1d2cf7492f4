// io.cpp — scenario JSON schema v1 and the solve outputs of the C++ drop-in.
//
// scenario_to_json / scenario_from_json restate scenario.cpp:296-378 (the
// state dimension follows the model kind, so the BASELINE extension kinds
// round-trip too — the reference's `Holo3D ? 6 : 4` only knows its own three);
// trajectory.json / denoise_trace.csv follow cmd_solve (tools/main.cpp:
// 309-377); read_trajectory_json replays an export.
#include <filesystem>
#include <fstream>
#include <stdexcept>

#include "../../include/d4orm/io.hpp"
#include "../../include/d4orm/reward.hpp"

namespace d4orm {

nlohmann::json scenario_to_json(const Scenario& s) {
  nlohmann::json j;
  j["schema_version"] = 1;
  j["id"] = s.id;
  j["model"] = to_string(s.model_kind);
  j["robots"] = s.robots;
  j["workspace_diameter"] = s.workspace_diameter;
  j["starts"] = nlohmann::json::array();
  j["goals"] = nlohmann::json::array();
  for (int k = 0; k < s.robots; ++k) {
    const double* st = s.starts.data() + static_cast<size_t>(k) * s.starts.rows();
    const double* go = s.goals.data() + static_cast<size_t>(k) * s.goals.rows();
    j["starts"].push_back(std::vector<double>(st, st + s.starts.rows()));
    j["goals"].push_back(std::vector<double>(go, go + s.goals.rows()));
  }
  j["obstacles"] = nlohmann::json::array();
  for (const Obstacle& o : s.obstacles.obstacles) {
    nlohmann::json e;
    e["center"] = std::vector<double>(o.center.data(), o.center.data() + o.center.size());
    e["radius"] = o.radius;
    j["obstacles"].push_back(e);
  }
  j["reward"] = {{"w_t", s.reward.w_t},
                 {"epsilon", s.reward.epsilon},
                 {"robot_radius", s.reward.robot_radius},
                 {"goal_tolerance", s.reward.goal_tolerance},
                 {"obstacle_weight", s.reward.obstacle_weight}};
  return j;
}

Scenario scenario_from_json(const nlohmann::json& j) {
  if (!j.contains("schema_version") || j.at("schema_version").get<int>() != 1)
    throw std::invalid_argument("scenario json: unsupported schema_version");
  Scenario s;
  s.id = j.at("id").get<std::string>();
  s.model_kind = model_kind_from_string(j.at("model").get<std::string>());
  s.robots = j.at("robots").get<int>();
  s.workspace_diameter = j.at("workspace_diameter").get<double>();
  const auto& starts = j.at("starts");
  const auto& goals = j.at("goals");
  if (starts.size() != static_cast<size_t>(s.robots) || goals.size() != static_cast<size_t>(s.robots))
    throw std::invalid_argument("scenario json: starts/goals count does not match robots");
  const int dx = state_dim_of(s.model_kind), pd = s.position_dim();
  s.starts = Matrix(dx, s.robots);
  s.goals = Matrix(pd, s.robots);
  for (int k = 0; k < s.robots; ++k) {
    const auto st = starts.at(k).get<std::vector<double>>();
    const auto go = goals.at(k).get<std::vector<double>>();
    if (static_cast<int>(st.size()) != dx || static_cast<int>(go.size()) != pd)
      throw std::invalid_argument("scenario json: state or goal dimension mismatch");
    for (int q = 0; q < dx; ++q) s.starts(q, k) = st[q];
    for (int q = 0; q < pd; ++q) s.goals(q, k) = go[q];
  }
  for (const auto& e : j.value("obstacles", nlohmann::json::array())) {
    Obstacle o;
    const auto c = e.at("center").get<std::vector<double>>();
    o.center = Vector(static_cast<Index>(c.size()));
    for (size_t q = 0; q < c.size(); ++q) o.center[static_cast<Index>(q)] = c[q];
    o.radius = e.at("radius").get<double>();
    s.obstacles.obstacles.push_back(o);
  }
  if (j.contains("reward")) {
    const auto& r = j.at("reward");
    s.reward.w_t = r.value("w_t", s.reward.w_t);
    s.reward.epsilon = r.value("epsilon", s.reward.epsilon);
    s.reward.robot_radius = r.value("robot_radius", s.reward.robot_radius);
    s.reward.goal_tolerance = r.value("goal_tolerance", s.reward.goal_tolerance);
    s.reward.obstacle_weight = r.value("obstacle_weight", s.reward.obstacle_weight);
  }
  validate_scenario(s);
  return s;
}

nlohmann::json trajectory_to_json(const JointTrajectory& tr) {
  nlohmann::json robots = nlohmann::json::array();
  const int H = tr.horizon();
  for (int k = 0; k < tr.robots; ++k) {
    nlohmann::json steps = nlohmann::json::array();
    for (int t = 0; t <= H; ++t) {
      const double* x = tr.states.data() + static_cast<size_t>(t) * tr.states.rows() + static_cast<size_t>(k) * tr.state_dim;
      const double* u =
          tr.controls.data() + static_cast<size_t>(t) * tr.controls.rows() + static_cast<size_t>(k) * tr.control_dim;
      steps.push_back({{"time", t * tr.dt},
                       {"state", std::vector<double>(x, x + tr.state_dim)},
                       {"control", std::vector<double>(u, u + tr.control_dim)}});
    }
    robots.push_back({{"robot", k}, {"steps", steps}});
  }
  return robots;
}

nlohmann::json solve_output_json(const Scenario& scenario, const SolveResult& result, const std::string& solver,
                                 const nlohmann::json& config) {
  nlohmann::json out;
  out["schema_version"] = 1;
  out["scenario"] = scenario_to_json(scenario);
  out["config"] = config.is_null() ? nlohmann::json::object() : config;
  out["config"]["solver.name"] = solver;
  out["result"] = {{"success", result.success},
                   {"reward", result.best_reward},
                   {"objective", objective(result.best_trajectory, scenario)},
                   {"iterations", result.iterations_used},
                   {"total_steps", result.total_denoise_steps},
                   {"dt", result.best_trajectory.dt}};
  out["result"]["robots"] = trajectory_to_json(result.best_trajectory);
  return out;
}

void write_solve_outputs(const std::string& out_dir, const Scenario& scenario, const SolveResult& result,
                         const std::string& solver, const nlohmann::json& config) {
  namespace fs = std::filesystem;
  fs::create_directories(out_dir);
  const fs::path traj = fs::path(out_dir) / "trajectory.json";
  std::ofstream tf(traj);
  if (!tf) throw std::runtime_error("cannot write " + traj.string());
  tf << solve_output_json(scenario, result, solver, config).dump(2) << '\n';
  const fs::path trace = fs::path(out_dir) / "denoise_trace.csv";
  std::ofstream cf(trace);
  if (!cf) throw std::runtime_error("cannot write " + trace.string());
  cf << "iteration,step,best_sample_reward,mean_sample_reward,weight_entropy\n";
  cf.precision(17);
  for (size_t it = 0; it < result.traces.size(); ++it)
    for (const auto& st : result.traces[it].steps)
      cf << it + 1 << ',' << st.step << ',' << st.best_reward << ',' << st.mean_reward << ',' << st.weight_entropy
         << '\n';
}

LoadedTrajectory read_trajectory_json(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw std::runtime_error("read_trajectory_json: cannot open " + path);
  const nlohmann::json j = nlohmann::json::parse(f);
  if (j.value("schema_version", 0) != 1) throw std::invalid_argument("trajectory json: unsupported schema_version");
  LoadedTrajectory out;
  out.scenario = scenario_from_json(j.at("scenario"));
  out.result = j.at("result");
  const nlohmann::json robots = out.result.at("robots");
  out.result.erase("robots");
  const Scenario& s = out.scenario;
  if (robots.size() != static_cast<size_t>(s.robots))
    throw std::invalid_argument("trajectory json: robot count does not match the scenario");
  const int dx = state_dim_of(s.model_kind);
  const int H = static_cast<int>(robots.at(0).at("steps").size()) - 1;
  const int du = static_cast<int>(robots.at(0).at("steps").at(0).at("control").size());
  JointTrajectory& tr = out.trajectory;
  tr.robots = s.robots;
  tr.state_dim = dx;
  tr.control_dim = du;
  tr.dt = out.result.at("dt").get<double>();
  tr.states = Matrix(static_cast<Index>(s.robots) * dx, H + 1);
  tr.controls = Matrix(static_cast<Index>(s.robots) * du, H + 1);
  for (int k = 0; k < s.robots; ++k) {
    const auto& steps = robots.at(k).at("steps");
    if (static_cast<int>(steps.size()) != H + 1) throw std::invalid_argument("trajectory json: ragged robot steps");
    for (int t = 0; t <= H; ++t) {
      const auto x = steps.at(t).at("state").get<std::vector<double>>();
      const auto u = steps.at(t).at("control").get<std::vector<double>>();
      if (static_cast<int>(x.size()) != dx || static_cast<int>(u.size()) != du)
        throw std::invalid_argument("trajectory json: state or control dimension mismatch");
      for (int q = 0; q < dx; ++q) tr.states(static_cast<Index>(k) * dx + q, t) = x[q];
      for (int q = 0; q < du; ++q) tr.controls(static_cast<Index>(k) * du + q, t) = u[q];
    }
  }
  return out;
}

}  // namespace d4orm
