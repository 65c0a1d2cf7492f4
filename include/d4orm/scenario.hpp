#pragma once
// Drop-in for proj/include/d4orm/scenario.hpp:17-61 (problem setup and the
// scenario JSON schema v1; the JSON functions are declared when nlohmann's
// single header json.hpp is on the include path, as in the reference build).
#include <cstdint>
#include <string>
#include <vector>

#include "d4orm/dynamics.hpp"
#include "d4orm/reward.hpp"
#include "d4orm/types.hpp"

namespace d4orm {

struct Scenario {
  std::string id;
  ModelKind model_kind{ModelKind::Holo2D};
  int robots{0};
  Matrix starts;  // state_dim x robots
  Matrix goals;   // position_dim x robots
  double workspace_diameter{4.0};
  ObstacleSet obstacles;
  RewardConfig reward;

  int position_dim() const {
    return (model_kind == ModelKind::Holo3D || model_kind == ModelKind::Holo3DVel) ? 3 : 2;
  }
  Vector start_position(int k) const { return starts.col(k).head(position_dim()); }
  Vector goal_position(int k) const { return goals.col(k); }
};

int state_dim_of(ModelKind kind);
void validate_scenario(const Scenario& scenario);
Scenario antipodal_circle(int robots, double diameter, ModelKind kind, const RewardConfig& reward = {});
Scenario antipodal_sphere(int robots, double diameter, const RewardConfig& reward = {},
                          ModelKind kind = ModelKind::Holo3D);
Scenario random_square(int robots, double diameter, std::uint64_t seed, ModelKind kind = ModelKind::Holo2D,
                       const RewardConfig& reward = {}, double min_separation = -1.0);
Scenario add_obstacles(const Scenario& scenario, const std::vector<Obstacle>& obstacles);
std::vector<Obstacle> obstacle_preset(const std::string& name, double diameter);
std::vector<std::string> obstacle_preset_names();

// ---- BASELINE.json problem generators (builder-defined)
/// 8 corners of an edge-length cube, goal = opposite corner (C4).
Scenario cube_corners(double edge, ModelKind kind = ModelKind::Holo3DVel, const RewardConfig& reward = {});
/// Seeded obstacles: centre ~ U[lo,hi]^p, radius ~ U[r_lo,r_hi], rejected when
/// the inflated disc touches a start or goal (C2, C5).
Scenario random_obstacles(const Scenario& scenario, int count, std::uint64_t seed, double lo, double hi, double r_lo,
                          double r_hi);

struct BaselineConfig {
  Scenario scenario;
  DynamicsModel model;
  int horizon;
  int samples;  // BASELINE "N samples/step" = DenoiserConfig::batch
  int steps;
  int iterations;
};
/// BASELINE.json configs[index-1], index 1..5.
BaselineConfig baseline_config(int index);

}  // namespace d4orm

#if __has_include(<json.hpp>)
#include <json.hpp>
namespace d4orm {
/// Scenario JSON schema v1 (scenario.cpp:296-378); "model" accepts the
/// extension kinds too, and the state dimension follows the kind.
nlohmann::json scenario_to_json(const Scenario& scenario);
Scenario scenario_from_json(const nlohmann::json& j);
}  // namespace d4orm
#endif
