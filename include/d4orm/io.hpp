#pragma once
// Result I/O of the reference CLI (tools/main.cpp:309-324,349-377):
// trajectory.json (scenario + config + result + per-robot states/controls)
// and denoise_trace.csv, plus the reader that replays an exported trajectory
// (check_success on an exported trajectory).
#include <string>

#include <json.hpp>

#include "d4orm/result.hpp"
#include "d4orm/scenario.hpp"

namespace d4orm {

/// Per-robot steps {time, state, control} (tools/main.cpp:309-324).
nlohmann::json trajectory_to_json(const JointTrajectory& trajectory);

/// trajectory.json document of cmd_solve (tools/main.cpp:349-362).
nlohmann::json solve_output_json(const Scenario& scenario, const SolveResult& result, const std::string& solver,
                                 const nlohmann::json& config);

/// Writes out_dir/trajectory.json and out_dir/denoise_trace.csv exactly as
/// cmd_solve does (tools/main.cpp:364-377).
void write_solve_outputs(const std::string& out_dir, const Scenario& scenario, const SolveResult& result,
                         const std::string& solver, const nlohmann::json& config);

struct LoadedTrajectory {
  Scenario scenario;
  JointTrajectory trajectory;
  nlohmann::json result;  // the "result" object minus "robots"
};
/// Reads a trajectory.json back (scenario + best trajectory) for replay.
LoadedTrajectory read_trajectory_json(const std::string& path);

}  // namespace d4orm
