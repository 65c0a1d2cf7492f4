#pragma once
// Drop-in for proj/include/d4orm/dynamics.hpp:11-155.  ModelKind keeps the
// reference's three kinds (same values) and adds the BASELINE extensions
// (SURVEY.md App. A), each a derivative functor in the rk4_with pattern.
#include <cmath>
#include <string>
#include <vector>

#include "d4orm/types.hpp"

namespace d4orm {

enum class ModelKind { DiffDrive = 0, Holo2D = 1, Holo3D = 2, Holo2DVel = 3, Holo3DVel = 4, Unicycle = 5 };

const char* to_string(ModelKind kind);
ModelKind model_kind_from_string(const std::string& name);

/// State layouts: DiffDrive [x,y,θ,v] u=[ω,a]; Holo2D [x,y,vx,vy] u=[ax,ay];
/// Holo3D [p(3),v(3)] u=a(3); Holo2DVel [x,y] u=v(2); Holo3DVel [p(3)] u=v(3);
/// Unicycle [x,y,θ] u=[v,ω].
struct DynamicsModel {
  ModelKind kind{ModelKind::Holo2D};
  int state_dim{4};
  int control_dim{2};
  Vector control_lower;
  Vector control_upper;

  int position_dim() const {
    return (kind == ModelKind::Holo3D || kind == ModelKind::Holo3DVel) ? 3 : 2;
  }

  /// ±control_limit on every axis (dynamics.hpp:33); asymmetric bounds (the
  /// BASELINE unicycle) are set on control_lower/control_upper directly.
  static DynamicsModel make(ModelKind kind, double control_limit = 2.0);
};

struct JointControls {
  int robots{0};
  int control_dim{0};
  Matrix u;  // (robots * control_dim) x horizon, column t = controls of step t

  int horizon() const { return static_cast<int>(u.cols()); }
  auto robot(int k) { return u.middleRows(k * control_dim, control_dim); }
  auto robot(int k) const { return u.middleRows(k * control_dim, control_dim); }

  static JointControls zeros(int robots, int control_dim, int horizon);
};

struct JointTrajectory {
  int robots{0};
  int state_dim{0};
  int control_dim{0};
  double dt{0.0};
  Matrix states;    // (robots * state_dim) x (H+1)
  Matrix controls;  // (robots * control_dim) x (H+1), column H zero

  int horizon() const { return static_cast<int>(states.cols()) - 1; }
  auto robot_states(int k) const { return states.middleRows(k * state_dim, state_dim); }
  auto robot_controls(int k) const { return controls.middleRows(k * control_dim, control_dim); }
  Vector state(int k, int t) const { return states.col(t).segment(k * state_dim, state_dim); }
  Vector control(int k, int t) const { return controls.col(t).segment(k * control_dim, control_dim); }
  Vector position(int k, int t, int position_dim) const { return states.col(t).segment(k * state_dim, position_dim); }

  JointControls executed_controls() const;
};

Vector derivative(const DynamicsModel& model, const Vector& x, const Vector& u);
Vector rk4_step(const DynamicsModel& model, const Vector& x, const Vector& u, double dt);

/// GPU: one rollout through the fp64 parity instantiation of the fused
/// rollout kernel (bitwise equal to the reference for the holonomic kinds).
JointTrajectory rollout(const DynamicsModel& model, const Matrix& starts, const JointControls& controls, double dt);

/// GPU: all members in one launch (dynamics.hpp:150-155).
std::vector<JointTrajectory> batch_rollout(const DynamicsModel& model, const Matrix& starts,
                                           const std::vector<JointControls>& batch, double dt, int workers = 0);

}  // namespace d4orm
