"""TEST HELPER: a numpy restatement of the per-iteration outcome of one
executed trajectory — objective (reward.cpp:136-156) and check_success
(reward.cpp:162-200) with the reference's messages — used by the GPU tests to
re-check the device's K6 outcome on a returned trajectory."""
from __future__ import annotations

import numpy as np

from paper_2503_12204_b200.scenarios import Problem


def objective(p: Problem, states: np.ndarray) -> float:
    """Fraction of robot-steps t=1..H inside the goal ball."""
    pos = states[1:, :, : p.pdim]
    d2 = ((pos - p.goals[None]) ** 2).sum(-1)
    return float((d2 <= p.goal_tolerance ** 2).sum()) / (p.robots * p.horizon)


def check_success(p: Problem, states: np.ndarray) -> tuple[bool, str]:
    """Strict 2R_a at every step (t=0..H), obstacles, terminal goal ball;
    the first violation in the reference's scan order is reported."""
    R, pd = p.robots, p.pdim
    safety_sq = 4.0 * p.robot_radius * p.robot_radius
    pos = states[:, :, :pd]                                   # (T+1, R, pd)
    diff = pos[:, :, None, :] - pos[:, None, :, :]
    d2 = (diff ** 2).sum(-1)                                  # (T+1, R, R)
    iu = np.triu(np.ones((R, R), dtype=bool), 1)
    pair_hit = (d2 <= safety_sq) & iu[None]
    if len(p.obs_radii):
        od2 = ((pos[:, :, None, :] - p.obs_centers[None, None]) ** 2).sum(-1)   # (T+1, R, O)
        lim = (p.obs_radii + p.robot_radius) ** 2
        obs_hit = od2 <= lim[None, None]
    else:
        obs_hit = np.zeros(pos.shape[:2] + (0,), dtype=bool)
    if pair_hit.any() or obs_hit.any():
        for t in range(states.shape[0]):
            for k in range(R):
                ls = np.nonzero(pair_hit[t, k])[0]
                if len(ls):
                    return False, f"safety: robots {k} and {ls[0]} within 2*R_a at step {t}"
                os_ = np.nonzero(obs_hit[t, k])[0]
                if len(os_):
                    return False, f"obstacle: robot {k} hits obstacle {os_[0]} at step {t}"
    end = np.sqrt(((pos[-1] - p.goals) ** 2).sum(-1))
    for k in range(R):
        if end[k] > p.goal_tolerance:
            return False, (f"terminal: robot {k} ends {end[k]:f} m from its goal "
                           f"(tolerance {p.goal_tolerance:f})")
    return True, ""
