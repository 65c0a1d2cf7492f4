"""The 32-step-window pair-list K2+K3 (csrc/k_pl32.cuh: 16-20 warps per SM, a
window's fitness split over the sample's two warps) against the 64-step
pair-list kernel it replaces on production launches (k_rollout_fitness<…, PL>,
knob D4ORM_PL32=0).

Positions are the same arithmetic, the fp32 goal partials are folded on the
same 64-step periods, and conflict / obstacle robot-steps are counts, so a
Philox denoising step must give the SAME BITS either way: rewards, weights,
the updated variable and the trace record (reward.cpp:88-127 through
denoiser.cpp:152-180).  Culling on == off likewise (D4ORM_CULL)."""
import os

import numpy as np
import pytest

import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S

pytestmark = pytest.mark.gpu


def _square(R, side, seed, kind=S.HOLO2D_VEL, n_obs=0, **kw):
    rng = np.random.default_rng(seed)
    dx, du, pd = S.DIMS[kind]
    starts = np.zeros((R, dx))
    starts[:, :pd] = rng.uniform(-side / 2, side / 2, size=(R, pd))
    if kind in (S.UNICYCLE, S.DIFFDRIVE):
        starts[:, 2] = rng.uniform(-np.pi, np.pi, R)
    goals = rng.uniform(-side / 2, side / 2, size=(R, pd))
    lo, hi = ([-1.0, -np.pi / 2], [1.0, np.pi / 2]) if kind == S.UNICYCLE else ([-1.0] * du, [1.0] * du)
    p = S.Problem(kind, starts=starts, goals=goals, lower=lo, upper=hi, **kw)
    if n_obs:
        p.obs_centers = rng.uniform(-side / 2, side / 2, (n_obs, pd))
        p.obs_radii = rng.uniform(0.3, 1.0, n_obs)
    return p


def _cases():
    c5 = S.baseline_config(5).problem
    return {
        # (problem, batch, denoising steps, step indices to run)
        "C5_R64_T256_O16": (c5, 4096, 100, (100, 57, 1)),
        "dense_R64_T96": (_square(64, 5.0, 1, horizon=96, robot_radius=0.2, n_obs=5), 1024, 20, (20, 3)),
        "R40_T40_pad_O19": (_square(40, 14.0, 2, horizon=40, robot_radius=0.25, n_obs=19), 1001, 10, (10, 2)),
        "R33_T100_O1": (_square(33, 10.0, 3, horizon=100, robot_radius=0.3, n_obs=1), 777, 10, (9,)),
        "R64_T31_no_obstacles": (_square(64, 9.0, 4, horizon=31, robot_radius=0.2), 512, 10, (10, 1)),
        "unicycle_R48_T64": (_square(48, 12.0, 5, kind=S.UNICYCLE, horizon=64, robot_radius=0.25, n_obs=4), 768, 10,
                             (10, 4)),
        "diffdrive_R64_T48": (_square(64, 12.0, 6, kind=S.DIFFDRIVE, horizon=48, robot_radius=0.2, n_obs=7), 512, 10,
                              (10,)),
        "R34_T5_tiny_horizon": (_square(34, 8.0, 9, horizon=5, robot_radius=0.2, n_obs=2), 300, 10, (10,)),
        "R64_T1_single_step": (_square(64, 8.0, 10, horizon=1, robot_radius=0.2), 257, 10, (10,)),
        "holo2d_R36_T70": (_square(36, 8.0, 7, kind=S.HOLO2D, horizon=70, robot_radius=0.2, n_obs=3), 600, 10, (10, 5)),
    }


CASES = _cases()


def _steps(p, batch, steps, idx, env):
    """Philox denoising steps `idx` from a fixed non-trivial variable, in a
    fresh context under `env`; → (per-step outputs, kernel id)."""
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    g = None
    try:
        g = d4.GpuDenoiser(p)
        cfg = d4.DenoiserConfig(steps=steps, batch=batch, seed=11)
        rng = np.random.default_rng(5)
        base = np.zeros((p.horizon, p.robots, p.du))
        var = 0.3 * rng.standard_normal(base.shape)
        outs = [g.denoise_step(base, var, i, cfg) for i in idx]
        return outs, g.last_fit_kernel(), g.fitness_path()
    finally:
        if g is not None:
            g.close()
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("case", list(CASES))
def test_pl32_equals_pl64_bitwise(case):
    p, batch, steps, idx = CASES[case]
    new, kn, path = _steps(p, batch, steps, idx, {"D4ORM_PL32": "1"})
    old, ko, _ = _steps(p, batch, steps, idx, {"D4ORM_PL32": "0"})
    assert path == 1 and kn == 2 and ko == 0
    hits = 0
    for (v1, r1, w1, t1), (v0, r0, w0, t0) in zip(new, old):
        np.testing.assert_array_equal(r1, r0)
        np.testing.assert_array_equal(w1, w0)
        np.testing.assert_array_equal(v1, v0)
        assert t1 == t0
        hits += int(np.unique(r0).size > 1)
    assert hits == len(idx)  # the rewards are not degenerate


@pytest.mark.parametrize("case", ["C5_R64_T256_O16", "dense_R64_T96", "R40_T40_pad_O19", "unicycle_R48_T64"])
def test_pl32_culling_changes_nothing(case):
    p, batch, steps, idx = CASES[case]
    on, k1, _ = _steps(p, batch, steps, idx[:1], {"D4ORM_PL32": "1", "D4ORM_CULL": "1"})
    off, k0, _ = _steps(p, batch, steps, idx[:1], {"D4ORM_PL32": "1", "D4ORM_CULL": "0"})
    assert k1 == 2 and k0 == 2
    np.testing.assert_array_equal(on[0][1], off[0][1])
    np.testing.assert_array_equal(on[0][0], off[0][0])


def test_pl32_effort_weight():
    """With an effort weight the per-robot Σ‖u‖² is summed in 8-step blocks here
    and 16-step blocks there: equal to fp32 association, not bitwise."""
    p = _square(64, 9.0, 8, horizon=64, robot_radius=0.2, n_obs=2, effort_weight=0.05)
    new, kn, _ = _steps(p, 512, 10, (10,), {"D4ORM_PL32": "1"})
    old, ko, _ = _steps(p, 512, 10, (10,), {"D4ORM_PL32": "0"})
    assert kn == 2 and ko == 0
    np.testing.assert_allclose(new[0][1], old[0][1], rtol=0, atol=1e-6)


def test_pl32_not_used_off_the_production_path():
    """Host-supplied controls (rollout_fitness) and fp64 keep k_rollout_fitness."""
    p = CASES["R64_T31_no_obstacles"][0]
    g = d4.GpuDenoiser(p)
    try:
        u = np.zeros((4, p.horizon, p.robots, p.du))
        g.rollout_fitness(u)
        assert g.last_fit_kernel() == 0
    finally:
        g.close()


@pytest.mark.parametrize("kind", [S.HOLO2D_VEL, S.UNICYCLE])
def test_pl32_reports_nonfinite_state(kind):
    """An infinite base control with unbounded controls: the window's watch (the
    goal sum for velocity kinds, the state sum otherwise) triggers the exact
    replay, which reports the first failing robot and step like
    dynamics.cpp:81-84 (second 32-step window, a padded team)."""
    p = _square(40, 14.0, 21, kind=kind, horizon=70, robot_radius=0.2, n_obs=2)
    du = p.du
    p = S.Problem(kind, starts=p.starts, goals=p.goals, horizon=70, lower=[-np.inf] * du, upper=[np.inf] * du,
                  robot_radius=0.2, obs_centers=p.obs_centers, obs_radii=p.obs_radii)
    base = np.zeros((70, 40, du))
    base[45, 7, 0] = np.inf
    g = d4.GpuDenoiser(p)
    try:
        with pytest.raises(d4.D4ormError,
                           match="run_denoising: sample 0 at step 5: rollout: non-finite state for robot 7 at step 46"):
            g.run_denoising(base, d4.DenoiserConfig(steps=5, batch=1024, seed=1))
        assert g.last_fit_kernel() == 2
    finally:
        g.close()
