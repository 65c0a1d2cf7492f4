"""The lean small-team K2+K3 (csrc/k_small.cuh: R <= 16, one wave of 7 CTAs per
SM) against the general kernel it replaces on production launches
(k_rollout_fitness<float, KIND, 8, 2, 1>, knob D4ORM_SMALL=0).

Same rollout block arithmetic, same robot tiles, same 16-step chunks and fold
order: a Philox denoising step must give the SAME BITS either way — rewards,
weights, the updated variable and the trace record (reward.cpp:88-127 through
denoiser.cpp:152-180) — on every model kind, with padding lanes, ragged
horizons and batches, and obstacles."""
import os

import numpy as np
import pytest

import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S

pytestmark = pytest.mark.gpu


def _square(R, side, seed, kind, n_obs=0, **kw):
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
    out = {}
    for c, batch in ((2, 8192), (3, 16384), (4, 16384)):
        rc = S.baseline_config(c)
        out[f"C{c}_full"] = (rc.problem, batch, rc.steps, (rc.steps, 37, 1))
    out["holo2d_R13_T50_O5"] = (_square(13, 5.0, 1, S.HOLO2D, horizon=50, robot_radius=0.2, n_obs=5), 1001, 10, (10, 3))
    out["diffdrive_R16_T33"] = (_square(16, 5.0, 2, S.DIFFDRIVE, horizon=33, robot_radius=0.2, n_obs=2), 777, 10, (10,))
    out["holo3d_R7_T21_O3"] = (_square(7, 4.0, 3, S.HOLO3D, horizon=21, robot_radius=0.3, n_obs=3), 500, 10, (10, 2))
    out["holo3dvel_R12_T64_O9"] = (_square(12, 4.0, 4, S.HOLO3D_VEL, horizon=64, robot_radius=0.3, n_obs=9), 640, 10, (5,))
    out["unicycle_R5_T17"] = (_square(5, 3.0, 5, S.UNICYCLE, horizon=17, robot_radius=0.25, n_obs=1), 333, 10, (10, 1))
    out["holo2dvel_R16_T3"] = (_square(16, 4.0, 7, S.HOLO2D_VEL, horizon=3, robot_radius=0.2, n_obs=1), 8192, 10, (10,))
    out["holo2dvel_R9_dense"] = (_square(9, 2.0, 6, S.HOLO2D_VEL, horizon=40, robot_radius=0.2, n_obs=4), 2048, 10, (10,))
    return out


CASES = _cases()


def _steps(p, batch, steps, idx, env):
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
        return outs, g.last_fit_kernel()
    finally:
        if g is not None:
            g.close()
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("case", list(CASES))
def test_small_equals_general_bitwise(case):
    p, batch, steps, idx = CASES[case]
    new, kn = _steps(p, batch, steps, idx, {"D4ORM_SMALL": "1"})
    old, ko = _steps(p, batch, steps, idx, {"D4ORM_SMALL": "0"})
    assert kn == 3 and ko == 0
    for (v1, r1, w1, t1), (v0, r0, w0, t0) in zip(new, old):
        np.testing.assert_array_equal(r1, r0)
        np.testing.assert_array_equal(w1, w0)
        np.testing.assert_array_equal(v1, v0)
        assert t1 == t0
        assert np.unique(r0).size > 1


def test_small_effort_weight():
    """Two-control kinds sum Σ‖u‖² in 4-step blocks here and 16-step blocks
    there: equal to fp32 association; the three-control kinds are sequential
    in both (bitwise)."""
    p = _square(16, 5.0, 8, S.HOLO2D_VEL, horizon=48, robot_radius=0.2, n_obs=2, effort_weight=0.05)
    new, kn = _steps(p, 8192, 10, (10,), {"D4ORM_SMALL": "1"})
    old, ko = _steps(p, 8192, 10, (10,), {"D4ORM_SMALL": "0"})
    assert kn == 3 and ko == 0
    np.testing.assert_allclose(new[0][1], old[0][1], rtol=0, atol=1e-6)
    p = _square(8, 4.0, 9, S.HOLO3D_VEL, horizon=48, robot_radius=0.2, effort_weight=0.05)
    new, _ = _steps(p, 16384, 10, (10,), {"D4ORM_SMALL": "1"})
    old, _ = _steps(p, 16384, 10, (10,), {"D4ORM_SMALL": "0"})
    np.testing.assert_array_equal(new[0][1], old[0][1])


def test_small_not_used_for_c1_or_host_controls():
    """C1 keeps the time-segmented kernel; host-supplied controls keep the general one."""
    rc = S.baseline_config(1)
    _, k = _steps(rc.problem, rc.samples, rc.steps, (rc.steps,), {})
    assert k == 1
    p = CASES["C2_full"][0]
    g = d4.GpuDenoiser(p)
    try:
        g.rollout_fitness(np.zeros((4, p.horizon, p.robots, p.du)))
        assert g.last_fit_kernel() == 0
    finally:
        g.close()


@pytest.mark.parametrize("kind", [S.HOLO2D_VEL, S.UNICYCLE, S.HOLO3D])
def test_small_reports_nonfinite_state(kind):
    """An infinite base control with unbounded controls: the chunk's watch
    triggers the exact replay, which reports the first failing robot and step
    like dynamics.cpp:81-84 (second 16-step chunk, padding lanes)."""
    p = _square(12, 8.0, 21, kind, horizon=40, robot_radius=0.2, n_obs=2)
    du = p.du
    p = S.Problem(kind, starts=p.starts, goals=p.goals, horizon=40, lower=[-np.inf] * du, upper=[np.inf] * du,
                  robot_radius=0.2, obs_centers=p.obs_centers, obs_radii=p.obs_radii)
    base = np.zeros((40, 12, du))
    base[21, 5, 0] = np.inf
    g = d4.GpuDenoiser(p)
    try:
        with pytest.raises(d4.D4ormError,
                           match="run_denoising: sample 0 at step 5: rollout: non-finite state for robot 5 at step 22"):
            g.run_denoising(base, d4.DenoiserConfig(steps=5, batch=8192, seed=1))
        assert g.last_fit_kernel() == 3
    finally:
        g.close()
