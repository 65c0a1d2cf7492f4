"""The time-segmented K2+K3 (csrc/k_seg.cu: a robot's horizon split over 8
threads, states from a scan of the segment sums) against the regular kernel
(one thread walks a robot's whole horizon) and against the reference's error
behaviour.  The segmented kernel serves latency-bound launches of the
velocity-input kinds (C1 by default); knob D4ORM_SEG=0/1 forces either.

Both kernels draw the same Philox normals, clamp the same controls and test
the same predicates; their states differ only by fp32 association
(x_0 + Σ dt·u as a scan vs the serial chain), so rewards agree to fp32
rounding except where a pair / obstacle test sits on its boundary."""
import os

import numpy as np
import pytest

import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S

pytestmark = pytest.mark.gpu


def _run(seg, fn):
    os.environ["D4ORM_SEG"] = "1" if seg else "0"
    g = d4.GpuDenoiser()
    try:
        return fn(g)
    finally:
        g.close()
        os.environ.pop("D4ORM_SEG", None)


def _square(kind, R, T, n_obs, seed, side=4.0):
    rng = np.random.default_rng(seed)
    dx, du, pd = S.DIMS[kind]
    st = rng.uniform(-side / 2, side / 2, (R, pd))
    go = rng.uniform(-side / 2, side / 2, (R, pd))
    p = S.Problem(kind, starts=st.copy(), goals=go, horizon=T, lower=[-1] * du, upper=[1] * du, robot_radius=0.2)
    if n_obs:
        p.obs_centers = rng.uniform(-side / 2, side / 2, (n_obs, pd))
        p.obs_radii = rng.uniform(0.2, 0.6, n_obs)
    return p


CASES = {
    "C1": lambda: S.baseline_config(1).problem,
    "2d_R1_T16": lambda: _square(S.HOLO2D_VEL, 1, 16, 2, 1),
    "2d_R2_T64_obs": lambda: _square(S.HOLO2D_VEL, 2, 64, 5, 2),
    "2d_R8_T128_obs": lambda: _square(S.HOLO2D_VEL, 8, 128, 4, 3),
    "2d_R16_T32_obs": lambda: _square(S.HOLO2D_VEL, 16, 32, 3, 4),
    "3d_R4_T32": lambda: _square(S.HOLO3D_VEL, 4, 32, 0, 5),
    "3d_R8_T64_obs": lambda: _square(S.HOLO3D_VEL, 8, 64, 3, 6),
}


def _step(p, M, noise):
    def run(g):
        g.set_problem(p)
        cfg = d4.DenoiserConfig(steps=10, batch=M, seed=11)
        rng = np.random.default_rng(2)
        base = 0.3 * rng.normal(size=(p.horizon, p.robots, p.du))
        var = 0.1 * rng.normal(size=base.shape)
        if noise is not None:
            g.set_options(d4.PREC_F32, d4.NOISE_HOST)
        return g.denoise_step(base, var, 7, cfg, noise)
    return run


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("host_noise", [False, True], ids=["philox", "host"])
def test_seg_matches_regular(case, host_noise):
    p = CASES[case]()
    M = 1000
    z = np.random.default_rng(5).normal(size=(M, p.horizon * p.robots * p.du)) if host_noise else None
    v1, r1, w1, t1 = _run(True, _step(p, M, z))
    v0, r0, w0, t0 = _run(False, _step(p, M, z))
    unit = max(p.w_t, p.obstacle_weight) / (p.robots * p.horizon)
    d = np.abs(r1 - r0)
    assert (d <= 1e-5 + 2 * unit).all(), (case, d.max())
    assert (d > 1e-5).mean() <= 0.01, (case, (d > 1e-5).mean())  # boundary flips are rare
    assert np.isfinite(r1).all() and r1.std() > 0
    # the same samples win: the update agrees to fp32 rounding of the states
    if (d <= 1e-5).all():
        np.testing.assert_allclose(v1, v0, rtol=1e-4, atol=1e-5)


def test_seg_is_the_default_for_c1_only():
    """C1 (32 regular CTAs) takes the segmented kernel; C2/C4 (1024 CTAs) and the
    unicycle C3 keep the regular one — visible as bitwise-equal rewards with the
    knob forced off."""
    for cfg, seg in [(1, True), (2, False), (4, False)]:
        p = S.baseline_config(cfg).problem
        M = S.baseline_config(cfg).samples

        def run(g):
            g.set_problem(p)
            return g.denoise_step(np.zeros((p.horizon, p.robots, p.du)), np.zeros((p.horizon, p.robots, p.du)), 50,
                                  d4.DenoiserConfig(steps=100, batch=M, seed=3), None)[1]

        os.environ.pop("D4ORM_SEG", None)
        g = d4.GpuDenoiser()
        try:
            r_default = run(g)
        finally:
            g.close()
        r_regular = _run(False, run)
        assert np.array_equal(r_default, r_regular) == (not seg), cfg


def test_seg_reports_nonfinite_state():
    """An infinite base control with unbounded controls: the first failing robot
    and step are reported as dynamics.cpp:81-84 does (the segment that holds
    the step finds it; later segments inherit the infinite offset)."""
    R, T = 4, 32
    st = np.array([[0, 0], [2, 0], [0, 2], [2, 2]], dtype=float)
    p = S.Problem(S.HOLO2D_VEL, starts=st, goals=-st + 0.5, horizon=T, lower=[-np.inf] * 2, upper=[np.inf] * 2)
    base = np.zeros((T, R, 2))
    base[7, 2, 0] = np.inf

    def run(g):
        g.set_problem(p)
        return g.run_denoising(base, d4.DenoiserConfig(steps=5, batch=64, seed=1))

    with pytest.raises(d4.D4ormError, match="run_denoising: sample 0 at step 5: rollout: non-finite state for robot 2 at step 8"):
        _run(True, run)
