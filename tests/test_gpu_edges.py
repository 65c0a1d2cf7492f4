"""Edge shapes for the fused rollout+fitness kernel: a single robot, two
robots, a long horizon cut into ragged chunks, horizons shorter than a chunk,
batches that leave a CTA partly empty, a 100-robot team (Rp 112: items
shared by two threads, 8 flag words, culling across 7 tiles), and pair-list
teams (33..64 robots: padding, ragged windows, a dead sample slot) — fp64
against the oracle to 1e-12, fp32 to the fp32 band, and culling on == off."""
import os

import numpy as np
import pytest

import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S

pytestmark = pytest.mark.gpu


def _problem(R, T, seed, kind=S.HOLO2D_VEL, side=10.0, n_obs=0, radius=0.2):
    rng = np.random.default_rng(seed)
    dx, du, pd = S.DIMS[kind]
    st = np.zeros((R, dx))
    st[:, :pd] = rng.uniform(-side / 2, side / 2, (R, pd))
    go = rng.uniform(-side / 2, side / 2, (R, pd))
    kw = {}
    if n_obs:
        kw = dict(obs_centers=rng.uniform(-side / 2, side / 2, (n_obs, pd)), obs_radii=rng.uniform(0.2, 1.0, n_obs))
    return S.Problem(kind, starts=st, goals=go, horizon=T, lower=[-1] * du, upper=[1] * du, robot_radius=radius, **kw)


SHAPES = {
    "R1_T3_M7": (1, 3, 7, S.HOLO2D_VEL, 0),
    "R2_T1_M2": (2, 1, 2, S.HOLO2D_VEL, 1),
    "R5_T70_M33": (5, 70, 33, S.UNICYCLE, 2),
    "R17_T9_M5": (17, 9, 5, S.HOLO3D_VEL, 3),
    "R100_T20_M6": (100, 20, 6, S.HOLO2D_VEL, 5),
    "R100_T70_M3_diffdrive": (100, 70, 3, S.DIFFDRIVE, 0),
    # pair-list fitness (planar, 33..64 robots): odd team padded to 64, ragged
    # chunks (T = 70: a partial window and an empty one), a dead sample slot
    "R33_T70_M5_pairlist": (33, 70, 5, S.HOLO2D_VEL, 4),
    "R64_T33_M3_pairlist": (64, 33, 3, S.HOLO2D_VEL, 6),
    "R49_T40_M7_pairlist_unicycle": (49, 40, 7, S.UNICYCLE, 3),
}


@pytest.fixture(scope="module")
def gpu():
    g = d4.GpuDenoiser()
    yield g
    g.close()


@pytest.mark.parametrize("name", list(SHAPES))
def test_edge_shapes_match_oracle(gpu, oracle, name):
    from test_gpu_parity import controls_for, explain_flips, oracle_rollout_batch
    R, T, M, kind, n_obs = SHAPES[name]
    side = 6.0 if R > 50 else 10.0
    p = _problem(R, T, sum(map(ord, name)), kind=kind, side=side, n_obs=n_obs)  # stable seed
    u = controls_for(p, M, 3, scale=1.0)
    ref = oracle_rollout_batch(oracle, p, u)
    gpu.set_options(d4.PREC_F64, d4.NOISE_HOST)
    gpu.set_problem(p)
    st, ct, rw, cnt = gpu.rollout_fitness(u)
    for m, (rs, rc, rr, nc, no) in enumerate(ref):
        np.testing.assert_allclose(st[m], rs, rtol=1e-12, atol=1e-12)
        assert (cnt[m, 0], cnt[m, 1]) == (nc, no), (m, cnt[m], nc, no)
        assert abs(rw[m] - rr) <= 1e-12, (m, rw[m], rr)
    gpu.set_options(d4.PREC_F32, d4.NOISE_HOST)
    gpu.set_problem(p)
    res = []
    for cull in ("1", "0"):
        os.environ["D4ORM_CULL"] = cull
        try:
            gpu.set_problem(p)
            res.append(gpu.rollout_fitness(u))
        finally:
            os.environ.pop("D4ORM_CULL", None)
    (st1, _, rw1, cnt1), (st0, _, rw0, cnt0) = res
    np.testing.assert_array_equal(cnt1, cnt0)
    np.testing.assert_array_equal(rw1, rw0)
    unit = max(p.w_t, p.obstacle_weight) / (p.robots * p.horizon)
    for m, (rs, rc, rr, nc, no) in enumerate(ref):
        np.testing.assert_allclose(st1[m], rs, atol=5e-5, rtol=1e-5)
        flips = abs(cnt1[m, 0] - nc) + abs(cnt1[m, 1] - no)
        if flips:
            assert explain_flips(oracle, p, st1[m], cnt1[m, 0], cnt1[m, 1]), (m, cnt1[m], nc, no)
        assert abs(rw1[m] - rr) <= 3e-5 + flips * unit, (m, rw1[m], rr, flips)


@pytest.mark.parametrize("kind", [S.HOLO2D_VEL, S.UNICYCLE])
def test_fused_path_reports_nonfinite_state(gpu, kind):
    """Throughput path (fp32, Philox drawn in the rollout): an infinite base
    control with unbounded controls makes the state non-finite; the chunk's
    watch (the goal sum for velocity kinds, the state sum otherwise) triggers
    the exact replay, which reports the first failing robot and step like
    dynamics.cpp:81-84 (sample 0 is the lowest failing index)."""
    dx, du, pd = S.DIMS[kind]
    R, T = 3, 20
    st = np.zeros((R, dx))
    st[:, :pd] = np.array([[0, 0], [2, 0], [0, 2]], dtype=float)[:, :pd]
    p = S.Problem(kind, starts=st, goals=np.array([[1, 1], [3, 3], [-2, 2]], dtype=float)[:, :pd], horizon=T,
                  lower=[-np.inf] * du, upper=[np.inf] * du)
    base = np.zeros((T, R, du))
    base[7, 2, 0] = np.inf
    gpu.set_options(d4.PREC_F32, d4.NOISE_PHILOX)
    gpu.set_problem(p)
    with pytest.raises(d4.D4ormError, match="run_denoising: sample 0 at step 5: rollout: non-finite state for robot 2 at step 8"):
        gpu.run_denoising(base, d4.DenoiserConfig(steps=5, batch=64, seed=1))


def _nan_msg(gpu, prec, p, base, var, i, cfg, noise):
    gpu.set_options(prec, d4.NOISE_HOST)
    gpu.set_problem(p)
    with pytest.raises(d4.D4ormError) as e:
        gpu.denoise_step(base, var, i, cfg, noise)
    return str(e.value)


@pytest.mark.parametrize("where", ["noise", "variable", "base"])
def test_f32_nan_inputs_fail_like_the_reference(gpu, oracle, where):
    """A NaN in the noise, the variable or the base reaches a candidate control;
    the reference's clamp (cwiseMax/cwiseMin) keeps it and the rollout throws
    for the first failing sample at its first NaN robot/step
    (dynamics.cpp:76-84, denoiser.cpp:163-164).  The fp32 path clamps with
    FMNMX, so it scans its inputs: same message as the fp64 path and the
    oracle."""
    p = CASES_NAN()
    M, N, i = 64, 6, 4
    cfg = d4.DenoiserConfig(steps=N, batch=M, seed=2)
    base = np.zeros((p.horizon, p.robots, p.du))
    var = 0.1 * np.ones_like(base)
    noise = oracle.step_noise(2, i, 0, M, p.elems)
    if where == "noise":
        noise.reshape(M, p.horizon, p.robots, p.du)[37, 5, 2, 1] = np.nan
        noise.reshape(M, p.horizon, p.robots, p.du)[41, 1, 0, 0] = np.nan
        want = "run_denoising: sample 37 at step 4: rollout: non-finite state for robot 2 at step 6"
    elif where == "variable":
        var[9, 1, 0] = np.nan
        want = "run_denoising: sample 0 at step 4: rollout: non-finite state for robot 1 at step 10"
    else:
        base[3, 3, 1] = np.nan
        want = "run_denoising: sample 0 at step 4: rollout: non-finite state for robot 3 at step 4"
    m32 = _nan_msg(gpu, d4.PREC_F32, p, base, var, i, cfg, noise)
    m64 = _nan_msg(gpu, d4.PREC_F64, p, base, var, i, cfg, noise)
    from oracle.oracle import make_config
    ab, _ = oracle.make_schedule(N, 0.05)
    with pytest.raises(RuntimeError) as e:
        oracle.denoise_step(p, base, var, ab, make_config(N, M, seed=2), i, noise)
    assert m32 == m64 == str(e.value) == want, (m32, m64, str(e.value))


def CASES_NAN():
    return S.antipodal_circle(5, 4.0, S.HOLO2D_VEL, robot_radius=0.1, horizon=12, lower=[-1, -1], upper=[1, 1])
