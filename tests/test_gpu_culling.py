"""The fp32 fitness culling (x-strip tile pairs, row pairs, obstacle bucket
ranges per half tile — csrc/k23.cuh) must not change any decision: on
scenarios built to stress it, culling ON equals culling OFF bitwise (rewards
and conflict / obstacle counts), and both match the fp64 oracle up to flips
explained by the fp32 band."""
import os

import numpy as np
import pytest

import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S

pytestmark = pytest.mark.gpu


def _square(R, side, seed, kind=S.HOLO2D_VEL, **kw):
    rng = np.random.default_rng(seed)
    pd = S.DIMS[kind][2]
    st = rng.uniform(-side / 2, side / 2, size=(R, pd))
    go = rng.uniform(-side / 2, side / 2, size=(R, pd))
    dx = S.DIMS[kind][0]
    starts = np.zeros((R, dx))
    starts[:, :pd] = st
    return S.Problem(kind, starts=starts, goals=go, lower=[-1] * S.DIMS[kind][1], upper=[1] * S.DIMS[kind][1], **kw)


def _stress():
    rng = np.random.default_rng(11)
    out = {}
    # dense: 64 robots in 6 m, conflicts everywhere (tiles overlap, little culls)
    out["dense"] = _square(64, 6.0, 1, horizon=40, robot_radius=0.2)
    # wide: 64 robots over 120 m, 9 obstacles clustered in one corner (most
    # strips lie outside the obstacle table's x-extent)
    p = _square(64, 120.0, 2, horizon=40, robot_radius=0.3)
    p.obs_centers = np.c_[rng.uniform(40, 55, 9), rng.uniform(40, 55, 9)]
    p.obs_radii = rng.uniform(0.5, 3.0, 9)
    out["wide_corner_obstacles"] = p
    # a vertical line: every robot at the same x (ranks by lane; strips coincide)
    starts = np.c_[np.zeros(48), np.linspace(-10, 10, 48)]
    goals = np.c_[np.full(48, 0.3), np.linspace(10, -10, 48)]
    out["same_x_line"] = S.Problem(S.HOLO2D_VEL, starts=starts, goals=goals, horizon=30, lower=[-1, -1],
                                   upper=[1, 1], robot_radius=0.15,
                                   obs_centers=np.array([[0.0, 0.0], [0.0, 5.0], [5.0, 5.0]]),
                                   obs_radii=np.array([0.5, 1.0, 0.7]))
    # R = 40 (Rp 48, padding lanes), 7 obstacles incl. one huge that covers all
    p = _square(40, 16.0, 3, horizon=32, robot_radius=0.2)
    p.obs_centers = np.r_[rng.uniform(-8, 8, (6, 2)), [[0.0, 0.0]]]
    p.obs_radii = np.r_[rng.uniform(0.3, 1.0, 6), [30.0]]
    out["R40_huge_obstacle"] = p
    # 3D velocity model, 64 robots, obstacles (culling on x only)
    p = _square(64, 12.0, 4, kind=S.HOLO3D_VEL, horizon=24, robot_radius=0.25)
    p.obs_centers = rng.uniform(-6, 6, (5, 3))
    p.obs_radii = rng.uniform(0.3, 1.2, 5)
    out["holo3d_64"] = p
    return out


CASES = _stress()


def _run(gpu, p, u, cull):
    os.environ["D4ORM_CULL"] = "1" if cull else "0"
    try:
        gpu.set_problem(p)
        return gpu.rollout_fitness(u)
    finally:
        os.environ.pop("D4ORM_CULL", None)


@pytest.fixture(scope="module")
def gpu():
    g = d4.GpuDenoiser()
    g.set_options(d4.PREC_F32, d4.NOISE_HOST)
    yield g
    g.close()


@pytest.mark.parametrize("case", list(CASES))
def test_culling_changes_nothing(gpu, oracle, case):
    from test_gpu_parity import controls_for, explain_flips, oracle_rollout_batch
    p = CASES[case]
    u = controls_for(p, 20, 5, scale=1.0)
    st1, _, rw1, cnt1 = _run(gpu, p, u, True)
    st0, _, rw0, cnt0 = _run(gpu, p, u, False)
    np.testing.assert_array_equal(cnt1, cnt0)
    np.testing.assert_array_equal(rw1, rw0)
    np.testing.assert_array_equal(st1, st0)
    assert cnt1[:, 0].sum() > 0 or case in ("wide_corner_obstacles",)  # the scenarios do conflict
    ref = oracle_rollout_batch(oracle, p, u)
    for m, (rs, rc, rr, nc, no) in enumerate(ref):
        if (cnt1[m, 0], cnt1[m, 1]) != (nc, no):
            assert explain_flips(oracle, p, st1[m], cnt1[m, 0], cnt1[m, 1]), (case, m, cnt1[m], nc, no)


def test_fitness_path_selection(gpu):
    """Planar teams of 33..64 run the pair-list fitness, the rest the tiles."""
    gpu.set_problem(S.baseline_config(5).problem.with_horizon(16))
    assert gpu.fitness_path() == 1
    gpu.set_problem(CASES["R40_huge_obstacle"])
    assert gpu.fitness_path() == 1
    gpu.set_problem(CASES["holo3d_64"])
    assert gpu.fitness_path() == 0
    gpu.set_problem(S.baseline_config(2).problem)
    assert gpu.fitness_path() == 0


@pytest.mark.parametrize("case", ["dense", "same_x_line", "R40_huge_obstacle"])
def test_pair_list_matches_tiles(gpu, oracle, case):
    """The pair-list fitness (direct-form tests) and the tile fitness
    (expanded-form tests) see the same states; their counts differ only by
    decisions inside the fp32 band, and both match the fp64 oracle up to
    explained flips."""
    from test_gpu_parity import controls_for, explain_flips
    p = CASES[case]
    u = controls_for(p, 16, 9, scale=1.0)
    os.environ["D4ORM_PL"] = "0"
    try:
        gpu.set_problem(p)
        assert gpu.fitness_path() == 0
        st0, _, rw0, cnt0 = gpu.rollout_fitness(u)
    finally:
        os.environ.pop("D4ORM_PL", None)
    gpu.set_problem(p)
    assert gpu.fitness_path() == 1
    st1, _, rw1, cnt1 = gpu.rollout_fitness(u)
    np.testing.assert_array_equal(st1, st0)
    unit = max(p.w_t, p.obstacle_weight) / (p.robots * p.horizon)
    for m in range(u.shape[0]):
        if (cnt1[m] != cnt0[m]).any():
            assert explain_flips(oracle, p, st1[m], cnt1[m, 0], cnt1[m, 1]), (case, m, cnt1[m], cnt0[m])
            assert explain_flips(oracle, p, st0[m], cnt0[m, 0], cnt0[m, 1]), (case, m, cnt1[m], cnt0[m])
        flips = abs(int(cnt1[m, 0]) - int(cnt0[m, 0])) + abs(int(cnt1[m, 1]) - int(cnt0[m, 1]))
        assert abs(rw1[m] - rw0[m]) <= 1e-5 + flips * unit, (case, m, rw1[m], rw0[m])
