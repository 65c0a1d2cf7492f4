"""CPU: pin the oracle before trusting it.

(1) Known-answer tests: every SPEC.md worked example on the path —
    the only known-answer values the reference holds (proj/tests/ is empty).
(2) Bitwise agreement with the reference's own sources (oracle/_ref, built from
    /root/reference/proj/src unchanged against oracle/eigen_shim).
(3) The committed golden vectors (tests/golden/, made by tests/golden/make_golden.py
    from oracle/_ref) — so the pin still holds where /root/reference is absent.
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

from paper_2503_12204_b200 import scenarios as S
from oracle.oracle import cem_config, make_config, mppi_config

GOLDEN = Path(__file__).parent / "golden"


# ------------------------------------------------------------------ (1) KATs
def test_kat_derivative(oracle):
    # SPEC.md:59-61
    np.testing.assert_allclose(oracle.derivative(S.DIFFDRIVE, [0, 0, 0, 1], [0, 0]), [1, 0, 0, 0], atol=0)
    np.testing.assert_allclose(oracle.derivative(S.HOLO2D, [0, 0, 0, 0], [0, 0]), [0, 0, 0, 0])
    np.testing.assert_allclose(oracle.derivative(S.DIFFDRIVE, [0, 0, math.pi / 2, 2], [0.5, -1]), [0, 2, 0.5, -1],
                               atol=1e-15)


def test_kat_rk4(oracle):
    # SPEC.md:68-70
    np.testing.assert_allclose(oracle.rk4_step(S.HOLO2D, [0, 0, 1, 0], [0, 0], 0.1), [0.1, 0, 1, 0], atol=1e-15)
    np.testing.assert_allclose(oracle.rk4_step(S.HOLO2D, [0, 0, 0, 0], [1, 0], 0.1), [0.005, 0, 0.1, 0], atol=1e-15)
    np.testing.assert_allclose(oracle.rk4_step(S.DIFFDRIVE, [0, 0, 0, 1], [1, 0], 0.1),
                               [math.sin(0.1), 1 - math.cos(0.1), 0.1, 1], atol=1e-6)
    # extensions: single integrator is exact, unicycle arc
    np.testing.assert_allclose(oracle.rk4_step(S.HOLO2D_VEL, [1, 2], [1, -1], 0.1), [1.1, 1.9], atol=1e-15)
    np.testing.assert_allclose(oracle.rk4_step(S.UNICYCLE, [0, 0, 0], [1, 1], 0.1),
                               [math.sin(0.1), 1 - math.cos(0.1), 0.1], atol=1e-6)


def test_kat_rollout(oracle):
    # const u=[1,0], H=10 → p_x = 0.5, v_x = 1.0; zero controls fixed point
    p = S.Problem(S.HOLO2D, starts=[[0, 0, 0, 0]], goals=[[1, 1]], horizon=10)
    st, ct = oracle.rollout(p, np.tile([1.0, 0.0], (10, 1, 1)))
    assert abs(st[-1, 0, 0] - 0.5) < 1e-9 and abs(st[-1, 0, 2] - 1.0) < 1e-12
    st, _ = oracle.rollout(p.with_horizon(3), np.zeros((3, 1, 2)))
    assert (st == 0).all()
    # clamping happens once, before integration, and is what is stored
    st, ct = oracle.rollout(p.with_horizon(2), np.full((2, 1, 2), 5.0))
    assert (ct[:2] == 2.0).all() and (ct[2] == 0).all()


def test_kat_reward(oracle):
    # SPEC.md:132-161
    base = dict(kind=S.HOLO2D_VEL, horizon=3, lower=[-1, -1], upper=[1, 1])
    p = S.Problem(starts=[[0, 0]], goals=[[4, 0]], **base)
    st = np.zeros((4, 1, 2))
    st[1:, 0] = [3, 0]  # distance 1 of start distance 4 → 0.75
    assert oracle.total_reward(p, st)[0] == pytest.approx(0.75)
    st[1:, 0] = [4, 0]  # parked at goal → 1.0
    assert oracle.total_reward(p, st)[0] == 1.0
    st[1:, 0] = [0, 0]  # parked at start → 0.0
    assert oracle.total_reward(p, st)[0] == 0.0
    # two robots parked at their goals within 2R_a+eps, w_t = 2 → -1.0
    p2 = S.Problem(starts=[[0, 0], [5, 5]], goals=[[1, 0], [1.2, 0]], **base)
    st2 = np.zeros((4, 2, 2))
    st2[:, 0] = [1, 0]
    st2[:, 1] = [1.2, 0]
    assert oracle.total_reward(p2, st2)[0] == pytest.approx(-1.0)
    # boundary: distance exactly 2R_a + eps counts (<=)
    p3 = S.Problem(starts=[[0, 0], [0.25, 0]], goals=[[1, 1], [2, 2]], robot_radius=0.1, epsilon=0.05, **base)
    st3 = np.zeros((4, 2, 2))
    st3[:, 1] = [0.25, 0]
    assert oracle.total_reward(p3, st3)[1] == 6
    st3[:, 1] = [0.26, 0]
    assert oracle.total_reward(p3, st3)[1] == 0
    # obstacle: R_a = 0.1, radius 0.5, centre distance 0.59 → hit
    p4 = S.Problem(starts=[[0, 0]], goals=[[3, 3]], obs_centers=[[0.59, 0]], obs_radii=[0.5], **base)
    st4 = np.zeros((4, 1, 2))
    assert oracle.total_reward(p4, st4)[2] == 3


def test_kat_check_success(oracle):
    # stationary pair at exactly 2R_a → fail at step 0 (strict)
    p = S.Problem(S.HOLO2D_VEL, starts=[[0, 0], [0.2, 0]], goals=[[0, 0.5], [0.5, 0.5]], horizon=2,
                  robot_radius=0.1)
    st = np.zeros((3, 2, 2))
    st[:, 1] = [0.2, 0]
    ok, msg = oracle.check_success(p, st)
    assert not ok and msg == "safety: robots 0 and 1 within 2*R_a at step 0"
    st[:, 1] = [0.2 + 1e-9, 0]
    st[2, 0] = [0, 0.5]
    st[2, 1] = [0.5, 0.5]
    ok, msg = oracle.check_success(p, st)
    assert ok, msg


def test_kat_schedule(oracle):
    # SPEC.md:220-231
    ab, a = oracle.make_schedule(2, 0.25)
    np.testing.assert_allclose(ab, [1, 0.5, 0.25], rtol=1e-15)
    np.testing.assert_allclose(a, [0.5, 0.5], rtol=1e-15)
    ab, a = oracle.make_schedule(100, 0.05)
    assert abs(np.prod(a) - 0.05) < 1e-12


def test_kat_weights(oracle):
    # SPEC.md:280-282,312
    np.testing.assert_array_equal(oracle.score_weights(np.full(5, 0.3), 0.1), np.full(5, 0.2))
    r = np.array([0.1, 0.5, -0.2, 0.9])
    np.testing.assert_allclose(oracle.score_weights(r, 0.1), oracle.score_weights(r + 3.0, 0.1), rtol=1e-12)
    # z = [-1, 1] (rewards [0, 2] have pop-std 1), λ = 1 → [0.1192, 0.8808]
    np.testing.assert_allclose(oracle.score_weights(np.array([0.0, 2.0]), 1.0), [0.11920292, 0.88079708], atol=1e-8)
    w = oracle.score_weights(np.random.default_rng(0).normal(size=1000), 0.1)
    assert abs(w.sum() - 1) < 1e-12
    with pytest.raises(ValueError):
        oracle.score_weights(np.ones(1), 0.1)
    with pytest.raises(RuntimeError, match="non-finite reward for sample 1"):
        oracle.score_weights(np.array([0.0, np.inf]), 0.1)


def test_kat_mc_average_and_step(reference):
    # SPEC.md:289-291, 298-300
    s = np.stack([np.zeros((3, 1, 2)), np.ones((3, 1, 2))])
    np.testing.assert_allclose(reference.mc_average(s, [0.25, 0.75]), np.full((3, 1, 2), 0.75))


def test_denoising_deterministic_and_single_step(oracle):
    # fixed seed → identical output; worker count does not matter
    p = S.antipodal_circle(4, 4.0, S.HOLO2D, horizon=12)
    base = np.zeros((12, 4, 2))
    v1, t1 = oracle.run_denoising(p, base, make_config(3, 16, seed=5, workers=1))
    v2, t2 = oracle.run_denoising(p, base, make_config(3, 16, seed=5, workers=4))
    np.testing.assert_array_equal(v1, v2)
    assert t1 == t2


# ------------------------------------------------- (2) bitwise vs reference
PIN_PROBLEMS = {
    "holo2d": lambda: S.antipodal_circle(6, 3.0, S.HOLO2D, horizon=20),
    "diffdrive": lambda: S.antipodal_circle(5, 3.0, S.DIFFDRIVE, horizon=20),
    "holo3d": lambda: S.antipodal_sphere(6, 3.0, horizon=20),
    "C2": lambda: S.baseline_config(2).problem.with_horizon(20),
    "C3": lambda: S.baseline_config(3).problem.with_horizon(20),
    "C4": lambda: S.baseline_config(4).problem.with_horizon(20),
    "C5": lambda: S.baseline_config(5).problem.with_horizon(8),
}


def test_pin_rng(oracle, reference):
    for seed in (0, 1, 12345, 2**63 + 7):
        np.testing.assert_array_equal(oracle.normal_fill(seed, 777), reference.normal_fill(seed, 777))
        assert oracle.mix_seed(seed, 3, 9) == reference.mix_seed(seed, 3, 9) == S.mix_seed(seed, 3, 9)


@pytest.mark.parametrize("name", list(PIN_PROBLEMS))
def test_pin_rollout_reward(oracle, reference, name):
    p = PIN_PROBLEMS[name]()
    rng = np.random.default_rng(1)
    for scale in (0.5, 3.0):
        u = rng.normal(size=(p.horizon, p.robots, p.du)) * scale
        s1, c1 = oracle.rollout(p, u)
        s2, c2 = reference.rollout(p, u)
        np.testing.assert_array_equal(s1, s2)
        np.testing.assert_array_equal(c1, c2)
        assert oracle.total_reward(p, s1)[0] == reference.total_reward(p, s2)
        assert oracle.objective(p, s1) == reference.objective(p, s2)
        assert oracle.check_success(p, s1) == reference.check_success(p, s2)


@pytest.mark.parametrize("name", ["holo2d", "diffdrive", "holo3d", "C2", "C3", "C4"])
@pytest.mark.parametrize("mode", [0, 1])
def test_pin_run_denoising(oracle, reference, name, mode):
    p = PIN_PROBLEMS[name]()
    base = np.random.default_rng(2).normal(size=(p.horizon, p.robots, p.du)) * 0.3
    cfg = make_config(4, 24, seed=77, mode=mode, workers=2)
    v1, t1 = oracle.run_denoising(p, base, cfg)
    v2, t2 = reference.run_denoising(p, base, cfg)
    np.testing.assert_array_equal(v1, v2)
    assert t1 == t2


def test_pin_sample_batch(oracle, reference):
    p = PIN_PROBLEMS["C2"]()
    cur = np.random.default_rng(3).normal(size=(p.horizon, p.robots, p.du))
    ab, _ = oracle.make_schedule(10, 0.05)
    ms, sd = 1 / math.sqrt(ab[6]), math.sqrt(1 / ab[6] - 1)
    assert (ms, sd) == reference.sampling_spread(10, 0.05, 6)
    z = oracle.step_noise(99, 6, 0, 5, p.elems)
    want = ms * cur.reshape(1, -1) + sd * z
    got = reference.sample_batch(p, cur, 10, 0.05, 6, 5, 99).reshape(5, -1)
    np.testing.assert_array_equal(got, want)


def test_pin_mc_average_and_weighted_update(oracle, reference):
    """or_mc_average is the reference's mc_average bitwise; or_weighted_update
    (sample_batch + mc_average + denoise_step for given weights, the stage the
    fp32 GPU parity tests feed the GPU's own rewards through) equals
    sqrt(ab[i-1]) * mc_average(sample_batch(...)) of the reference bitwise."""
    p = PIN_PROBLEMS["C2"]()
    M, N, i, seed = 37, 10, 6, 99
    cur = np.random.default_rng(4).normal(size=(p.horizon, p.robots, p.du))
    smp = reference.sample_batch(p, cur, N, 0.05, i, M, seed)
    w = oracle.score_weights(np.random.default_rng(5).normal(size=M), 0.1)
    want = reference.mc_average(smp, w)
    np.testing.assert_array_equal(oracle.mc_average(smp, w), want)
    ab, _ = oracle.make_schedule(N, 0.05)
    ms, sd = reference.sampling_spread(N, 0.05, i)
    z = oracle.step_noise(seed, i, 0, M, p.elems)
    got = oracle.weighted_update(cur, z, w, ms, sd, math.sqrt(ab[i - 1]))
    np.testing.assert_array_equal(got, math.sqrt(ab[i - 1]) * want)
    with pytest.raises(ValueError, match="weights must sum to 1"):
        oracle.mc_average(smp, w * 1.01)


def test_oracle_step_chain_equals_run_denoising(oracle):
    """The GPU free-running parity tests drive the oracle one denoise_step at a
    time with given noise; that chain is run_denoising bitwise."""
    p = PIN_PROBLEMS["C4"]()
    N, M, seed = 5, 40, 12
    base = np.random.default_rng(6).normal(size=(p.horizon, p.robots, p.du)) * 0.3
    cfg = make_config(N, M, seed=seed, workers=2)
    want, tr_want = oracle.run_denoising(p, base, cfg)
    ab, _ = oracle.make_schedule(N, 0.05)
    v = np.zeros_like(base)
    tr = []
    for i in range(N, 0, -1):
        v, _, _, rec = oracle.denoise_step(p, base, v, ab, cfg, i, oracle.step_noise(seed, i, 0, M, p.elems))
        tr.append(rec)
    np.testing.assert_array_equal(v, want)
    assert tr == tr_want


@pytest.mark.parametrize("name", ["holo2d", "C3"])
def test_pin_solve(oracle, reference, name):
    p = PIN_PROBLEMS[name]()
    cfg = make_config(3, 16, seed=1)
    a = oracle.solve(p, cfg, max_iterations=3, stop_on_success=False)
    b = reference.solve(p, cfg, max_iterations=3, stop_on_success=False)
    np.testing.assert_array_equal(a["states"], b["states"])
    assert a["best_reward"] == b["best_reward"] and a["per_iteration"] == b["per_iteration"]


@pytest.mark.parametrize("name", ["holo2d", "C2", "C3"])
def test_pin_mppi_cem(oracle, reference, name):
    """MPPI / CEM baselines (baselines.cpp:99-173): the C restatement bitwise
    against the reference's own mppi_solve / cem_solve (native kinds) or the
    same statements with the extension rollout."""
    p = PIN_PROBLEMS[name]()
    mc = mppi_config(24, sigma=0.7, iterations=3, seed=5, stop_on_success=False)
    a, b = oracle.mppi_solve(p, mc), reference.mppi_solve(p, mc)
    np.testing.assert_array_equal(a["states"], b["states"])
    assert a["best_reward"] == b["best_reward"] and a["per_iteration"] == b["per_iteration"]
    assert a["iterations"] == b["iterations"] == 3
    cc = cem_config(40, elite_fraction=0.2, initial_std=0.8, min_std=0.05, iterations=3, seed=9, stop_on_success=False)
    a, b = oracle.cem_solve(p, cc), reference.cem_solve(p, cc)
    np.testing.assert_array_equal(a["states"], b["states"])
    assert a["best_reward"] == b["best_reward"] and a["per_iteration"] == b["per_iteration"]


def test_pin_select_elites(oracle, reference):
    rng = np.random.default_rng(3)
    for m, k in [(10, 3), (64, 6), (257, 25), (5, 5), (7, 1)]:
        r = np.round(rng.normal(size=m), 1)  # many ties: lower index wins
        assert oracle.select_elites(r, k) == reference.select_elites(r, k)
    with pytest.raises(ValueError, match="elite count out of range"):
        oracle.select_elites(np.zeros(4), 5)
    with pytest.raises(ValueError, match="elite count out of range"):
        reference.select_elites(np.zeros(4), 0)


def test_pin_generators(reference):
    for n, d in [(4, 8.0), (16, 12.0), (7, 5.0)]:
        st, go = reference.antipodal_circle(n, d, 1, 0.25)
        q = S.antipodal_circle(n, d, S.HOLO2D, 0.25)
        np.testing.assert_array_equal(st, q.starts)
        np.testing.assert_array_equal(go, q.goals)
    st, go = reference.antipodal_circle(8, 10.0, 0, 0.3)
    q = S.antipodal_circle(8, 10.0, S.DIFFDRIVE, 0.3)
    np.testing.assert_array_equal(st, q.starts)
    st, go = reference.antipodal_sphere(9, 6.0, 0.1)
    q = S.antipodal_sphere(9, 6.0, 0.1)
    np.testing.assert_array_equal(st, q.starts)
    np.testing.assert_array_equal(go, q.goals)
    st, go = reference.random_square(12, 6.0, 5, 1, 0.2)
    q = S.random_square(12, 6.0, 5, S.HOLO2D, 0.2)
    np.testing.assert_array_equal(st, q.starts)
    np.testing.assert_array_equal(go, q.goals)


# ------------------------------------------------------ (3) golden vectors
def _golden():
    f = GOLDEN / "golden.npz"
    if not f.exists():
        pytest.skip("tests/golden/golden.npz missing")
    return np.load(f, allow_pickle=False), json.loads((GOLDEN / "golden.json").read_text())


def test_golden_vectors(oracle):
    g, meta = _golden()
    for seed in meta["normal_seeds"]:
        np.testing.assert_array_equal(oracle.normal_fill(seed, meta["normal_count"]), g[f"normal_{seed}"])
    for case in meta["cases"]:
        p = S.baseline_config(case["config"]).problem.with_horizon(case["horizon"])
        u = g[f"{case['id']}_u"]
        st, ct = oracle.rollout(p, u)
        np.testing.assert_array_equal(st, g[f"{case['id']}_states"])
        r, nc, no = oracle.total_reward(p, st)
        assert r == float(g[f"{case['id']}_reward"])
        cfg = make_config(case["steps"], case["batch"], seed=case["seed"])
        v, tr = oracle.run_denoising(p, g[f"{case['id']}_base"], cfg)
        np.testing.assert_array_equal(v, g[f"{case['id']}_variable"])
        np.testing.assert_array_equal(np.array(tr), g[f"{case['id']}_trace"])
