"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle on
identical inputs and identical noise.

Tolerances (written here):
  * fp64 parity mode: states rel 1e-12 (holonomic kinds are exact sums;
    sin/cos kinds differ from glibc by ulps), rewards abs 1e-12, collision /
    obstacle counts exact, weights rel 1e-9, variable rel 1e-9.
  * fp32 throughput mode: states abs 2e-5 m, rewards abs 2e-5 (+ one
    w_t/(R·T) per explained decision flip) for arbitrary control batches; a
    denoising step: rewards 1e-6 after whole flips, ≤ 2 % flips, K4 on the
    GPU's rewards 1e-11 rel, K5 on them 5e-6 of max|v|, the whole step 1e-4 of
    max|v| without flips, else the flips' own effect + 5e-6
    (tests/e2e_f32.py::check_step_f32).
"""
import numpy as np
import pytest

import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
from oracle.oracle import make_config

pytestmark = pytest.mark.gpu

CASES = {
    "holo2d": lambda: S.antipodal_circle(6, 4.0, S.HOLO2D, horizon=24),
    "diffdrive": lambda: S.antipodal_circle(5, 4.0, S.DIFFDRIVE, horizon=24),
    "holo3d": lambda: S.antipodal_sphere(7, 4.0, horizon=24),
    "C1": lambda: S.baseline_config(1).problem,
    "C2": lambda: S.baseline_config(2).problem.with_horizon(40),
    "C3": lambda: S.baseline_config(3).problem.with_horizon(40),
    "C4": lambda: S.baseline_config(4).problem.with_horizon(40),
    "C5": lambda: S.baseline_config(5).problem.with_horizon(24),
    "R40": lambda: S.random_square(40, 8.0, 3, S.HOLO2D_VEL, robot_radius=0.15, horizon=16, lower=[-1, -1], upper=[1, 1]),
    # 20 robots: a tile width that is not a multiple of the 16-step rollout block (TC widened, choose_tc)
    "R20": lambda: S.random_square(20, 7.0, 5, S.HOLO2D_VEL, robot_radius=0.15, horizon=40, lower=[-1, -1], upper=[1, 1]),
}


def controls_for(p, count, seed, scale=1.5):
    rng = np.random.default_rng(seed)
    # biased toward the goals so robots meet (collisions happen) + noise
    d = (p.goals - p.starts[:, : p.pdim])
    drift = np.zeros((p.robots, p.du))
    if p.kind in (S.HOLO2D_VEL, S.HOLO3D_VEL):
        drift = d / (p.horizon * p.dt)
    return drift[None, None] + scale * rng.normal(size=(count, p.horizon, p.robots, p.du))


@pytest.fixture(scope="module")
def gpu():
    g = d4.GpuDenoiser()
    yield g
    g.close()


def oracle_rollout_batch(oracle, p, u):
    out = []
    for m in range(u.shape[0]):
        st, ct = oracle.rollout(p, u[m])
        r, nc, no = oracle.total_reward(p, st)
        out.append((st, ct, r, nc, no))
    return out


@pytest.mark.parametrize("case", list(CASES))
def test_rollout_fitness_f64_matches_oracle(gpu, oracle, case):
    p = CASES[case]()
    gpu.set_options(d4.PREC_F64, d4.NOISE_HOST)
    gpu.set_problem(p)
    u = controls_for(p, 24, 1)
    st, ct, rw, cnt = gpu.rollout_fitness(u)
    ref = oracle_rollout_batch(oracle, p, u)
    for m, (rs, rc, rr, nc, no) in enumerate(ref):
        if p.kind in (S.DIFFDRIVE, S.UNICYCLE):
            np.testing.assert_allclose(st[m], rs, rtol=1e-12, atol=1e-12)
        else:
            np.testing.assert_array_equal(st[m], rs)
        np.testing.assert_array_equal(ct[m], rc)
        assert abs(rw[m] - rr) <= 1e-12, (m, rw[m], rr)
        assert (cnt[m, 0], cnt[m, 1]) == (nc, no), (m, cnt[m], nc, no)


def _counts(p, st, delta):
    """Conflict / obstacle robot-steps (t >= 1) with the squared thresholds
    shifted by delta (numpy, fp64)."""
    pos = st[1:, :, : p.pdim]
    m2 = (2 * p.robot_radius + p.epsilon) ** 2 + delta
    d2 = ((pos[:, :, None, :] - pos[:, None, :, :]) ** 2).sum(-1)
    R = p.robots
    d2[:, np.arange(R), np.arange(R)] = np.inf
    nc = int((d2 <= m2).any(-1).sum())
    no = 0
    if len(p.obs_radii):
        od2 = ((pos[:, :, None, :] - p.obs_centers[None, None]) ** 2).sum(-1)
        no = int((od2 <= (p.obs_radii + p.robot_radius)[None, None] ** 2 + delta).any(-1).sum())
    return nc, no


# fp32 decisions use the expanded form |a|²+|b|²−2a·b on fp32 positions: a flip
# is 'explained' when the GPU count lies between the counts with the squared
# margin shifted by ∓FLIP_BAND on the GPU's own positions.
FLIP_BAND = 2e-4


def explain_flips(oracle, p, st_gpu, nc_gpu, no_gpu):
    lo = _counts(p, st_gpu, -FLIP_BAND)
    hi = _counts(p, st_gpu, FLIP_BAND)
    return lo[0] <= nc_gpu <= hi[0] and lo[1] <= no_gpu <= hi[1]


@pytest.mark.parametrize("case", list(CASES))
def test_rollout_fitness_f32_matches_oracle(gpu, oracle, case):
    p = CASES[case]()
    gpu.set_options(d4.PREC_F32, d4.NOISE_HOST)
    gpu.set_problem(p)
    u = controls_for(p, 24, 2)
    st, ct, rw, cnt = gpu.rollout_fitness(u)
    ref = oracle_rollout_batch(oracle, p, u)
    unit = max(p.w_t, p.obstacle_weight) / (p.robots * p.horizon)
    for m, (rs, rc, rr, nc, no) in enumerate(ref):
        np.testing.assert_allclose(st[m], rs, atol=2e-5, rtol=1e-5)
        np.testing.assert_allclose(ct[m], rc, atol=1e-6, rtol=1e-6)
        flips = abs(cnt[m, 0] - nc) + abs(cnt[m, 1] - no)
        if flips:
            assert explain_flips(oracle, p, st[m], cnt[m, 0], cnt[m, 1]), (m, cnt[m], nc, no)
        assert abs(rw[m] - rr) <= 2e-5 + flips * unit, (m, rw[m], rr, flips)


def test_collisions_are_counted(gpu, oracle):
    """Robots parked in conflict, and exactly on the (2R_a+eps) boundary: the
    reference's `<=` counts it."""
    p = S.Problem(S.HOLO2D_VEL, starts=[[0, 0], [0.25, 0], [3, 3]], goals=[[1, 1], [2, 2], [-3, -3]],
                  horizon=4, lower=[-1, -1], upper=[1, 1], robot_radius=0.1, epsilon=0.05)
    u = np.zeros((1, 4, 3, 2))
    for prec in (d4.PREC_F64, d4.PREC_F32):
        gpu.set_options(prec, d4.NOISE_HOST)
        gpu.set_problem(p)
        st, ct, rw, cnt = gpu.rollout_fitness(u)
        r, nc, no = oracle.total_reward(p, st[0].astype(np.float64))
        assert nc == 8 and cnt[0, 0] == 8, (prec, cnt, nc)
        assert abs(rw[0] - r) < 1e-6


@pytest.mark.parametrize("m", [2, 3, 1000, 8192, 16384, 70001, 400000])
def test_score_weights(gpu, oracle, m):
    rng = np.random.default_rng(m)
    r = rng.normal(size=m) * 0.01 + 0.3
    w, t3 = gpu.score_weights(r, 0.1)
    wo = oracle.score_weights(r, 0.1)
    np.testing.assert_allclose(w, wo, rtol=1e-9, atol=1e-300)
    assert abs(t3[2] - oracle.weight_entropy(wo)) < 1e-9 * max(1, abs(t3[2]))
    assert t3[0] == r.max() and abs(t3[1] - r.mean()) < 1e-12


def test_score_weights_degenerate_and_errors(gpu):
    w, _ = gpu.score_weights(np.full(10, 0.5), 0.1)
    np.testing.assert_array_equal(w, np.full(10, 0.1))
    with pytest.raises(ValueError):
        gpu.score_weights(np.ones(1), 0.1)
    with pytest.raises(ValueError):
        gpu.score_weights(np.ones(4), 0.0)
    with pytest.raises(d4.D4ormError, match="non-finite reward for sample 2"):
        gpu.score_weights(np.array([0.1, 0.2, np.nan, 0.3]), 0.1)


@pytest.mark.parametrize("case", ["holo2d", "C2", "C3", "C4", "R40"])
@pytest.mark.parametrize("prec", [d4.PREC_F64, d4.PREC_F32])
def test_denoise_step_teacher_forced(gpu, oracle, case, prec):
    p = CASES[case]()
    M, N, i = 512, 10, 7
    cfg = d4.DenoiserConfig(steps=N, batch=M, seed=11)
    ocfg = make_config(N, M, seed=11)
    ab, _ = oracle.make_schedule(N, 0.05)
    rng = np.random.default_rng(5)
    base = controls_for(p, 1, 3, scale=0.3)[0]
    var = 0.2 * rng.normal(size=base.shape)
    noise = oracle.step_noise(11, i, 0, M, p.elems)
    if prec == d4.PREC_F32:  # the fp32 path consumes fp32 normals: give the oracle exactly those
        noise = noise.astype(np.float32).astype(np.float64)
    gpu.set_options(prec, d4.NOISE_HOST)
    gpu.set_problem(p)
    v_g, r_g, w_g, rec_g = gpu.denoise_step(base, var, i, cfg, noise)
    v_o, r_o, w_o, rec_o = oracle.denoise_step(p, base, var, ab, ocfg, i, noise)
    if prec == d4.PREC_F64:
        np.testing.assert_allclose(r_g, r_o, atol=1e-12)
        np.testing.assert_allclose(w_g, w_o, rtol=1e-8, atol=1e-300)
        np.testing.assert_allclose(v_g, v_o, rtol=1e-9, atol=1e-12)
    else:
        from e2e_f32 import check_step_f32
        m = check_step_f32(oracle, p, var, i, ab, cfg.lam, noise, v_g, r_g, w_g, v_o, r_o, tag=case)
        print(case, m)
    assert rec_g[0] == i


@pytest.mark.parametrize("case", ["holo2d", "C1", "C3"])
def test_run_denoising_host_noise_f64(gpu, oracle, case):
    """Free-running N steps with the oracle's own NormalStream noise: fp64 GPU
    path tracks the reference within 1e-9 relative."""
    p = CASES[case]()
    M, N = 256, 8
    for mode in (d4.DEFORMATION, d4.FROM_SCRATCH):
        cfg = d4.DenoiserConfig(steps=N, batch=M, seed=4, mode=mode)
        base = controls_for(p, 1, 4, scale=0.3)[0]
        gpu.set_options(d4.PREC_F64, d4.NOISE_HOST)
        gpu.set_problem(p)
        gpu.set_noise_provider(lambda step, m0, count, elems: (
            oracle.normal_fill(oracle.mix_seed(4, 0, 0), elems)[None] if step == 0 else
            oracle.step_noise(4, step, m0, count, elems)))
        v_g, tr_g = gpu.run_denoising(base, cfg)
        v_o, tr_o = oracle.run_denoising(p, base, make_config(N, M, seed=4, mode=mode))
        np.testing.assert_allclose(v_g, v_o, rtol=1e-9, atol=1e-12)
        for a, b in zip(tr_g, tr_o):
            assert a[0] == b[0]
            np.testing.assert_allclose(a[1:], b[1:], rtol=1e-9, atol=1e-12)


def test_run_denoising_philox_deterministic(gpu):
    p = CASES["C2"]()
    cfg = d4.DenoiserConfig(steps=6, batch=1024, seed=9)
    base = np.zeros((p.horizon, p.robots, p.du))
    gpu.set_options(d4.PREC_F32, d4.NOISE_PHILOX, graphs=True)
    gpu.set_problem(p)
    v1, t1 = gpu.run_denoising(base, cfg)
    v2, t2 = gpu.run_denoising(base, cfg)
    gpu.set_options(d4.PREC_F32, d4.NOISE_PHILOX, graphs=False)
    v3, t3 = gpu.run_denoising(base, cfg)
    np.testing.assert_array_equal(v1, v2)
    np.testing.assert_array_equal(v1, v3)
    assert t1 == t2 == t3
    assert np.abs(v1).max() > 0


def test_philox_noise_is_standard_normal_and_shard_invariant(gpu):
    p = CASES["C2"]()
    gpu.set_options(d4.PREC_F32, d4.NOISE_PHILOX)
    gpu.set_problem(p)
    z = gpu.philox_noise(123, 50, 0, 64)
    # K1 and the fused in-rollout draw are the same function: run one fp32
    # Philox step and one fp64 step (K1) with identical inputs → same rewards
    # up to fp32 rounding
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01
    z2 = gpu.philox_noise(123, 50, 32, 32)
    np.testing.assert_array_equal(z[32:], z2)
    z3 = gpu.philox_noise(123, 49, 0, 64)
    assert not np.array_equal(z, z3)
    big = gpu.philox_noise(7, 3, 0, 2048)  # 8.4M normals: finite, tails bounded by Box-Muller on 23-bit uniforms
    assert np.isfinite(big).all() and np.abs(big).max() < 6.5


def test_nonfinite_state_error_message(gpu):
    p = S.Problem(S.HOLO2D_VEL, starts=[[0, 0], [1, 1]], goals=[[1, 0], [0, 1]], horizon=5,
                  lower=[-np.inf, -np.inf], upper=[np.inf, np.inf])
    u = np.zeros((2, 5, 2, 2))
    u[1, 2, 1, 0] = np.inf
    gpu.set_options(d4.PREC_F32, d4.NOISE_HOST)
    gpu.set_problem(p)
    with pytest.raises(d4.D4ormError, match="member 1: rollout: non-finite state for robot 1 at step 3"):
        gpu.rollout_fitness(u)


def test_invalid_arguments(gpu):
    p = CASES["holo2d"]()
    gpu.set_problem(p)
    with pytest.raises(ValueError, match="batch must be >= 2"):
        gpu.run_denoising(np.zeros((p.horizon, p.robots, p.du)), d4.DenoiserConfig(steps=2, batch=1))
    with pytest.raises(ValueError, match="lambda must be > 0"):
        gpu.run_denoising(np.zeros((p.horizon, p.robots, p.du)), d4.DenoiserConfig(steps=2, batch=4, lam=0))
    bad = S.Problem(S.HOLO2D, starts=[[0, 0, 0, 0]], goals=[[0, 0]], horizon=3)
    with pytest.raises(ValueError, match="starts on its goal"):
        gpu.set_problem(bad)


@pytest.mark.parametrize("case", ["C2", "C3", "C4"])
def test_fused_philox_equals_k1_noise(gpu, case):
    """The fp32 hot path draws its noise inside K2+K3; feeding K1's output for
    the same (seed, step) through the host-noise path must give bitwise the
    same rewards, weights and updated variable."""
    p = CASES[case]()
    M, N, i, seed = 512, 10, 6, 21
    cfg = d4.DenoiserConfig(steps=N, batch=M, seed=seed)
    base = controls_for(p, 1, 8, scale=0.3)[0]
    var = 0.1 * np.random.default_rng(1).normal(size=base.shape)
    gpu.set_options(d4.PREC_F32, d4.NOISE_PHILOX)
    gpu.set_problem(p)
    v1, r1, w1, _ = gpu.denoise_step(base, var, i, cfg, None)
    key_seed = seed
    z = gpu.philox_noise(key_seed, i, 0, M).astype(np.float64)
    gpu.set_options(d4.PREC_F32, d4.NOISE_HOST)
    v2, r2, w2, _ = gpu.denoise_step(base, var, i, cfg, z)
    np.testing.assert_array_equal(r1, r2)
    np.testing.assert_array_equal(w1, w2)
    np.testing.assert_array_equal(v1, v2)


def test_nccl_protocol_on_one_rank():
    """The sharded protocol (reward all-gather, chunk-tree roots all-gather, all
    inside the step graphs) on a 1-rank NCCL communicator: bitwise the result of
    the single-GPU path."""
    import ctypes as C
    from paper_2503_12204_b200._lib import lib
    buf = C.create_string_buffer(128)
    assert lib().d4orm_cuda_nccl_id(buf) == 0
    p = CASES["C2"]()
    cfg = d4.DenoiserConfig(steps=5, batch=1024, seed=13)
    base = controls_for(p, 1, 2, scale=0.3)[0]
    a = d4.GpuDenoiser(p)
    b = d4.GpuDenoiser(p, rank=0, world=1, nccl_id=bytes(buf.raw))
    va, ta = a.run_denoising(base, cfg)
    vb, tb = b.run_denoising(base, cfg)
    # sharded: K2+K3, K4, K5a, K5b, root tree; one GPU: the same 4, or K2+K3 +
    # the fused small-batch tail (bitwise the same result, checked below)
    assert b.launches_per_step() == 5 and a.launches_per_step() in (2, 4)
    np.testing.assert_array_equal(va, vb)
    assert ta == tb
    a.close()
    b.close()


def test_nccl_protocol_solve_and_baselines_on_one_rank():
    """solve / MPPI / CEM (the bench's solve leg and the sharded baselines) on a
    1-rank NCCL communicator: bitwise the single-GPU results."""
    import ctypes as C
    from paper_2503_12204_b200._lib import lib
    p = CASES["C2"]()
    buf = C.create_string_buffer(128)
    assert lib().d4orm_cuda_nccl_id(buf) == 0
    a = d4.GpuDenoiser(p)
    b = d4.GpuDenoiser(p, rank=0, world=1, nccl_id=bytes(buf.raw))
    try:
        cfg = d4.DenoiserConfig(steps=6, batch=1024, seed=5)
        ra = a.solve(cfg, max_iterations=3, stop_on_success=False)
        rb = b.solve(cfg, max_iterations=3, stop_on_success=False)
        assert [x[:3] for x in ra.per_iteration] == [x[:3] for x in rb.per_iteration]
        np.testing.assert_array_equal(ra.best_states, rb.best_states)
        assert ra.traces == rb.traces
        for fn in ("mppi_solve", "cem_solve"):
            xa = getattr(a, fn)(batch=1024, iterations=4, seed=3, stop_on_success=False)
            xb = getattr(b, fn)(batch=1024, iterations=4, seed=3, stop_on_success=False)
            assert [x[:3] for x in xa.per_iteration] == [x[:3] for x in xb.per_iteration], fn
            np.testing.assert_array_equal(xa.best_controls, xb.best_controls)
    finally:
        a.close()
        b.close()


def test_philox_noise_matches_cpu_model(gpu):
    """K1 / the fused draw against the numpy model (tests/philox_model.py,
    itself pinned to the Philox4x32-10 known-answer vectors): the integer stream
    is exact, so the normals agree to the MUFU approximations (~1e-6)."""
    import philox_model
    for case, seed, step, m0, count in [("C2", 123, 50, 0, 64), ("C4", 9, 1, 1000, 16), ("C3", 2**63 + 5, 99, 2**33, 8)]:
        p = CASES[case]()
        gpu.set_options(d4.PREC_F32, d4.NOISE_PHILOX)
        gpu.set_problem(p)
        z = gpu.philox_noise(seed, step, m0, count).reshape(count, p.horizon, p.robots, p.du)
        ref = philox_model.normals(seed, step, m0, count, p.robots, p.horizon, p.du)
        err = np.abs(z.astype(np.float64) - ref)
        assert err.max() < 5e-5 * (1 + np.abs(ref).max()), (case, err.max())
        assert np.median(err) < 1e-6


@pytest.mark.parametrize("case", ["holo2d", "C2", "C3"])
def test_device_solve_matches_oracle(gpu, oracle, case):
    """The anytime loop on the device (K7 + steps + K6 per iteration) against
    the oracle's solve (optimizer.cpp:49-102) in correctness mode: same noise,
    fp64; the final rollout, total_reward, objective and check_success are
    computed in the reference's own order, so they agree to the Δ parity."""
    p = CASES[case]()
    N, M, seed, its = 6, 256, 7, 3
    cfg = d4.DenoiserConfig(steps=N, batch=M, seed=seed)
    cur = {"seed": None}
    gpu.set_options(d4.PREC_F64, d4.NOISE_HOST)
    gpu.set_problem(p)
    gpu.set_noise_provider(lambda step, m0, count, elems: oracle.step_noise(cur["seed"], step, m0, count, elems))
    res = gpu.solve(cfg, max_iterations=its, stop_on_success=False,
                    on_iteration=lambda it, seed_it: cur.__setitem__("seed", seed_it))
    ref = oracle.solve(p, make_config(N, M, seed=seed), max_iterations=its, stop_on_success=False)
    assert res.iterations_used == ref["iterations"] == its
    for a, b in zip(res.per_iteration, ref["per_iteration"]):
        assert abs(a[0] - b[0]) < 1e-9 and a[1] == b[1] and a[2] == b[2]
    assert abs(res.best_reward - ref["best_reward"]) < 1e-9
    assert res.success == ref["success"]
    np.testing.assert_allclose(res.best_states, ref["states"], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(res.best_controls, ref["controls"], rtol=1e-9, atol=1e-9)
    assert len(res.traces) == its and len(res.traces[0]) == N


def test_device_solve_philox_stops_on_success(gpu):
    """Throughput mode: Philox noise, one graph per iteration.  Deterministic
    for a seed; stop_on_success ends the loop at the first collision-free,
    goal-reaching iterate (C1-style swap that is reachable)."""
    p = S.antipodal_circle(4, 4.0, S.HOLO2D_VEL, robot_radius=0.1, horizon=48, lower=[-1, -1], upper=[1, 1])
    cfg = d4.DenoiserConfig(steps=40, batch=1024, seed=3)
    gpu.set_options(d4.PREC_F32, d4.NOISE_PHILOX)
    gpu.set_problem(p)
    r1 = gpu.solve(cfg, max_iterations=8, stop_on_success=True)
    r2 = gpu.solve(cfg, max_iterations=8, stop_on_success=True)
    assert r1.iterations_used == r2.iterations_used
    assert r1.best_reward == r2.best_reward
    np.testing.assert_array_equal(r1.best_states, r2.best_states)
    rewards = [it[0] for it in r1.per_iteration]
    assert r1.best_reward == max(rewards)
    if r1.success:
        assert r1.per_iteration[-1][2] and not any(it[2] for it in r1.per_iteration[:-1])
    # the device outcome equals the host restatement on the returned trajectory
    from outcome_model import check_success, objective
    assert check_success(p, r1.best_states)[0] == r1.success
    best_it = rewards.index(r1.best_reward)
    assert objective(p, r1.best_states) == r1.per_iteration[best_it][1]


@pytest.mark.parametrize("kind", ["C3", "diffdrive"])
def test_heading_kinds_f32_full_horizon(gpu, oracle, kind):
    """fp32 heading kinds (unicycle, diff-drive) over a full 128-step horizon
    with headings wound far from [−π, π]: the fast reduced sin/cos and the
    k2 = k3 stage sharing keep positions within 2e-5 m of the fp64 oracle."""
    p = (S.baseline_config(3).problem if kind == "C3"
         else S.antipodal_circle(5, 4.0, S.DIFFDRIVE, horizon=128))
    gpu.set_options(d4.PREC_F32, d4.NOISE_HOST)
    gpu.set_problem(p)
    u = controls_for(p, 16, 5, scale=2.5)   # clamped: |ω| at the limit most of the time
    st, ct, rw, cnt = gpu.rollout_fitness(u)
    worst = 0.0
    for m in range(u.shape[0]):
        rs, rc = oracle.rollout(p, u[m])
        worst = max(worst, float(np.abs(st[m][..., :2] - rs[..., :2]).max()))
        np.testing.assert_allclose(st[m], rs, atol=2e-5, rtol=1e-5)
    print(f"{kind}: max |Δposition| = {worst:.3g} m over {p.horizon} steps")


@pytest.mark.parametrize("case", ["C1", "C2", "C5"])
def test_run_graph_equals_eager_steps(gpu, case):
    """run_denoising replays ONE graph for the whole run in Philox mode; the
    eager per-step launches (graphs off) give bitwise the same variable and
    trace — both modes (FromScratch draws its initial variable with K1 first),
    and a second call reuses the graph."""
    p = CASES[case]()
    base = controls_for(p, 1, 9, scale=0.3)[0]
    M = 2048 if case != "C1" else 1024
    for mode in (d4.DEFORMATION, d4.FROM_SCRATCH):
        cfg = d4.DenoiserConfig(steps=7, batch=M, seed=4, mode=mode)
        gpu.set_options(d4.PREC_F32, d4.NOISE_PHILOX, graphs=True)
        gpu.set_problem(p)
        v1, t1 = gpu.run_denoising(base, cfg)
        v1b, t1b = gpu.run_denoising(base, cfg)
        gpu.set_options(d4.PREC_F32, d4.NOISE_PHILOX, graphs=False)
        v2, t2 = gpu.run_denoising(base, cfg)
        np.testing.assert_array_equal(v1, v2)
        np.testing.assert_array_equal(v1, v1b)
        assert t1 == t2 == t1b
