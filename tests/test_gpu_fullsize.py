"""Every BASELINE config at its full size.  C1–C4: one denoising step against
the oracle on the oracle's own noise (fp64 to 1e-9; fp32 by
tests/e2e_f32.py::check_step_f32: rewards, flips, K4 and K5 on the GPU's own
rewards, the whole step 1e-4 without flips).
C5 (R = 64, T = 256, N = 262144 samples, 16 obstacles) through size-independent
properties — the oracle cannot run a full C5 step in test time (≈ 2 min on 8
cores, 68.7 GB), so:

  * K4 at full size equals the oracle's score_weights on the step's own rewards
    (rel 1e-9), and the trace record is consistent with them;
  * single samples picked across the whole batch (first, last, both shard
    boundaries of an 8-way split) re-run on the host from their Philox noise
    agree with the fp64 oracle: reward 1e-6 after removing whole decision
    flips, each flip inside the fp32 band of the sample's own positions;
  * the step is deterministic, and the sharded protocol on a 1-rank NCCL
    communicator gives bitwise the same variable, rewards and weights;
  * a full 100-step run_denoising stays finite with entropies in [0, log N].
"""
import ctypes as C

import numpy as np
import pytest

import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S

pytestmark = pytest.mark.gpu

RC = S.baseline_config(5)
P = RC.problem
M = RC.samples
STEP = 100          # the first denoising step (largest sampling spread)
SEED = 21


def _variable():
    rng = np.random.default_rng(5)
    return 0.2 * rng.normal(size=(P.horizon, P.robots, P.du))


@pytest.fixture(scope="module")
def full_step():
    g = d4.GpuDenoiser(P)
    cfg = d4.DenoiserConfig(steps=RC.steps, batch=M, seed=SEED)
    base = np.zeros((P.horizon, P.robots, P.du))
    var = _variable()
    v1, r1, w1, rec1 = g.denoise_step(base, var, STEP, cfg)
    v2, r2, w2, rec2 = g.denoise_step(base, var, STEP, cfg)
    yield g, cfg, base, var, (v1, r1, w1, rec1), (v2, r2, w2, rec2)
    g.close()


def test_full_size_step_is_deterministic(full_step):
    _, _, _, _, a, b = full_step
    for x, y in zip(a[:3], b[:3]):
        np.testing.assert_array_equal(x, y)
    assert a[3] == b[3]


def test_full_size_weights_match_oracle(full_step, oracle):
    _, cfg, _, _, (v, r, w, rec), _ = full_step
    assert r.shape == (M,) and np.isfinite(r).all() and np.isfinite(v).all()
    wo = oracle.score_weights(r, cfg.lam)
    np.testing.assert_allclose(w, wo, rtol=1e-9, atol=1e-300)
    assert abs(w.sum() - 1.0) < 1e-9 and (w >= 0).all()
    step, best, mean, ent = rec
    assert step == STEP and best == r.max() and abs(mean - r.mean()) < 1e-12
    assert abs(ent - oracle.weight_entropy(wo)) < 1e-9 * max(1.0, abs(ent))
    assert 0.0 <= ent <= np.log(M)


@pytest.mark.parametrize("m", [0, 1, 32767, 32768, 131071, 131072, 262143])
def test_full_size_samples_match_oracle(full_step, oracle, m):
    """Sample m of the full-size step, rebuilt from its own Philox noise."""
    g, cfg, base, var, (_, r, _, _), _ = full_step
    ab = d4.make_schedule(cfg.steps, cfg.alpha_bar_final)
    ms, sd = 1.0 / np.sqrt(ab[STEP]), np.sqrt(1.0 / ab[STEP] - 1.0)
    z = g.philox_noise(cfg.seed, STEP, m, 1)[0].astype(np.float64).reshape(P.horizon, P.robots, P.du)
    u = base + ms * var + sd * z
    st_o, _ = oracle.rollout(P, u)
    r_o, nc, no = oracle.total_reward(P, st_o)
    g.set_options(d4.PREC_F32, d4.NOISE_HOST)
    st_g, _, r_g, cnt = g.rollout_fitness(u[None])
    g.set_options(d4.PREC_F32, d4.NOISE_PHILOX)
    np.testing.assert_allclose(st_g[0], st_o, atol=2e-5, rtol=1e-5)
    unit = max(P.w_t, P.obstacle_weight) / (P.robots * P.horizon)
    # the full-size step's reward for sample m against the oracle's on the same
    # noise: a continuous part (fp32 positions) plus k whole decision flips
    # (w_t = w_o, so a flip of either kind moves the reward by one unit); the
    # step kernel's count nc + no − k must lie in the fp32 band of the counts
    # on the GPU's positions of this sample
    from test_gpu_parity import _counts, FLIP_BAND
    k = round((r_o - r[m]) / unit)
    assert abs((r[m] - r_o) + k * unit) <= 1e-6, (m, r[m], r_o, k)
    lo, hi = _counts(P, st_g[0], -FLIP_BAND), _counts(P, st_g[0], FLIP_BAND)
    assert lo[0] + lo[1] <= nc + no + k <= hi[0] + hi[1], (m, nc, no, k, lo, hi)


def test_full_size_sharded_protocol_is_bitwise(full_step):
    """The step through a 1-rank NCCL communicator (reward all-gather and the
    chunk-tree root all-gather inside the step) at full size."""
    from paper_2503_12204_b200._lib import lib
    g, cfg, base, var, (v, r, w, rec), _ = full_step
    buf = C.create_string_buffer(128)
    assert lib().d4orm_cuda_nccl_id(buf) == 0
    b = d4.GpuDenoiser(P, rank=0, world=1, nccl_id=bytes(buf.raw))
    try:
        vb, rb, wb, recb = b.denoise_step(base, var, STEP, cfg)
    finally:
        b.close()
    np.testing.assert_array_equal(rb, r)
    np.testing.assert_array_equal(wb, w)
    np.testing.assert_array_equal(vb, v)
    assert recb == rec


def test_full_size_run_denoising(full_step):
    g, cfg, base, _, _, _ = full_step
    v, tr = g.run_denoising(base, cfg)
    assert np.isfinite(v).all() and len(tr) == cfg.steps
    assert [t[0] for t in tr] == list(range(cfg.steps, 0, -1))
    for step, best, mean, ent in tr:
        assert best >= mean and 0.0 <= ent <= np.log(M) + 1e-9


@pytest.mark.parametrize("cfg_index", [1, 2, 3, 4])
@pytest.mark.parametrize("prec", [d4.PREC_F64, d4.PREC_F32])
def test_full_size_teacher_forced_step_c1_c4(oracle, cfg_index, prec):
    """C1–C4 are small enough for the oracle: one denoising step at the full
    BASELINE shape (N, T, R, obstacles) with the oracle's own noise, GPU vs
    oracle — fp64 to 1e-9, fp32 within the stated band."""
    from oracle.oracle import make_config
    rc = S.baseline_config(cfg_index)
    p, M, N, i = rc.problem, rc.samples, rc.steps, 63
    cfg = d4.DenoiserConfig(steps=N, batch=M, seed=17)
    ocfg = make_config(N, M, seed=17)
    ab, _ = oracle.make_schedule(N, 0.05)
    rng = np.random.default_rng(cfg_index)
    base = 0.3 * rng.normal(size=(p.horizon, p.robots, p.du))
    var = 0.2 * rng.normal(size=base.shape)
    noise = oracle.step_noise(17, i, 0, M, p.elems)
    if prec == d4.PREC_F32:  # the fp32 path consumes fp32 normals: give the oracle exactly those
        noise = noise.astype(np.float32).astype(np.float64)
    g = d4.GpuDenoiser(p, precision=prec, noise=d4.NOISE_HOST)
    try:
        v_g, r_g, w_g, rec_g = g.denoise_step(base, var, i, cfg, noise)
    finally:
        g.close()
    v_o, r_o, w_o, rec_o = oracle.denoise_step(p, base, var, ab, ocfg, i, noise)
    assert rec_g[0] == i
    if prec == d4.PREC_F64:
        np.testing.assert_allclose(r_g, r_o, atol=1e-12)
        np.testing.assert_allclose(w_g, w_o, rtol=1e-8, atol=1e-300)
        np.testing.assert_allclose(v_g, v_o, rtol=1e-9, atol=1e-12)
    else:
        from e2e_f32 import check_step_f32
        print(rc.name, check_step_f32(oracle, p, var, i, ab, 0.1, noise, v_g, r_g, w_g, v_o, r_o, tag=rc.name))
