"""d4orm_cuda_weighted_mean — mc_average (denoiser.cpp:92-108) as a device
stage (K5a chunk partials + K5b pairwise tree) — against the oracle's
mc_average, itself pinned bitwise to the reference's
(tests/test_oracle_pin.py::test_pin_mc_average_and_weighted_update).

Tolerances: fp64 — the per-chunk sums are the reference's ascending-m sums,
only the order in which the 256-sample chunks combine differs, so the error
is bounded by a few ulps of Σ_m |w_m·x_m|: 1e-13 of that.  fp32 — samples
and weights rounded to fp32, fp32 accumulation: 2e-6 of Σ_m |w_m·x_m|.
Shapes cover both K5a forms (E < 16384: 16 lanes per element group; E ≥
16384: one sequential walk per thread with the compacted non-zero weights),
ragged E (not a multiple of 4), M below / at / above one chunk and
non-multiples of 256, and zero weights.
"""
import numpy as np
import pytest

import paper_2503_12204_b200 as d4

pytestmark = pytest.mark.gpu

SHAPES = [(1, 1), (2, 3), (255, 7), (256, 64), (257, 4096), (1000, 2050), (3000, 16384), (700, 32771)]


@pytest.fixture(scope="module")
def gpu():
    g = d4.GpuDenoiser()
    yield g
    g.close()


def _case(M, E, seed, sparse=False):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(M, E)) * 3.0 + 0.5
    w = rng.exponential(size=M)
    if sparse and M > 4:
        w[rng.random(M) < 0.6] = 0.0
        w[0] = max(w[0], 1.0)
    return x, w / w.sum()


@pytest.mark.parametrize("prec,rel", [(d4.PREC_F64, 1e-13), (d4.PREC_F32, 2e-6)])
@pytest.mark.parametrize("M,E", SHAPES)
def test_weighted_mean_matches_oracle(gpu, oracle, prec, rel, M, E):
    gpu.set_options(prec, d4.NOISE_HOST, False)
    for sparse in (False, True):
        x, w = _case(M, E, M * 31 + E, sparse)
        want = oracle.mc_average(x, w)
        got = gpu.weighted_mean(x, w)
        bound = rel * (np.abs(w)[:, None] * np.abs(x)).sum(0) + 1e-300
        err = np.abs(got - want)
        assert (err <= bound).all(), (prec, M, E, sparse, float((err / bound).max()))


def test_weighted_mean_errors(gpu):
    gpu.set_options(d4.PREC_F64, d4.NOISE_HOST, False)
    x = np.ones((4, 5))
    with pytest.raises(ValueError, match="weights must sum to 1"):
        gpu.weighted_mean(x, np.array([0.5, 0.5, 0.5, 0.0]))
    with pytest.raises(ValueError, match="weight count does not match"):
        gpu.weighted_mean(x, np.array([0.5, 0.5]))
    # the reference's tolerance on Σw is 1e-9 (denoiser.cpp:97-101)
    w = np.full(4, 0.25)
    w[0] += 5e-10
    np.testing.assert_allclose(gpu.weighted_mean(x, w), np.ones(5) * (1 + 5e-10), rtol=1e-15)


def test_weighted_mean_is_the_step_reduction(gpu, oracle):
    """The same K5 the denoising step runs: feeding the step's own samples
    (mean_scale·var + std·z) and weights through weighted_mean gives the step's
    update / √ᾱ_{i−1} (fp64: within rounding)."""
    from paper_2503_12204_b200 import scenarios as S
    p = S.baseline_config(2).problem.with_horizon(24)
    M, N, i, seed = 512, 10, 4, 3
    gpu.set_options(d4.PREC_F64, d4.NOISE_HOST, False)
    gpu.set_problem(p)
    cfg = d4.DenoiserConfig(steps=N, batch=M, seed=seed)
    rng = np.random.default_rng(0)
    var = 0.2 * rng.normal(size=(p.horizon, p.robots, p.du))
    z = oracle.step_noise(seed, i, 0, M, p.elems)
    v, r, w, _ = gpu.denoise_step(np.zeros_like(var), var, i, cfg, z)
    ab = d4.make_schedule(N, 0.05)
    smp = (1 / np.sqrt(ab[i])) * var.reshape(1, -1) + np.sqrt(1 / ab[i] - 1) * z
    avg = gpu.weighted_mean(smp, w)
    np.testing.assert_allclose(np.sqrt(ab[i - 1]) * avg, v.ravel(), rtol=1e-12, atol=1e-14)
