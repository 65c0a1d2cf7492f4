"""K4's fp32 weights (the input of K5) and their adaptive floor
(csrc/d4orm_kernels.cuh, kW32Mass): a sample's w32 is zeroed only when it lies
below a power-of-two floor 2^-b chosen so that ALL the zeroed weights add up to
at most 2^-24 of the total.  Checked on reward distributions of the path's
shapes (Gaussian, a collision-penalty mixture, heavy tails, ties, a degenerate
batch) over both K4 variants (one CTA for M <= 8192, the cooperative grid)."""
import numpy as np
import pytest

import paper_2503_12204_b200 as d4

MASS = 2.0 ** -24  # kW32Mass (csrc/d4orm_kernels.cuh): half an ulp of the fp32 weight sum

pytestmark = pytest.mark.gpu


def _rewards(kind, M, seed):
    rng = np.random.default_rng(seed)
    if kind == "gauss":
        return rng.normal(-0.3, 0.05, M)
    if kind == "collisions":  # goal term + penalty for a random number of conflict robot-steps
        return rng.normal(0.2, 0.02, M) - 2.0 / 512 * rng.poisson(rng.uniform(0, 40, M))
    if kind == "heavy":
        return -np.abs(rng.standard_cauchy(M)) * 0.01
    if kind == "ties":
        return np.round(rng.normal(0, 1, M), 1)
    if kind == "constant":
        return np.full(M, 0.25)
    raise ValueError(kind)


@pytest.fixture(scope="module")
def gpu():
    g = d4.GpuDenoiser()
    yield g
    g.close()


@pytest.mark.parametrize("M", [1000, 8192, 16384, 262144])
@pytest.mark.parametrize("kind", ["gauss", "collisions", "heavy", "ties", "constant"])
def test_w32_floor(gpu, kind, M):
    r = _rewards(kind, M, M + len(kind))
    w, _ = gpu.score_weights(r, 0.1)
    w32 = gpu.last_w32(M)
    kept = w32 != 0
    assert kept[np.argmax(w)]
    # kept weights are the fp64 weights rounded to fp32
    np.testing.assert_array_equal(w32[kept], w[kept].astype(np.float32))
    # the zeroed weights add up to at most 2^-24 of the total (Σw = 1)
    assert w[~kept].sum() <= MASS * (1 + 1e-12)
    # and the floor is a threshold: every zeroed weight lies below every kept one
    if (~kept).any():
        assert w[~kept].max() < w[kept].min()
    if kind == "constant":
        assert kept.all()


def test_w32_floor_drops_most_at_c5_like_spread(gpu):
    """At λ = 0.1 on z-scores the floor removes most of a Gaussian batch (that
    is what K5 saves), while the kept set still carries 1 − 2^-24 of the mass."""
    r = _rewards("gauss", 262144, 3)
    w, _ = gpu.score_weights(r, 0.1)
    kept = gpu.last_w32(len(r)) != 0
    assert kept.mean() < 0.25
    assert w[kept].sum() >= 1 - MASS
