"""MPPI / CEM baselines (baselines.cpp:99-173) on the device vs the oracle.

Correctness mode: fp64 arithmetic and the oracle's NormalStream noise (the
host provider's `step` is the iteration), so the GPU loop must reproduce the
oracle's per-iteration reward / objective / success and the best trajectory
(the oracle is pinned bitwise to the reference's own mppi_solve / cem_solve in
tests/test_oracle_pin.py).  Throughput mode (fp32, Philox) is checked for
determinism and for the device outcome against the host restatement."""
import numpy as np
import pytest

import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
from oracle.oracle import cem_config, mppi_config

pytestmark = pytest.mark.gpu

CASES = {
    "holo2d": lambda: S.antipodal_circle(6, 4.0, S.HOLO2D, horizon=24),
    "C2": lambda: S.baseline_config(2).problem.with_horizon(32),
    "C3": lambda: S.baseline_config(3).problem.with_horizon(32),
    "C4": lambda: S.baseline_config(4).problem.with_horizon(24),
}


@pytest.fixture(scope="module")
def gpu():
    g = d4.GpuDenoiser()
    yield g
    g.close()


def _host_noise(gpu, oracle, seed):
    gpu.set_options(d4.PREC_F64, d4.NOISE_HOST)
    gpu.set_noise_provider(lambda step, m0, count, elems: oracle.step_noise(seed, step, m0, count, elems))


def _compare(res, ref, iters):
    assert res.iterations_used == ref["iterations"] == iters
    for a, b in zip(res.per_iteration, ref["per_iteration"]):
        assert abs(a[0] - b[0]) < 1e-9 and abs(a[1] - b[1]) < 1e-12 and a[2] == b[2]
    assert abs(res.best_reward - ref["best_reward"]) < 1e-9
    assert res.success == ref["success"]
    np.testing.assert_allclose(res.best_states, ref["states"], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(res.best_controls, ref["controls"], rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("case", ["holo2d", "C2", "C3"])
def test_mppi_matches_oracle(gpu, oracle, case):
    p = CASES[case]()
    M, it, seed, sigma = 300, 4, 5, 0.7
    gpu.set_problem(p)
    _host_noise(gpu, oracle, seed)
    res = gpu.mppi_solve(batch=M, sigma=sigma, iterations=it, seed=seed, stop_on_success=False)
    ref = oracle.mppi_solve(p, mppi_config(M, sigma=sigma, iterations=it, seed=seed, stop_on_success=False))
    _compare(res, ref, it)


@pytest.mark.parametrize("case", ["holo2d", "C2", "C4"])
def test_cem_matches_oracle(gpu, oracle, case):
    p = CASES[case]()
    M, it, seed = 300, 4, 9
    gpu.set_problem(p)
    _host_noise(gpu, oracle, seed)
    res = gpu.cem_solve(batch=M, elite_fraction=0.1, initial_std=0.8, min_std=0.05, iterations=it, seed=seed,
                        stop_on_success=False)
    ref = oracle.cem_solve(p, cem_config(M, elite_fraction=0.1, initial_std=0.8, min_std=0.05, iterations=it,
                                         seed=seed, stop_on_success=False))
    _compare(res, ref, it)


def test_baseline_argument_errors(gpu):
    gpu.set_problem(CASES["holo2d"]())
    gpu.set_options(d4.PREC_F32, d4.NOISE_PHILOX)
    with pytest.raises(ValueError, match="mppi_solve: sigma must be positive"):
        gpu.mppi_solve(batch=8, sigma=0.0, iterations=1)
    with pytest.raises(ValueError, match="mppi_solve: batch must be >= 2"):
        gpu.mppi_solve(batch=1, iterations=1)
    with pytest.raises(ValueError, match="cem_solve: elite_fraction must lie in"):
        gpu.cem_solve(batch=8, elite_fraction=1.0, iterations=1)
    with pytest.raises(ValueError, match="cem_solve: elite_fraction \\* batch must be >= 1"):
        gpu.cem_solve(batch=8, elite_fraction=0.05, iterations=1)
    with pytest.raises(ValueError, match="cem_solve: stds must be positive"):
        gpu.cem_solve(batch=20, min_std=0.0, iterations=1)


@pytest.mark.parametrize("method", ["mppi", "cem"])
def test_baselines_philox_throughput_mode(gpu, method):
    """fp32 + Philox, one graph per iteration: deterministic, best = max, and
    the device outcome equals the host restatement on the returned trajectory."""
    from outcome_model import check_success, objective
    p = CASES["C2"]()
    gpu.set_problem(p)
    gpu.set_options(d4.PREC_F32, d4.NOISE_PHILOX)
    run = (lambda: gpu.mppi_solve(batch=2048, sigma=0.5, iterations=6, seed=1, stop_on_success=False)) \
        if method == "mppi" else \
        (lambda: gpu.cem_solve(batch=2048, elite_fraction=0.05, iterations=6, seed=1, stop_on_success=False))
    a, b = run(), run()
    assert a.iterations_used == 6 and a.best_reward == b.best_reward
    np.testing.assert_array_equal(a.best_states, b.best_states)
    rewards = [r[0] for r in a.per_iteration]
    assert a.best_reward == max(rewards)
    assert check_success(p, a.best_states)[0] == a.success
    assert objective(p, a.best_states) == a.per_iteration[rewards.index(a.best_reward)][1]
    assert rewards[-1] > rewards[0]  # the mean improves over the iterations
