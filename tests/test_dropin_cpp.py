"""The C++ drop-in (include/d4orm/*.hpp — the reference planner interface) on
the GPU, checked against the CPU oracle.  The C++ program is compiled here with
g++ against the in-tree libd4orm_b200.so."""
import json
import math
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2503_12204_b200 import scenarios as S
from oracle.oracle import cem_config, make_config, mppi_config

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dropin(tmp_path_factory):
    exe = tmp_path_factory.mktemp("cpp") / "test_dropin"
    pkg = ROOT / "paper_2503_12204_b200"
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tests/cpp/test_dropin.cpp"),
                    f"-L{pkg}", "-ld4orm_b200", f"-Wl,-rpath,{pkg}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    return json.loads(out)


def test_generators_match_python_mirror(dropin):
    for c in (2, 5):
        p = S.baseline_config(c).problem
        np.testing.assert_array_equal(np.array(dropin[f"c{c}_starts"]), p.starts.ravel())
        np.testing.assert_array_equal(np.array(dropin[f"c{c}_obs"]), p.obs_centers.ravel())
        np.testing.assert_array_equal(np.array(dropin[f"c{c}_rad"]), p.obs_radii)


def test_rollout_kat(dropin):
    assert abs(dropin["kat_px"] - 0.5) < 1e-9 and abs(dropin["kat_vx"] - 1.0) < 1e-12


def _small():
    p = S.baseline_config(2).problem.with_horizon(16)
    base = 0.3 * np.sin(0.7 * np.arange(p.elems)).reshape(p.horizon, p.robots, p.du)
    return p, base


def test_run_denoising_correctness_mode(dropin, oracle):
    p, base = _small()
    v, tr = oracle.run_denoising(p, base, make_config(6, 256, seed=7))
    np.testing.assert_allclose(np.array(dropin["rd_variable"]), v.ravel(), rtol=1e-9, atol=1e-12)
    for a, b in zip(dropin["rd_trace"], tr):
        assert a[0] == b[0]
        np.testing.assert_allclose(a[1:], b[1:], rtol=1e-9, atol=1e-12)


def test_solve_correctness_mode(dropin, oracle):
    p, _ = _small()
    r = oracle.solve(p, make_config(6, 256, seed=7), max_iterations=2, stop_on_success=False)
    assert dropin["solve_iters"] == r["iterations"]
    assert abs(dropin["solve_best"] - r["best_reward"]) < 1e-9
    assert bool(dropin["solve_success"]) == r["success"]
    np.testing.assert_allclose(np.array(dropin["solve_states"]), r["states"].ravel(), rtol=1e-9, atol=1e-9)


def test_throughput_mode_deterministic_and_errors(dropin):
    assert dropin["f32_repeat_maxdiff"] == 0.0
    assert dropin["err_batch"] == "run_denoising: batch must be >= 2"


def test_baselines_correctness_mode(dropin, oracle):
    """mppi_solve / cem_solve through the C++ drop-in (baselines.hpp) vs the oracle."""
    p = S.baseline_config(2).problem.with_horizon(16)
    r = oracle.mppi_solve(p, mppi_config(200, sigma=0.6, iterations=3, seed=4, stop_on_success=False))
    assert dropin["mppi_iters"] == r["iterations"] == 3
    assert abs(dropin["mppi_best"] - r["best_reward"]) < 1e-9
    np.testing.assert_allclose(np.array(dropin["mppi_states"]), r["states"].ravel(), rtol=1e-9, atol=1e-9)
    r = oracle.cem_solve(p, cem_config(200, elite_fraction=0.1, initial_std=0.7, iterations=3, seed=4,
                                       stop_on_success=False))
    assert dropin["cem_iters"] == r["iterations"] == 3
    assert abs(dropin["cem_best"] - r["best_reward"]) < 1e-9
    np.testing.assert_allclose(np.array(dropin["cem_states"]), r["states"].ravel(), rtol=1e-9, atol=1e-9)
    assert dropin["elites"] == oracle.select_elites(np.array([0.5, 0.9, 0.5, -1.0, 0.9, 0.2, 0.9]), 3) == [1, 4, 6]


def test_mc_average_on_device(dropin, oracle):
    """d4orm::mc_average → d4orm_cuda_weighted_mean (K5a + K5b, fp64) against
    the oracle's mc_average (pinned bitwise to the reference's)."""
    M = 600
    j = np.arange(30)
    smp = np.stack([np.sin(0.37 * m + 1.3 * j) * (1.0 + 0.01 * m) for m in range(M)])
    w = np.exp(-0.01 * np.arange(M))
    w = w / w.sum()
    want = oracle.mc_average(smp, w)
    np.testing.assert_allclose(np.array(dropin["mc_avg"]), want, rtol=1e-12, atol=1e-14)
    assert dropin["mc_err"] == "mc_average: weights must sum to 1"
