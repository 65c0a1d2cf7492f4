"""K5a with regenerated noise (k_wmean_regen, csrc/d4orm_kernels.cuh) against
K5a reading the z rows K2+K3 stored (k_wmean_partial).

The normals are a pure function of (seed, step, m, k, n), the per-element sums
run in the same ascending-m fmaf order and the sub-range tree is the same, so
the two must agree BIT FOR BIT: denoised variable, trace, and (through `solve`
and MPPI) the whole anytime loop.  Knob: D4ORM_K5REGEN=0/1 (read per step; a
fresh context per setting so no captured graph carries the other choice)."""
import os

import numpy as np
import pytest

import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S

pytestmark = pytest.mark.gpu


def _with_regen(flag, fn):
    os.environ["D4ORM_K5REGEN"] = "1" if flag else "0"
    g = None
    try:
        g = d4.GpuDenoiser()
        return fn(g)
    finally:
        if g is not None:
            g.close()
        os.environ.pop("D4ORM_K5REGEN", None)


def _denoise(p, batch, steps, seed):
    def run(g):
        g.set_problem(p)
        cfg = d4.DenoiserConfig(steps=steps, batch=batch, seed=seed)
        return g.run_denoising(np.zeros((p.horizon, p.robots, p.du)), cfg)
    return run


# (config, batch, steps): every BASELINE shape (C5 at its full batch, both K5a
# shapes: E >= 16384 one walk per thread, smaller E 16 sub-ranges), plus
# ragged cases (batch not a multiple of the 256-sample chunk, T·du % 4 != 0)
CASES = [(1, 1024, 20), (2, 8192, 6), (3, 16384, 4), (4, 16384, 4), (5, 262144, 2), (5, 4096, 5)]


@pytest.mark.parametrize("cfg,batch,steps", CASES, ids=[f"C{c}-N{b}" for c, b, _ in CASES])
def test_regen_equals_stored(cfg, batch, steps):
    p = S.baseline_config(cfg).problem
    v0, tr0 = _with_regen(False, _denoise(p, batch, steps, 3))
    v1, tr1 = _with_regen(True, _denoise(p, batch, steps, 3))
    np.testing.assert_array_equal(v1, v0)
    assert tr1 == tr0
    assert np.abs(v0).max() > 0


@pytest.mark.parametrize("kind,T,batch", [(S.HOLO2D_VEL, 33, 1000), (S.HOLO3D_VEL, 17, 777), (S.UNICYCLE, 9, 300)])
def test_regen_ragged(kind, T, batch):
    """Ragged shapes: T·du not a multiple of 4 (a robot's last Philox group is
    partial), a batch that leaves the last chunk part-filled.  (R = 4 keeps E
    a multiple of 4: the stored path's fused float4 walk, which regen is
    enabled for.)"""
    du = S.DIMS[kind][1]
    if S.DIMS[kind][2] == 3:
        p = S.cube_corners(6.0, kind, robot_radius=0.2, horizon=T, lower=[-1] * du, upper=[1] * du)
    else:
        p = S.antipodal_circle(4, 6.0, kind, robot_radius=0.2, horizon=T, lower=[-1] * du, upper=[1] * du)
    assert (T * du) % 4 != 0 and (p.robots * T * du) % 4 == 0
    v0, tr0 = _with_regen(False, _denoise(p, batch, 5, 7))
    v1, tr1 = _with_regen(True, _denoise(p, batch, 5, 7))
    np.testing.assert_array_equal(v1, v0)
    assert tr1 == tr0


def test_regen_solve_and_mppi():
    """The anytime loop (one graph per iteration) and MPPI on the same
    kernels: regenerated noise changes nothing."""
    p = S.baseline_config(2).problem

    def solve(g):
        g.set_problem(p)
        r = g.solve(d4.DenoiserConfig(steps=8, batch=2048, seed=1), max_iterations=2, stop_on_success=False)
        return r

    def mppi(g):
        g.set_problem(p)
        return g.mppi_solve(batch=2048, iterations=6, stop_on_success=False)

    a, b = _with_regen(False, solve), _with_regen(True, solve)
    np.testing.assert_array_equal(a.best_controls, b.best_controls)
    assert a.best_reward == b.best_reward and a.traces == b.traces
    assert [r[:3] for r in a.per_iteration] == [r[:3] for r in b.per_iteration]
    a, b = _with_regen(False, mppi), _with_regen(True, mppi)
    np.testing.assert_array_equal(a.best_controls, b.best_controls)
    assert a.best_reward == b.best_reward
    assert [r[:3] for r in a.per_iteration] == [r[:3] for r in b.per_iteration]


def test_regen_switch_in_one_context():
    """One context, the K5a mode switched between runs: the captured graphs are
    keyed on the mode (and the z buffer grows when the stored path needs rows),
    so every run gives the same bits."""
    p = S.baseline_config(4).problem
    g = d4.GpuDenoiser()
    try:
        g.set_problem(p)
        cfg = d4.DenoiserConfig(steps=4, batch=4096, seed=5)
        base = np.zeros((p.horizon, p.robots, p.du))
        outs, modes = [], []
        for flag in ("1", "0", "1", "0"):
            os.environ["D4ORM_K5REGEN"] = flag
            outs.append(g.run_denoising(base, cfg))
            modes.append(g.k5_regen())
        assert modes == [1, 0, 1, 0]
        for v, tr in outs[1:]:
            np.testing.assert_array_equal(v, outs[0][0])
            assert tr == outs[0][1]
    finally:
        os.environ.pop("D4ORM_K5REGEN", None)
        g.close()
