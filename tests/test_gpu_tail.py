"""The fused small-batch step tail (d4k::k_small_step_tail: K4 + K5a + K5b in
one launch for M ≤ 2048, fp32, stored noise, one rank — C1) against the
three-kernel path (D4ORM_FUSE_TAIL=0): bitwise the same variable, rewards,
weights and trace, over batch sizes below / at / across the 256-sample chunk
and up to the 2048 limit, both noise sources."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu

CHILD = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
out = {}
for name, p in (("C1", S.baseline_config(1).problem),
                ("C2s", S.baseline_config(2).problem.with_horizon(24)),
                ("C3s", S.baseline_config(3).problem.with_horizon(20))):
    for M in (2, 255, 300, 1024, 2048):
        g = d4.GpuDenoiser(p)
        base = 0.1 * np.cos(np.arange(p.elems)).reshape(p.horizon, p.robots, p.du)
        v, tr = g.run_denoising(base, d4.DenoiserConfig(steps=5, batch=M, seed=M))
        out[f"{name}_{M}_run"] = v
        out[f"{name}_{M}_trace"] = np.array(tr, dtype=float)
        g.set_options(d4.PREC_F32, d4.NOISE_HOST, False)
        z = np.random.default_rng(M).normal(size=(M, p.elems))
        v2, r2, w2, rec = g.denoise_step(base, 0.2 * base, 3, d4.DenoiserConfig(steps=5, batch=M, seed=1), z)
        out[f"{name}_{M}_step"] = v2
        out[f"{name}_{M}_r"] = r2
        out[f"{name}_{M}_w"] = w2
        out[f"{name}_{M}_rec"] = np.array(rec, dtype=float)
        out[f"{name}_{M}_launches"] = np.array(g.launches_per_step())
        g.close()
np.savez(sys.argv[2], **out)
'''


def _run(fuse, path):
    env = dict(os.environ, D4ORM_FUSE_TAIL=str(fuse))
    r = subprocess.run([sys.executable, "-c", CHILD, str(ROOT), str(path)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(path)


def test_fused_tail_is_bitwise_the_three_kernel_path(tmp_path):
    fused = _run(1, tmp_path / "fused.npz")
    plain = _run(0, tmp_path / "plain.npz")
    assert set(fused.files) == set(plain.files)
    n_fused = 0
    for k in fused.files:
        if k.endswith("_launches"):
            assert int(plain[k]) == 4
            n_fused += int(fused[k]) == 2
            continue
        np.testing.assert_array_equal(fused[k], plain[k], err_msg=k)
    assert n_fused >= 10  # the fused tail actually ran


CHILD_K4 = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
out = {}
g = d4.GpuDenoiser()
for M in (2049, 5000, 12000, 16384):
    for kind, r in (("normal", np.random.default_rng(M).normal(size=M) * 0.01 + 0.3),
                    ("skewed", np.random.default_rng(M + 1).exponential(size=M) * 0.05),
                    ("flat", np.full(M, 0.25))):
        w, t3 = g.score_weights(r, 0.1)
        out[f"{M}_{kind}_w"] = w
        out[f"{M}_{kind}_w32"] = g.last_w32(M)
        out[f"{M}_{kind}_t"] = t3
p = S.baseline_config(4).problem.with_horizon(32)   # du = 3: the adaptive floor
g.set_problem(p)
v, r, w, rec = g.denoise_step(np.zeros((32, 8, 3)), np.full((32, 8, 3), 0.1), 4, d4.DenoiserConfig(steps=6, batch=16384, seed=3))
out["step_v"], out["step_w"], out["step_rec"] = v, w, np.array(rec, dtype=float)
np.savez(sys.argv[2], **out)
'''


def test_cluster_k4_is_bitwise_the_grid_k4(tmp_path):
    """K4 for 2048 < M ≤ 16384 as one thread-block cluster (DSMEM folds) vs the
    cooperative grid (global scratch + grid barriers): the same fold order, so
    bitwise the same weights, fp32 weights (incl. the adaptive floor), trace."""
    res = []
    for on in (1, 0):
        env = dict(os.environ, D4ORM_K4CLUSTER=str(on))
        f = tmp_path / f"k4_{on}.npz"
        r = subprocess.run([sys.executable, "-c", CHILD_K4, str(ROOT), str(f)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        res.append(np.load(f))
    for k in res[0].files:
        np.testing.assert_array_equal(res[0][k], res[1][k], err_msg=k)


CHILD_TREE = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
out = {}
for name, p, M in (("C2", S.baseline_config(2).problem.with_horizon(32), 8192),
                   ("C4", S.baseline_config(4).problem.with_horizon(32), 16384),
                   ("C5", S.baseline_config(5).problem.with_horizon(32), 262144),
                   ("odd", S.baseline_config(2).problem.with_horizon(20), 256 * 37)):
    g = d4.GpuDenoiser(p)
    v, tr = g.run_denoising(np.zeros((p.horizon, p.robots, p.du)), d4.DenoiserConfig(steps=3, batch=M, seed=5))
    out[name] = v
    for prec in (d4.PREC_F64,):
        g.set_options(prec, d4.NOISE_HOST, False)
        z = np.random.default_rng(1).normal(size=(min(M, 8192), p.elems))
        v2, _, _, _ = g.denoise_step(np.zeros_like(v), 0.1 + 0 * v, 2, d4.DenoiserConfig(steps=3, batch=len(z), seed=1), z)
        out[name + "_f64"] = v2
    g.set_options(d4.PREC_F32, d4.NOISE_PHILOX, True)
    mr = g.mppi_solve(batch=min(M, 8192), iterations=2, seed=3, stop_on_success=False)
    cr = g.cem_solve(batch=min(M, 8192), iterations=2, seed=3, stop_on_success=False)
    out[name + "_mppi"], out[name + "_cem"] = mr.best_controls, cr.best_controls
    g.close()
np.savez(sys.argv[2], **out)
'''


def test_parallel_tree_is_bitwise_the_serial_tree(tmp_path):
    """K5b with the 8-leaf block roots in parallel vs the serial walk (D4ORM_TREEPAR=0):
    denoising runs (fp32, fp64), MPPI and CEM (the CEM finalisations) at chunk
    counts 32, 64, 1024 and 37 (not a power of two: leftover leaves)."""
    res = []
    for on in (1, 0):
        env = dict(os.environ, D4ORM_TREEPAR=str(on))
        f = tmp_path / f"tree_{on}.npz"
        r = subprocess.run([sys.executable, "-c", CHILD_TREE, str(ROOT), str(f)], env=env, capture_output=True,
                           text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        res.append(np.load(f))
    for k in res[0].files:
        np.testing.assert_array_equal(res[0][k], res[1][k], err_msg=k)
