"""Small workloads that reach every kernel family of the library, for
compute-sanitizer (memcheck / racecheck / synccheck; one tool per run):

  python tools/sanitize.py            # all cases
  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize.py

Cases: the fused K2+K3 with the pair list (C5 shape: R = 64, O = 16), the tile
path with x-strip culling (R = 40) and small tiles (C2/C4 shapes), the
time-segmented K2+K3 (C1), the fp64 parity instantiation with K1, K4 as one CTA
and as the cooperative grid (shared-memory histogram of the adaptive floor),
K5a stored and regenerating, K5b, K6/K7 (solve), MPPI and CEM (CUB sort),
d4orm_cuda_weighted_mean, and the host-exchange multi-rank path is exercised
by tests/test_gpu_multirank.py.  Shapes are kept tiny (racecheck is slow).
"""
import sys
import os
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2503_12204_b200 as d4  # noqa: E402
from paper_2503_12204_b200 import scenarios as S  # noqa: E402


def run(name, fn):
    t = time.time()
    fn()
    print(f"{name}: ok ({time.time() - t:.1f}s)", flush=True)


def main():
    g = d4.GpuDenoiser()

    def denoise(p, M, steps=2, prec=d4.PREC_F32, noise=d4.NOISE_PHILOX, graphs=False):
        g.set_options(prec, noise, graphs)
        g.set_problem(p)
        if noise == d4.NOISE_HOST:
            rng = np.random.default_rng(1)
            g.set_noise_provider(lambda step, m0, count, elems: rng.normal(size=(count, elems)))
        v, tr = g.run_denoising(np.zeros((p.horizon, p.robots, p.du)), d4.DenoiserConfig(steps=steps, batch=M, seed=3))
        assert np.isfinite(v).all()

    c5 = S.baseline_config(5).problem.with_horizon(64)
    run("C5 pair list, 32-step windows (k_pl32) + K5a regen + adaptive floor (fp32, Philox)", lambda: denoise(c5, 512))
    run("C5 pair list, ragged horizon / odd batch (k_pl32)", lambda: denoise(c5.with_horizon(41), 511))
    os.environ["D4ORM_PL32"] = "0"
    run("C5 pair list, 64-step kernel (D4ORM_PL32=0)", lambda: denoise(c5, 512))
    os.environ.pop("D4ORM_PL32")
    run("C5 stored z (host noise)", lambda: denoise(c5, 512, noise=d4.NOISE_HOST))
    r40 = S.random_square(40, 8.0, 3, S.HOLO2D_VEL, robot_radius=0.15, horizon=32, lower=[-1, -1], upper=[1, 1])
    run("R40 pair list with padding lanes (k_pl32, runtime row stride)", lambda: denoise(r40, 512))
    run("C2 small tiles + obstacles", lambda: denoise(S.baseline_config(2).problem.with_horizon(32), 1024))
    run("C3 unicycle", lambda: denoise(S.baseline_config(3).problem.with_horizon(32), 1024))
    run("C4 3-D (du = 3, K5a regen)", lambda: denoise(S.baseline_config(4).problem.with_horizon(32), 1024))
    run("C1 time-segmented K2+K3", lambda: denoise(S.baseline_config(1).problem, 1024))
    run("fp64 parity path + K1", lambda: denoise(S.baseline_config(2).problem.with_horizon(16), 512, prec=d4.PREC_F64))
    run("CUDA graphs", lambda: denoise(S.baseline_config(2).problem.with_horizon(16), 512, graphs=True))
    # K4 as one CTA and as the cooperative grid
    g.set_options(d4.PREC_F32, d4.NOISE_PHILOX, False)
    for m in (1000, 8192, 20000, 300000):
        run(f"K4 score_weights M={m}", lambda m=m: g.score_weights(np.random.default_rng(m).normal(size=m) * 0.01, 0.1))
    run("K4 grid inside a step (M = 16384)", lambda: denoise(S.baseline_config(4).problem.with_horizon(8), 16384))
    # K5 as an operator
    for prec in (d4.PREC_F64, d4.PREC_F32):
        g.set_options(prec, d4.NOISE_HOST, False)
        run(f"weighted_mean prec={prec}", lambda: g.weighted_mean(np.ones((300, 16390)), np.full(300, 1 / 300)))
    # the anytime loop and the baselines
    p = S.baseline_config(2).problem.with_horizon(24)
    g.set_options(d4.PREC_F32, d4.NOISE_PHILOX, False)
    g.set_problem(p)
    run("solve (K7 + steps + K6)", lambda: g.solve(d4.DenoiserConfig(steps=3, batch=512, seed=1), max_iterations=2,
                                                   stop_on_success=False))
    run("MPPI", lambda: g.mppi_solve(batch=512, iterations=2, seed=1, stop_on_success=False))
    run("CEM (CUB radix sort)", lambda: g.cem_solve(batch=512, iterations=2, seed=1, stop_on_success=False))
    g.close()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
