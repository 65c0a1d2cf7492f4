"""fp32 production path end to end against the fp64 oracle — the measurement
helpers behind tests/test_gpu_e2e_f32.py (and its __main__ report).

Reference semantics followed (via the oracle, oracle/d4orm_oracle.c):
run_denoising's loop body (denoiser.cpp:152-180): sample_batch (:34-48),
rollout (dynamics.cpp:122-169), total_reward (reward.cpp:67-130),
score_weights (denoiser.cpp:50-90), mc_average (:92-108), denoise_step
(:110-117); the anytime loop solve (optimizer.cpp:48-102).

Per denoising step three comparisons, all on identical noise (the oracle gets
exactly the fp32 normals the GPU consumed):

  shadow   the oracle runs step i from the GPU's own variable: per-sample
           rewards (continuous part + decision flips at the collision
           boundary, each flip re-counted on the GPU's positions), weights,
           variable;
  stage    the oracle's score_weights + weighted mean + update on the GPU's
           own rewards against the GPU's weights (K4) and variable (K5a/K5b):
           isolates the reduction kernels from the rollout's fp32 rounding;
  free     the GPU's free-running run (production kernels, CUDA graphs) and
           the oracle's free-running run from the same start and noise:
           per-step drift max|Δv| / max|v|.
"""
from __future__ import annotations

import math
import time

import numpy as np

import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
from oracle.oracle import make_config

C5_SAMPLES = 4096   # full C5 R/T/O; E = 32768 keeps the E >= 16384 K5 instantiations


def run_config(ci: int):
    rc = S.baseline_config(ci)
    M = C5_SAMPLES if ci == 5 else rc.samples
    return rc, rc.problem, M


def unit_of(p) -> float:
    """One decision flip changes a reward by w/(R·T) (reward.cpp:104-125,129)."""
    return max(p.w_t, p.obstacle_weight) / (p.robots * p.horizon)


FLIP_BAND = 2e-4   # squared-distance band (m²) an fp32 decision may sit in


def _counts(p, st, delta):
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


def explain_flip(g, oracle, p, u):
    """Re-run one candidate u through the fp32 kernel (states out) and the
    oracle; the GPU's counts must lie between the oracle's counts on the GPU's
    own positions with the squared margin shifted by ∓FLIP_BAND."""
    st_g, _, r_g, cnt = g.rollout_fitness(u[None])
    lo = _counts(p, st_g[0], -FLIP_BAND)
    hi = _counts(p, st_g[0], FLIP_BAND)
    return lo[0] <= cnt[0, 0] <= hi[0] and lo[1] <= cnt[0, 1] <= hi[1]


class StepLog:
    def __init__(self):
        self.rows = []

    def add(self, **kw):
        self.rows.append(kw)

    def col(self, k):
        return np.array([r[k] for r in self.rows])


def f32_noise(noise64):
    return noise64.astype(np.float32).astype(np.float64)


def gpu_chain(g, p, base, cfg, noise_of):
    """The GPU's free run as a chain of denoise_step calls (returns every
    step's input variable, output, rewards, weights, record).  noise_of(i) is
    the host noise or None for the in-kernel Philox draw."""
    v = np.zeros((p.horizon, p.robots, p.du))
    out = []
    for i in range(cfg.steps, 0, -1):
        z = noise_of(i)
        v2, r, w, rec = g.denoise_step(base, v, i, cfg, z)
        out.append((i, v, v2, r, w, rec))
        v = v2
    return out


def compare_run(g, oracle, ci: int, source: str, steps: int = 100, seed: int = 0, base=None, explain_max: int = 4,
                log=print):
    """Run `steps` denoising steps of config ci on the GPU (fp32) and the
    oracle (fp64), with noise `source` in {"host", "philox"}.  Returns a dict of
    per-step measurements (see module docstring)."""
    rc, p, M = run_config(ci)
    cfg = d4.DenoiserConfig(steps=steps, batch=M, lam=rc.lam, alpha_bar_final=rc.alpha_bar_final, seed=seed)
    ocfg = make_config(steps, M, lam=rc.lam, abf=rc.alpha_bar_final, seed=seed)
    ab, _ = oracle.make_schedule(steps, rc.alpha_bar_final)
    if base is None:
        base = np.zeros((p.horizon, p.robots, p.du))
    E = p.elems
    philox = source == "philox"
    g.set_options(d4.PREC_F32, d4.NOISE_PHILOX if philox else d4.NOISE_HOST, True)
    g.set_problem(p)
    cache = {}

    def noise64(i):          # exactly the fp32 normals the GPU consumes, as fp64
        if i not in cache:
            cache.clear()
            if philox:
                cache[i] = g.philox_noise(seed, i, 0, M).astype(np.float64)
            else:
                cache[i] = f32_noise(oracle.step_noise(seed, i, 0, M, E))
        return cache[i]

    t0 = time.perf_counter()
    chain = gpu_chain(g, p, base, cfg, (lambda i: None) if philox else noise64)
    # the production call (graphs in Philox mode) is the chain bitwise
    if not philox:
        g.set_noise_provider(lambda step, m0, count, elems: noise64(step)[m0:m0 + count])
    v_run, tr_run = g.run_denoising(base, cfg)
    run_equal = bool(np.array_equal(v_run, chain[-1][2])) and tr_run == [c[5] for c in chain]
    t_gpu = time.perf_counter() - t0

    unit = unit_of(p)
    log_ = StepLog()
    v_free = np.zeros_like(base)
    first_flip = None
    t_or = 0.0
    for (i, v_in, v_out, r_g, w_g, rec_g) in chain:
        z = noise64(i)
        t1 = time.perf_counter()
        # shadow: the oracle's step i from the GPU's variable
        v_sh, r_o, w_o, rec_o = oracle.denoise_step(p, base, v_in, ab, ocfg, i, z)
        # free: the oracle's own trajectory
        v_free, r_f, _, _ = oracle.denoise_step(p, base, v_free, ab, ocfg, i, z)
        # stage: the oracle's weights + mean + update on the GPU's rewards
        w_st = oracle.score_weights(r_g, rc.lam)
        ms, sd = 1.0 / math.sqrt(ab[i]), math.sqrt(1.0 / ab[i] - 1.0)
        v_st = oracle.weighted_update(v_in, z, w_st, ms, sd, math.sqrt(ab[i - 1]))
        t_or += time.perf_counter() - t1
        dr = r_g - r_o
        k = np.rint(dr / unit)
        cont = np.abs(dr - k * unit)
        flips = np.flatnonzero(k != 0)
        explained = 0
        if len(flips):
            g.set_options(d4.PREC_F32, d4.NOISE_HOST, True)
        for m in flips[:explain_max]:
            u = base + ms * v_in + sd * z[m].reshape(base.shape)
            explained += bool(explain_flip(g, oracle, p, u))
        g.set_options(d4.PREC_F32, d4.NOISE_PHILOX if philox else d4.NOISE_HOST, True)
        if len(flips) and first_flip is None:
            first_flip = i
        scale = float(np.abs(v_st).max())
        log_.add(i=i, rew_cont=float(cont.max()), rew_flips=int(len(flips)), flips_explained=explained,
                 flips_checked=int(min(len(flips), explain_max)),
                 w_stage=float(np.max(np.abs(w_g - w_st) / np.maximum(w_st, 1e-300) * (w_st > 1e-12))),
                 v_stage=float(np.abs(v_out - v_st).max()) / scale,
                 v_shadow=float(np.abs(v_out - v_sh).max()) / float(np.abs(v_sh).max()),
                 v_shadow_from_rewards=float(np.abs(v_st - v_sh).max()) / float(np.abs(v_sh).max()),
                 v_free=float(np.abs(v_out - v_free).max()) / float(np.abs(v_free).max()),
                 best=(rec_g[1], rec_o[1]), ent=(rec_g[3], rec_o[3]))
    res = dict(config=ci, source=source, M=M, steps=steps, run_equal=run_equal, first_flip=first_flip, log=log_,
               v_gpu=chain[-1][2], v_oracle=v_free, t_gpu=t_gpu, t_oracle=t_or, p=p, base=base)
    # outcome of the final variable: fp64 rollout of base + Δ, total_reward /
    # objective / check_success (optimizer.cpp:26-28,81-83) on both
    out = {}
    for name, v in (("gpu", chain[-1][2]), ("oracle", v_free)):
        st, _ = oracle.rollout(p, base + v)
        out[name] = (oracle.total_reward(p, st)[0], oracle.objective(p, st), oracle.check_success(p, st)[0])
    res["outcome"] = out
    log(f"C{ci} {source:6s} M={M} steps={steps}: gpu {t_gpu:.1f}s oracle {t_or:.1f}s run==chain {run_equal} "
        f"first flip at step {first_flip} | max rew_cont {log_.col('rew_cont').max():.2e} "
        f"flips/step max {log_.col('rew_flips').max()} | w_stage {log_.col('w_stage').max():.2e} "
        f"v_stage {log_.col('v_stage').max():.2e} | v_shadow {log_.col('v_shadow').max():.2e} "
        f"(from rewards {log_.col('v_shadow_from_rewards').max():.2e}) | v_free final "
        f"{log_.rows[-1]['v_free']:.2e} max {log_.col('v_free').max():.2e} | outcome {out}")
    return res


def drift_table(res) -> str:
    L = res["log"]
    lines = ["step  rew_cont  flips  v_stage   v_shadow  v_free"]
    for r in L.rows:
        lines.append(f"{r['i']:4d}  {r['rew_cont']:.2e}  {r['rew_flips']:5d}  {r['v_stage']:.2e}  "
                     f"{r['v_shadow']:.2e}  {r['v_free']:.2e}")
    return "\n".join(lines)


if __name__ == "__main__":
    import argparse
    import json
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle.oracle import Oracle
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--sources", default="philox,host")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    o = Oracle()
    g = d4.GpuDenoiser()
    allres = []
    for ci in map(int, a.configs.split(",")):
        for src in a.sources.split(","):
            r = compare_run(g, o, ci, src, steps=a.steps)
            print(drift_table(r), flush=True)
            allres.append({"config": ci, "source": src, "M": r["M"], "first_flip": r["first_flip"],
                           "run_equal": r["run_equal"], "outcome": r["outcome"], "t_oracle": r["t_oracle"],
                           "rows": r["log"].rows})
    if a.json:
        Path(a.json).write_text(json.dumps(allres, default=float))
