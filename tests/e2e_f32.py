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


def gpu_chain(g, p, base, cfg, noise_of, run_steps=None):
    """The GPU's free run as a chain of denoise_step calls (returns every
    step's input variable, output, rewards, weights, record) over the first
    run_steps steps i = N, N-1, ... of the schedule.  noise_of(i) is the host
    noise or None for the in-kernel Philox draw."""
    v = np.zeros((p.horizon, p.robots, p.du))
    out = []
    last = cfg.steps - (run_steps or cfg.steps)
    for i in range(cfg.steps, last, -1):
        z = noise_of(i)
        v2, r, w, rec = g.denoise_step(base, v, i, cfg, z)
        out.append((i, v, v2, r, w, rec))
        v = v2
    return out


def outcome_of(oracle, p, base, v):
    """fp64 rollout of base + Δ and the reference's outcome (optimizer.cpp:26-28,
    81-83): total_reward, objective, check_success, and its two parts —
    collision-free (no pair conflict at t = 0..T, no obstacle overlap) and
    goal-reached (every robot inside the goal ball at T), reward.cpp:162-200."""
    st, _ = oracle.rollout(p, base + v)
    pos = st[:, :, : p.pdim]
    d2 = ((pos[:, :, None, :] - pos[:, None, :, :]) ** 2).sum(-1)
    R = p.robots
    d2[:, np.arange(R), np.arange(R)] = np.inf
    free = bool((d2 > 4 * p.robot_radius ** 2).all())
    if len(p.obs_radii):
        od2 = ((pos[:, :, None, :] - p.obs_centers[None, None]) ** 2).sum(-1)
        free = free and bool((od2 > (p.obs_radii + p.robot_radius)[None, None] ** 2).all())
    goal = bool((np.sqrt(((pos[-1] - p.goals) ** 2).sum(-1)) <= p.goal_tolerance).all())
    ok = oracle.check_success(p, st)[0]
    return dict(reward=oracle.total_reward(p, st)[0], objective=oracle.objective(p, st), success=ok,
                collision_free=free, goal_reached=goal)


# the fp32 step tolerances (tests/test_gpu_e2e_f32.py documents how they were measured)
REW_CONT = 1e-6        # |Δreward| after removing whole decision flips
FLIP_RATE = 0.02       # decision flips per step, fraction of the samples
W_STAGE = 1e-11        # K4 vs the oracle's score_weights on the GPU's rewards (relative)
V_STAGE = 5e-6         # K5 vs the oracle's weighted mean + update on the GPU's rewards (of max|v|)
V_STEP_NOFLIP = 1e-4   # whole step vs the oracle, steps without a flip (of max|v|)


def check_step_f32(oracle, p, var, i, ab, lam, noise, v_g, r_g, w_g, v_o, r_o, tag=""):
    """One fp32 denoising step i (from `var`, with `noise`) against the
    oracle's step from the same inputs: rewards (continuous part + flip
    count), K4 and K5 in isolation on the GPU's own rewards, and the whole step
    — within V_STEP_NOFLIP when no decision flipped, else within what the flips
    themselves move the reference's own update (+ V_STAGE).  Returns the
    measured numbers."""
    unit = unit_of(p)
    M = len(r_g)
    dr = r_g - r_o
    k = np.rint(dr / unit)
    cont = float(np.abs(dr - k * unit).max())
    flips = int((k != 0).sum())
    assert cont <= REW_CONT, (tag, "reward", cont)
    assert flips <= FLIP_RATE * M, (tag, "flips", flips)
    w_st = oracle.score_weights(r_g, lam)
    wrel = float(np.max(np.abs(w_g - w_st) / np.maximum(w_st, 1e-300) * (w_st > 1e-12)))
    assert wrel <= W_STAGE, (tag, "weights", wrel)
    ms, sd = 1.0 / math.sqrt(ab[i]), math.sqrt(1.0 / ab[i] - 1.0)
    v_st = oracle.weighted_update(var, noise, w_st, ms, sd, math.sqrt(ab[i - 1])).reshape(v_g.shape)
    scale = float(np.abs(v_o).max())
    vst = float(np.abs(v_g - v_st).max()) / scale
    assert vst <= V_STAGE, (tag, "K5 stage", vst)
    vstep = float(np.abs(v_g - v_o).max()) / scale
    from_rewards = float(np.abs(v_st - v_o).max()) / scale
    if flips == 0:
        assert vstep <= V_STEP_NOFLIP, (tag, "step", vstep)
    else:
        assert vstep <= from_rewards + V_STAGE, (tag, "step with flips", vstep, from_rewards)
    return dict(rew_cont=cont, flips=flips, w_stage=wrel, v_stage=vst, v_step=vstep, v_from_rewards=from_rewards)


def compare_run(g, oracle, ci: int, source: str, steps: int = 100, seed: int = 0, base=None, explain_max: int = 4,
                run_steps=None, free_steps=None, control=False, check_run=True, log=print):
    """Run denoising steps i = steps .. steps-run_steps+1 of config ci on the
    GPU (fp32) and the oracle (fp64), with noise `source` in {"host",
    "philox"}.  The oracle's free run covers the first free_steps of them
    (default all); control=True adds a second free oracle run on the same noise
    perturbed at the fp32-rounding level (z·(1 + 2^-24·u), u = ±1 per
    element): the reference's own sensitivity, against which the GPU's drift is
    read.  Returns a dict of per-step measurements (see module docstring)."""
    rc, p, M = run_config(ci)
    run_steps = run_steps or steps
    free_steps = run_steps if free_steps is None else free_steps
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
    # the GPU runs the whole schedule in Philox mode (cheap; run == chain is
    # checked on it); the oracle compares the first run_steps steps
    chain = gpu_chain(g, p, base, cfg, (lambda i: None) if philox else noise64, None if philox else run_steps)
    run_equal = None
    if check_run and len(chain) == steps:
        # the production call (graphs in Philox mode) is the chain bitwise
        if not philox:
            g.set_noise_provider(lambda step, m0, count, elems: noise64(step)[m0:m0 + count])
        v_run, tr_run = g.run_denoising(base, cfg)
        run_equal = bool(np.array_equal(v_run, chain[-1][2])) and tr_run == [c[5] for c in chain]
    t_gpu = time.perf_counter() - t0

    unit = unit_of(p)
    log_ = StepLog()
    v_free = np.zeros_like(base)
    v_ctrl = np.zeros_like(base)
    sign = np.where(np.random.default_rng(99).random(M * E) < 0.5, -1.0, 1.0).reshape(M, E) if control else None
    first_flip = None
    t_or = 0.0
    for n, (i, v_in, v_out, r_g, w_g, rec_g) in enumerate(chain[:run_steps]):
        z = noise64(i)
        t1 = time.perf_counter()
        # shadow: the oracle's step i from the GPU's variable
        v_sh, r_o, w_o, rec_o = oracle.denoise_step(p, base, v_in, ab, ocfg, i, z)
        free = n < free_steps
        if free:  # the oracle's own trajectory
            v_free, r_f, _, _ = oracle.denoise_step(p, base, v_free, ab, ocfg, i, z)
            if control:
                v_ctrl, _, _, _ = oracle.denoise_step(p, base, v_ctrl, ab, ocfg, i, z * (1.0 + sign * 2.0 ** -24))
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
        row = dict(i=i, rew_cont=float(cont.max()), rew_flips=int(len(flips)), flips_explained=explained,
                   flips_checked=int(min(len(flips), explain_max)),
                   w_stage=float(np.max(np.abs(w_g - w_st) / np.maximum(w_st, 1e-300) * (w_st > 1e-12))),
                   v_stage=float(np.abs(v_out - v_st).max()) / scale,
                   v_shadow=float(np.abs(v_out - v_sh).max()) / float(np.abs(v_sh).max()),
                   v_shadow_from_rewards=float(np.abs(v_st - v_sh).max()) / float(np.abs(v_sh).max()),
                   best=(rec_g[1], rec_o[1]), ent=(rec_g[3], rec_o[3]))
        if free:
            row["v_free"] = float(np.abs(v_out - v_free).max()) / float(np.abs(v_free).max())
            if control:
                row["v_ctrl"] = float(np.abs(v_ctrl - v_free).max()) / float(np.abs(v_free).max())
        log_.add(**row)
    res = dict(config=ci, source=source, M=M, steps=steps, run_steps=run_steps, free_steps=free_steps,
               run_equal=run_equal, first_flip=first_flip, log=log_, v_gpu=chain[run_steps - 1][2], v_oracle=v_free,
               t_gpu=t_gpu, t_oracle=t_or, p=p, base=base)
    if free_steps == run_steps:
        res["outcome"] = {"gpu": outcome_of(oracle, p, base, chain[run_steps - 1][2]),
                          "oracle": outcome_of(oracle, p, base, v_free)}
        if control:
            res["outcome"]["oracle_perturbed"] = outcome_of(oracle, p, base, v_ctrl)
    fr = [r.get("v_free") for r in log_.rows if "v_free" in r]
    ct = [r.get("v_ctrl") for r in log_.rows if "v_ctrl" in r]
    log(f"C{ci} {source:6s} M={M} steps {run_steps}/{steps} (free {free_steps}): gpu {t_gpu:.1f}s oracle {t_or:.1f}s "
        f"run==chain {run_equal} first flip at step {first_flip} | max rew_cont {log_.col('rew_cont').max():.2e} "
        f"flips/step max {log_.col('rew_flips').max()} | w_stage {log_.col('w_stage').max():.2e} "
        f"v_stage {log_.col('v_stage').max():.2e} | v_shadow {log_.col('v_shadow').max():.2e} "
        f"(from rewards {log_.col('v_shadow_from_rewards').max():.2e}) | v_free last {fr[-1] if fr else None} "
        f"| v_ctrl last {ct[-1] if ct else None} | outcome {res.get('outcome')}")
    return res


def drift_table(res) -> str:
    L = res["log"]
    lines = ["step  rew_cont  flips  v_stage   v_shadow  v_free    v_ctrl"]
    for r in L.rows:
        lines.append(f"{r['i']:4d}  {r['rew_cont']:.2e}  {r['rew_flips']:5d}  {r['v_stage']:.2e}  "
                     f"{r['v_shadow']:.2e}  {r.get('v_free', float('nan')):.2e}  {r.get('v_ctrl', float('nan')):.2e}")
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
    ap.add_argument("--run-steps", type=int, default=None)
    ap.add_argument("--free-steps", type=int, default=None)
    ap.add_argument("--control", action="store_true")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    o = Oracle()
    g = d4.GpuDenoiser()
    allres = []
    for ci in map(int, a.configs.split(",")):
        for src in a.sources.split(","):
            r = compare_run(g, o, ci, src, steps=a.steps, run_steps=a.run_steps, free_steps=a.free_steps,
                            control=a.control)
            print(drift_table(r), flush=True)
            allres.append({"config": ci, "source": src, "M": r["M"], "first_flip": r["first_flip"],
                           "run_equal": r["run_equal"], "outcome": r.get("outcome"), "t_oracle": r["t_oracle"],
                           "rows": r["log"].rows})
    if a.json:
        Path(a.json).write_text(json.dumps(allres, default=float))
