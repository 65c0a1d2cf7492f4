"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes access to the CPU checkers:
  * ``Oracle``    — the plain-C fp64 restatement (oracle/d4orm_oracle.c)
  * ``Reference`` — the reference's own proj/src compiled unchanged
                    (oracle/_ref/libd4orm_ref.so, built by oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import
this module.  The product path (paper_2503_12204_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "build" / "libd4orm_oracle.so"
REF_SO = HERE / "_ref" / "libd4orm_ref.so"


class OrProblem(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("dx", C.c_int), ("du", C.c_int), ("pdim", C.c_int),
        ("robots", C.c_int), ("horizon", C.c_int), ("dt", C.c_double),
        ("lower", C.c_double * 3), ("upper", C.c_double * 3),
        ("starts", C.POINTER(C.c_double)), ("goals", C.POINTER(C.c_double)),
        ("n_obstacles", C.c_int), ("obs_centers", C.POINTER(C.c_double)), ("obs_radii", C.POINTER(C.c_double)),
        ("w_t", C.c_double), ("epsilon", C.c_double), ("robot_radius", C.c_double),
        ("goal_tolerance", C.c_double), ("obstacle_weight", C.c_double),
    ]


class OrConfig(C.Structure):
    _fields_ = [("steps", C.c_int), ("batch", C.c_int64), ("lambda_", C.c_double), ("alpha_bar_final", C.c_double),
                ("seed", C.c_uint64), ("mode", C.c_int), ("workers", C.c_int)]


class OrTrace(C.Structure):
    _fields_ = [("step", C.c_int), ("best_reward", C.c_double), ("mean_reward", C.c_double),
                ("weight_entropy", C.c_double)]


class OrOptConfig(C.Structure):
    _fields_ = [("max_iterations", C.c_int), ("stop_on_success", C.c_int), ("deadline_seconds", C.c_double)]


class OrIterStats(C.Structure):
    _fields_ = [("reward", C.c_double), ("objective", C.c_double), ("success", C.c_int),
                ("wall_seconds", C.c_double)]


class OrMppiConfig(C.Structure):
    _fields_ = [("batch", C.c_int64), ("lambda_", C.c_double), ("sigma", C.c_double), ("iterations", C.c_int),
                ("seed", C.c_uint64), ("stop_on_success", C.c_int), ("deadline_seconds", C.c_double),
                ("workers", C.c_int)]


class OrCemConfig(C.Structure):
    _fields_ = [("batch", C.c_int64), ("elite_fraction", C.c_double), ("initial_std", C.c_double),
                ("min_std", C.c_double), ("iterations", C.c_int), ("seed", C.c_uint64), ("stop_on_success", C.c_int),
                ("deadline_seconds", C.c_double), ("workers", C.c_int)]


def mppi_config(batch, lam=0.1, sigma=1.0, iterations=10, seed=0, stop_on_success=True, workers=0):
    return OrMppiConfig(batch, lam, sigma, iterations, seed & ((1 << 64) - 1), int(stop_on_success), 0.0, workers)


def cem_config(batch, elite_fraction=0.1, initial_std=1.0, min_std=0.05, iterations=10, seed=0,
               stop_on_success=True, workers=0):
    return OrCemConfig(batch, elite_fraction, initial_std, min_std, iterations, seed & ((1 << 64) - 1),
                       int(stop_on_success), 0.0, workers)


def _dp(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(C.POINTER(C.c_double))


def make_problem(p) -> tuple[OrProblem, tuple]:
    """Build the C struct from a scenarios.Problem-like object (keep-alive tuple returned)."""
    dx, du, pd = p.dims
    starts = np.ascontiguousarray(p.starts, dtype=np.float64)
    goals = np.ascontiguousarray(p.goals, dtype=np.float64)
    oc = np.ascontiguousarray(p.obs_centers, dtype=np.float64).reshape(-1) if len(p.obs_radii) else np.zeros(3)
    orr = np.ascontiguousarray(p.obs_radii, dtype=np.float64) if len(p.obs_radii) else np.zeros(1)
    s = OrProblem()
    s.kind, s.dx, s.du, s.pdim = p.kind, dx, du, pd
    s.robots, s.horizon, s.dt = p.robots, p.horizon, p.dt
    for d in range(du):
        s.lower[d], s.upper[d] = p.lower[d], p.upper[d]
    s.starts, s.goals = _dp(starts), _dp(goals)
    s.n_obstacles = len(p.obs_radii)
    s.obs_centers, s.obs_radii = _dp(oc), _dp(orr)
    s.w_t, s.epsilon, s.robot_radius = p.w_t, p.epsilon, p.robot_radius
    s.goal_tolerance, s.obstacle_weight = p.goal_tolerance, p.obstacle_weight
    return s, (starts, goals, oc, orr)


def make_config(steps, batch, lam=0.1, abf=0.05, seed=0, mode=1, workers=0) -> OrConfig:
    return OrConfig(steps, batch, lam, abf, seed & ((1 << 64) - 1), mode, workers)


class _Base:
    prefix = ""

    def __init__(self, path: Path):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (python -m paper_2503_12204_b200.build --oracle)")
        self.L = C.CDLL(str(path))
        self._sig()

    def _sig(self):
        pass


class Oracle(_Base):
    """The plain-C fp64 restatement."""

    def __init__(self, path: Path = ORACLE_SO):
        super().__init__(path)

    def _sig(self):
        L, dp, i64, vp = self.L, C.POINTER(C.c_double), C.c_int64, C.c_void_p
        L.or_splitmix64.restype = C.c_uint64
        L.or_splitmix64.argtypes = [C.c_uint64]
        L.or_mix_seed.restype = C.c_uint64
        L.or_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.or_mix_seed3.restype = C.c_uint64
        L.or_mix_seed3.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.or_normal_fill.argtypes = [C.c_uint64, dp, i64]
        L.or_step_noise.argtypes = [C.c_uint64, C.c_int, i64, i64, i64, dp, C.c_int]
        L.or_make_schedule.argtypes = [C.c_int, C.c_double, dp, dp]
        L.or_rk4_step.argtypes = [C.c_int, dp, dp, C.c_double, dp]
        L.or_derivative.argtypes = [C.c_int, dp, dp, dp]
        L.or_rollout.argtypes = [C.POINTER(OrProblem), dp, dp, dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.or_total_reward.argtypes = [C.POINTER(OrProblem), dp, dp, C.POINTER(i64), C.POINTER(i64)]
        L.or_objective.argtypes = [C.POINTER(OrProblem), dp]
        L.or_objective.restype = C.c_double
        L.or_check_success.argtypes = [C.POINTER(OrProblem), dp, C.c_char_p, C.c_int]
        L.or_score_weights.argtypes = [dp, i64, C.c_double, dp]
        L.or_weight_entropy.argtypes = [dp, i64]
        L.or_weight_entropy.restype = C.c_double
        L.or_denoise_step.argtypes = [C.POINTER(OrProblem), dp, dp, C.POINTER(OrConfig), C.c_int, dp, dp, dp, dp,
                                      C.POINTER(OrTrace)]
        L.or_run_denoising.argtypes = [C.POINTER(OrProblem), dp, C.POINTER(OrConfig), dp, C.POINTER(OrTrace)]
        L.or_mc_average.argtypes = [dp, dp, i64, i64, dp]
        L.or_weighted_update.argtypes = [dp, dp, dp, i64, i64, C.c_double, C.c_double, C.c_double, dp]
        L.or_solve.argtypes = [C.POINTER(OrProblem), C.POINTER(OrConfig), C.POINTER(OrOptConfig), dp, dp, dp,
                               C.POINTER(C.c_int), C.POINTER(OrIterStats), C.POINTER(OrTrace)]
        L.or_select_elites.argtypes = [dp, i64, C.c_int, C.POINTER(C.c_int)]
        L.or_mppi_solve.argtypes = [C.POINTER(OrProblem), C.POINTER(OrMppiConfig), dp, dp, dp, C.POINTER(C.c_int),
                                    C.POINTER(OrIterStats)]
        L.or_cem_solve.argtypes = [C.POINTER(OrProblem), C.POINTER(OrCemConfig), dp, dp, dp, C.POINTER(C.c_int),
                                   C.POINTER(OrIterStats)]
        L.or_last_error.restype = C.c_char_p

    def err(self):
        return self.L.or_last_error().decode()

    # --- rng
    def mix_seed(self, a, b, c=None):
        return self.L.or_mix_seed(a, b) if c is None else self.L.or_mix_seed3(a, b, c)

    def normal_fill(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n)
        self.L.or_normal_fill(seed, _dp(out), n)
        return out

    def step_noise(self, seed: int, i: int, m0: int, count: int, elems: int, workers: int = 0) -> np.ndarray:
        out = np.empty((count, elems))
        self.L.or_step_noise(seed, i, m0, count, elems, _dp(out), workers)
        return out

    def make_schedule(self, steps, abf):
        ab = np.empty(steps + 1)
        a = np.empty(steps)
        if self.L.or_make_schedule(steps, abf, _dp(ab), _dp(a)):
            raise ValueError(self.err())
        return ab, a

    def rk4_step(self, kind, x, u, dt):
        x = np.ascontiguousarray(x, dtype=np.float64)
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty_like(x)
        self.L.or_rk4_step(kind, _dp(x), _dp(u), dt, _dp(out))
        return out

    def derivative(self, kind, x, u):
        x = np.ascontiguousarray(x, dtype=np.float64)
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty_like(x)
        self.L.or_derivative(kind, _dp(x), _dp(u), _dp(out))
        return out

    def rollout(self, p, u):
        s, keep = make_problem(p)
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(p.horizon, p.robots, p.du)
        states = np.empty((p.horizon + 1, p.robots, p.dx))
        controls = np.empty((p.horizon + 1, p.robots, p.du))
        br, bs = C.c_int(-1), C.c_int(-1)
        rc = self.L.or_rollout(C.byref(s), _dp(u), _dp(states), _dp(controls), C.byref(br), C.byref(bs))
        if rc:
            raise RuntimeError(self.err())
        return states, controls

    def total_reward(self, p, states):
        s, keep = make_problem(p)
        states = np.ascontiguousarray(states, dtype=np.float64)
        r = C.c_double()
        nc, no = C.c_int64(), C.c_int64()
        rc = self.L.or_total_reward(C.byref(s), _dp(states), C.byref(r), C.byref(nc), C.byref(no))
        if rc:
            raise ValueError(self.err())
        return r.value, nc.value, no.value

    def objective(self, p, states):
        s, keep = make_problem(p)
        return self.L.or_objective(C.byref(s), _dp(np.ascontiguousarray(states, dtype=np.float64)))

    def check_success(self, p, states):
        s, keep = make_problem(p)
        buf = C.create_string_buffer(256)
        ok = self.L.or_check_success(C.byref(s), _dp(np.ascontiguousarray(states, dtype=np.float64)), buf, 256)
        return bool(ok), buf.value.decode()

    def score_weights(self, rewards, lam):
        r = np.ascontiguousarray(rewards, dtype=np.float64)
        w = np.empty_like(r)
        rc = self.L.or_score_weights(_dp(r), len(r), lam, _dp(w))
        if rc == 1:
            raise ValueError(self.err())
        if rc:
            raise RuntimeError(self.err())
        return w

    def weight_entropy(self, w):
        return self.L.or_weight_entropy(_dp(np.ascontiguousarray(w, dtype=np.float64)), len(w))

    def denoise_step(self, p, base, variable, ab, cfg: OrConfig, i, noise=None):
        s, keep = make_problem(p)
        base = np.ascontiguousarray(base, dtype=np.float64)
        var = np.array(variable, dtype=np.float64, copy=True, order="C")
        nz = None if noise is None else np.ascontiguousarray(noise, dtype=np.float64)
        rw = np.empty(cfg.batch)
        w = np.empty(cfg.batch)
        rec = OrTrace()
        ab = np.ascontiguousarray(ab, dtype=np.float64)
        rc = self.L.or_denoise_step(C.byref(s), _dp(base), _dp(ab), C.byref(cfg), i, _dp(var), _dp(nz), _dp(rw),
                                    _dp(w), C.byref(rec))
        if rc:
            raise RuntimeError(self.err())
        return var, rw, w, (rec.step, rec.best_reward, rec.mean_reward, rec.weight_entropy)

    def mc_average(self, samples, weights):
        """mc_average (denoiser.cpp:92-108) of M sample rows."""
        smp = np.ascontiguousarray(samples, dtype=np.float64)
        M = smp.shape[0]
        w = np.ascontiguousarray(weights, dtype=np.float64)
        out = np.empty(smp.shape[1:])
        if self.L.or_mc_average(_dp(smp), _dp(w), M, smp[0].size, _dp(out)):
            raise ValueError(self.err())
        return out

    def weighted_update(self, variable, noise, weights, mean_scale, std_dev, update_scale):
        """sample_batch + mc_average + denoise_step for given weights:
        update_scale · Σ_m w_m (mean_scale·variable + std_dev·z_m)."""
        var = np.ascontiguousarray(variable, dtype=np.float64)
        nz = np.ascontiguousarray(noise, dtype=np.float64).reshape(len(weights), var.size)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        out = np.empty_like(var)
        if self.L.or_weighted_update(_dp(var), _dp(nz), _dp(w), len(w), var.size, mean_scale, std_dev,
                                     update_scale, _dp(out)):
            raise ValueError(self.err())
        return out

    def run_denoising(self, p, base, cfg: OrConfig):
        s, keep = make_problem(p)
        base = np.ascontiguousarray(base, dtype=np.float64)
        out = np.empty((p.horizon, p.robots, p.du))
        tr = (OrTrace * cfg.steps)()
        rc = self.L.or_run_denoising(C.byref(s), _dp(base), C.byref(cfg), _dp(out), tr)
        if rc:
            raise RuntimeError(self.err())
        return out, [(t.step, t.best_reward, t.mean_reward, t.weight_entropy) for t in tr]

    def solve(self, p, cfg: OrConfig, max_iterations=10, stop_on_success=True):
        s, keep = make_problem(p)
        oc = OrOptConfig(max_iterations, int(stop_on_success), 0.0)
        states = np.empty((p.horizon + 1, p.robots, p.dx))
        controls = np.empty((p.horizon + 1, p.robots, p.du))
        best = C.c_double()
        ok = C.c_int()
        its = (OrIterStats * max_iterations)()
        used = self.L.or_solve(C.byref(s), C.byref(cfg), C.byref(oc), _dp(states), _dp(controls), C.byref(best),
                               C.byref(ok), its, None)
        if used < 0:
            raise RuntimeError(self.err())
        return dict(states=states, controls=controls, best_reward=best.value, success=bool(ok.value),
                    iterations=used, per_iteration=[(its[j].reward, its[j].objective, bool(its[j].success))
                                                    for j in range(used)])


    def select_elites(self, rewards, count):
        r = np.ascontiguousarray(rewards, dtype=np.float64)
        out = (C.c_int * count)()
        if self.L.or_select_elites(_dp(r), len(r), count, out):
            raise ValueError(self.err())
        return list(out)

    def _baseline(self, fn, p, cfg, iterations):
        s, keep = make_problem(p)
        states = np.empty((p.horizon + 1, p.robots, p.dx))
        controls = np.empty((p.horizon + 1, p.robots, p.du))
        best = C.c_double()
        ok = C.c_int()
        its = (OrIterStats * iterations)()
        used = fn(C.byref(s), C.byref(cfg), _dp(states), _dp(controls), C.byref(best), C.byref(ok), its)
        if used < 0:
            raise RuntimeError(self.err())
        return dict(states=states, controls=controls, best_reward=best.value, success=bool(ok.value),
                    iterations=used, per_iteration=[(its[j].reward, its[j].objective, bool(its[j].success))
                                                    for j in range(used)])

    def mppi_solve(self, p, cfg: OrMppiConfig):
        return self._baseline(self.L.or_mppi_solve, p, cfg, cfg.iterations)

    def cem_solve(self, p, cfg: OrCemConfig):
        return self._baseline(self.L.or_cem_solve, p, cfg, cfg.iterations)

class Reference(_Base):
    """The reference's own library (proj/src, unchanged) behind ref_* C entry points."""

    def __init__(self, path: Path = REF_SO):
        super().__init__(path)

    def _sig(self):
        L, dp, i64 = self.L, C.POINTER(C.c_double), C.c_int64
        L.ref_last_error.restype = C.c_char_p
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_mix_seed3.restype = C.c_uint64
        L.ref_mix_seed3.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.ref_normal_fill.argtypes = [C.c_uint64, dp, i64]
        L.ref_sample_batch.argtypes = [C.POINTER(OrProblem), dp, C.c_int, C.c_double, C.c_int, C.c_int, C.c_uint64, dp]
        L.ref_make_schedule.argtypes = [C.c_int, C.c_double, dp, dp]
        L.ref_sampling_spread.argtypes = [C.c_int, C.c_double, C.c_int, dp, dp]
        L.ref_rk4_step.argtypes = [C.c_int, dp, dp, C.c_double, dp]
        L.ref_rollout.argtypes = [C.POINTER(OrProblem), dp, dp, dp]
        L.ref_total_reward.argtypes = [C.POINTER(OrProblem), dp, dp]
        L.ref_objective.argtypes = [C.POINTER(OrProblem), dp]
        L.ref_objective.restype = C.c_double
        L.ref_check_success.argtypes = [C.POINTER(OrProblem), dp, C.c_char_p, C.c_int]
        L.ref_score_weights.argtypes = [dp, i64, C.c_double, dp]
        L.ref_mc_average.argtypes = [dp, dp, i64, C.c_int, C.c_int, dp]
        L.ref_run_denoising.argtypes = [C.POINTER(OrProblem), dp, C.POINTER(OrConfig), dp, C.POINTER(OrTrace)]
        L.ref_solve.argtypes = [C.POINTER(OrProblem), C.POINTER(OrConfig), C.POINTER(OrOptConfig), dp, dp,
                                C.POINTER(C.c_int), C.POINTER(OrIterStats)]
        L.ref_select_elites.argtypes = [dp, i64, C.c_int, C.POINTER(C.c_int)]
        L.ref_mppi_solve.argtypes = [C.POINTER(OrProblem), C.POINTER(OrMppiConfig), dp, dp, C.POINTER(C.c_int),
                                     C.POINTER(OrIterStats)]
        L.ref_cem_solve.argtypes = [C.POINTER(OrProblem), C.POINTER(OrCemConfig), dp, dp, C.POINTER(C.c_int),
                                    C.POINTER(OrIterStats)]
        L.ref_antipodal_circle.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double, dp, dp]
        L.ref_antipodal_sphere.argtypes = [C.c_int, C.c_double, C.c_double, dp, dp]
        L.ref_random_square.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_double, dp, dp]

    def err(self):
        return self.L.ref_last_error().decode()

    def _ok(self, rc):
        if rc:
            raise RuntimeError(self.err())

    def mix_seed(self, a, b, c=None):
        return self.L.ref_mix_seed(a, b) if c is None else self.L.ref_mix_seed3(a, b, c)

    def normal_fill(self, seed, n):
        out = np.empty(n)
        self.L.ref_normal_fill(seed, _dp(out), n)
        return out

    def make_schedule(self, steps, abf):
        ab, a = np.empty(steps + 1), np.empty(steps)
        self._ok(self.L.ref_make_schedule(steps, abf, _dp(ab), _dp(a)))
        return ab, a

    def sampling_spread(self, steps, abf, i):
        ms, sd = C.c_double(), C.c_double()
        self._ok(self.L.ref_sampling_spread(steps, abf, i, C.byref(ms), C.byref(sd)))
        return ms.value, sd.value

    def sample_batch(self, p, current, steps, abf, i, batch, seed):
        s, keep = make_problem(p)
        cur = np.ascontiguousarray(current, dtype=np.float64)
        out = np.empty((batch, p.horizon, p.robots, p.du))
        self._ok(self.L.ref_sample_batch(C.byref(s), _dp(cur), steps, abf, i, batch, seed, _dp(out)))
        return out

    def rk4_step(self, kind, x, u, dt):
        x = np.ascontiguousarray(x, dtype=np.float64)
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty_like(x)
        self._ok(self.L.ref_rk4_step(kind, _dp(x), _dp(u), dt, _dp(out)))
        return out

    def rollout(self, p, u):
        s, keep = make_problem(p)
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(p.horizon, p.robots, p.du)
        states = np.empty((p.horizon + 1, p.robots, p.dx))
        controls = np.empty((p.horizon + 1, p.robots, p.du))
        self._ok(self.L.ref_rollout(C.byref(s), _dp(u), _dp(states), _dp(controls)))
        return states, controls

    def total_reward(self, p, states):
        s, keep = make_problem(p)
        r = C.c_double()
        self._ok(self.L.ref_total_reward(C.byref(s), _dp(np.ascontiguousarray(states, dtype=np.float64)), C.byref(r)))
        return r.value

    def objective(self, p, states):
        s, keep = make_problem(p)
        return self.L.ref_objective(C.byref(s), _dp(np.ascontiguousarray(states, dtype=np.float64)))

    def check_success(self, p, states):
        s, keep = make_problem(p)
        buf = C.create_string_buffer(256)
        ok = self.L.ref_check_success(C.byref(s), _dp(np.ascontiguousarray(states, dtype=np.float64)), buf, 256)
        return bool(ok), buf.value.decode()

    def score_weights(self, rewards, lam):
        r = np.ascontiguousarray(rewards, dtype=np.float64)
        w = np.empty_like(r)
        self._ok(self.L.ref_score_weights(_dp(r), len(r), lam, _dp(w)))
        return w

    def mc_average(self, samples, weights):
        s = np.ascontiguousarray(samples, dtype=np.float64)
        m = s.shape[0]
        e = s[0].size
        out = np.empty(s.shape[1:])
        self._ok(self.L.ref_mc_average(_dp(s.reshape(m, e)), _dp(np.ascontiguousarray(weights, dtype=np.float64)), m,
                                       e, 1, _dp(out)))
        return out

    def run_denoising(self, p, base, cfg: OrConfig):
        s, keep = make_problem(p)
        base = np.ascontiguousarray(base, dtype=np.float64)
        out = np.empty((p.horizon, p.robots, p.du))
        tr = (OrTrace * cfg.steps)()
        self._ok(self.L.ref_run_denoising(C.byref(s), _dp(base), C.byref(cfg), _dp(out), tr))
        return out, [(t.step, t.best_reward, t.mean_reward, t.weight_entropy) for t in tr]

    def solve(self, p, cfg: OrConfig, max_iterations=10, stop_on_success=True):
        s, keep = make_problem(p)
        oc = OrOptConfig(max_iterations, int(stop_on_success), 0.0)
        states = np.empty((p.horizon + 1, p.robots, p.dx))
        best = C.c_double()
        ok = C.c_int()
        its = (OrIterStats * max_iterations)()
        used = self.L.ref_solve(C.byref(s), C.byref(cfg), C.byref(oc), _dp(states), C.byref(best), C.byref(ok), its)
        if used < 0:
            raise RuntimeError(self.err())
        return dict(states=states, best_reward=best.value, success=bool(ok.value), iterations=used,
                    per_iteration=[(its[j].reward, its[j].objective, bool(its[j].success)) for j in range(used)])

    def select_elites(self, rewards, count):
        r = np.ascontiguousarray(rewards, dtype=np.float64)
        out = (C.c_int * count)()
        if self.L.ref_select_elites(_dp(r), len(r), count, out):
            raise ValueError(self.err())
        return list(out)

    def _baseline(self, fn, p, cfg, iterations):
        s, keep = make_problem(p)
        states = np.empty((p.horizon + 1, p.robots, p.dx))
        best = C.c_double()
        ok = C.c_int()
        its = (OrIterStats * iterations)()
        used = fn(C.byref(s), C.byref(cfg), _dp(states), C.byref(best), C.byref(ok), its)
        if used < 0:
            raise RuntimeError(self.err())
        return dict(states=states, best_reward=best.value, success=bool(ok.value), iterations=used,
                    per_iteration=[(its[j].reward, its[j].objective, bool(its[j].success)) for j in range(used)])

    def mppi_solve(self, p, cfg: OrMppiConfig):
        return self._baseline(self.L.ref_mppi_solve, p, cfg, cfg.iterations)

    def cem_solve(self, p, cfg: OrCemConfig):
        return self._baseline(self.L.ref_cem_solve, p, cfg, cfg.iterations)

    def antipodal_circle(self, robots, diameter, kind, robot_radius):
        dx = 4
        st, go = np.empty((robots, dx)), np.empty((robots, 2))
        self._ok(self.L.ref_antipodal_circle(robots, diameter, kind, robot_radius, _dp(st), _dp(go)))
        return st, go

    def antipodal_sphere(self, robots, diameter, robot_radius):
        st, go = np.empty((robots, 6)), np.empty((robots, 3))
        self._ok(self.L.ref_antipodal_sphere(robots, diameter, robot_radius, _dp(st), _dp(go)))
        return st, go

    def random_square(self, robots, diameter, seed, kind, robot_radius):
        st, go = np.empty((robots, 4)), np.empty((robots, 2))
        self._ok(self.L.ref_random_square(robots, diameter, seed, kind, robot_radius, _dp(st), _dp(go)))
        return st, go


def available_reference() -> bool:
    return REF_SO.exists()
