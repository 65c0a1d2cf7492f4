"""Host-side mirror of the reference planner interface over the CUDA C-ABI.

``GpuDenoiser`` owns one d4orm_cuda_ctx (one GPU, one stream) and exposes the
reference's operators with the same argument meaning and error behaviour:

  run_denoising   denoiser.hpp:68-70  / denoiser.cpp:119-184
  denoise_step    one loop body        denoiser.cpp:152-180 (teacher-forced)
  rollout_fitness rollout + total_reward  dynamics.cpp:122-169, reward.cpp:67-130
  score_weights   denoiser.cpp:50-90 (+ weight_entropy :24-30)
  solve           optimizer.cpp:48-102 (anytime loop, every iteration on the device)

Arrays use the reference's layouts: a joint control sequence is (T, R, du)
C-contiguous == Eigen (R*du) x T column-major.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import (DEFORMATION, FROM_SCRATCH, NOISE_HOST, NOISE_PHILOX, PREC_F32, PREC_F64, DenoiserConfig_C,
                   Problem_C, TraceRec_C, dptr, lib, raise_for)
from .scenarios import Problem


@dataclass
class DenoiserConfig:
    """DenoiserConfig (denoiser.hpp:19-27); batch = BASELINE "N samples"."""
    steps: int = 100
    batch: int = 2048
    lam: float = 0.1
    alpha_bar_final: float = 0.05
    seed: int = 0
    mode: int = DEFORMATION

    def c(self) -> DenoiserConfig_C:
        return DenoiserConfig_C(self.steps, self.batch, self.lam, self.alpha_bar_final, self.seed & ((1 << 64) - 1),
                                self.mode)


def make_schedule(steps: int, alpha_bar_final: float) -> np.ndarray:
    """schedule.cpp:9-27 — alpha_bar[0..N]."""
    if steps < 1:
        raise ValueError(f"make_schedule: steps must be >= 1, got {steps}")
    if not (0.0 < alpha_bar_final < 1.0):
        raise ValueError(f"make_schedule: alpha_bar_final must lie in (0, 1), got {alpha_bar_final}")
    ab = np.empty(steps + 1)
    ab[0] = 1.0
    for i in range(1, steps + 1):
        ab[i] = alpha_bar_final ** (i / steps)
    return ab


class GpuDenoiser:
    def __init__(self, problem: Problem | None = None, device: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, precision: int = PREC_F32, noise: int = NOISE_PHILOX,
                 graphs: bool = True, exchange=None):
        """world > 1: the step's two all-gathers run over NCCL (nccl_id, the
        128 bytes rank 0 got from d4orm_cuda_nccl_id) or through `exchange`,
        a host function exchange(local: bytes) -> bytes (all ranks' blocks
        concatenated in rank order), e.g. torch.distributed over gloo."""
        L = lib()
        self._L = L
        h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        rc = L.d4orm_cuda_create(device, rank, world, idbuf, C.byref(h))
        if rc != 0:
            raise _lib.D4ormError(rc, f"d4orm_cuda_create failed (code {rc}) on device {device}")
        self._h = h
        self.world, self.rank = world, rank
        self._noise_cb = None
        self._noise_provider = None
        self._xcb = None
        self.problem = None
        if exchange is not None:
            self.set_exchange(exchange)
        self.set_options(precision, noise, graphs)
        if problem is not None:
            self.set_problem(problem)

    def close(self):
        if getattr(self, "_h", None):
            self._L.d4orm_cuda_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc:
            raise_for(rc, self._L.d4orm_cuda_last_error(self._h).decode())

    # ---------------------------------------------------------- setup
    def set_options(self, precision: int = PREC_F32, noise: int = NOISE_PHILOX, graphs: bool = True):
        self.precision, self.noise, self.graphs = precision, noise, graphs
        self._check(self._L.d4orm_cuda_set_options(self._h, precision, noise, int(graphs)))

    def set_problem(self, p: Problem):
        self._keep = (p.starts, p.goals, p.obs_centers, p.obs_radii)
        pc = Problem_C()
        pc.kind = p.kind
        pc.dx, pc.du, pc.pdim = p.dims
        pc.robots, pc.horizon, pc.dt = p.robots, p.horizon, p.dt
        for d in range(p.du):
            pc.lower[d], pc.upper[d] = p.lower[d], p.upper[d]
        pc.starts, pc.goals = dptr(p.starts), dptr(p.goals)
        pc.n_obstacles = len(p.obs_radii)
        pc.obs_centers = dptr(p.obs_centers) if len(p.obs_radii) else dptr(np.zeros(3))
        pc.obs_radii = dptr(p.obs_radii) if len(p.obs_radii) else dptr(np.zeros(1))
        pc.w_t, pc.epsilon, pc.robot_radius = p.w_t, p.epsilon, p.robot_radius
        pc.goal_tolerance, pc.obstacle_weight, pc.effort_weight = p.goal_tolerance, p.obstacle_weight, p.effort_weight
        self._check(self._L.d4orm_cuda_set_problem(self._h, C.byref(pc)))
        self.problem = p

    def set_exchange(self, fn):
        """Host-mediated all-gather for world > 1 without NCCL (see __init__)."""
        def cb(user, local, nbytes, gathered):
            try:
                out = fn(C.string_at(local, nbytes))
                if len(out) != nbytes * self.world:
                    return 1
                C.memmove(gathered, out, len(out))
                return 0
            except Exception:
                return 1

        self._xcb = _lib.EXCHANGE_FN(cb)
        self._check(self._L.d4orm_cuda_set_exchange_fn(self._h, self._xcb, None))

    def set_noise_provider(self, fn):
        """fn(step, m0, count, elems) -> (count, elems) float64 normals (host noise mode)."""
        self._noise_provider = fn

        def cb(user, step, m0, count, elems, dst):
            try:
                arr = np.ascontiguousarray(fn(step, m0, count, elems), dtype=np.float64).reshape(count * elems)
                C.memmove(dst, arr.ctypes.data, arr.nbytes)
                return 0
            except Exception:  # surfaced as a runtime error by the library
                return 1

        self._noise_cb = _lib.NOISE_FN(cb)
        self._check(self._L.d4orm_cuda_set_noise_fn(self._h, self._noise_cb, None))

    # ---------------------------------------------------------- the path
    def _shape(self):
        p = self.problem
        return (p.horizon, p.robots, p.du)

    def run_denoising(self, base: np.ndarray, cfg: DenoiserConfig):
        """run_denoising (denoiser.cpp:119-184) → (variable (T,R,du), trace)."""
        base = np.ascontiguousarray(base, dtype=np.float64).reshape(self._shape())
        out = np.empty(self._shape())
        trace = (TraceRec_C * cfg.steps)()
        c = cfg.c()
        self._check(self._L.d4orm_cuda_run_denoising(self._h, dptr(base), C.byref(c), dptr(out), trace))
        return out, [(t.step, t.best_reward, t.mean_reward, t.weight_entropy) for t in trace]

    def denoise_step(self, base, variable, i: int, cfg: DenoiserConfig, noise: np.ndarray | None = None):
        """One loop body (denoiser.cpp:152-180): → (variable', rewards, weights, trace record)."""
        base = np.ascontiguousarray(base, dtype=np.float64).reshape(self._shape())
        var = np.ascontiguousarray(variable, dtype=np.float64).reshape(self._shape())
        nz = None if noise is None else np.ascontiguousarray(noise, dtype=np.float64).reshape(cfg.batch, -1)
        out = np.empty(self._shape())
        rw = np.empty(cfg.batch)
        w = np.empty(cfg.batch)
        rec = TraceRec_C()
        c = cfg.c()
        self._check(self._L.d4orm_cuda_denoise_step(self._h, dptr(base), dptr(var), dptr(nz), i, C.byref(c), dptr(out),
                                                   dptr(rw), dptr(w), C.byref(rec)))
        return out, rw, w, (rec.step, rec.best_reward, rec.mean_reward, rec.weight_entropy)

    def rollout_fitness(self, u: np.ndarray, want_states: bool = True):
        """rollout + total_reward for `count` control sequences u (count,T,R,du)."""
        p = self.problem
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1, p.horizon, p.robots, p.du)
        n = u.shape[0]
        states = np.empty((n, p.horizon + 1, p.robots, p.dx)) if want_states else None
        controls = np.empty((n, p.horizon + 1, p.robots, p.du)) if want_states else None
        rewards = np.empty(n)
        counts = np.empty((n, 2), dtype=np.int64)
        self._check(self._L.d4orm_cuda_rollout_fitness(self._h, dptr(u), n, dptr(states), dptr(controls), dptr(rewards),
                                                      counts.ctypes.data_as(C.POINTER(C.c_int64))))
        return states, controls, rewards, counts

    def score_weights(self, rewards: np.ndarray, lam: float):
        r = np.ascontiguousarray(rewards, dtype=np.float64)
        w = np.empty_like(r)
        t3 = np.empty(3)
        self._check(self._L.d4orm_cuda_score_weights(self._h, dptr(r), len(r), lam, dptr(w), dptr(t3)))
        return w, t3

    def weighted_mean(self, samples: np.ndarray, weights: np.ndarray) -> np.ndarray:
        """mc_average (denoiser.cpp:92-108) on the device (K5a + K5b) in the
        context's precision: Σ_m w_m·samples[m] → samples.shape[1:]."""
        smp = np.ascontiguousarray(samples, dtype=np.float64)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        m = smp.shape[0] if smp.ndim else 0
        if m != len(w):
            raise ValueError("mc_average: weight count does not match sample count")
        out = np.empty(smp.shape[1:])
        self._check(self._L.d4orm_cuda_weighted_mean(self._h, dptr(smp), dptr(w), m, int(np.prod(smp.shape[1:])),
                                                     dptr(out)))
        return out

    def philox_noise(self, seed: int, step: int, m0: int, count: int) -> np.ndarray:
        out = np.empty((count, self.problem.elems), dtype=np.float32)
        self._check(self._L.d4orm_cuda_philox_noise(self._h, seed, step, m0, count,
                                                    out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def bench_steps(self, base, cfg: DenoiserConfig, warmup: int, steps: int, kernels: bool = True):
        base = np.ascontiguousarray(base, dtype=np.float64).reshape(self._shape())
        ms = C.c_double()
        kms = np.zeros(6)
        c = cfg.c()
        self._check(self._L.d4orm_cuda_bench_steps(self._h, dptr(base), C.byref(c), warmup, steps, C.byref(ms),
                                                  dptr(kms) if kernels else None))
        return ms.value, kms

    def launches_per_step(self) -> int:
        return self._L.d4orm_cuda_launches_per_step(self._h)

    def last_w32(self, m: int) -> np.ndarray:
        """The fp32 weights K4 left for K5 (zero below the adaptive floor)."""
        out = np.empty(m, dtype=np.float32)
        self._check(self._L.d4orm_cuda_last_w32(self._h, out.ctypes.data_as(C.POINTER(C.c_float)), m))
        return out

    def k5_regen(self) -> int:
        """1: the last run's K5a regenerated the Philox noise (no z rows), 0: it
        read the stored z rows, -1: no run yet."""
        return self._L.d4orm_cuda_k5_regen(self._h)

    def fitness_path(self) -> int:
        """fp32 fitness form for the current problem: 1 pair list, 0 tiles."""
        return self._L.d4orm_cuda_fitness_path(self._h)

    def last_fit_kernel(self) -> int:
        """K2+K3 kernel of the last fitness launch: 0 k_rollout_fitness, 1 the
        time-segmented kernel, 2 k_rollout_fitness_pl32 (32-step windows)."""
        return self._L.d4orm_cuda_last_fit_kernel(self._h)

    # ---------------------------------------------------------- anytime loop
    def solve(self, cfg: DenoiserConfig, max_iterations: int = 10, stop_on_success: bool = True,
              deadline_seconds: float | None = None, on_iteration=None):
        """solve (optimizer.cpp:48-102) on the device (d4orm_cuda_solve): zero-
        control start, per-iteration seed mix_seed(seed, it), denoise a
        deformation, fp64 rollout of base+Δ, total_reward / objective /
        check_success and best tracking in K6; one CUDA graph per iteration in
        Philox mode.  on_iteration(it, seed_it) runs before each iteration (host
        noise providers reseed there)."""
        if max_iterations < 1:
            raise ValueError("solve: max_iterations must be >= 1")
        p = self.problem
        sc = _lib.SolveConfig_C()
        sc.max_iterations = max_iterations
        sc.stop_on_success = int(stop_on_success)
        sc.deadline_seconds = float(deadline_seconds) if deadline_seconds is not None else 0.0
        sc.denoiser = cfg.c()
        cb = None
        if on_iteration is not None:
            def _cb(user, it, seed_it):
                try:
                    on_iteration(it, seed_it)
                    return 0
                except Exception:
                    return 1
            cb = _lib.ITER_FN(_cb)
            sc.on_iteration = cb
        best_states = np.empty((p.horizon + 1, p.robots, p.dx))
        best_controls = np.empty((p.horizon + 1, p.robots, p.du))
        recs = (_lib.IterationRec_C * max_iterations)()
        traces = (TraceRec_C * (max_iterations * cfg.steps))()
        used, ok = C.c_int(), C.c_int()
        best = C.c_double()
        t0 = time.perf_counter()
        self._check(self._L.d4orm_cuda_solve(self._h, C.byref(sc), dptr(best_states), dptr(best_controls), recs,
                                             traces, C.byref(used), C.byref(best), C.byref(ok)))
        result = SolveResult()
        result.iterations_used = used.value
        result.total_denoise_steps = used.value * cfg.steps
        result.per_iteration = [(r.reward, r.objective, bool(r.success), r.elapsed) for r in recs[: used.value]]
        result.traces = [[(t.step, t.best_reward, t.mean_reward, t.weight_entropy)
                          for t in traces[i * cfg.steps:(i + 1) * cfg.steps]] for i in range(used.value)]
        result.best_reward = best.value
        result.best_states, result.best_controls = best_states, best_controls
        result.success = bool(ok.value)
        result.wall_time = time.perf_counter() - t0
        return result


    # ---------------------------------------------------------- baselines
    def _baseline(self, fn, cfg_c, iterations, batch):
        p = self.problem
        best_states = np.empty((p.horizon + 1, p.robots, p.dx))
        best_controls = np.empty((p.horizon + 1, p.robots, p.du))
        recs = (_lib.IterationRec_C * iterations)()
        used, ok = C.c_int(), C.c_int()
        best = C.c_double()
        t0 = time.perf_counter()
        self._check(fn(self._h, C.byref(cfg_c), dptr(best_states), dptr(best_controls), recs, C.byref(used),
                       C.byref(best), C.byref(ok)))
        result = SolveResult()
        result.iterations_used = used.value
        result.total_denoise_steps = used.value
        result.per_iteration = [(r.reward, r.objective, bool(r.success), r.elapsed) for r in recs[: used.value]]
        result.best_reward = best.value
        result.best_states, result.best_controls = best_states, best_controls
        result.success = bool(ok.value)
        result.wall_time = time.perf_counter() - t0
        return result

    def mppi_solve(self, batch: int = 2048, lam: float = 0.1, sigma: float = 1.0, iterations: int = 1000,
                   seed: int = 0, stop_on_success: bool = True, deadline_seconds: float | None = None):
        """mppi_solve (baselines.cpp:99-129) on the device; host-noise providers
        receive the iteration as `step` (stream mix_seed(seed, it, m))."""
        c = _lib.MppiConfig_C(batch, lam, sigma, iterations, seed & ((1 << 64) - 1), int(stop_on_success),
                              float(deadline_seconds or 0.0))
        return self._baseline(self._L.d4orm_cuda_mppi_solve, c, iterations, batch)

    def cem_solve(self, batch: int = 2048, elite_fraction: float = 0.1, initial_std: float = 1.0,
                  min_std: float = 0.05, iterations: int = 1000, seed: int = 0, stop_on_success: bool = True,
                  deadline_seconds: float | None = None):
        """cem_solve (baselines.cpp:131-173) on the device."""
        c = _lib.CemConfig_C(batch, elite_fraction, initial_std, min_std, iterations, seed & ((1 << 64) - 1),
                             int(stop_on_success), float(deadline_seconds or 0.0))
        return self._baseline(self._L.d4orm_cuda_cem_solve, c, iterations, batch)


@dataclass
class SolveResult:
    """SolveResult (result.hpp:20-29)."""
    best_states: np.ndarray | None = None
    best_controls: np.ndarray | None = None
    best_reward: float = 0.0
    success: bool = False
    iterations_used: int = 0
    total_denoise_steps: int = 0
    wall_time: float = 0.0
    per_iteration: list = field(default_factory=list)
    traces: list = field(default_factory=list)
