#!/usr/bin/env python
"""bench.py — the denoise-step hot path on B200, one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--impl ours|reference]

A "step" is one denoising step (denoiser.cpp:152-180) over the whole batch of
samples: Philox noise, rollout+fitness of every sample, softmax weights, the
weighted mean and the update.  Default workload: BASELINE config C5 (2D
velocity-input holonomic, R=64, T=256, N=262144 samples/step, 16 obstacles),
the configuration the FP32-roofline target and the 1/2/4/8-GPU scaling are
quoted on; --config selects another BASELINE shape.  Samples are sharded
across ranks (one process per GPU, torchrun); total work is fixed → "strong".

value    rollouts+fitness evaluations/s with inputs resident in HBM (device
         CUDA-event timing of exactly K steps, max over ranks)
e2e      the same metric through the public C-ABI call d4orm_cuda_run_denoising
         with host buffers (H2D base, D2H variable+trace inside the region)
solve    the same metric through d4orm_cuda_solve (the anytime loop, every
         iteration on the device), the config's iteration count
roofline dominant kernel K2+K3 (rollout+fitness), FP32-bound: algorithmic
         FLOPs per launch / its CUDA-event launch time, against the
         FP32 peak measured live on this GPU (d4orm_cuda_fp32_peak)
--impl reference  the reference's own CPU implementation (oracle/_ref: proj/src
         compiled unchanged) on all host cores, bounded sample per step
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "joint-trajectory rollouts+fitness evals/sec"
UNIT = "evals/s"


def algorithmic_flops_per_eval(p) -> float:
    """F = T·[R·(f_dyn + 3·du + 3p + 3) + 3p·R(R−1)/2 + 3p·R·O]."""
    R, T, du, pd, O = p.robots, p.horizon, p.du, p.pdim, len(p.obs_radii)
    f_dyn = {0: 40, 1: 2 * 4, 2: 2 * 6, 3: 2 * du, 4: 2 * du, 5: 40}[p.kind]
    return T * (R * (f_dyn + 3 * du + 3 * pd + 3) + 3 * pd * R * (R - 1) / 2 + 3 * pd * R * O)


class ClockSampler:
    """nvidia-smi-equivalent clocks / throttle reasons sampled during the timed region (NVML)."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x10: "sync_boost"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz, self.ok = [], set(), None, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # reported, never fatal
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "note": "NVML unavailable"}
        load = [s for s in self.samples if s > 0.5 * (self.max_mhz or 1)] or self.samples
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def dist_setup(world: int):
    """Control plane only (barrier, 128-byte NCCL id broadcast, max-over-ranks):
    gloo over 127.0.0.1.  The per-step data exchange is NCCL inside the library."""
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo", rank=int(os.environ["RANK"]), world_size=world)
    return dist


def reduce_max(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_reference_step(ref, p, batch: int, seed: int, workers: int = 0) -> float:
    """One denoising step of the reference's own run_denoising (steps=1) over
    `batch` samples on all host cores; returns seconds."""
    from oracle.oracle import make_config
    base = np.zeros((p.horizon, p.robots, p.du))
    t0 = time.perf_counter()
    ref.run_denoising(p, base, make_config(1, batch, seed=seed, workers=workers))
    return time.perf_counter() - t0


def reference_checker():
    from oracle.oracle import REF_SO, ORACLE_SO, Oracle, Reference
    if REF_SO.exists():
        return Reference(), "reference", "oracle/_ref: reference proj/src compiled unchanged"
    if not ORACLE_SO.exists():
        import subprocess
        subprocess.run(["make", "-s", "-f", str(ROOT / "oracle" / "Makefile")], check=True)
    return Oracle(), "port", "oracle/d4orm_oracle.c (plain-C restatement, pinned bitwise to the reference)"


def size_cpu_sample(ref, p, M: int, budget_s: float) -> tuple[int, float]:
    """Largest power-of-two sample ≤ M whose reference step takes ≈budget_s."""
    b = min(M, 256)
    t = cpu_reference_step(ref, p, b, 1)
    while b < M and t * 2 <= budget_s:
        b = min(M, b * 2)
        t = cpu_reference_step(ref, p, b, 1)
    return b, t


def config_json(rc, world: int) -> dict:
    p = rc.problem
    return {"workload": rc.name, "model": p.name, "robots": p.robots, "horizon": p.horizon, "samples_per_step": rc.samples,
            "denoising_steps": rc.steps, "iterations": rc.iterations, "obstacles": int(len(p.obs_radii)),
            "global_batch": rc.samples, "seq_len": p.horizon, "parallelism": f"samples-sharded x{world}",
            "l2": "no flush needed: every step draws fresh noise (Philox keyed by step), so no step re-reads inputs "
                  "a previous step left in L2 except the %d KB base/variable; per-step chunk partials %.0f MB "
                  "(+ z rows %.0f MB when stored) vs 126 MB L2" % (p.elems * 4 // 1024,
                                                                 (rc.samples // world + 255) // 256 * p.elems * 4 / 1e6,
                                                                 rc.samples // world * p.elems * 4 / 1e6)}


def run_reference_arm(args, rc, rank: int, world: int):
    if rank != 0:
        return
    p = rc.problem
    ref, kind, what = reference_checker()
    cores = os.cpu_count() or 1
    per_step_budget = max(0.5, min(2.0, 150.0 / max(1, args.steps + args.warmup)))
    batch, _ = size_cpu_sample(ref, p, rc.samples, per_step_budget)
    for j in range(args.warmup):
        cpu_reference_step(ref, p, batch, 100 + j)
    times = [cpu_reference_step(ref, p, batch, 200 + j) for j in range(args.steps)]
    total = sum(times)
    value = batch * args.steps / total
    sample = (f"{batch} of {rc.samples} samples per step ({what}; velocity-input/unicycle kinds via the "
              f"reference's rk4_with extension point), run_denoising steps=1, workers=0 (all {cores} threads)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup,
            # a full step of the config at the measured rate; the bounded sample's own time beside it
            "ms_per_step": 1e3 * rc.samples / value, "sample_ms_per_step": 1e3 * total / args.steps,
            "sample_per_step": batch, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_json(rc, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def self_launch(args_list, n: int) -> int:
    """--gpus N without a launcher: start N ranks (one process per GPU) with
    torch.distributed.run on this node, exactly as the driver would, and pass
    the exit code through.  Rank 0 prints the JSON line."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()), *args_list]
    sys.stderr.write("bench.py: self-launching %d ranks: %s\n" % (n, " ".join(cmd)))
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1-C4 step-latency keys")
    ap.add_argument("--no-f64", action="store_true", help="skip the fp64 (reference arithmetic) throughput key")
    ap.add_argument("--graphs", type=int, default=1)
    ap.add_argument("--force-comm", action="store_true",
                    help="N = 1 through the sharded protocol (1-rank NCCL communicator): exercises the N > 1 path")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check: every rank prints its rank/world/device as JSON and exits (no GPU work)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(sys.argv[1:], args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: refusing to measure a different "
                         f"GPU count than asked\n")
        sys.exit(2)
    if args.dry_run:
        print(json.dumps({"dry_run": True, "rank": rank, "world": world, "local_rank": local_rank,
                          "device": f"cuda:{local_rank}", "impl": args.impl,
                          "master": f"{os.environ.get('MASTER_ADDR', '-')}:{os.environ.get('MASTER_PORT', '-')}"}),
              flush=True)
        return
    if world > 1:
        # the NCCL communicator-init lines (one "Init COMPLETE" per rank) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    from paper_2503_12204_b200 import scenarios as S
    rc = S.baseline_config(args.config)

    if args.impl == "reference":
        run_reference_arm(args, rc, rank, world)
        return

    import paper_2503_12204_b200 as d4
    from paper_2503_12204_b200._lib import lib
    dist = dist_setup(world) if world > 1 else None
    nccl_id = None
    if world == 1 and args.force_comm:
        buf = C.create_string_buffer(128)
        assert lib().d4orm_cuda_nccl_id(buf) == 0, "ncclGetUniqueId failed"
        nccl_id = bytes(buf.raw)
    if world > 1:
        buf = C.create_string_buffer(128)
        obj = [None]
        if rank == 0:
            assert lib().d4orm_cuda_nccl_id(buf) == 0, "ncclGetUniqueId failed"
            obj = [bytes(buf.raw)]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    p = rc.problem
    M = rc.samples
    Ml = M // world
    g = d4.GpuDenoiser(p, device=local_rank, rank=rank, world=world, nccl_id=nccl_id, precision=d4.PREC_F32,
                       noise=d4.NOISE_PHILOX, graphs=bool(args.graphs))
    if world > 1:
        sys.stderr.write(f"bench.py: rank {rank}/{world} on cuda:{local_rank}: NCCL communicator initialised "
                         f"(samples [{rank * Ml}, {(rank + 1) * Ml}))\n")
    cfg = d4.DenoiserConfig(steps=rc.steps, batch=M, lam=rc.lam, alpha_bar_final=rc.alpha_bar_final, seed=rc.seed)
    base = np.zeros((p.horizon, p.robots, p.du))

    L = lib()
    L.d4orm_cuda_fp32_peak.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    peak_tf, peak_clk = C.c_double(), C.c_double()
    L.d4orm_cuda_fp32_peak(local_rank, 5, C.byref(peak_tf), C.byref(peak_clk))

    if dist:
        dist.barrier()
    with ClockSampler(local_rank) as clk:
        ms, kms = g.bench_steps(base, cfg, args.warmup, args.steps, kernels=True)
    ms = reduce_max(dist, ms)
    if dist:
        dist.barrier()
    value = M * args.steps / (ms / 1e3)

    # e2e through the public C-ABI call with host buffers
    e2e = None
    if not args.no_e2e:
        g.run_denoising(base, cfg)  # untimed: builds the run's graph (one per shape, reused by every later call)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        g.run_denoising(base, cfg)
        dt = reduce_max(dist, time.perf_counter() - t0)
        E = p.elems
        # per call: base (fp32 upload of the fp64 host array), variable init, Philox key table, error word in;
        # variable + trace + error word out.  The noise never crosses the bus (drawn in-kernel).
        h2d_call = int(E * 4 + E * 8 + (cfg.steps + 1) * 8 + 8)
        d2h_call = int(E * 8 + cfg.steps * 32 + 8)
        e2e = {"value": M * cfg.steps / dt, "unit": UNIT, "h2d_bytes_per_step": h2d_call / cfg.steps,
               "d2h_bytes_per_step": d2h_call / cfg.steps, "h2d_bytes_per_call": h2d_call,
               "d2h_bytes_per_call": d2h_call,
               "step": f"one public call d4orm_cuda_run_denoising = {cfg.steps} denoising steps (host base in, host "
                       f"variable + trace out); bytes per step = per call / {cfg.steps}",
               "ms_per_call": dt * 1e3}

    # the anytime loop (solve, optimizer.cpp:49-102) on the device: every
    # iteration's denoising + final rollout/outcome in one graph per iteration
    solve = None
    if not args.no_e2e:
        g.solve(cfg, max_iterations=rc.iterations, stop_on_success=False)  # graph build (untimed)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        sr = g.solve(cfg, max_iterations=rc.iterations, stop_on_success=False)
        dt = reduce_max(dist, time.perf_counter() - t0)
        solve = {"value": M * cfg.steps * sr.iterations_used / dt, "unit": UNIT, "iterations": sr.iterations_used,
                 "wall_ms": dt * 1e3, "best_reward": sr.best_reward, "success": sr.success,
                 "call": "d4orm_cuda_solve: max_iterations=%d, stop_on_success=false (SURVEY 8d throughput runs)"
                         % rc.iterations}

    F = algorithmic_flops_per_eval(p)
    k23_ms = kms[1]
    achieved = Ml * F / (k23_ms * 1e-3) / 1e12
    traffic, traffic_src = None, None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        tj = json.loads(tf.read_text())
        traffic, traffic_src = tj.get(rc.name), (tj.get("_sources") or {}).get(rc.name)
    E = p.elems
    # K5a: algorithmic bytes (every sample's z row) and the bytes it actually
    # moves — z rows of samples with a non-zero fp32 weight only (K4's floor:
    # for shapes whose K5a skips zero weights — E >= 16384 or du = 3, C4/C5 —
    # the adaptive floor dropping <= 2^-24 of the weight mass; elsewhere
    # weights below 2^-48 of the largest), + weights + partials
    parts = (Ml + 255) // 256 * E * 4
    k5_alg = Ml * E * 4 + Ml * 4 + parts
    k5_nz = float(kms[5])
    k5_read = int(k5_nz * E * 4) + Ml * 4 + parts
    if g.k5_regen() == 1:
        # K5a regenerates the Philox normals of the samples that keep a weight
        # (no z rows in HBM): instruction-issue bound, reported as normals/s
        k5_info = {"kernel": "k_wmean_regen (K5a)", "bound": "issue (Philox4x32-10 + Box-Muller per normal)",
                   "normals_per_launch": int(k5_nz * E), "samples_with_weight": k5_nz, "samples": Ml,
                   "gnormals_per_s": k5_nz * E / (kms[3] * 1e-3) / 1e9 if kms[3] > 0 else None,
                   "note": "z is not stored by K2+K3 nor read here; see DESIGN.md 3 (K5a) for the stored-vs-regenerated A/B"}
    else:
        k5_info = {"kernel": "k_wmean_partial (K5a)", "bound": "hbm",
                   "achieved_gbs": k5_read / (kms[3] * 1e-3) / 1e9 if kms[3] > 0 else None,
                   "peak_gbs": _hbm_peak(), "frac": (k5_read / (kms[3] * 1e-3) / 1e9) / _hbm_peak() if kms[3] > 0 else None,
                   "bytes_moved_per_launch": k5_read, "samples_with_weight": k5_nz, "samples": Ml,
                   "algorithmic_bytes_per_launch": k5_alg,
                   "note": "bytes moved = z rows of samples with non-zero fp32 weight + weights + chunk partials; "
                           "rows of zero-weight samples are skipped, so the algorithmic all-rows count over-states the rate"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded scenario generators, Philox noise)", "config": config_json(rc, world),
        "roofline": {"kernel": K23_KERNELS.get(g.last_fit_kernel(), "k_rollout_fitness") + " (K2+K3)", "bound": "fp32", "achieved": achieved, "peak": peak_tf.value,
                     "unit": "TFLOP/s", "frac": achieved / peak_tf.value if peak_tf.value else None,
                     "traffic": traffic, "traffic_source": traffic_src, "flops_per_eval": F, "evals_per_launch": Ml,
                     "launch_ms": k23_ms, "ncu": _ncu_summary(rc.name),
                     "peak_source": "measured live: d4orm_cuda_fp32_peak (FFMA2 over all SMs); MEASURED_PEAKS.json has no FP32 figure",
                     "note": "achieved = SURVEY 8d algorithmic FLOPs (every unordered pair and robot-obstacle test counted) / "
                             "launch time — frac can exceed 1: it is not a hardware utilisation; "
                             "launch time; the kernel culls tests exactly, so the executed FMA-pipe utilisation is lower "
                             "(the `ncu` key: the committed ncu --set full capture of this kernel)"},
        "kernel_ms": {"K1_philox": None, "K2K3_rollout_fitness": kms[1], "K4_weights": kms[2],
                      "K5_wmean_partial": kms[3], "K5_tree_update": kms[4],
                      "note": "K1 (Philox + Box-Muller) is fused into K2+K3 on the fp32 path: the noise is drawn in "
                              "registers there (and regenerated by K5a where k5.kernel says k_wmean_regen)"},
        "k5": k5_info,
        "gpu_launches": args.steps * g.launches_per_step(),
        "clocks": clk.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if solve:
        line["solve"] = solve
    if world == 1 and args.config == 5 and not args.no_configs:
        line["configs"] = other_configs(d4, local_rank, args)
    if world == 1 and not args.no_f64:
        line["f64"] = f64_throughput(d4, rc, local_rank)
    if rank == 0 and world == 1 and not args.no_cpu:
        ref, kind, what = reference_checker()
        batch, t = size_cpu_sample(ref, p, M, 2.0)
        reps = max(1, int(math.ceil(4.0 / max(t, 1e-3))))
        tt = sum(cpu_reference_step(ref, p, batch, 300 + j) for j in range(min(reps, 5)))
        n = min(reps, 5)
        line["cpu_baseline"] = {"value": batch * n / tt, "unit": UNIT, "cores": os.cpu_count(), "kind": kind,
                                "sample": f"{n} denoising step(s) x {batch} of {M} samples ({what}), all host threads"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    g.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def other_configs(d4, device: int, args) -> dict:
    """BASELINE's second metric, denoise-step latency, on C1-C4 (full shapes,
    fp32, Philox, CUDA graphs), measured in this run like the headline: W
    warm-up steps, then K steps timed with CUDA events on the context stream."""
    from paper_2503_12204_b200 import scenarios as S
    out = {}
    for ci in (1, 2, 3, 4):
        rc = S.baseline_config(ci)
        p = rc.problem
        g = d4.GpuDenoiser(p, device=device, precision=d4.PREC_F32, noise=d4.NOISE_PHILOX, graphs=True)
        cfg = d4.DenoiserConfig(steps=rc.steps, batch=rc.samples, lam=rc.lam, alpha_bar_final=rc.alpha_bar_final,
                                seed=rc.seed)
        base = np.zeros((p.horizon, p.robots, p.du))
        ms, kms = g.bench_steps(base, cfg, args.warmup, args.steps, kernels=True)
        F = algorithmic_flops_per_eval(p)
        out[f"C{ci}"] = {"workload": rc.name, "ms_per_step": ms / args.steps,
                         "value": rc.samples * args.steps / (ms / 1e3), "unit": UNIT,
                         "k23_ms": kms[1], "k4_ms": kms[2], "k5a_ms": kms[3], "k5b_ms": kms[4],
                         "k23_tflops": rc.samples * F / (kms[1] * 1e-3) / 1e12,
                         "gpu_launches_per_step": g.launches_per_step()}
        g.close()
    return out


def f64_throughput(d4, rc, device: int) -> dict:
    """The same workload in the fp64 parity instantiation (the reference's
    arithmetic: separately rounded mul/add, no FMA contraction, the reference's
    loop/break order in the fitness), W = 3 warm-up + 2 timed steps: the speed-up
    at the reference's own precision."""
    p = rc.problem
    g = d4.GpuDenoiser(p, device=device, precision=d4.PREC_F64, noise=d4.NOISE_PHILOX, graphs=True)
    cfg = d4.DenoiserConfig(steps=rc.steps, batch=rc.samples, lam=rc.lam, alpha_bar_final=rc.alpha_bar_final,
                            seed=rc.seed)
    steps = 2
    ms, _ = g.bench_steps(np.zeros((p.horizon, p.robots, p.du)), cfg, 3, steps, kernels=False)
    g.close()
    return {"value": rc.samples * steps / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
            "warmup": 3, "dtype": "f64",
            "note": "fp64 parity instantiation (PREC_F64: z stored and read, no culling, reference loop order)"}


# d4orm_cuda_last_fit_kernel: which K2+K3 kernel the captured step launches
K23_KERNELS = {0: "k_rollout_fitness", 1: "k_rollout_fitness_seg", 2: "k_rollout_fitness_pl32",
               3: "k_rollout_fitness_small"}


def _ncu_summary(name: str):
    """Hardware counters of K2+K3 from this round's committed `ncu --set full`
    capture (profiles/ncu_summary.json): FMA-pipe and issue utilisation beside
    the algorithmic fraction (the kernel culls pair tests exactly, so executed
    FMA work is below the algorithmic count)."""
    f = ROOT / "profiles" / "ncu_summary.json"
    try:
        return json.loads(f.read_text()).get(name)
    except Exception:
        return None


def _hbm_peak():
    f = ROOT / "MEASURED_PEAKS.json"
    try:
        return json.loads(f.read_text())["hbm_gbs"]
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


if __name__ == "__main__":
    main()
