"""Projected C5 strong scaling (G = 1, 2, 4, 8 ranks), from measurements on ONE
B200 (this pool has one GPU per call, so the NCCL path cannot be timed here).

A rank of G owns M/G contiguous samples; its step is K2+K3 + K5a on M/G samples,
K4 on all M rewards (replicated after the reward all-gather), K5b over its M/G/256
chunk partials plus the root tree, and two all-gathers.  This tool times a
single-GPU run of M/G samples (bench_steps: K steps, CUDA events), replaces its
K4 by the full-M K4 measured in the G = 1 run, and adds an all-gather
allowance (ALLGATHER_US per exchange, NVLink 5 latency-bound messages of 2 MB and
G x 128 KB).  Prints one JSON line per G.  A projection, not a measurement."""
import json
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S

ALLGATHER_US = 20.0
rc = S.baseline_config(5)
p = rc.problem
base = np.zeros((p.horizon, p.robots, p.du))
k4_full = None
for G in (1, 2, 4, 8):
    M = rc.samples // G
    g = d4.GpuDenoiser(p)
    cfg = d4.DenoiserConfig(steps=rc.steps, batch=M, seed=rc.seed)
    ms, k = g.bench_steps(base, cfg, 3, 20, kernels=True)
    g.close()
    step = ms / 20
    if G == 1:
        k4_full = k[2]
    proj = step - k[2] + k4_full + (2 * ALLGATHER_US / 1e3 if G > 1 else 0.0)
    print(json.dumps({"G": G, "samples_per_rank": M, "local_step_ms": step, "k23_ms": k[1], "k5a_ms": k[3],
                      "k4_local_ms": k[2], "k4_full_ms": k4_full, "projected_step_ms": proj,
                      "projected_evals_per_s": rc.samples / (proj / 1e3)}), flush=True)
