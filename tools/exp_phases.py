"""Experiment: split K2+K3 time into rollout (phase A) and fitness (phase B) shares."""
import sys, json
sys.path.insert(0, '.')
import numpy as np
import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
from dataclasses import replace
rc = S.baseline_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
for label, p in [("full", rc.problem), ("no-obstacles", replace(rc.problem, obs_centers=np.zeros((0, 2)), obs_radii=np.zeros(0)))]:
    g = d4.GpuDenoiser(p)
    cfg = d4.DenoiserConfig(steps=rc.steps, batch=rc.samples, seed=0)
    ms, k = g.bench_steps(np.zeros((p.horizon, p.robots, p.du)), cfg, 3, 5)
    print(label, "K23 ms", round(k[1], 3), "step ms", round(ms / 5, 3))
    g.close()
