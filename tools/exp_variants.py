"""Experiment: K2+K3 time of library variants (built by tools/build_variants.sh).

Usage: python tools/exp_variants.py CONFIG lib1.so lib2.so ...  (each lib in a
fresh process via D4ORM_LIB)."""
import os, subprocess, sys

CHILD = r'''
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
rc = S.baseline_config(int(sys.argv[1]))
p = rc.problem
g = d4.GpuDenoiser(p)
cfg = d4.DenoiserConfig(steps=rc.steps, batch=rc.samples, seed=0)
best = None
for _ in range(3):
    ms, k = g.bench_steps(np.zeros((p.horizon, p.robots, p.du)), cfg, 3, 10)
    best = k if best is None or k[1] < best[1] else best
print("K23 %.4f ms  K5p %.4f ms  K4 %.4f ms" % (best[1], best[3], best[2]))
'''

cfg = sys.argv[1]
for lib in sys.argv[2:]:
    env = dict(os.environ, D4ORM_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", CHILD, cfg], env=env, capture_output=True, text=True)
    print(f"C{cfg} {os.path.basename(lib):40s} {r.stdout.strip()} {r.stderr.strip()[-300:] if r.returncode else ''}", flush=True)
