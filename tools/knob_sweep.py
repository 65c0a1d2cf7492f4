"""K2+K3 time of BASELINE configs under the tuning knobs (each setting in a fresh
process): python tools/knob_sweep.py CONFIG 'ENV=V,ENV2=V2' ...  ('' = default)."""
import os, subprocess, sys

CHILD = r'''
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
rc = S.baseline_config(int(sys.argv[1]))
p = rc.problem
g = d4.GpuDenoiser(p)
import os as _os
cfg = d4.DenoiserConfig(steps=rc.steps, batch=int(_os.environ.get("KS_BATCH", rc.samples)), seed=0)
import os
reps, n = int(os.environ.get("KS_REPS", "3")), int(os.environ.get("KS_STEPS", "10"))
best, steps = None, []
for _ in range(reps):
    ms, k = g.bench_steps(np.zeros((p.horizon, p.robots, p.du)), cfg, 3, n)
    steps.append(ms / n)
    best = (ms / n, k) if best is None or k[1] < best[1][1] else best
print("step %.4f ms (min %.4f median %.4f)  K23 %.4f ms  K5a %.4f ms  K4 %.4f ms" % (
    best[0], min(steps), sorted(steps)[len(steps) // 2], best[1][1], best[1][3], best[1][2]))
'''
cfg = sys.argv[1]
for spec in sys.argv[2:]:
    env = dict(os.environ)
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        env[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD, cfg], env=env, capture_output=True, text=True)
    print(f"C{cfg} {spec or 'default':40s} {r.stdout.strip()} {r.stderr.strip()[-300:] if r.returncode else ''}", flush=True)
