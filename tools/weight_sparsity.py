"""Fraction of samples whose fp32 weight survives the 2^-48 floor, per denoising
step of a full run (BASELINE config, Philox, fp32) — how much of z K5 reads."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S

rc = S.baseline_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
p = rc.problem
g = d4.GpuDenoiser(p)
cfg = d4.DenoiserConfig(steps=rc.steps, batch=rc.samples, seed=0)
ab = d4.make_schedule(cfg.steps, cfg.alpha_bar_final)
base = np.zeros((p.horizon, p.robots, p.du))
var = np.zeros_like(base)
fr, fa = [], {30: [], 40: []}
for i in range(cfg.steps, 0, -1):
    var, r, w, rec = g.denoise_step(base, var, i, cfg, None)
    fr.append(float(np.mean(w >= w.max() * 2.0 ** -48)))
    # adaptive alternative: drop the smallest weights whose total is <= 2^-b of the sum
    cs = np.cumsum(np.sort(w))
    for b in fa:
        fa[b].append(1.0 - np.searchsorted(cs, cs[-1] * 2.0 ** -b, side="right") / len(w))
print("significant fraction per step (i = N..1), floor 2^-48 of the max:")
print(" ".join("%.3f" % f for f in fr))
print("mean %.3f  min %.3f  max %.3f" % (np.mean(fr), np.min(fr), np.max(fr)))
for b, v in fa.items():
    print("adaptive (dropped mass <= 2^-%d of the sum): mean %.3f  min %.3f  max %.3f" % (b, np.mean(v), np.min(v), np.max(v)))
