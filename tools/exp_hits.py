import sys
sys.path.insert(0,'.')
import numpy as np
import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
rc = S.baseline_config(5); p = rc.problem
g = d4.GpuDenoiser(p)
cfg = d4.DenoiserConfig(steps=rc.steps, batch=4096, seed=0)
base = np.zeros((p.horizon, p.robots, p.du))
sched = d4.make_schedule(rc.steps, cfg.alpha_bar_final) if hasattr(cfg,'alpha_bar_final') else None
v, tr = g.run_denoising(base, cfg)
# early step: var = 0, sd = sqrt(1-ab[N])... use sd=1 approx; late: var = v (final), small sd
for label, var, sd in (("early", np.zeros_like(base), 1.0), ("mid", 0.5*v, 0.5), ("late", v, 0.1)):
    z = g.philox_noise(0, 50, 0, 64).reshape(64, p.horizon, p.robots, p.du).astype(np.float64)
    u = np.clip(var[None] + sd*z, -1, 1)
    st, ct, rw, cnt = g.rollout_fitness(u, want_states=True)
    # per (sample, 32-step window): any conflict robot-step?
    print(label, "mean nconf", cnt[:,0].mean(), "mean nobs", cnt[:,1].mean(), "of", p.robots*p.horizon)
