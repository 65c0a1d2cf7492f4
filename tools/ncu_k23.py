"""One denoising step of a BASELINE config (default C5), for ncu captures of K2+K3."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
rc = S.baseline_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
p = rc.problem
g = d4.GpuDenoiser(p)
g.set_options(graphs=False)
cfg = d4.DenoiserConfig(steps=rc.steps, batch=rc.samples, seed=0)
g.bench_steps(np.zeros((p.horizon, p.robots, p.du)), cfg, 2, 1, kernels=False)  # 3 launches: profile with -s 2 -c 1
g.close()
print("done")
