"""Per-step time across the denoising schedule (i = N..1) of a BASELINE config:
bench_steps(warmup=j, steps=1) times step i = N - j alone (CUDA events) and its
instrumented pass gives the kernel split and the samples K5a keeps."""
import json, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 5
stride = int(sys.argv[2]) if len(sys.argv) > 2 else 5
rc = S.baseline_config(ci)
p = rc.problem
g = d4.GpuDenoiser(p)
cfg = d4.DenoiserConfig(steps=rc.steps, batch=rc.samples, seed=rc.seed)
base = np.zeros((p.horizon, p.robots, p.du))
rows = []
for j in range(0, rc.steps, stride):
    ms, k = g.bench_steps(base, cfg, j, 1, kernels=True)
    rows.append({"i": rc.steps - j, "ms": ms, "k23": k[1], "k5a": k[3], "kept": k[5] / rc.samples})
    print(json.dumps(rows[-1]), flush=True)
print("mean step ms %.3f" % np.mean([r["ms"] for r in rows]))
