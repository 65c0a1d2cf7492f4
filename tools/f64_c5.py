"""fp64 (parity instantiation: the reference's arithmetic, no FMA contraction)
throughput of the C5 step, for the bench's `f64` key: python tools/f64_c5.py [steps] [samples]"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rc = S.baseline_config(5)
p = rc.problem
M = int(sys.argv[2]) if len(sys.argv) > 2 else rc.samples
g = d4.GpuDenoiser(p, precision=d4.PREC_F64, noise=d4.NOISE_PHILOX)
cfg = d4.DenoiserConfig(steps=rc.steps, batch=M, seed=0)
t = time.time()
ms, kms = g.bench_steps(np.zeros((p.horizon, p.robots, p.du)), cfg, 3, steps)
print(f"f64 C5 M={M}: {ms / steps:.2f} ms/step, {M * steps / (ms / 1e3) / 1e6:.3f} M evals/s, kernels {kms}, wall {time.time() - t:.1f}s")
