"""The library built with its device-side bounds checks (-DD4K_CHECKED:
libd4orm_b200_checked.so) over the sanitizer workload (tools/sanitize.py) —
every kernel family, tiny shapes.  compute-sanitizer is not available on the
GPU pool (runs under it left GPUs needing a reset), so the repo carries its
own checks: shared-memory tile rows / robot columns, the pair-list window
boxes, K4's octave bins, K5a/K5 compaction slots, K5b's stack.  A failed check
prints "d4k check failed: file:line: condition" and traps.
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CHECKED = ROOT / "paper_2503_12204_b200" / "libd4orm_b200_checked.so"

pytestmark = pytest.mark.gpu


def test_checked_build_runs_the_sanitizer_workload_clean():
    if not CHECKED.exists():
        pytest.fail("libd4orm_b200_checked.so missing: run __graft_entry__.build()")
    env = dict(os.environ, D4ORM_LIB=str(CHECKED))
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize.py")], env=env, capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    assert "d4k check failed" not in out, out[-4000:]
    assert r.returncode == 0 and "sanitize workload done" in r.stdout, out[-4000:]


def test_checked_build_is_loaded_and_same_results():
    """The checked library is a different .so with the same arithmetic: one C5
    step (pair list, regenerating K5a) gives the same variable."""
    code = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S
from paper_2503_12204_b200._lib import LIB_PATH
p = S.baseline_config(5).problem.with_horizon(64)
g = d4.GpuDenoiser(p)
v, r, w, rec = g.denoise_step(np.zeros((64, 64, 2)), np.full((64, 64, 2), 0.1), 7, d4.DenoiserConfig(steps=10, batch=1024, seed=2))
np.save(sys.argv[2], v)
print(LIB_PATH)
'''
    outs = []
    for lib, tag in ((CHECKED, "chk"), (ROOT / "paper_2503_12204_b200" / "libd4orm_b200.so", "prod")):
        f = f"/tmp/d4_{tag}.npy"
        r = subprocess.run([sys.executable, "-c", code, str(ROOT), f], env=dict(os.environ, D4ORM_LIB=str(lib)),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        assert r.stdout.strip().endswith(lib.name)
        import numpy as np
        outs.append(np.load(f))
    import numpy as np
    np.testing.assert_allclose(outs[0], outs[1], rtol=1e-6, atol=1e-7)
