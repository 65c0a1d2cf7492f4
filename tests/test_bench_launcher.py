"""bench.py's multi-GPU launch contract, checked on CPU with --dry-run (every
rank reports rank / world / device and exits before any GPU work):

  * `bench.py --gpus N` without WORLD_SIZE self-launches N ranks through
    torch.distributed.run on 127.0.0.1 (the driver's own launch for N > 1);
  * under a launcher, WORLD_SIZE must equal --gpus (else exit 2, so a run can
    never silently measure fewer GPUs than asked);
  * the reference arm follows the same launch.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(args, env=None, timeout=300):
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True, env=e,
                          timeout=timeout, cwd=ROOT)


def _ranks(out):
    return sorted((json.loads(l) for l in out.splitlines() if l.startswith("{")), key=lambda d: d["rank"])


@pytest.mark.parametrize("n", [1, 2, 4])
def test_self_launch_starts_n_ranks(n):
    r = _run(["--gpus", str(n), "--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    ranks = _ranks(r.stdout)
    assert [d["rank"] for d in ranks] == list(range(n))
    assert all(d["world"] == n for d in ranks)
    assert [d["device"] for d in ranks] == [f"cuda:{i}" for i in range(n)]
    if n > 1:
        assert "self-launching" in r.stderr and all(d["master"].startswith("127.0.0.1:") for d in ranks)


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "2", "--dry-run"], env={"WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=3 but --gpus 2" in r.stderr
    r = _run(["--dry-run"], env={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert r.returncode == 2


def test_reference_arm_launch():
    r = _run(["--impl", "reference", "--gpus", "2", "--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    ranks = _ranks(r.stdout)
    assert len(ranks) == 2 and all(d["impl"] == "reference" for d in ranks)
