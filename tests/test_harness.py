"""The C++ drop-in's trial harness and I/O (include/d4orm/{bench,io}.hpp,
scenario JSON v1) against the reference's own bench.cpp / scenario.cpp
(compiled unchanged into oracle/_ref).  Host part runs on CPU; the batching
and solve-output part needs the GPU."""
import ctypes as C
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2503_12204_b200"


def _json_dir():
    import sys
    for sp in sys.path:
        d = Path(sp) / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"
        if (d / "json.hpp").exists():
            return d
    pytest.skip("json.hpp not available")


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    if not (PKG / "libd4orm_b200.so").exists():
        pytest.skip("libd4orm_b200.so not built")
    exe = tmp_path_factory.mktemp("cpp") / "test_harness"
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{ROOT / 'include'}", f"-I{_json_dir()}",
                    str(ROOT / "tests/cpp/test_harness.cpp"), f"-L{PKG}", "-ld4orm_b200", f"-Wl,-rpath,{PKG}",
                    "-o", str(exe)], check=True)
    return exe


def _run(exe, mode, d):
    out = subprocess.run([str(exe), mode, str(d)], check=True, capture_output=True, text=True).stdout
    return json.loads(out)


def _ref_lib():
    from oracle.oracle import REF_SO
    if not REF_SO.exists():
        pytest.skip("oracle/_ref not built")
    L = C.CDLL(str(REF_SO))
    L.ref_last_error.restype = C.c_char_p
    return L


def test_trial_csv_and_aggregate_match_reference(harness, tmp_path):
    got = _run(harness, "host", tmp_path)
    L = _ref_lib()
    paths = got["csv_paths"]
    arr = (C.c_char_p * len(paths))(*[p.encode() for p in paths])
    buf = C.create_string_buffer(1 << 20)
    assert L.ref_aggregate_csv(arr, len(paths), buf, len(buf)) == 0, L.ref_last_error()
    assert got["aggregate"] == json.loads(buf.value.decode())
    # the CSV text itself: the reference re-writes what it read, byte for byte
    for p in paths:
        q = p + ".ref"
        assert L.ref_csv_roundtrip(p.encode(), q.encode()) == 0
        assert Path(p).read_bytes() == Path(q).read_bytes()


def test_scenario_json_matches_reference(harness, tmp_path):
    got = _run(harness, "host", tmp_path)
    L = _ref_lib()
    buf = C.create_string_buffer(1 << 16)
    assert L.ref_antipodal_circle_json(4, C.c_double(6.0), 1, buf, len(buf)) == 0
    assert json.loads(got["circle_json"]) == json.loads(buf.value.decode())
    # the reference parses and re-writes ours identically (native kind)
    assert L.ref_scenario_json_roundtrip(got["circle_json"].encode(), buf, len(buf)) == 0
    assert json.loads(buf.value.decode()) == json.loads(got["circle_json"])
    assert got["c3_roundtrip_equal"] and got["c5_roundtrip_equal"]  # extension kinds round-trip
    assert got["bad_schema"] == "scenario json: unsupported schema_version"


@pytest.mark.gpu
def test_run_trials_batch_and_solve_outputs(harness, tmp_path):
    got = _run(harness, "gpu", tmp_path)
    assert got["batch_errors"] == ""
    assert got["batch_identical"], "concurrent trials must equal one-at-a-time trials"
    assert got["iterations"] == 3
    assert got["replay_success"] and got["replay_objective"] and got["replay_reward"]
    head = (tmp_path / "denoise_trace.csv").read_text().splitlines()
    assert head[0] == "iteration,step,best_sample_reward,mean_sample_reward,weight_entropy"
    assert len(head) == 1 + 2 * 10
    doc = json.loads((tmp_path / "trajectory.json").read_text())
    assert doc["schema_version"] == 1 and doc["config"]["solver.name"] == "d4orm"
    print("run_trials: sequential %.3f s, 8 concurrent %.3f s" % (got["seq_s"], got["par_s"]))
