"""CPU: the C-ABI library loads without a GPU and exports every symbol
include/d4orm_cuda.h declares; the C++ drop-in symbols are present too."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2503_12204_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def _declared(header):
    text = (ROOT / "include" / header).read_text()
    return sorted(set(re.findall(r"\b(d4orm_cuda_\w+)\s*\(", text)))


def test_header_declarations_match_binding():
    assert set(_declared("d4orm_cuda.h")) == set(_lib.EXPORTS)


def test_library_exports_all_symbols():
    if not _lib.LIB_PATH.exists():
        from paper_2503_12204_b200 import build
        build.build()
    L = C.CDLL(str(_lib.LIB_PATH))
    for name in _declared("d4orm_cuda.h") + _declared("d4orm_cuda_bench.h"):
        assert hasattr(L, name), name
    assert L.d4orm_cuda_version
    syms = subprocess.run(["nm", "-DC", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    for fn in ("d4orm::run_denoising(", "d4orm::solve(", "d4orm::iterate(", "d4orm::rollout(", "d4orm::batch_rollout(",
               "d4orm::score_weights(", "d4orm::make_schedule(", "d4orm::validate_scenario(", "d4orm::antipodal_circle(",
               "d4orm::total_reward(", "d4orm::check_success(", "d4orm::mppi_solve(", "d4orm::cem_solve(",
               "d4orm::select_elites("):
        assert fn in syms, fn


def test_no_gpu_fails_loudly():
    """Without a GPU the product path raises; it never computes on the CPU."""
    import paper_2503_12204_b200 as d4
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is visible")
    except ImportError:
        pass
    with pytest.raises(d4.D4ormError):
        d4.GpuDenoiser()
