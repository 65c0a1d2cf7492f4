import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a library)")
    config.addinivalue_line("markers", "slow: longer parity runs")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle, ORACLE_SO
    if not ORACLE_SO.exists():
        import subprocess
        subprocess.run(["make", "-s", "-f", str(ROOT / "oracle" / "Makefile"), str(ORACLE_SO)], check=True)
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, REF_SO
    if not REF_SO.exists():
        pytest.skip("oracle/_ref/libd4orm_ref.so not built (needs /root/reference at build time)")
    return Reference()
