"""In-tree build of the sm_100a library ``libd4orm_b200.so`` (and the oracle).

Compiles every ``csrc/*.cu`` and ``csrc/*.cpp`` with nvcc for
``-gencode arch=compute_100a,code=sm_100a`` in parallel, links one shared
object next to this file, and (when asked) builds the test-only oracle via
``oracle/Makefile``.  No PyTorch extension machinery: the product boundary is
the C-ABI in ``include/d4orm_cuda.h``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB = PKG / "libd4orm_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
def _json_dir() -> list[str]:
    """nlohmann json.hpp (header-only, shipped in the image's cudnn_frontend
    package) for the scenario / trajectory / trial I/O of the C++ drop-in — the
    same single header the reference vendors (proj/CMakeLists.txt:5)."""
    for sp in sys.path:
        d = Path(sp) / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"
        if (d / "json.hpp").exists():
            return [f"-I{d}"]
    return []


NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              f"-I{ROOT / 'include'}", f"-I{CSRC}", *_json_dir()]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def _newer(src: Path, obj: Path, deps: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, jobs: int | None = None, defines: tuple[str, ...] = (),
          out: Path | None = None) -> Path:
    """Build the library.  ``defines``/``out`` produce experiment variants
    (``-D`` flags, separate object dir and output .so) for tools/."""
    nvcc = _nvcc()
    obj_dir = OBJ if not defines else OBJ.parent / ("build_" + "_".join(d.lower().replace("=", "") for d in defines))
    lib = out or LIB
    obj_dir.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list((ROOT / "include").rglob("*.h*"))
    srcs = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    cmds = []
    objs = []
    for s in srcs:
        o = obj_dir / (s.name + ".o")
        objs.append(o)
        if _newer(s, o, headers):
            cmds.append([nvcc, *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", str(s), "-o", str(o)])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"compile failed: {cmd[-3]}")
        return r

    with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        list(ex.map(run, cmds))
    if cmds or not lib.exists():
        run([nvcc, *ARCH, "-shared", "-o", str(lib), *map(str, objs), "-ldl", "-lcudart"])
    return lib


CHECKED_LIB = PKG / "libd4orm_b200_checked.so"


def build_checked(verbose: bool = False) -> Path:
    """The same library with the device-side bounds checks on (-DD4K_CHECKED,
    d4orm_common.cuh): test infrastructure for tests/test_gpu_checked.py."""
    return build(verbose=verbose, defines=("D4K_CHECKED",), out=CHECKED_LIB)


def build_oracle() -> None:
    """Test-only checker: oracle/build/libd4orm_oracle.so and, where
    /root/reference exists, oracle/_ref/libd4orm_ref.so."""
    subprocess.run(["make", "-s", "-f", str(ROOT / "oracle" / "Makefile")], check=True)


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(verbose="-v" in sys.argv, defines=defs, out=Path(outs[0]) if outs else None))
    if "--oracle" in sys.argv:
        build_oracle()
