"""In-tree build of libdbsp_b200.so (host planner + sm_100a kernels + C ABI).

The host planner is compiled by g++ with -ffp-contract=off so every double
expression is evaluated exactly as written (bit-exact with the reference);
the CUDA sources are compiled by nvcc for sm_100a only.  The result lands next
to this file so it travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "dbsp_b200"
LIB = PKG / "libdbsp_b200.so"

CXX_SOURCES = ["planner_core.cpp", "schedule.cpp", "capi.cpp", "mask_io.cpp"]
CU_SOURCES = ["attention.cu", "schedule_device.cu", "planner_device.cu", "sp_exec.cu", "qkv_proj.cu"]
GENCODE = "-gencode=arch=compute_100a,code=sm_100a"


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libdbsp_b200.so")


def _run(cmd: list[str]) -> None:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd)}")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    """Compile (incrementally) and link libdbsp_b200.so; returns its path."""
    nvcc = _nvcc()
    BUILD.mkdir(parents=True, exist_ok=True)
    headers = sorted(CSRC.glob("*.hpp")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "dbsp_b200.h"]
    objs: list[Path] = []
    for src in CXX_SOURCES:
        obj = BUILD / (src + ".o")
        if force or _stale(obj, [CSRC / src] + headers):
            # -mpopcnt/-mbmi: hardware popcount/tzcnt for the mask walks (integer
            # only; no effect on any double, which -ffp-contract=off keeps exact)
            cmd = ["g++", "-std=c++20", "-O3", "-fPIC", "-ffp-contract=off", "-mpopcnt", "-mbmi",
                   "-mbmi2", "-mlzcnt", "-Wall", "-Wextra",
                   "-Wno-unused-parameter", f"-I{ROOT / 'include'}", "-c", str(CSRC / src), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd))
            _run(cmd)
        objs.append(obj)
    for src in CU_SOURCES:
        obj = BUILD / (src + ".o")
        if force or _stale(obj, [CSRC / src] + headers):
            extra = os.environ.get("DBSP_NVCC_FLAGS", "").split()
            cmd = [nvcc, GENCODE, "-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC",
                   *extra,
                   "-Xcompiler", "-ffp-contract=off", f"-I{ROOT / 'include'}", "-c", str(CSRC / src),
                   "-o", str(obj)]
            if verbose:
                print(" ".join(cmd))
            _run(cmd)
        objs.append(obj)
    if force or _stale(LIB, objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc, GENCODE, "-shared", "-o", str(tmp)] + [str(o) for o in objs] + ["-ldl", "-lcuda"]
        if verbose:
            print(" ".join(cmd))
        try:
            _run(cmd)
        except RuntimeError:
            # libcuda.so may be absent on a CPU-only build host; the driver
            # entry point is resolved through cudart at run time anyway.
            cmd = cmd[:-1]
            _run(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
