"""Build the in-tree sm_100a shared library ``_lib/libpcirc_b200.so``.

One nvcc invocation per translation unit, then a shared link; sources are
rebuilt only when newer than the library.  The library travels with the
repo snapshot to the GPU box (built files are git-ignored, not
gpurun-ignored).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libpcirc_b200.so"
SOURCES = ["pcb_simt.cu", "pcb_tc.cu", "pcb_tc_ws.cu", "pcb_tc_pf.cu", "pcb_capi.cu"]
HEADERS = ["pcb_internal.cuh", "pcb_tc.cuh", "pcb_ws.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build pcirc_b200")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "pcirc_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


HOST_SRC = CSRC / "host" / "pcc_compile.cpp"
HOST_LIB = OUT_DIR / "libpcirc_host.so"


def build_host(force: bool = False) -> Path:
    """The native host-compiler core (plain C++17, std::thread)."""
    deps = [HOST_SRC, PKG.parent / "include" / "pcirc_host.h"]
    if not force and HOST_LIB.exists() and all(HOST_LIB.stat().st_mtime >= d.stat().st_mtime
                                               for d in deps):
        return HOST_LIB
    OUT_DIR.mkdir(exist_ok=True)
    cxx = os.environ.get("CXX") or shutil.which("g++") or "g++"
    tmp = HOST_LIB.with_suffix(".so.tmp")
    cmd = [cxx, "-O3", "-std=c++17", "-fPIC", "-shared", "-Wall", "-o", str(tmp), str(HOST_SRC),
           "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("g++ failed on pcc_compile.cpp")
    os.replace(tmp, HOST_LIB)
    return HOST_LIB


def build(force: bool = False, verbose: bool = False) -> Path:
    build_host(force)
    if not force and not _stale():
        return LIB
    OUT_DIR.mkdir(exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = OUT_DIR / (Path(src).stem + ".o")
        cmd = [nvcc(), *ARCH, *FLAGS, "-c", str(CSRC / src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(res.stderr)
        (OUT_DIR / (Path(src).stem + ".ptxas.txt")).write_text(res.stderr)
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
