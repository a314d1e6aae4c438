"""Build the sm_100a extension in-tree: paper_2512_16134_b200/lib/libsbs_b200.so.

nvcc cross-compiles without a GPU.  Device code is built with -fmad=false so
no FMA contraction can change an FP64 timestamp expression, host code with
-ffp-contract=off for the same reason ("bit-exactness").
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
PROF = os.environ.get("SBS_PROF") == "1"   # development: clock64 region counters
CHECK = os.environ.get("SBS_CHECK") == "1"  # development: device bounds checks (trap)
LIB = LIB_DIR / ("libsbs_b200_prof.so" if PROF else "libsbs_b200_check.so" if CHECK else "libsbs_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["des.cu", "alloc.cu", "gen.cu"]
CPP_SOURCES = ["sbs_host.cpp"]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + [PKG.parent / "include" / "sbs_b200.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    obj_dir = LIB_DIR / ("obj_prof" if PROF else "obj_check" if CHECK else "obj")
    obj_dir.mkdir(exist_ok=True)
    objs = []
    common = ["-O3", "-std=c++17", "-lineinfo", f"-I{PKG.parent / 'include'}"]
    for src in CU_SOURCES:
        obj = obj_dir / (src + ".o")
        cmd = [NVCC, *ARCH, *common, *(["-DSBS_PROF"] if PROF else []), *(["-DSBS_CHECK"] if CHECK else []),
               "-fmad=false", "-Xptxas", "-v", "-Xcompiler",
               "-fPIC,-ffp-contract=off", "-c", str(CSRC / src), "-o", str(obj)]
        _run(cmd, verbose)
        objs.append(obj)
    for src in CPP_SOURCES:
        obj = obj_dir / (src + ".o")
        cmd = [NVCC, *common, "-x", "cu", *ARCH, "-fmad=false", "-Xcompiler",
               "-fPIC,-ffp-contract=off,-Wall", "-c", str(CSRC / src), "-o", str(obj)]
        _run(cmd, verbose)
        objs.append(obj)
    tmp = LIB.with_suffix(".so.tmp")
    _run([NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lpthread"], verbose)
    os.replace(tmp, LIB)
    return LIB


def _run(cmd, verbose):
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = LIB_DIR / "build.log"
    with open(log, "a") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr + "\n")
    if verbose or r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd[:4])} ... (see {log})")


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
