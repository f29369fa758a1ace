"""In-tree build of libdbag.so (CUDA kernels + C-ABI + host scene generator)
for sm_100a only. The .so lands next to this file so it travels to the GPU box
with the repo snapshot."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdbag.so")
# (source, extra flags): the exact-numerics TU must not contract a*b+c into
# FMA — it is a bit-for-bit twin of the oracle's arithmetic.
NCCL_HOME = None
for _p in sys.path + [os.path.join(sys.prefix, "lib", "python3.12", "site-packages")]:
    _c = os.path.join(_p, "nvidia", "nccl")
    if os.path.exists(os.path.join(_c, "include", "nccl.h")):
        NCCL_HOME = _c
        break
NCCL_INC = ["-I", os.path.join(NCCL_HOME, "include")] if NCCL_HOME else []
SOURCES = [("dbag_capi.cu", NCCL_INC), ("dbag_exact.cu", ["-fmad=false"]),
           ("dbag_blocks.cu", ["-fmad=false"]), ("dbag_metrics.cu", ["-fmad=false"]),
           ("dbag_lm.cu", ["-fmad=false"]),
           ("dbag_scenes.cpp", []), ("dbag_shard.cpp", []), ("dbag_io.cpp", [])]
HEADERS = ["dbag_common.cuh", "dbag_local.cuh", "dbag_lbfgs.cuh", "dbag_consensus.cuh",
           "dbag_index.cuh", "dbag_exact.h", "dbag_shard.h", "dbag_exact_geom.cuh", "dbag_blocks.h",
           "dbag_metrics.h", "dbag_errors.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; cannot build libdbag.so")
    return cand


def _inputs():
    files = [os.path.join(CSRC, s) for s, _ in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
    files.append(os.path.join(HERE, "..", "include", "dbag.h"))
    files.append(os.path.abspath(__file__))
    return files


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _inputs() if os.path.exists(f))


def build(force=False, verbose=False, extra=(), only=None):
    """only: recompile just these sources (with `extra`) into a scratch object
    dir and link them with the main build's objects (variant A/B builds)."""
    if not force and up_to_date():
        return LIB
    objdir = os.path.join(HERE, "_obj")
    os.makedirs(objdir, exist_ok=True)
    vardir = os.path.join(HERE, "_obj_var")
    objs = []
    for src, flags in SOURCES:
        if only is not None and src not in only:
            objs.append(os.path.join(objdir, src + ".o"))
            continue
        if only is not None:
            os.makedirs(vardir, exist_ok=True)
        obj = os.path.join(vardir if only is not None else objdir, src + ".o")
        cmd = [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v" if verbose else "-O3", *flags, *extra, "-c",
               os.path.join(CSRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(res.stderr)
        objs.append(obj)
    if not NCCL_HOME:
        raise RuntimeError("NCCL headers/library (nvidia/nccl in site-packages) not found")
    ncclib = os.path.join(NCCL_HOME, "lib")
    cudalib = os.path.join(os.path.dirname(os.path.dirname(nvcc())), "lib64")
    cmd = [nvcc(), *ARCH, "-shared", *objs, "-o", LIB + ".tmp", "-L", ncclib, "-l:libnccl.so.2",
           "-Xlinker", "-rpath," + ncclib, "-L", cudalib, "-lcusolver", "-lcublas",
           "-Xlinker", "-rpath," + cudalib]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed for libdbag.so")
    os.replace(LIB + ".tmp", LIB)
    if os.path.dirname(LIB) == HERE:
        build_tools()
    return LIB


TOOL_SRC = os.path.join(HERE, "..", "tools", "dbag_solve.cpp")
TOOL_BIN = os.path.join(HERE, "dbag_solve")


def build_tools():
    """C++ host driver over include/dbag.hpp, linked against the in-tree lib."""
    cxx = shutil.which("g++") or "g++"
    cmd = [cxx, "-O2", "-std=c++17", "-I", os.path.join(HERE, "..", "include"), TOOL_SRC,
           "-o", TOOL_BIN, "-L", HERE, "-ldbag", "-Wl,-rpath,$ORIGIN"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("g++ failed building tools/dbag_solve.cpp against dbag.hpp")
    return TOOL_BIN


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
