"""Build the native library libxrt.so in-tree (sm_100a only).

    python -m paper_2006_00686_b200.build [--force] [--verbose]

nvcc compiles every csrc/*.cu for ``-gencode arch=compute_100a,code=sm_100a`` with
``-lineinfo`` (so ncu's source page maps to the code) and links one shared library with
a static CUDA runtime.  The .so is git-ignored but travels to the GPU box with gpurun.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libxrt.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-Xptxas", "-v" if os.environ.get("XRT_PTXAS_VERBOSE") else "-O3", "-cudart", "static"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(INCLUDE, "xrt.h")]


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(f) > t for f in deps())


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libxrt.so (``out`` / ``defines`` for A/B experiment builds)."""
    global OUT
    target = out or OUT
    if out is None and not force and not stale():
        return OUT
    objs = []
    bdir = os.path.join(HERE, "build")
    os.makedirs(bdir, exist_ok=True)
    for src in sources():
        tag = ("." + "_".join(d.replace("=", "") for d in defines)) if defines else ""
        obj = os.path.join(bdir, os.path.basename(src) + tag + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = target + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
