"""Build libvks.so (the C-ABI library) in-tree with nvcc for sm_100a.

Every translation unit is compiled with `-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`.
project.cu, binning.cu and validate.cu additionally use `-fmad=false`: their fp32 operation order is pinned
 so projection outputs, tile rects and keys are bit-exact with the oracle.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libvks.so")
BUILD_DIR = os.path.join(ROOT, "build", "vks")
# debug build: the same sources with -DVKS_DEBUG_CHECKS (device bounds / invariant checks that trap;
# the stand-in for compute-sanitizer, which the GPU pool does not run), loaded when
# VKS_DEBUG_CHECKS=1 is set in the environment (paper_2605_00219_b200/_vks.py)
LIB_DEBUG = os.path.join(HERE, "libvks_debug.so")
BUILD_DIR_DEBUG = os.path.join(ROOT, "build", "vks_debug")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
          "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
PINNED = {"project.cu", "binning.cu", "validate.cu"}
SOURCES = ["project.cu", "project_bwd.cu", "binning.cu", "raster.cu", "adam.cu", "loss.cu", "mcmc.cu", "densify.cu", "validate.cu", "api.cu"]
HEADERS = ["vks_common.cuh", "vks_sh.cuh"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False, debug: bool = False) -> str:
    build_dir, lib = (BUILD_DIR_DEBUG, LIB_DEBUG) if debug else (BUILD_DIR, LIB)
    os.makedirs(build_dir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "vks.h"), __file__]
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [path] + hdrs):
            cmd = [nvcc(), *ARCH, *COMMON, *os.environ.get("VKS_NVCC_EXTRA", "").split(), "-c", path, "-o", obj]
            if debug:
                cmd.insert(1, "-DVKS_DEBUG_CHECKS")
            if src in PINNED:
                cmd.insert(1, "-fmad=false")
            if ptxas_v:
                cmd += ["-Xptxas", "-v"]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.check_call(cmd)
    if force or _stale(lib, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", lib, *objs, "-cudart", "static"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_v="-v" in sys.argv, debug="--debug" in sys.argv)
