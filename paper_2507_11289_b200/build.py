"""Build libdsea.so in-tree: nvcc for the sm_100a kernels, g++ for the host runtime
(-ffp-contract=off so the host lattice/velocity generator is bit-reproducible).

Usage: python -m paper_2507_11289_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libdsea.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES_CU = ["dsea_kernels.cu", "dsea_force.cu", "dsea_grid_kernels.cu"]
SOURCES_CPP = ["dsea_host.cpp", "dsea_grid.cpp"]
HEADERS = ["dsea_internal.h", "dsea_device.cuh", "dsea_plan.h", os.path.join("..", "..", "include", "dsea.h"),
           os.path.join("..", "..", "include", "dsea_grid.h")]


def _nccl_include() -> str:
    cands = [os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl", "include"),
             "/usr/include"]
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stdout.write(r.stdout)
        sys.stderr.write(r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}")


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.abspath(__file__)]
    objs = []
    for src in SOURCES_CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs):
            _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xptxas", "-v", "-fmad=true",
                  *os.environ.get("DSEA_NVCC_EXTRA", "").split(),   # -D sweeps (use --force)
                  "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o], verbose)
        objs.append(o)
    for src in SOURCES_CPP:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs):
            _run(["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
                  "-Wall", "-Wno-unused-function",
                  "-I", os.path.join(CUDA_HOME, "include"), "-I", _nccl_include(),
                  "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o], verbose)
        objs.append(o)
    if force or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-ldl", "-lpthread",
              "-lrt"], verbose)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
