"""In-tree build of libqcsim_b200.so (sm_100a) and the C++ API shim.

    python -m paper_1811_05630_b200.build

nvcc cross-compiles without a GPU; the resulting .so files travel with the
repository snapshot to the GPU box (they are git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                  "-Xptxas", "-warn-spills"]

LIB = os.path.join(HERE, "libqcsim_b200.so")
SOURCES = ["qcsim_b200.cu"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith(".cuh"))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


API_LIB = os.path.join(HERE, "libqcsim.so")           # C++ API shim (include/qcsim/*.hpp)
API_SRC = os.path.join(CSRC, "host", "qcsim_api.cpp")
API_SMOKE_SRC = os.path.join(ROOT, "tests", "cpp", "api_smoke.cpp")
API_SMOKE = os.path.join(ROOT, "tests", "cpp", "api_smoke")
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include")]


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build(force: bool = False, verbose: bool = True) -> str:
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "qcsim_c.h")]
    if force or _stale(LIB, deps):
        _run([NVCC] + NVFLAGS + ["-shared", "-o", LIB] + [os.path.join(CSRC, f) for f in SOURCES], verbose)
    hdrs = [os.path.join(ROOT, "include", "qcsim", h) for h in os.listdir(os.path.join(ROOT, "include", "qcsim"))]
    if force or _stale(API_LIB, [API_SRC, LIB] + hdrs):
        _run(["g++"] + CXXFLAGS + ["-shared", "-o", API_LIB, API_SRC, "-L" + HERE, "-lqcsim_b200",
                                   "-Wl,-rpath,$ORIGIN"], verbose)
    if force or _stale(API_SMOKE, [API_SMOKE_SRC, API_LIB] + hdrs):
        _run(["g++"] + CXXFLAGS + ["-o", API_SMOKE, API_SMOKE_SRC, "-L" + HERE, "-lqcsim", "-lqcsim_b200",
                                   "-Wl,-rpath," + HERE], verbose)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
