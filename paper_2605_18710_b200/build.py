"""Build the in-tree CUDA library paper_2605_18710_b200/libmosaic_gpu.so (sm_100a).

nvcc cross-compiles here (no GPU needed).  Flags:
  * -gencode arch=compute_100a,code=sm_100a  (B200 only; no other targets)
  * -fmad=false / -ffp-contract=off          (fp64 bit parity with the reference,
                                              BASELINE.md §2: FMA contraction changes bits)
  * -lineinfo                                (ncu source page)
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libmosaic_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX_HOST", "g++")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["engine.cu", "eval.cu", "nccl_plane.cu", "pack.cu", "sim.cu", "calib.cu"]
# engine_fast.cu is compiled once per search mode (specialised MIN / FIRST kernels)
CU_VARIANTS = [("engine_fast.cu", "engine_fast_min", ["-DMG_FAST_MODE=0"]),
               ("engine_fast.cu", "engine_fast_first", ["-DMG_FAST_MODE=1"]),
               ("engine_fast.cu", "engine_fast_any", ["-DMG_FAST_MODE=2"])]
CPP_SOURCES = ["model.cpp", "planner.cpp", "capi.cpp"]
HEADERS = ["engine.hpp", "search_core.cuh", "search_warp.cuh", "search_kernel.cuh", "spec_build.hpp", "model.hpp",
           "planner.hpp", "pack.hpp", "sim.hpp"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build(verbose_ptxas: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(HERE, "..", "include", "mosaic_gpu.h")
    ]
    objs = []
    units = [(src, src, []) for src in CU_SOURCES] + [(a, b + ".cu", c) for a, b, c in CU_VARIANTS]
    for src, name, defs in units:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, name + ".o")
        objs.append(o)
        if _newer(o, [s] + hdrs + [__file__]):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++20", *defs,
                   "-Xcompiler", "-fPIC,-ffp-contract=off", "-c", s, "-o", o]
            if verbose_ptxas:
                cmd.insert(1, "-Xptxas=-v")
            _run(cmd)
    for src in CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if _newer(o, [s] + hdrs + [__file__]):
            _run([CXX, "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-Wall",
                  "-I/usr/local/cuda/include", "-c", s, "-o", o])
    if _newer(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-Xcompiler", "-fPIC", "-ldl"])
    return LIB


if __name__ == "__main__":
    build(verbose_ptxas="-v" in sys.argv)
