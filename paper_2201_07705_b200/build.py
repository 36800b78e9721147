"""Build the CUDA path: libgemel.so (C ABI in include/gemel.h) for sm_100a.

    python -m paper_2201_07705_b200.build        # or __graft_entry__.build()

Compiles every translation unit with nvcc (-gencode arch=compute_100a,code=sm_100a
-lineinfo) in parallel, links one shared library in-tree (it travels to the GPU
box with the repo snapshot), plus the developer self-test binary.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libgemel.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["registry.cpp", "plan.cpp", "swap.cpp", "runtime.cpp", "tmap.cpp", "kernels/gemm_sm100.cu", "kernels/memops.cu",
           "kernels/detect.cu", "kernels/stem_sm100.cu"]
HEADERS = ["internal.h", "tmap.h", "kernels/gemm.h", "kernels/memops.h", "kernels/sm100_ptx.cuh", "kernels/stem.h", "kernels/select.cuh", "kernels/smem_attr.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src):
    obj = os.path.join(BUILD, src.replace("/", "_") + ".o")
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "gemel.h")]
    if _newer(obj, deps):
        cmd = [NVCC, *ARCH, *FLAGS, "-x", "cu" if src.endswith(".cu") else "c++", "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose=False, selftest=True):
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if _newer(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if selftest:
        exe = os.path.join(BUILD, "gemm_selftest")
        srcs = [os.path.join(CSRC, "tools", "gemm_selftest.cu"), os.path.join(CSRC, "kernels", "gemm_sm100.cu"),
                os.path.join(CSRC, "tmap.cpp")]
        if _newer(exe, srcs + [os.path.join(CSRC, h) for h in HEADERS]):
            r = subprocess.run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-DGEMEL_DEV_PROBES", "-I" + CSRC, "-o", exe,
                                *srcs],
                               capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"selftest build failed:\n{r.stderr}")
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
