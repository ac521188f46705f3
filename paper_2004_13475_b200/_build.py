"""In-tree build of the product library (libnbbgpu.so) and the test-only checkers.

nvcc cross-compiles sm_100a without a GPU, so this runs in the CPU container and
on the GPU box alike. The .so lands next to the package so it travels with the
repo snapshot (git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
LIB = os.path.join(PKG_DIR, "libnbbgpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["nbb_capi.cu", "nbb_host.cpp"]
HEADERS = ["common.cuh", "tile_kernels.cuh", "ca_pipe_kernel.cuh", "bits_kernels.cuh",
           "compact_kernels.cuh", "compact_pass.cuh", "compact_sliced.cuh", "compact_cluster.cuh",
           "percell_kernels.cuh",
           "util_kernels.cuh", "nbb_host.hpp", "nbb_multi.inc", "nbb_comm.inc"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "nbb_gpu.h"))
    if not force and _newer(LIB, deps):
        return LIB
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v" if verbose else "-O3",
           f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}",
           "-shared", "-o", LIB + ".tmp",
           *[os.path.join(CSRC, f) for f in SOURCES], "-ldl"]
    subprocess.run(cmd, check=True, cwd=ROOT)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_oracle() -> None:
    """TEST INFRASTRUCTURE: oracle/_ref/liboracle.so always; oracle/_ref/libnbbref.so
    (the unmodified reference) only where /root/reference exists (this container)."""
    odir = os.path.join(ROOT, "oracle")
    subprocess.run(["make", "-s", "oracle"], check=True, cwd=odir)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "ref"], check=True, cwd=odir)


if __name__ == "__main__":
    build_library(force="--force" in sys.argv, verbose="-v" in sys.argv)
    build_oracle()
    print(LIB)
