"""Build libhood_b200.so in-tree with nvcc for sm_100a (no JIT, no torch ext).

    python -m paper_1203_5004_b200.build [--verbose]

The shared library lands in paper_1203_5004_b200/lib/ (git-ignored, shipped to
the GPU box with the snapshot).  The C++ drop-in test driver
(tests/cpp/test_dropin.cpp -> lib/test_dropin) is built alongside.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
SO = os.path.join(LIB, "libhood_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["hood_kernels.cu", "hood_capi.cu", "hood_host.cpp"]
HEADERS = ["hood_device.cuh", "hood_kernels.cuh"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "hood_b200.h"),
                                                                  os.path.abspath(__file__)]
    if force or _stale(SO, deps):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared",
               "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-o", SO]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        cmd += os.environ.get("HOOD_NVCC_EXTRA", "").split()  # experiments only (e.g. -DHOOD_RING_COUNTERS)
        cmd += [os.path.join(CSRC, f) for f in SOURCES]
        cmd += ["-lcuda"] if False else []
        subprocess.run(cmd, check=True)
    drv_src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    drv = os.path.join(LIB, "test_dropin")
    if os.path.exists(drv_src) and (force or _stale(drv, [drv_src, SO, os.path.join(ROOT, "include", "hood_b200.hpp")])):
        subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-o", drv, drv_src,
                        "-L", LIB, "-lhood_b200", f"-Wl,-rpath,{LIB}", "-Wl,-rpath,$ORIGIN"], check=True)
    return SO


def build_checked(force: bool = False) -> str:
    """Bounds-checked build (-DHOOD_CHECKED: device-side invariant checks that
    trap), as lib/libhood_b200_checked.so; the GPU suite runs against it with
    HOOD_B200_LIB pointing at it (compute-sanitizer is closed on the pool)."""
    os.makedirs(LIB, exist_ok=True)
    so = os.path.join(LIB, "libhood_b200_checked.so")
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "hood_b200.h")]
    if force or _stale(so, deps):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared",
               "--expt-relaxed-constexpr", "-DHOOD_CHECKED", "-I", os.path.join(ROOT, "include"), "-o", so]
        cmd += [os.path.join(CSRC, f) for f in SOURCES]
        subprocess.run(cmd, check=True)
    return so


def build_trace(force: bool = False) -> str:
    """Profiling build (tools/trace_ring.py, tools/trace_finalize.py): the same
    sources with -DHOOD_TRACE (in-kernel globaltimer/clock64 stamps), as
    lib/libhood_b200_trace.so -- never loaded by the package unless
    HOOD_B200_LIB points at it."""
    os.makedirs(LIB, exist_ok=True)
    so = os.path.join(LIB, "libhood_b200_trace.so")
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "hood_b200.h")]
    if force or _stale(so, deps):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared",
               "--expt-relaxed-constexpr", "-DHOOD_TRACE", "-I", os.path.join(ROOT, "include"), "-o", so]
        cmd += [os.path.join(CSRC, f) for f in SOURCES]
        subprocess.run(cmd, check=True)
    return so


if __name__ == "__main__":
    if "--trace" in sys.argv:
        print(build_trace(force="--force" in sys.argv))
        sys.exit(0)
    if "--checked" in sys.argv:
        print(build_checked(force="--force" in sys.argv))
        sys.exit(0)
    build(verbose="--verbose" in sys.argv, force="--force" in sys.argv)
    print(SO)
