"""In-tree build of libsgi.so for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.path.join(PKG, "libsgi.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-fmad=false",            # no contraction: each fl() is one rounding
              "-Xptxas", "-v", "-Xcompiler", "-fPIC", "-shared", "-std=c++17"]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) +
                  glob.glob(os.path.join(PKG, "csrc", "*.cuh")) +
                  [os.path.join(ROOT, "include", "sgi.h")])


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/*.cu into paper_2510_09892_b200/libsgi.so if any source is newer."""
    srcs = sources()
    if (not force and os.path.exists(LIB_PATH)
            and all(os.path.getmtime(LIB_PATH) >= os.path.getmtime(s) for s in srcs)):
        return LIB_PATH
    cu = [s for s in srcs if s.endswith(".cu")]
    cmd = ["nvcc", *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB_PATH, *cu]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
        f.write(res.stderr)
    if verbose:
        print(res.stderr)
    return LIB_PATH


DEVTEST_SRC = os.path.join(ROOT, "tests", "native", "devtests.cu")
DEVTEST_LIB = os.path.join(ROOT, "tests", "native", "libsgi_devtest.so")


def build_devtests(force: bool = False) -> str:
    """Test-only library: device unit tests of the EFT primitives (tests/native)."""
    deps = [DEVTEST_SRC] + sources()
    if (not force and os.path.exists(DEVTEST_LIB)
            and all(os.path.getmtime(DEVTEST_LIB) >= os.path.getmtime(s) for s in deps)):
        return DEVTEST_LIB
    cmd = ["nvcc", *[f for f in NVCC_FLAGS if f not in ("-Xptxas", "-v")], "-o", DEVTEST_LIB,
           DEVTEST_SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    return DEVTEST_LIB


DEBUG_LIB = os.path.join(ROOT, "build", "debug", "libsgi_debug.so")


def build_debug(force: bool = False) -> str:
    """Test-only variant of libsgi.so with device-side checks (-DSGI_DEBUG_CHECKS=1: asserts on
    every queue / table / tile index, poisoned shared scratch; csrc/sgi_tma.cuh) — the stand-in
    for compute-sanitizer, which this GPU pool does not run."""
    srcs = sources()
    if (not force and os.path.exists(DEBUG_LIB)
            and all(os.path.getmtime(DEBUG_LIB) >= os.path.getmtime(s) for s in srcs)):
        return DEBUG_LIB
    os.makedirs(os.path.dirname(DEBUG_LIB), exist_ok=True)
    cu = [s for s in srcs if s.endswith(".cu")]
    flags = [f for f in NVCC_FLAGS if f not in ("-Xptxas", "-v")]
    cmd = ["nvcc", *flags, "-DSGI_DEBUG_CHECKS=1", "-I", os.path.join(ROOT, "include"), "-o",
           DEBUG_LIB, *cu]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    return DEBUG_LIB
