"""oracle — the CPU oracles for the arc/latitude intersection path.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` leg may
import this package.  It shares no code with the CUDA path (paper_2510_09892_b200/) and imports
nothing from it; the product path never imports it.

  (a) eft_oracle.c  — sequential IEEE binary64 evaluation of the paper's AccuX / naive formula,
                      the same op order the GPU must reproduce bit for bit (loaded via ctypes).
  (b) exact.py      — exact-rational evaluation of the closed form Eq.FINAL
                      with a >=400-bit square root, exact counts and the paper's error metric.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "liboracle_eft.so")
SRC = os.path.join(_HERE, "eft_oracle.c")

MODE_NAIVE, MODE_EFT, MODE_EFT_LITERAL = 0, 1, 2
MODE_YAC, MODE_BASE, MODE_NAIVE_KAHAN = 3, 4, 5
DEGENERATE = 0xFF

TRACE_FIELDS = ("nx", "ex", "ny", "ey", "nz", "ez", "S2", "s2", "S3", "s3", "C", "eC", "D", "eD",
                "sh", "sl", "s", "es", "Fx", "eFx", "Fy", "eFy", "Xp", "Yp", "Xm", "Ym",
                "Ppx", "Ppy", "Pmx", "Pmy",
                "Xp_p", "Xp_s", "Yp_p", "Yp_s", "Xm_p", "Xm_s", "Ym_p", "Ym_s")

PRIM = {"two_sum": 0, "fast_two_sum": 1, "two_prod": 2, "kahan_dop": 3, "accu_dop": 4,
        "sum_non_neg": 5, "sum_of_squares": 6, "sum_of_squares_c": 7, "acc_sqrt": 8,
        "comp_dot_c": 9, "comp_dot": 10}


def build() -> None:
    """Compile oracle (a) with the paper's no-contraction contract."""
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                           "-fno-fast-math", "-fopenmp", "-o", LIB, SRC, "-lm"])


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        L.oracle_intersect_batch.restype = ctypes.c_int
        L.oracle_intersect_batch.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_intersect_dw_batch.restype = ctypes.c_int
        L.oracle_intersect_dw_batch.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_int]
        L.oracle_trace.restype = ctypes.c_int
        L.oracle_trace.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_double, ctypes.c_void_p]
        L.oracle_prim_batch.restype = ctypes.c_int
        L.oracle_prim_batch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_int64, ctypes.c_void_p]
        _lib = L
    return _lib


def intersect(mode: int, a: np.ndarray, b: np.ndarray, z0: np.ndarray, n: int | None = None,
              nthreads: int = 1):
    """Oracle (a) over SoA planes a[3, ld], b[3, ld], z0[ld].

    Returns (out_xyz[2, 3, ld] float64, out_count[ld] uint8); columns >= n are untouched (NaN/0).
    """
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    z0 = np.ascontiguousarray(z0, np.float64)
    ld = z0.shape[0]
    n = ld if n is None else n
    assert a.shape == (3, ld) and b.shape == (3, ld)
    out = np.full((2, 3, ld), np.nan)
    cnt = np.zeros(ld, np.uint8)
    rc = lib().oracle_intersect_batch(mode, a.ctypes.data, b.ctypes.data, z0.ctypes.data, n, ld,
                                      out.ctypes.data, cnt.ctypes.data, nthreads)
    if rc != 0:
        raise ValueError("oracle_intersect_batch rejected its arguments")
    return out, cnt


def intersect_dw(mode: int, a: np.ndarray, b: np.ndarray, z0: np.ndarray, nthreads: int = 1):
    """Oracle (a) with double-word points (EFT modes): (out_xyz[2,3,n], out_lo[2,2,n], count[n]);
    P ~ out_xyz + out_lo per x/y coordinate (reading R11)."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    z0 = np.ascontiguousarray(z0, np.float64)
    ld = z0.shape[0]
    out = np.empty((2, 3, ld), np.float64)
    lo = np.empty((2, 2, ld), np.float64)
    cnt = np.empty(ld, np.uint8)
    rc = lib().oracle_intersect_dw_batch(mode, a.ctypes.data, b.ctypes.data, z0.ctypes.data, ld,
                                         ld, out.ctypes.data, lo.ctypes.data, cnt.ctypes.data,
                                         nthreads)
    if rc != 0:
        raise ValueError("oracle_intersect_dw_batch rejected its arguments")
    return out, lo, cnt


def trace(mode: int, x1, x2, z0: float) -> tuple[int, dict]:
    """Every intermediate of one query (Appendix-A style)."""
    x1 = np.ascontiguousarray(x1, np.float64)
    x2 = np.ascontiguousarray(x2, np.float64)
    out = np.zeros(len(TRACE_FIELDS), np.float64)
    c = lib().oracle_trace(mode, x1.ctypes.data, x2.ctypes.data, float(z0), out.ctypes.data)
    return c, dict(zip(TRACE_FIELDS, out.tolist()))


def prim(name: str, rows: np.ndarray, k: int = 0) -> np.ndarray:
    """Apply one EFT operator of oracle (a) to each row of `rows`; returns [n, 2] (hi, lo)."""
    rows = np.ascontiguousarray(rows, np.float64)
    n, width = rows.shape
    out = np.zeros((n, 2), np.float64)
    rc = lib().oracle_prim_batch(PRIM[name], k, rows.ctypes.data, width, n, out.ctypes.data)
    if rc != 0:
        raise ValueError(name)
    return out
