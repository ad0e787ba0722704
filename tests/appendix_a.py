"""Appendix-A statistics (tests only): mean relative error of each intermediate of
the x-coordinate formula -(z0 nx nz + s ny)/|n_xy|^2 over a dataset, as the paper plots in its
Fig. 6 (Appendix A).  Pairs are scored by their exact sum (P:1169-1176:
"computed the relative error between their exact sum and the ground-truth quantity"); the ground
truth is exact rational arithmetic (oracle (b)'s integer model), s to ~2^-400.
"""
from __future__ import annotations

import csv
import os
from fractions import Fraction

from oracle import exact

# (label, hi field, lo field or None, exact-value key), left to right as in Fig. 6
ITEMS = (("n_x", "nx", "ex", "nx"), ("|n|^2", "S3", "s3", "N"), ("|n_xy|^2", "S2", "s2", "S"),
         ("z0^2", "C", "eC", "C"), ("|n|^2 z0^2", "D", "eD", "D"), ("s^2", "sh", "sl", "sigma"),
         ("s", "s", "es", "s"), ("n_x n_z", "Fx", "eFx", "F"),
         ("z0 n_x n_z + s n_y", "Xp_p", "Xp_s", "X"), ("fl(numerator)", "Xp", None, "X"),
         ("fl(|n_xy|^2)", "S2", None, "S"), ("p_x", "Ppx", None, "px"))


def exact_values(x1, x2, z0) -> dict | None:
    """Exact intermediates of the + root's x coordinate (None when s^2 <= 0 or n_xy = 0)."""
    q = exact.Query(x1, x2, z0)
    if q.sigma <= 0 or q.S == 0:
        return None
    L = q.L
    s_int, K = q.s_scaled()
    nx, ny, nz = (Fraction(v, 1 << (2 * L)) for v in q.n)
    zz = Fraction(q.Z, 1 << L)
    S, N = Fraction(q.S, 1 << (4 * L)), Fraction(q.N, 1 << (4 * L))
    s = Fraction(s_int, 1 << (3 * L + K))
    X = zz * nx * nz + s * ny
    return {"nx": nx, "N": N, "S": S, "C": zz * zz, "D": N * zz * zz,
            "sigma": Fraction(q.sigma, 1 << (6 * L)), "s": s, "F": nx * nz, "X": X, "px": -X / S}


def rel_errors(trace: dict, ex: dict) -> dict:
    """Relative error of each ITEM whose fields the mode fills (zero exact values skipped)."""
    out = {}
    for label, hi, lo, key in ITEMS:
        v = Fraction(trace[hi]) + (Fraction(trace[lo]) if lo else 0)
        if trace[hi] == 0.0 and ex[key] != 0:
            continue                            # not produced by this mode (plain binary64)
        if ex[key] == 0:
            continue
        out[label] = float(abs(v - ex[key]) / abs(ex[key]))
    return out


def mean_table(traces, exacts) -> dict:
    """label -> (mean relative error, samples) over the queries with an exact value."""
    acc = {}
    for t, e in zip(traces, exacts):
        if e is None:
            continue
        for k, v in rel_errors(t, e).items():
            s, c = acc.get(k, (0.0, 0))
            acc[k] = (s + v, c + 1)
    return {k: (s / c, c) for k, (s, c) in acc.items()}


def write_csv(path, tables: dict, source: str) -> None:
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["# Appendix A (P:1161-1211) mean relative error per intermediate", source])
        w.writerow(["intermediate", *[f"{m} mean_rel_err" for m in tables], "samples"])
        for label, *_ in ITEMS:
            row = [label]
            n = 0
            for m, tab in tables.items():
                v = tab.get(label)
                row.append(f"{v[0]:.3e}" if v else "")
                n = max(n, v[1] if v else 0)
            w.writerow(row + [n])
