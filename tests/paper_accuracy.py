"""Per-group accuracy report on the paper's two accuracy datasets (tests only).

The paper groups its primary dataset by latitude band and plots the worst (maximum) relative
error per band (Fig. 2 and Fig. 3), and groups its secondary ill-conditioned dataset
by the interval of the offset r (Fig. 4).  Here the ground truth is oracle (b)
(exact rationals, P:937's Mathematica replaced) and the computed points come either from oracle
(a) (CPU tests) or from the CUDA path (GPU tests; bitwise equal to oracle (a) there).

Relative error = |dP| = sqrt(dPx^2 + dPy^2) (|P| = 1), taken over the in-arc points
whose count agrees with the exact count; count disagreements are tallied per group.
"""
from __future__ import annotations

import csv
import os

import numpy as np

import sgi_inputs
from oracle import exact

MODE_NAMES = ("eft", "eft_literal", "naive", "yac", "base", "naive_kahan")


def exact_results(a, b, z0, idx):
    """Oracle (b) for the queries `idx` (global = local indices)."""
    return {int(i): exact.exact_query(a[:, i], b[:, i], z0[i]) for i in idx}


def group_stats(config, idx, exact_by_i, out, cnt, z0):
    """Per group: [n_queries, n_points, max |dP|, max err_u, count mismatches]."""
    ng = len(sgi_inputs.PRIMARY_BAND_EDGES) - 1 if config == 6 else len(sgi_inputs.SECONDARY_DECADES)
    st = np.zeros((ng, 5))
    for i in idx:
        g = int(sgi_inputs.group_of(config, int(i)))
        e = exact_by_i[int(i)]
        st[g, 0] += 1
        if e.count != int(cnt[i]):
            st[g, 4] += 1
            continue
        if e.count in (0, exact.DEGENERATE):
            continue
        for k in range(e.count):
            p = (out[k, 0, i], out[k, 1, i])
            st[g, 1] += 1
            st[g, 2] = max(st[g, 2], exact.point_error(p, e.points[k]))
            st[g, 3] = max(st[g, 3], exact.err_u(p, e.points[k], z0[i]))
    return st


def write_csv(path, config, stats_by_mode, source):
    """One row per (group, mode), the paper's plot-ready layout."""
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["# config", config, "source", source, "metric",
                    "|dP| = sqrt(dPx^2 + dPy^2) vs oracle (b); err_u = |dP| / (u sqrt(1 - z0^2))"])
        w.writerow(["group", "label", "mode", "queries", "points", "max_rel_err", "max_err_u",
                    "count_mismatches"])
        for mode, st in stats_by_mode.items():
            for g in range(st.shape[0]):
                w.writerow([g, sgi_inputs.group_label(config, g), mode, int(st[g, 0]),
                            int(st[g, 1]), f"{st[g, 2]:.3e}", f"{st[g, 3]:.3f}", int(st[g, 4])])


def check_paper_claims(config, stats):
    """The shapes the paper reports, as assertions (each cites its passage)."""
    eft, lit, naive, base = stats["eft"], stats["eft_literal"], stats["naive"], stats["base"]
    for st in (eft, lit):
        # Eq.BOUND: AccuX within 3 sqrt(1 - z0^2) u everywhere, counts exact
        assert st[:, 3].max() <= 3.0, st[:, 3]
        assert st[:, 4].sum() == 0
        assert (st[:, 1] > 0).all()
    if config == 6:
        # double precision loses digits approaching the north pole, AccuX does not
        assert naive[-1, 2] >= 100 * naive[8, 2] and naive[-1, 2] >= 1e-13
        assert eft[-1, 2] <= 1e-16
        # Eq.BASE cancels as n^z^2 -> 1, i.e. for arcs near the equator
        assert base[0, 2] >= 1e-7 and base[0, 2] >= 1e6 * eft[0, 2]
    else:
        # on the ill-conditioned decades only AccuX keeps acceptable accuracy
        assert naive[0, 2] >= 1e-12 and naive[0, 2] >= 1e4 * eft[0, 2]
        assert base[0, 2] >= 1e-6
