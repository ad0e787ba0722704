"""Pins for the paper's comparison formulas in oracle (a): Eq.YAC,
Eq.BASE and Eq.FINAL with Kahan's DiffOfProd normal (Alg.3), all in plain
binary64 (reading R9).

  * hand cases: the exact counts, and points within a few ulps of the closed forms (the
    normalisation n/|n| rounds);
  * the paper's accuracy claims for Fig. 2 on its secondary dataset shape: Eq.BASE
    "suffers from catastrophic cancellation when n^z^2 approaches 1" — near-equatorial arcs
    (endpoints in (0, 1e-4 deg]) lose >= 100x more than Eq.FINAL (SPEC acceptance 7);
    Eq.YAC's normalisation is "numerically stable": within 100x of Eq.FINAL there;
  * Kahan's normal tightens the naive formula on near-coincident endpoints.
"""
import math

import numpy as np
import pytest

import oracle
import sgi_inputs
from oracle import exact
from test_oracle_exact import closed_form, hand_cases

U = 2.0 ** -53
VARIANTS = {"yac": oracle.MODE_YAC, "base": oracle.MODE_BASE, "naive_kahan": oracle.MODE_NAIVE_KAHAN}


@pytest.mark.parametrize("mode", list(VARIANTS))
@pytest.mark.parametrize("case", hand_cases(), ids=lambda c: c["name"])
def test_hand_cases(case, mode):
    a = np.array(case["x1"], float).reshape(3, 1)
    b = np.array(case["x2"], float).reshape(3, 1)
    out, cnt = oracle.intersect(VARIANTS[mode], a, b, np.array([case["z0"]]))
    assert cnt[0] == case["count"]
    for k, (px, py) in enumerate(case["points"]):
        assert abs(out[k, 0, 0] - closed_form(px)) <= 8 * U
        assert abs(out[k, 1, 0] - closed_form(py)) <= 8 * U
        assert out[k, 2, 0] == case["z0"]


def _equatorial_band(n, seed=21):
    """Arcs with both endpoints in the latitude band (0, 1e-4 deg], z0 between them."""
    rng = np.random.default_rng(seed)
    lat = np.radians(rng.uniform(0, 1e-4, (2, n)))
    lon = np.radians(rng.uniform(0, 360, (2, n)))
    lon[1] = lon[0] + np.radians(rng.uniform(1, 170, n))
    pts = np.stack([np.cos(lat) * np.cos(lon), np.cos(lat) * np.sin(lon), np.sin(lat)])
    a, b = pts[:, 0], pts[:, 1]
    lo, hi = np.minimum(a[2], b[2]), np.maximum(a[2], b[2])
    z0 = lo + rng.uniform(0, 1, n) * (hi - lo)
    return np.ascontiguousarray(a), np.ascontiguousarray(b), z0


def _max_err(mode, a, b, z0):
    out, cnt = oracle.intersect(mode, a, b, z0)
    worst = 0.0
    for i in range(len(z0)):
        ex = exact.exact_query(a[:, i], b[:, i], z0[i])
        if ex.count != cnt[i] or ex.count in (0, exact.DEGENERATE):
            continue
        for k in range(ex.count):
            worst = max(worst, exact.point_error((out[k, 0, i], out[k, 1, i]), ex.points[k]))
    return worst


def test_base_formula_cancellation_near_equator():
    a, b, z0 = _equatorial_band(400)
    final = _max_err(oracle.MODE_NAIVE, a, b, z0)
    base = _max_err(oracle.MODE_BASE, a, b, z0)
    yac = _max_err(oracle.MODE_YAC, a, b, z0)
    assert base >= 100 * final, (base, final)
    assert yac <= 100 * final + 1e-15, (yac, final)


def test_kahan_normal_on_near_coincident_arcs():
    a, b, z0 = sgi_inputs.generate_host(3, 1500)
    idx = np.arange(2, 1500, 3)                       # C3 near-coincident class
    a, b, z0 = a[:, idx].copy(), b[:, idx].copy(), z0[idx].copy()
    errs = {}
    for name, mode in (("naive", oracle.MODE_NAIVE), ("kahan", oracle.MODE_NAIVE_KAHAN)):
        out, cnt = oracle.intersect(mode, a, b, z0)
        e = []
        for i in range(len(z0)):
            ex = exact.exact_query(a[:, i], b[:, i], z0[i])
            if ex.count == cnt[i] and ex.count == 1:
                e.append(exact.point_error((out[0, 0, i], out[0, 1, i]), ex.points[0]))
        errs[name] = np.median(e)
    assert errs["kahan"] < errs["naive"] / 10, errs
