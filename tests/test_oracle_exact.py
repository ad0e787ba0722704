"""Pins for oracle (b) (oracle/exact.py): the closed form computed exactly.

Oracle (b) is checked against things other than itself: the hand cases' closed forms, an
independent transcription of the geometry (Eq.YAC with a normalised normal), the
invariants the exact intersection must satisfy (|P| = 1, n.P = 0, P_z = z0),
brute-force crossing search along the arc (no use of the formula or of the containment
identity), power-of-two and arbitrary positive scaling of endpoints, and the
polynomial identities its sqrt-free containment test relies on.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import sgi_inputs
from helpers import F, random_unit
from oracle import exact

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_cases.json")


def closed_form(expr: str) -> float:
    """RN of a golden closed form: '0', '1', 'sqrt:p/q', 'neg_sqrt:p/q'."""
    import mpmath as mp
    with mp.workdps(60):
        if expr.startswith("sqrt:") or expr.startswith("neg_sqrt:"):
            sign = -1 if expr.startswith("neg") else 1
            p, q = expr.split(":")[1].split("/")
            return float(sign * mp.sqrt(mp.mpf(int(p)) / int(q)))
        return float(mp.mpf(expr))


def hand_cases():
    with open(GOLDEN) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", hand_cases(), ids=lambda c: c["name"])
def test_hand_cases(case):
    ex = exact.exact_query(case["x1"], case["x2"], case["z0"])
    assert ex.count == case["count"]
    want = [(closed_form(px), closed_form(py)) for px, py in case["points"]]
    assert ex.rounded == want
    for h, (px, _) in zip(case.get("hex", []), want):
        assert px.hex() == h


def _mixed_queries(n, seed=7):
    """Long, short and non-unit arcs with z0 spanning [-1, 1] (0/1/2 intersections occur)."""
    rng = np.random.default_rng(seed)
    x1, x2 = random_unit(rng, n), random_unit(rng, n)
    short = rng.random(n) < 0.3
    x2[short] = x1[short] + 10 ** rng.uniform(-6, -1, (short.sum(), 1)) * random_unit(rng, short.sum())
    scale = rng.random(n) < 0.25
    x1[scale] *= 1.75
    x2[scale & (rng.random(n) < 0.5)] *= 0.3
    z0 = rng.uniform(-1, 1, n)
    between = rng.random(n) < 0.5
    lo, hi = np.minimum(x1[:, 2] / np.linalg.norm(x1, axis=1), x2[:, 2] / np.linalg.norm(x2, axis=1)), \
        np.maximum(x1[:, 2] / np.linalg.norm(x1, axis=1), x2[:, 2] / np.linalg.norm(x2, axis=1))
    z0[between] = (lo + rng.random(n) * (hi - lo))[between]
    return x1, x2, z0


def test_eq_yac_agrees_with_eq_final():
    """Eq.FINAL and Eq.YAC are the same geometry."""
    import mpmath as mp
    x1, x2, z0 = _mixed_queries(300, seed=11)
    checked = 0
    for i in range(len(z0)):
        ex = exact.exact_query(x1[i], x2[i], z0[i])
        if ex.sigma_sign <= 0 or ex.count == exact.DEGENERATE:
            continue
        q = exact.Query(x1[i], x2[i], z0[i])
        s_int, K = q.s_scaled()
        den = q.S << (q.L + K)
        bx, by = (q.Z * q.n[0] * q.n[2]) << K, (q.Z * q.n[1] * q.n[2]) << K
        final = [(-(bx + s_int * q.n[1]) / Fraction(den), -(by - s_int * q.n[0]) / Fraction(den)),
                 (-(bx - s_int * q.n[1]) / Fraction(den), -(by + s_int * q.n[0]) / Fraction(den))]
        yac = exact.yac_points(x1[i], x2[i], z0[i])
        with mp.workdps(120):
            for (fx, fy), (yx, yy) in zip(final, yac):
                assert abs(mp.mpf(fx.numerator) / fx.denominator - yx) < mp.mpf(2) ** -300
                assert abs(mp.mpf(fy.numerator) / fy.denominator - yy) < mp.mpf(2) ** -300
        checked += 1
    assert checked > 100


def test_invariants_unit_norm_and_on_plane():
    """|P|^2 = Px^2 + Py^2 + z0^2 = 1 and n.P = 0 for the exact points."""
    x1, x2, z0 = _mixed_queries(400, seed=12)
    seen = 0
    for i in range(len(z0)):
        ex = exact.exact_query(x1[i], x2[i], z0[i])
        if ex.count in (0, exact.DEGENERATE):
            continue
        q = exact.Query(x1[i], x2[i], z0[i])
        nvec = [Fraction(c, 2 ** (2 * q.L)) for c in q.n]
        nn = sum(c * c for c in nvec)
        for (px, py, den) in ex.points:
            Px, Py, Pz = Fraction(px, den), Fraction(py, den), F(z0[i])
            assert abs(Px * Px + Py * Py + Pz * Pz - 1) < Fraction(1, 2 ** 350)
            dot = nvec[0] * Px + nvec[1] * Py + nvec[2] * Pz
            assert abs(dot) ** 2 < nn * Fraction(1, 2 ** 700)
            seen += 1
    assert seen > 150


def test_brute_force_counts_and_points():
    """Sign changes of z(t) - z0 along the arc, bisected at 60 digits (no Eq.FINAL used)."""
    import mpmath as mp
    x1, x2, z0 = _mixed_queries(150, seed=13)
    hist = {0: 0, 1: 0, 2: 0}
    for i in range(len(z0)):
        ex = exact.exact_query(x1[i], x2[i], z0[i])
        if ex.count == exact.DEGENERATE:
            continue
        crossings, min_gap = exact.brute_force(x1[i], x2[i], z0[i], samples=401, dps=40)
        if min_gap < 1e-9:          # grazing: sampling cannot see a touch reliably
            continue
        assert len(crossings) == ex.count, (i, crossings, ex.count)
        hist[ex.count] += 1
        for (bx, by), (px, py, den) in zip(crossings, ex.points):
            with mp.workdps(40):
                assert abs(bx - mp.mpf(px) / den) < 1e-30
                assert abs(by - mp.mpf(py) / den) < 1e-30
    assert hist[0] > 10 and hist[1] > 10 and hist[2] >= 1, hist


def test_brute_force_two_point_order():
    """Arc order of two crossings (P+ first iff g1 >= 0) against the brute-force walk."""
    import mpmath as mp
    cfg_a, cfg_b, cfg_z = sgi_inputs.generate_host(3, 90)
    checked = 0
    for i in range(0, 90, 3):                          # near-tangent class: two points
        ex = exact.exact_query(cfg_a[:, i], cfg_b[:, i], cfg_z[i])
        if ex.count != 2:
            continue
        crossings, _ = exact.brute_force(cfg_a[:, i], cfg_b[:, i], cfg_z[i], samples=2001, dps=40)
        if len(crossings) != 2:
            continue                                   # crossings closer than the grid
        with mp.workdps(40):
            for (bx, by), (px, py, den) in zip(crossings, ex.points):
                assert abs(bx - mp.mpf(px) / den) < 1e-20
        checked += 1
    assert checked >= 5


def test_sqrt_free_containment_identities():
    """(z0 g_k)^2 - s^2 z_k^2 = S * D_k and g_k^2 + N z_k^2 = S |x_k|^2 (integer-exact)."""
    rng = np.random.default_rng(14)
    for _ in range(500):
        v = rng.integers(-2 ** 20, 2 ** 20, 7).astype(np.float64) / 2 ** 20
        q = exact.Query(v[:3], v[3:6], v[6])
        for k, X in ((1, q.X1), (2, q.X2)):
            g = q.g(k)
            # every term below carries the same scale 2^8L (resp. 2^6L)
            assert (q.Z * g) ** 2 - q.sigma * X[2] ** 2 == q.S * q.D(k)
            assert g * g + q.N * X[2] ** 2 == q.S * (X[0] ** 2 + X[1] ** 2 + X[2] ** 2)


@pytest.mark.parametrize("k", [-30, -7, 5, 30])
def test_scale_invariance(k):
    """Eq.FINAL is invariant to |x1| and |x2| (footnote P:298-306)."""
    x1, x2, z0 = _mixed_queries(120, seed=15)
    for i in range(len(z0)):
        ref = exact.exact_query(x1[i], x2[i], z0[i])
        for a, b in ((x1[i] * 2.0 ** k, x2[i]), (x1[i], x2[i] * 2.0 ** k)):
            ex = exact.exact_query(a, b, z0[i])
            assert ex.count == ref.count
            assert ex.rounded == ref.rounded


def test_scale_invariance_non_dyadic():
    """Integer endpoints scaled exactly by 3 and 5: same count and points."""
    rng = np.random.default_rng(16)
    for _ in range(300):
        v = rng.integers(-2 ** 12, 2 ** 12, 6).astype(np.float64)
        z0 = rng.uniform(-1, 1)
        ref = exact.exact_query(v[:3], v[3:], z0)
        ex = exact.exact_query(v[:3] * 3, v[3:] * 5, z0)
        assert (ex.count, ex.rounded) == (ref.count, ref.rounded)


def test_err_u_metric():
    """err_u (P:333 metric / (u sqrt(1-z0^2))): a 3-4-5 displacement gives 5u."""
    u = 2.0 ** -53
    p_exact = (3 << 60, 0, 1 << 62)                     # P = (0.75, 0)
    assert exact.point_error((0.75 + 3 * u, 4 * u), p_exact) == 5 * u
    assert exact.err_u((0.75 + 3 * u, 4 * u), p_exact, 0.6) == pytest.approx(5 / 0.8, rel=1e-15)
    assert exact.err_u((0.75, 0.0), p_exact, 0.0) == 0.0
