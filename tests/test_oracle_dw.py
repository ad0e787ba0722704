"""Double-word points of oracle (a) (reading R11) against oracle (b).

The paper rounds each coordinate once; the double-word output keeps the low part
the AccuX pairs already carry.  Pinned here: the high part is the EFT output bit for bit, the
low part is within the rounded result's own error (|lo| <= 4 ulp(hi): Eq.BOUND, puts
hi within 3 ulps of P), hi + lo is within 1e-6 u of the exact point on every dataset shape, and
(test_double_word_first_order_bound) within the first-order bound DESIGN.md R11 derives from
the operator bounds of the pieces (CompDotC Eq.5.1, AccuDOP P:636-639, SumOfSquaresC P:1563,
AccSqrt P:826, the carried s^2 error); tools/oracle_mutation_check.py's four low-part mutations
(dropped hi s2, dropped dl, sign of s2, dropped sigma) are caught."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import sgi_inputs
from oracle import exact

U = 2.0 ** -53


@pytest.mark.parametrize("config,n", [(1, 2000), (2, 2000), (3, 3000), (6, 17 * 60), (7, 13 * 60)])
@pytest.mark.parametrize("mode", [oracle.MODE_EFT, oracle.MODE_EFT_LITERAL])
def test_double_word_points(config, n, mode):
    a, b, z0 = sgi_inputs.generate_host(config, n)
    out, lo, cnt = oracle.intersect_dw(mode, a, b, z0)
    ref, rcnt = oracle.intersect(mode, a, b, z0)
    assert np.array_equal(cnt, rcnt)
    assert np.array_equal(out.view(np.int64), ref.view(np.int64)) or (
        ((out == ref) | (np.isnan(out) & np.isnan(ref))).all())
    checked = 0
    for i in range(n):
        c = int(cnt[i])
        used = c if c in (1, 2) else 0
        assert np.isnan(lo[used:, :, i]).all()
        if used == 0:
            continue
        if mode == oracle.MODE_EFT_LITERAL and config == 3 and i % 3 == 2:
            continue          # literal mode on near-coincident arcs: outside the paper's bound (R6)
        ex = exact.exact_query(a[:, i], b[:, i], z0[i])
        if ex.count != c:
            continue          # rounded-predicate ties (reading R7'), counted by other tests
        for k in range(used):
            px, py, den = ex.points[k]
            for d, num in ((0, px), (1, py)):
                assert abs(lo[k, d, i]) <= 4 * abs(np.spacing(out[k, d, i]))
            dx = Fraction(out[k, 0, i]) + Fraction(lo[k, 0, i]) - Fraction(px, den)
            dy = Fraction(out[k, 1, i]) + Fraction(lo[k, 1, i]) - Fraction(py, den)
            err_dw = float(dx * dx + dy * dy) ** 0.5
            assert err_dw <= 1e-6 * U, (i, k, err_dw / U)
            checked += 1
    assert checked > n // 2


def _first_order_bound_terms(a, b, z0, t):
    """Exact geometry and the pair magnitudes the double-word bound is stated in (R11):
    kappa_n = max over the normal's components of (|ad| + |bc|) / |ad - bc| (AccuDOP's condition,
    P:636-639), S = |n_xy|^2, D = |n|^2 z0^2, sigma = S - D (exact), and A_x, A_y = the sums of
    the absolute terms of the two CompDotC numerators (Eq.5.1)."""
    x1 = [Fraction(v) for v in a]
    x2 = [Fraction(v) for v in b]
    Z = Fraction(z0)
    prods = [(x1[1] * x2[2], x1[2] * x2[1]), (x1[2] * x2[0], x1[0] * x2[2]),
             (x1[0] * x2[1], x1[1] * x2[0])]
    n = [p - q for p, q in prods]
    kn = max(float((abs(p) + abs(q)) / abs(p - q)) if p != q else 0.0 for p, q in prods)
    S = n[0] ** 2 + n[1] ** 2
    D = (S + n[2] ** 2) * Z * Z
    z = float(z0)
    ax = (abs(t["Fx"] * z) + abs(t["eFx"] * z) + abs(t["ny"] * t["s"]) + abs(t["ey"] * t["s"])
          + abs(t["ny"] * t["es"]) + abs(t["ey"] * t["es"]))
    ay = (abs(t["Fy"] * z) + abs(t["eFy"] * z) + abs(t["nx"] * t["s"]) + abs(t["ex"] * t["s"])
          + abs(t["nx"] * t["es"]) + abs(t["ex"] * t["es"]))
    return kn, S, D, S - D, ax, ay


@pytest.mark.parametrize("config,n", [(1, 500), (2, 500), (3, 900), (6, 17 * 20), (7, 13 * 20)])
def test_double_word_first_order_bound(config, n):
    """The double-word point against the exact one, within the bound derived in DESIGN.md (R11)
    from the operator bounds the pieces carry — the numerator's CompDotC (Eq.5.1, 36u^2 A), the
    normal's AccuDOP ((1 + 2 kappa_n) u^2 per component), SumOfSquaresC,
    AccSqrt (25/8 u^2) plus the s^2 error carried into s ((S + D) / sigma), and the low
    part's own roundings:
        |hi + lo - P_c| <= 64 u^2 [ (A_c / S2)(1 + kappa_n) + |P| (1 + kappa_n + (S + D)/sigma) ]
    per coordinate c (higher-order terms dropped, as in Eq.BOUND).  A dropped or
    misplaced low-part term (the remainder t, the CompDot error dl, hi s2) is an O(u) error and
    fails it by a factor ~1e14."""
    a, b, z0 = sgi_inputs.generate_host(config, n)
    out, lo, cnt = oracle.intersect_dw(oracle.MODE_EFT, a, b, z0)
    worst, checked = 0.0, 0
    for i in range(n):
        c = int(cnt[i])
        used = c if c in (1, 2) else 0
        if not used:
            continue
        ex = exact.exact_query(a[:, i], b[:, i], z0[i])
        if ex.count != c:
            continue
        _, t = oracle.trace(oracle.MODE_EFT, a[:, i], b[:, i], z0[i])
        kn, S, D, sig, ax, ay = _first_order_bound_terms(a[:, i], b[:, i], z0[i], t)
        if sig <= 0:
            continue
        cond = float((S + D) / sig)
        for k in range(used):
            px, py, den = ex.points[k]
            pn = float((Fraction(px, den) ** 2 + Fraction(py, den) ** 2)) ** 0.5
            for d, num, A in ((0, px, ax), (1, py, ay)):
                err = abs(float(Fraction(out[k, d, i]) + Fraction(lo[k, d, i]) - Fraction(num, den)))
                bound = U * U * ((A / t["S2"]) * (1 + kn) + pn * (1 + kn + cond))
                worst = max(worst, err / bound)
                checked += 1
    assert checked > n // 2
    assert worst <= 64.0, worst
