"""Pins for oracle (a)'s EFT operators (§5) against exact rational arithmetic.

Each operator is checked against what the paper (or the mathematics) fixes: exactness of the
error-free transformations, and the published error bounds of the compensated operators.  A
plausible transcription mistake (a dropped term, a wrong sign, a swapped operand) breaks one of
these.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from helpers import F, U, exact_sqrt, random_doubles, random_unit

RNG_SEED = 20251010
N = 20000


def _pairs(rng, n):
    a = random_doubles(rng, n)
    b = random_doubles(rng, n)
    # a slice of near and exact cancellations, zeros and equal magnitudes
    k = n // 8
    b[:k] = -a[:k] * (1 + rng.integers(-4, 5, k) * U)
    b[k:2 * k] = -a[k:2 * k]
    a[2 * k:2 * k + 10] = 0.0
    return a, b


# ---------------------------------------------------------------------------- SPEC examples
@pytest.mark.parametrize("name,row,expect", [
    ("two_sum", [1.0, 2.0 ** -60], (1.0, 2.0 ** -60)),
    ("two_sum", [3.5, 0.0], (3.5, 0.0)),
    ("fast_two_sum", [2.0, 1.0], (3.0, 0.0)),
    ("fast_two_sum", [1.0, 2.0 ** -53], (1.0, 2.0 ** -53)),          # S:55 (tie to even)
    ("two_prod", [134217729.0, 134217729.0], (18014398777917440.0, 1.0)),
    ("two_prod", [0.3, 1.0], (0.3, 0.0)),
    ("kahan_dop", [3.0, 2.0, 2.0, 3.0], (5.0, 0.0)),
    ("accu_dop", [0.7, 0.3, 0.7, 0.3], (0.0, 0.0)),                  # a*d - b*c with a=c, b=d
    ("accu_dop", [1.0, 0.0, 0.0, 1.0], (1.0, 0.0)),                  # a*d - b*c = 1
    ("sum_non_neg", [1.0, 0.0, 2.0, 0.0], (3.0, 0.0)),
    ("acc_sqrt", [4.0, 0.0], (2.0, 0.0)),
    ("acc_sqrt", [2.25, 0.0], (1.5, 0.0)),
    ("acc_sqrt", [0.0, 0.0], (0.0, 0.0)),                            # S:141 (H = 0)
])
def test_spec_examples(name, row, expect):
    out = oracle.prim(name, np.array([row]))
    assert tuple(out[0]) == expect


@pytest.mark.parametrize("name,k,row,expect", [
    ("sum_of_squares", 2, [3.0, 4.0], (25.0, 0.0)),
    ("sum_of_squares", 3, [0.0, 0.0, 1.0], (1.0, 0.0)),
    ("sum_of_squares_c", 2, [3.0, 4.0, 0.0, 0.0], (25.0, 0.0)),
    ("sum_of_squares_c", 3, [1.0, 0.0, 0.0, 0.0, 0.0, 0.0], (1.0, 0.0)),
    ("comp_dot_c", 1, [1.0, 1.0], (1.0, 0.0)),
    ("comp_dot_c", 2, [2.0, 3.0, 3.0, -2.0], (0.0, 0.0)),
    ("comp_dot", 1, [7.0, 0.0], (0.0, 0.0)),
])
def test_spec_vector_examples(name, k, row, expect):
    out = oracle.prim(name, np.array([row]), k)
    assert tuple(out[0]) == expect


# ------------------------------------------------------------------------- exactness (E1-E3)
@pytest.mark.parametrize("name", ["two_sum", "two_prod"])
def test_eft_exactness(name):
    rng = np.random.default_rng(RNG_SEED)
    a, b = _pairs(rng, N)
    out = oracle.prim(name, np.stack([a, b], 1))
    for x, y, (hi, lo) in zip(a, b, out):
        exact = F(x) + F(y) if name == "two_sum" else F(x) * F(y)
        assert F(hi) + F(lo) == exact
        assert hi == float(exact)            # hi = RN(a o b): the pair is normalised


def test_fast_two_sum_exactness_with_precondition():
    rng = np.random.default_rng(RNG_SEED + 1)
    a, b = _pairs(rng, N)
    swap = np.abs(a) < np.abs(b)
    a2, b2 = np.where(swap, b, a), np.where(swap, a, b)
    out = oracle.prim("fast_two_sum", np.stack([a2, b2], 1))
    for x, y, (hi, lo) in zip(a2, b2, out):
        assert F(hi) + F(lo) == F(x) + F(y)


# --------------------------------------------------------------- compensated-operator bounds
def _unit_quads(rng, n):
    """Components of random unit vectors, as the cross product feeds them."""
    x1, x2 = random_unit(rng, n), random_unit(rng, n)
    # near-parallel pairs give the heavy cancellations the bound is about
    k = n // 4
    x2[:k] = x1[:k] + 1e-9 * random_unit(rng, k)
    return x1, x2


def test_accu_dop_bound_and_printed_sign_typo():
    """AccuDOP (Alg.4): |err| <= (1 + 2(|ad|+|bc|)/|ad-bc|) u^2 |ad-bc| + O(u^3).

    Reading R1: the residual is r1 - r2.  The printed r1 + r2 must violate the bound,
    which is how this test tells the two apart."""
    rng = np.random.default_rng(RNG_SEED + 2)
    x1, x2 = _unit_quads(rng, N)
    a, b, c, d = x1[:, 1], x1[:, 2], x2[:, 1], x2[:, 2]
    out = oracle.prim("accu_dop", np.stack([a, b, c, d], 1))
    worst = 0.0
    printed_violations = 0
    for i in range(N):
        ad, bc = F(a[i]) * F(d[i]), F(b[i]) * F(c[i])
        exact = ad - bc
        got = F(out[i, 0]) + F(out[i, 1])
        if exact == 0:
            assert got == 0
            continue
        bound = (1 + 2 * (abs(ad) + abs(bc)) / abs(exact)) * Fraction(U) ** 2 * abs(exact)
        ratio = abs(got - exact) / bound
        worst = max(worst, float(ratio))
        # the printed variant err = s + (r1 + r2)
        p1, p2 = a[i] * d[i], b[i] * c[i]
        r1 = F(a[i]) * F(d[i]) - F(p1)
        r2 = F(b[i]) * F(c[i]) - F(p2)
        dop = p1 - p2
        s = (F(p1) - F(p2)) - F(dop)
        printed = F(dop) + F(float(s) + float(float(r1) + float(r2)))
        if abs(printed - exact) > bound * (1 + 64 * U):
            printed_violations += 1
    assert worst <= 1 + 64 * U, worst
    assert printed_violations > N // 10


def test_kahan_dop_bound():
    """Kahan's DiffOfProd (Alg.3): relative error <= 2u."""
    rng = np.random.default_rng(RNG_SEED + 3)
    x1, x2 = _unit_quads(rng, N // 4)
    a, b, c, d = x1[:, 0], x1[:, 1], x2[:, 1], x2[:, 0]
    out = oracle.prim("kahan_dop", np.stack([a, b, c, d], 1))
    for i in range(len(a)):
        exact = F(a[i]) * F(d[i]) - F(b[i]) * F(c[i])
        err = abs(F(out[i, 0]) - exact)
        assert err <= 2 * Fraction(U) * abs(exact) * (1 + 8 * Fraction(U))


def _gamma(n):
    return n * Fraction(U) / (1 - n * Fraction(U))


@pytest.mark.parametrize("n", [2, 4, 6])
def test_comp_dot_bounds(n):
    """CompDotC Eq.5.1 and CompDot Eq.5.2."""
    rng = np.random.default_rng(RNG_SEED + 10 + n)
    m = 4000
    x = random_doubles(rng, m * n, -20, 20).reshape(m, n)
    y = random_doubles(rng, m * n, -20, 20).reshape(m, n)
    # ill-conditioned rows: make the last product cancel the rest
    for i in range(m // 2):
        partial = sum(F(x[i, j]) * F(y[i, j]) for j in range(n - 1))
        y[i, n - 1] = -float(partial) / x[i, n - 1]
    rows = np.concatenate([x, y], 1)
    cdc = oracle.prim("comp_dot_c", rows, n)
    cd = oracle.prim("comp_dot", rows, n)
    u = Fraction(U)
    for i in range(m):
        exact = sum(F(x[i, j]) * F(y[i, j]) for j in range(n))
        absdot = sum(abs(F(x[i, j]) * F(y[i, j])) for j in range(n))
        bound_c = _gamma(n) * n * u / (1 - (n - 1) * u) * absdot
        assert abs(F(cdc[i, 0]) + F(cdc[i, 1]) - exact) <= bound_c
        assert abs(F(cd[i, 0]) - exact) <= u * abs(exact) + bound_c


def test_sum_non_neg_bound():
    """SumNonNeg (Alg.6): relative error <= 3u^2 for normalised inputs."""
    rng = np.random.default_rng(RNG_SEED + 4)
    A = np.abs(random_doubles(rng, N, -10, 10))
    B = np.abs(random_doubles(rng, N, -10, 10))
    a = A * rng.uniform(-1, 1, N) * U
    b = B * rng.uniform(-1, 1, N) * U
    out = oracle.prim("sum_non_neg", np.stack([A, a, B, b], 1))
    u2 = Fraction(U) ** 2
    for i in range(N):
        exact = F(A[i]) + F(a[i]) + F(B[i]) + F(b[i])
        got = F(out[i, 0]) + F(out[i, 1])
        assert abs(got - exact) <= 3 * u2 * exact
        assert abs(out[i, 1]) <= U * abs(out[i, 0])           # FastTwoSum output is normalised


@pytest.mark.parametrize("k,coef", [(2, 3), (3, 6)])
def test_sum_of_squares_bound(k, coef):
    """SumOfSquares (Alg.5): 3u^2 (n=2) and 6u^2 (n=3)."""
    rng = np.random.default_rng(RNG_SEED + 20 + k)
    x = random_unit(rng, N)[:, :k] * rng.uniform(0.5, 1.0, (N, 1))
    out = oracle.prim("sum_of_squares", x, k)
    u2 = Fraction(U) ** 2
    for i in range(N):
        exact = sum(F(v) ** 2 for v in x[i])
        assert abs(F(out[i, 0]) + F(out[i, 1]) - exact) <= coef * u2 * exact


@pytest.mark.parametrize("k,coef", [(2, 3), (3, 6)])
def test_sum_of_squares_c_bound(k, coef):
    """SumOfSquaresC (Alg.7) on compensated vectors from real cross products
    (renormalised AccuDOP pairs, |e| <= u|x|): relative error vs sum (x+e)^2 within the
    S2 bounds, checked as coef*u^2 with slack 2 (SPEC acceptance 3)."""
    rng = np.random.default_rng(RNG_SEED + 30 + k)
    x1, x2 = _unit_quads(rng, N // 2)
    comps = []
    for (i, j) in ((1, 2), (2, 0), (0, 1))[:k]:
        pr = oracle.prim("accu_dop", np.stack([x1[:, i], x1[:, j], x2[:, i], x2[:, j]], 1))
        pr = oracle.prim("two_sum", pr)      # renormalise (reading R6)
        comps.append(pr)
    xs = np.stack([c[:, 0] for c in comps], 1)
    es = np.stack([c[:, 1] for c in comps], 1)
    out = oracle.prim("sum_of_squares_c", np.concatenate([xs, es], 1), k)
    u2 = Fraction(U) ** 2
    for i in range(len(xs)):
        exact = sum((F(xs[i, j]) + F(es[i, j])) ** 2 for j in range(k))
        if exact == 0:
            continue
        assert abs(F(out[i, 0]) + F(out[i, 1]) - exact) <= 2 * coef * u2 * exact


def test_acc_sqrt_bound():
    """AccSqrt (bound 25/8 u^2 P:826) for normalised (H, h), |h| <= u H."""
    rng = np.random.default_rng(RNG_SEED + 5)
    H = np.abs(random_doubles(rng, N, -60, 10))
    h = H * rng.uniform(-1, 1, N) * U
    out = oracle.prim("acc_sqrt", np.stack([H, h], 1))
    for i in range(N):
        exact = exact_sqrt(F(H[i]) + F(h[i]))
        got = F(out[i, 0]) + F(out[i, 1])
        assert abs(got - exact) <= Fraction(25, 8) * Fraction(U) ** 2 * exact * (1 + 64 * Fraction(U))
