"""Policy Cert's certificates (DESIGN.md §5 L7-L8, reading R12) emulated on the CPU with exactly
rounded binary64 operations (Python floats; fma through exact rationals), against oracle (a)'s
operators.  This pins the mathematics of the certificates independently of the GPU:
  * the cheap evaluations stay inside the proven budgets (numerators: |T' - V| <= 26.9 u^2 A and
    the listing's |p + sigma - V| <= 36.01 u^2 A, Eq.5.1; |n_xy|^2: |T' - T_o| <= 19.2 u^2 S;
    s^2: |T' - T_o| <= 75.3 u^2 (S + D));
  * wherever a certificate passes, the certified value equals the listing's bit for bit, also on
    rows placed on rounding boundaries (where the certificates must and do fire).
The device code is the same op sequence (tests/test_gpu_device_units.py runs it on the B200)."""
import math
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle

U = 2.0 ** -53
UF = Fr(U)


def fma(a, b, c):
    return float(Fr(a) * Fr(b) + Fr(c))


def tp(a, b):
    p = a * b
    return p, fma(a, b, -p)


def ts(a, b):
    s = a + b
    v = s - a
    return s, (a - (s - v)) + (b - v)


def fts(a, b):
    s = a + b
    return s, b - (s - a)


def numerators_cert(F, eF, v, ev, z0, s, es):
    """Emulation of sgi_query.cuh numerators_cert (es_dev = 0): (X+, X-) or None per root, and
    the unevaluated sums H + sigma'."""
    P1, e1 = tp(F, z0)
    P3, e3 = tp(v, s)
    c = fma(eF, z0, e1)
    w = fma(ev, es, fma(v, es, fma(ev, s, e3)))
    M2 = (abs(P1) + abs(P3)) * 2.0 ** -97
    out, sums = [], []
    for sg in (1.0, -1.0):
        H, q = ts(P1, sg * P3)
        sig = (q + c) + sg * w
        up, dn = H + (sig + M2), H + (sig - M2)
        out.append(up if up - dn == 0 else None)
        sums.append(Fr(H) + Fr(sig))
    return out, sums, abs(P1) + abs(P3)


def numerator_cert_one(F, eF, v, ev, z0, s, es):
    """Emulation of sgi_query.cuh numerator_cert_one (es_dev = 0): one root, its sign folded
    into s and es."""
    P1, e1 = tp(F, z0)
    P3, e3 = tp(v, s)
    c = fma(eF, z0, e1)
    w = fma(ev, es, fma(v, es, fma(ev, s, e3)))
    M2 = (abs(P1) + abs(P3)) * 2.0 ** -97
    H, q = ts(P1, P3)
    sig = (q + c) + w
    up, dn = H + (sig + M2), H + (sig - M2)
    return up if up - dn == 0 else None


def cert_front(nx, ex, ny, ey, nz, ez, z0):
    """Emulation of cert_sums + cert_sigma: (S2 or None, sigma_h or None) and the sums."""
    a2, b2, c2 = tp(nx, nx), tp(ny, ny), tp(nz, nz)
    Q2 = ts(a2[0], b2[0])
    l = (a2[1] + b2[1]) + Q2[1]
    R2 = fma(nx, ex, ny * ey)
    Q3 = ts(Q2[0], c2[0])
    R3 = fma(nz, ez, R2)
    l2 = fma(2.0, R2, l)
    l3 = fma(2.0, R3, (l + c2[1]) + Q3[1])
    m2 = Q2[0] * 2.0 ** -98
    S2 = Q2[0] + (l2 + m2)
    ok2 = S2 - (Q2[0] + (l2 - m2)) == 0
    S2l = l2 - (S2 - Q2[0])
    C = tp(z0, z0)
    d1 = tp(Q3[0], C[0])
    Ds = fma(Q3[0], C[1], fma(l3, C[0], d1[1]))
    E = fts(S2, -d1[0])
    e = (S2l - Ds) + E[1]
    ms = (S2 + d1[0]) * 2.0 ** -97
    sh = E[0] + (e + ms)
    oks = sh - (E[0] + (e - ms)) == 0
    return (S2 if ok2 else None, sh if (ok2 and oks) else None,
            Fr(Q2[0]) + Fr(l2), Fr(E[0]) + Fr(e))


def numerator_rows(rng, n, near_ties):
    F = rng.uniform(0.5, 1, n) * 2.0 ** rng.integers(-40, 10, n) * rng.choice([-1, 1], n)
    z0 = rng.uniform(-1, 1, n)
    v = rng.uniform(0.5, 1, n) * 2.0 ** rng.integers(-40, 10, n) * rng.choice([-1, 1], n)
    s = np.abs(F * z0 / v) * rng.uniform(0.01, 4, n)
    eF = F * rng.uniform(-3, 3, n) * U
    ev = v * rng.uniform(-1, 1, n) * U
    es = s * rng.uniform(-1, 1, n) * U
    if near_ties:          # move V onto a midpoint of X+ through es (exact rationals)
        for i in range(n):
            K = (Fr(F[i]) + Fr(eF[i])) * Fr(z0[i]) + (Fr(v[i]) + Fr(ev[i])) * Fr(s[i])
            cv = Fr(v[i]) + Fr(ev[i])
            X0 = float(K + cv * Fr(es[i]))
            if X0 == 0.0:
                continue
            m = Fr(X0) + Fr(math.ulp(X0)) / 2 * (1 if rng.random() < 0.5 else -1)
            e2 = float((m - K) / cv)
            if abs(e2) <= 1.5 * U * abs(s[i]):
                es[i] = e2
    return np.stack([F, eF, v, ev, z0, s, es], axis=1)


@pytest.mark.parametrize("near_ties", [False, True])
def test_numerator_certificate(near_ties):
    rng = np.random.default_rng(31 + near_ties)
    rows = numerator_rows(rng, 1500, near_ties)
    F, eF, v, ev, z0, s, es = rows.T
    w = np.stack([z0, z0, s, s, es, es], axis=1)
    fired = 0
    for sg, k in ((1.0, 0), (-1.0, 1)):
        x = np.stack([F, eF, sg * v, sg * ev, sg * v, sg * ev], axis=1)
        xw = np.ascontiguousarray(np.hstack([x, w]))
        X = oracle.prim("comp_dot", xw, 6)[:, 0]
        pc = oracle.prim("comp_dot_c", xw, 6)
        for i in range(len(F)):
            got, sums, A = numerators_cert(*rows[i])
            V = sum(Fr(x[i, j]) * Fr(w[i, j]) for j in range(6))
            A = Fr(A)
            assert abs(sums[k] - V) <= Fr(269, 10) * UF * UF * A          # E' <= 26.9 u^2 A
            assert abs(Fr(pc[i, 0]) + Fr(pc[i, 1]) - V) <= Fr(3601, 100) * UF * UF * A   # Eq.5.1
            if got[k] is None:
                fired += 1
            else:
                assert got[k] == X[i], (i, k)
    if near_ties:
        assert fired > 300
    else:
        assert fired == 0


@pytest.mark.parametrize("near_ties", [False, True])
def test_one_root_numerator_is_the_two_root_one(near_ties):
    """L10: the - root's certified numerator computed as the + root's with s and e_s negated
    (TwoProd(v, -s) = -TwoProd(v, s), RN odd) equals the two-root form bit for bit, certificate
    decision included — also on rows placed on rounding boundaries."""
    rng = np.random.default_rng(41 + near_ties)
    rows = numerator_rows(rng, 3000, near_ties)
    fired = 0
    for r in rows:
        both, _, _ = numerators_cert(*r)
        F, eF, v, ev, z0, s, es = r
        one = (numerator_cert_one(F, eF, v, ev, z0, s, es),
               numerator_cert_one(F, eF, v, ev, z0, -s, -es))
        for k in range(2):
            assert (one[k] is None) == (both[k] is None)
            if one[k] is not None:
                assert math.copysign(1.0, one[k]) == math.copysign(1.0, both[k]) and one[k] == both[k]
            fired += one[k] is None
    assert (fired > 300) if near_ties else fired == 0


def front_rows(rng, n, target):
    n3 = rng.normal(size=(n, 3)) * 2.0 ** rng.integers(-30, 1, (n, 1))
    e3 = n3 * rng.uniform(-1, 1, (n, 3)) * U
    S = n3[:, 0] ** 2 + n3[:, 1] ** 2
    z0 = rng.uniform(-1, 1, n) * np.sqrt(S / (S + n3[:, 2] ** 2))
    for i in range(n if target else 0):
        nx, ny, nz = (Fr(t) for t in n3[i])
        ex, ey, ez = (Fr(t) for t in e3[i])
        z2 = Fr(z0[i]) ** 2
        S2 = nx * nx + ny * ny + 2 * (nx * ex + ny * ey)
        sgn = 1 if rng.random() < 0.5 else -1
        if target == "S2":
            h = float(S2)
            m = Fr(h) + sgn * Fr(math.ulp(h)) / 2
            new = float((m - nx * nx - ny * ny - 2 * nx * ex) / (2 * ny))
            if abs(new) <= U * abs(n3[i, 1]):
                e3[i, 1] = new
        else:
            h = float(S2 - (S2 + nz * nz + 2 * nz * ez) * z2)
            if h <= 0 or z2 == 0 or nz == 0:
                continue
            m = Fr(h) + sgn * Fr(math.ulp(h)) / 2
            new = float((S2 - (S2 + nz * nz) * z2 - m) / (2 * nz * z2))
            if abs(new) <= U * abs(n3[i, 2]):
                e3[i, 2] = new
    return np.stack([n3[:, 0], e3[:, 0], n3[:, 1], e3[:, 1], n3[:, 2], e3[:, 2], z0], axis=1)


@pytest.mark.parametrize("target", [None, "S2", "sigma"])
def test_front_certificates(target):
    rng = np.random.default_rng({None: 41, "S2": 42, "sigma": 43}[target])
    rows = front_rows(rng, 1200, target)
    nx, ex, ny, ey, nz, ez, z0 = rows.T
    S2o = oracle.prim("sum_of_squares_c", np.ascontiguousarray(np.stack([nx, ny, ex, ey], 1)), 2)
    S3o = oracle.prim("sum_of_squares_c",
                      np.ascontiguousarray(np.stack([nx, ny, nz, ex, ey, ez], 1)), 3)
    fired = 0
    for i in range(len(z0)):
        C = tp(z0[i], z0[i])
        Do = oracle.prim("comp_dot_c", np.array([[S3o[i, 0], S3o[i, 0], S3o[i, 1], S3o[i, 1],
                                                  C[0], C[1], C[0], C[1]]]), 4)[0]
        Eo = ts(S2o[i, 0], -Do[0])
        eo = (S2o[i, 1] - Do[1]) + Eo[1]
        sho = Eo[0] + eo
        S2c, shc, T2, Ts = cert_front(*rows[i])
        S = Fr(nx[i]) ** 2 + Fr(ny[i]) ** 2
        D = (S + Fr(nz[i]) ** 2) * Fr(z0[i]) ** 2
        assert abs(T2 - (Fr(S2o[i, 0]) + Fr(S2o[i, 1]))) <= Fr(192, 10) * UF * UF * S
        if S2c is not None:
            assert S2c == S2o[i, 0]
            assert abs(Ts - (Fr(Eo[0]) + Fr(eo))) <= Fr(753, 10) * UF * UF * (S + D)
        if shc is None:
            fired += 1
        else:
            assert shc == sho, i
    if target is None:
        assert fired <= 2
    else:
        assert fired > 150
