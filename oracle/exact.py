"""oracle/exact.py — ORACLE (b): the closed form Eq.FINAL evaluated exactly.  TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py may import this module; it shares no code with
the CUDA path.

What it computes (PAPER.md, "Fast and Accurate Intersections on a Sphere"):
  * n = x1 x x2, S = |n_xy|^2, N = |n|^2, sigma = s^2 = S - N z0^2:
    polynomials in the 7 dyadic inputs, evaluated EXACTLY with Python integers (every double is
    m * 2^e, so all inputs are scaled to one common power of two).
  * Existence: intersections iff sigma >= 0, two iff sigma > 0 — exact signs.
  * Eq.FINAL: P+- = (-(z0 nx nz +- s ny)/S, -(z0 ny nz -+ s nx)/S, z0), both roots
    (P:923-931), with s = sqrt(sigma) to >= 400 bits (integer isqrt), so the reference point is
    accurate far below binary64's 2^-53.
  * Containment (points "must still be checked to ensure they lie between x1 and x2"):
    P lies on the closed minor arc iff (x1 x P).n >= 0 and (P x x2).n >= 0.  With
    g_k = nx y_k - ny x_k the identity P+-.(n x x_k) = (N/S)(z0 g_k -+ s z_k) holds, and the sign
    of z0 g_k -+ s z_k is decided without a square root: when both terms share a sign, it is
    sign(z0 g_k) * sign(D_k) because (z0 g_k)^2 - sigma z_k^2 = S D_k with
    D_k = z0^2 |x_k|^2 - z_k^2 (a polynomial identity, pinned in tests against brute force).
  * Degenerate inputs: n = 0 -> 0xFF; n_xy = 0 -> 0xFF if z0 = 0 else 0.
  * Error metric: |dP| = sqrt(dPx^2 + dPy^2); the build's ulp figure is
    err_u = |dP| / (2^-53 sqrt(1 - z0^2)) so that the paper's bound 3 sqrt(1-z0^2) u
    (Eq.BOUND) reads err_u <= 3.
"""
from __future__ import annotations

import math
from fractions import Fraction
from dataclasses import dataclass, field

U = 2.0 ** -53
DEGENERATE = 0xFF
SQRT_BITS = 420          # isqrt guard bits: s is accurate to ~2^-400 relative


def _split(x: float) -> tuple[int, int]:
    """x = m * 2^e with integer m (e <= 0 whenever x has a fractional part)."""
    p, q = float(x).as_integer_ratio()       # q is a power of two
    return p, -(q.bit_length() - 1)


@dataclass
class ExactResult:
    count: int                     # 0, 1, 2 or 0xFF (exact)
    sigma_sign: int                # sign of s^2 = S - N z0^2 (0 when degenerate)
    points: list = field(default_factory=list)   # [(num_x, num_y, den)] in arc order, exact-ish
    rounded: list = field(default_factory=list)  # [(RN(Px), RN(Py))] in arc order
    inside: tuple = (False, False)               # (P+ in arc, P- in arc)
    margins: tuple = ()            # |A-B|/(|A|+|B|) of the four deciding comparisons (floats)


class Query:
    """Exact integer model of one query (x1, x2, z0), all scaled by 2^L."""

    def __init__(self, x1, x2, z0):
        vals = [float(v) for v in (*x1, *x2, z0)]
        parts = [_split(v) for v in vals]
        L = max(0, max(-e for _, e in parts))
        ints = [m << (e + L) for m, e in parts]
        self.L = L
        self.X1 = ints[0:3]
        self.X2 = ints[3:6]
        self.Z = ints[6]
        self.z0 = vals[6]
        X1, X2 = self.X1, self.X2
        # n = x1 x x2 (scale 2^2L)
        self.n = (X1[1] * X2[2] - X1[2] * X2[1],
                  X1[2] * X2[0] - X1[0] * X2[2],
                  X1[0] * X2[1] - X1[1] * X2[0])
        nx, ny, nz = self.n
        self.S = nx * nx + ny * ny                     # scale 2^4L
        self.N = self.S + nz * nz                      # scale 2^4L
        self.sigma = (self.S << (2 * L)) - self.N * self.Z * self.Z   # scale 2^6L

    def g(self, k: int) -> int:
        """g_k = nx y_k - ny x_k (scale 2^3L)."""
        X = self.X1 if k == 1 else self.X2
        return self.n[0] * X[1] - self.n[1] * X[0]

    def D(self, k: int) -> int:
        """D_k = z0^2 |x_k|^2 - z_k^2 (scale 2^4L)."""
        X = self.X1 if k == 1 else self.X2
        return self.Z * self.Z * (X[0] ** 2 + X[1] ** 2 + X[2] ** 2) - (X[2] ** 2 << (2 * self.L))

    def s_scaled(self) -> tuple[int, int]:
        """(s_int, K) with s ~= s_int / 2^(3L + K), relative error < 2^-400."""
        if self.sigma <= 0:
            return 0, 0
        K = max(SQRT_BITS - self.sigma.bit_length() // 2, 0) + 64
        return math.isqrt(self.sigma << (2 * K)), K


def _sgn(v: int) -> int:
    return (v > 0) - (v < 0)


def _sign_diff(A: int, B_sign: int, D: int) -> int:
    """sign(A - B) given sign(A) exactly, sign(B), and A^2 - B^2 = S*D with S > 0."""
    sa = _sgn(A)
    if B_sign == 0:
        return sa
    if sa == 0:
        return -B_sign
    if sa != B_sign:
        return sa
    return sa * _sgn(D)


def exact_query(x1, x2, z0) -> ExactResult:
    """Exact count, containment and >=400-bit points of one query (see module docstring)."""
    q = Query(x1, x2, z0)
    nx, ny, nz = q.n
    if nx == 0 and ny == 0 and nz == 0:
        return ExactResult(DEGENERATE, 0)
    if q.S == 0:
        return ExactResult(DEGENERATE if q.Z == 0 else 0, 0)
    ss = _sgn(q.sigma)
    if ss < 0:
        return ExactResult(0, -1)
    g1, g2 = q.g(1), q.g(2)
    D1, D2 = q.D(1), q.D(2)
    A1, A2 = q.Z * g1, q.Z * g2                        # z0 g_k (scale 2^4L)
    z1s, z2s = _sgn(q.X1[2]), _sgn(q.X2[2])
    sgn_s = 1 if ss > 0 else 0
    # P+: z0 g1 - s z1 >= 0 and z0 g2 - s z2 <= 0;  P-: z0 g1 + s z1 >= 0 and z0 g2 + s z2 <= 0
    t1p = _sign_diff(A1, sgn_s * z1s, D1)
    t2p = _sign_diff(A2, sgn_s * z2s, D2)
    t1m = _sign_diff(A1, -sgn_s * z1s, D1)
    t2m = _sign_diff(A2, -sgn_s * z2s, D2)
    inp = t1p >= 0 and t2p <= 0
    inm = ss > 0 and t1m >= 0 and t2m <= 0
    count = int(inp) + int(inm)
    # high-precision points
    s_int, K = q.s_scaled()
    L = q.L
    den = q.S << (L + K)                               # P = -num / den
    base_x = (q.Z * nx * nz) << K                      # z0 nx nz at scale 2^(5L+K)
    base_y = (q.Z * ny * nz) << K
    Pp = (-(base_x + s_int * ny), -(base_y - s_int * nx), den)
    Pm = (-(base_x - s_int * ny), -(base_y + s_int * nx), den)
    order = []
    if count == 2:
        order = [Pp, Pm] if g1 >= 0 else [Pm, Pp]
    elif count == 1:
        order = [Pp if inp else Pm]
    res = ExactResult(count, ss, order, [(px / d, py / d) for px, py, d in order], (inp, inm))
    # margins of the deciding comparisons, for reporting count mismatches (floats are enough)
    # (integer / 2^k as a correctly rounded float: 2.0 ** k overflows for scaled inputs)
    def f2(num, k):
        return float(Fraction(num, 1 << k))
    sf = math.sqrt(f2(q.sigma, 6 * L)) if q.sigma > 0 else 0.0
    A1f, A2f = f2(A1, 4 * L), f2(A2, 4 * L)
    z1f, z2f = f2(q.X1[2], L), f2(q.X2[2], L)
    def margin(A, B):
        den_ = abs(A) + abs(B)
        return abs(A - B) / den_ if den_ > 0 else 0.0
    res.margins = (margin(A1f, sf * z1f), margin(A2f, sf * z2f),
                   margin(A1f, -sf * z1f), margin(A2f, -sf * z2f))
    return res


def point_error(p_tilde: tuple[float, float], p_exact: tuple[int, int, int]) -> float:
    """|P~ - P| with P~ a binary64 point and P = (num_x, num_y, den) exact-ish."""
    px, py, den = p_exact
    out = []
    for v, num in ((p_tilde[0], px), (p_tilde[1], py)):
        a, b = float(v).as_integer_ratio()
        out.append((a * den - b * num) / (b * den))
    return math.hypot(out[0], out[1])


def err_u(p_tilde, p_exact, z0: float) -> float:
    """err_u = |P~ - P| / (u sqrt(1 - z0^2)); Eq.BOUND is err_u <= 3."""
    scale = U * math.sqrt(max(0.0, (1.0 - z0) * (1.0 + z0)))
    e = point_error(p_tilde, p_exact)
    if scale == 0.0:
        return 0.0 if e == 0.0 else math.inf
    return e / scale


def check_query(x1, x2, z0, count: int, slots) -> dict:
    """Compare one computed result (count, [(x, y), (x, y)]) against the exact oracle."""
    ex = exact_query(x1, x2, z0)
    out = {"count_exact": ex.count, "count_match": ex.count == count, "err_u": [],
           "margins": ex.margins}
    if ex.count == count and count not in (0, DEGENERATE):
        for k in range(count):
            out["err_u"].append(err_u(slots[k], ex.points[k], z0))
    return out


# ------------------------------------------------------------------ independent cross-checks
def yac_points(x1, x2, z0, dps: int = 120):
    """Eq.YAC with the normalised normal, evaluated in mpmath at `dps` digits.

    A second transcription of the same geometry: on non-degenerate inputs it must
    agree with Eq.FINAL to far below 2^-53.  Returns [(Px, Py) of the +s root, of the -s root].
    """
    import mpmath as mp
    with mp.workdps(dps):
        a = [mp.mpf(float(v)) for v in x1]
        b = [mp.mpf(float(v)) for v in x2]
        z = mp.mpf(float(z0))
        n = [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]
        nn = mp.sqrt(n[0] ** 2 + n[1] ** 2 + n[2] ** 2)
        h = [c / nn for c in n]
        t2 = h[0] ** 2 + h[1] ** 2
        sh = mp.sqrt(t2 - z * z)
        out = []
        for sg in (1, -1):
            px = -(z * h[0] * h[2] + sg * sh * h[1]) / t2
            py = -(z * h[1] * h[2] - sg * sh * h[0]) / t2
            out.append((px, py))
        return out


def brute_force(x1, x2, z0, samples: int = 2001, dps: int = 60):
    """Count crossings of the latitude z = z0 along the arc by sampling + bisection.

    Independent of Eq.FINAL and of the containment identity: walks the normalised chord
    p(t) = (1-t) x1^ + t x2^ (t in [0,1], a monotone reparametrisation of the minor arc),
    records sign changes of z(p(t)/|p(t)|) - z0, bisects each, and returns
    (crossings in arc order as (Px, Py) mpf pairs, minimum |z - z0| seen on the grid).
    """
    import mpmath as mp
    with mp.workdps(dps):
        a = [mp.mpf(float(v)) for v in x1]
        b = [mp.mpf(float(v)) for v in x2]
        na = mp.sqrt(sum(c * c for c in a))
        nb = mp.sqrt(sum(c * c for c in b))
        a = [c / na for c in a]
        b = [c / nb for c in b]
        z = mp.mpf(float(z0))

        def f(t):
            p = [(1 - t) * a[i] + t * b[i] for i in range(3)]
            r = mp.sqrt(sum(c * c for c in p))
            return p[2] / r - z, p, r

        ts = [mp.mpf(i) / (samples - 1) for i in range(samples)]
        vals = [f(t)[0] for t in ts]
        crossings = []
        for i in range(samples - 1):
            v0, v1 = vals[i], vals[i + 1]
            if v0 == 0:
                t = ts[i]
            elif v0 * v1 < 0 or (v1 == 0 and i == samples - 2):
                lo, hi = ts[i], ts[i + 1]
                flo = v0
                for _ in range(dps * 4):
                    mid = (lo + hi) / 2
                    fm = f(mid)[0]
                    if fm == 0:
                        lo = hi = mid
                        break
                    if (fm < 0) == (flo < 0):
                        lo, flo = mid, fm
                    else:
                        hi = mid
                t = (lo + hi) / 2
            else:
                continue
            _, p, r = f(t)
            crossings.append((p[0] / r, p[1] / r))
        return crossings, min(abs(v) for v in vals)
