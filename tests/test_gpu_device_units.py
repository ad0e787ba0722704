"""Device unit tests of the EFT primitives (tests/native/devtests.cu), bitwise on the B200:
the ordered-FastTwoSum TwoSum equals Knuth's TwoSum and is exact; the AccuDOP renormalisation
as a FastTwoSum equals Knuth's TwoSum (cancelling quadruples included); the high-word sign and
zero tests equal the double comparisons; the shared-reciprocal
division and the fast-path sqrt equal __ddiv_rn / __dsqrt_rn whenever their guards pass."""
import ctypes

import pytest

torch = pytest.importorskip("torch")
from paper_2510_09892_b200._build import build_devtests  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_primitives_bitwise_on_device(seed):
    lib = ctypes.CDLL(build_devtests())
    lib.sgi_devtest.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p]
    out = torch.zeros(10, dtype=torch.int64, device="cuda")
    n = 1 << 24
    assert lib.sgi_devtest(seed, n, ctypes.c_void_p(out.data_ptr())) == 0
    c = out.cpu().tolist()
    assert c[0] == 0, f"two_sum value mismatches: {c}"
    assert c[2] == 0, f"two_sum not exact: {c}"
    assert c[3] == 0, f"div mismatches: {c}"
    assert c[5] == 0, f"sqrt mismatches: {c}"
    assert c[7] == 0, f"AccuDOP renormalisation: FastTwoSum != TwoSum: {c}"
    assert c[8] > n // 64, f"too few cancelling AccuDOP cases exercised: {c}"
    assert c[9] == 0, f"is_zero/is_pos/is_neg/is_nonneg != double comparisons: {c}"
    # the guards do fire on the tiny numerators / radicands the test feeds on purpose
    assert c[4] > 0 and c[6] > 0


# ------------------------------------------ device primitives vs oracle (a), op by op
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from helpers import random_doubles  # noqa: E402

PRIM_ROWS = {            # name: (width, k, exponent range of the entries)
    "two_sum": (2, 0, (-200, 200)), "fast_two_sum": (2, 0, (-200, 200)),
    "two_prod": (2, 0, (-200, 200)), "kahan_dop": (4, 0, (-100, 100)),
    "accu_dop": (4, 0, (-100, 100)), "sum_non_neg": (4, 0, (-100, 100)),
    "sum_of_squares": (3, 3, (-60, 60)), "sum_of_squares_c": (6, 3, (-60, 60)),
    "acc_sqrt": (2, 0, (-300, 300)), "comp_dot_c": (12, 6, (-60, 60)),
    "comp_dot": (12, 6, (-60, 60)),
}


def _rows(name, n, rng):
    width, k, (lo, hi) = PRIM_ROWS[name]
    r = random_doubles(rng, n * width, lo, hi).reshape(n, width)
    if name == "fast_two_sum":                     # its precondition: |a| >= |b|
        big = np.maximum(np.abs(r[:, 0]), np.abs(r[:, 1]))
        small = np.minimum(np.abs(r[:, 0]), np.abs(r[:, 1]))
        r[:, 0] = big * np.sign(r[:, 0]); r[:, 1] = small * np.sign(r[:, 1])
    if name in ("accu_dop", "kahan_dop"):          # a*b close to c*d for a third of the rows
        m = rng.random(n) < 1 / 3
        r[m, 3] = r[m, 0] * r[m, 1] / r[m, 2] * (1 + rng.integers(-4, 5, m.sum()) * 2.0 ** -52)
    if name == "sum_non_neg":                      # two non-negative pairs (hi, lo), |lo| <= u|hi|
        r[:, 0] = np.abs(r[:, 0]); r[:, 2] = np.abs(r[:, 2])
        r[:, 1] = r[:, 0] * rng.uniform(-1, 1, n) * 2.0 ** -54
        r[:, 3] = r[:, 2] * rng.uniform(-1, 1, n) * 2.0 ** -54
    if name == "sum_of_squares_c":                 # (x, e) with |e| <= u |x|
        r[:, 3:] = r[:, :3] * rng.uniform(-1, 1, (n, 3)) * 2.0 ** -53
    if name == "acc_sqrt":                         # (H, h) with |h| <= u|H|, some H <= 0
        r[:, 1] = r[:, 0] * rng.uniform(-1, 1, n) * 2.0 ** -53
        r[:, 0] = np.where(rng.random(n) < 0.9, np.abs(r[:, 0]), r[:, 0])
        r[: n // 50, 0] = 0.0
    return np.ascontiguousarray(r), k


@pytest.mark.parametrize("name", list(PRIM_ROWS))
def test_device_primitives_equal_oracle(name):
    lib = ctypes.CDLL(build_devtests())
    lib.sgi_devprim.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]
    rng = np.random.default_rng(hash(name) % 2**32)
    n = 200_000
    rows, k = _rows(name, n, rng)
    ref = oracle.prim(name, rows, k)
    din = torch.from_numpy(rows).cuda()
    for fast in ((0, 1) if name == "acc_sqrt" else (0,)):
        dout = torch.empty((n, 2), dtype=torch.float64, device="cuda")
        assert lib.sgi_devprim(oracle.PRIM[name], k, ctypes.c_void_p(din.data_ptr()), rows.shape[1],
                               n, ctypes.c_void_p(dout.data_ptr()), fast) == 0
        got = dout.cpu().numpy()
        keep = ~np.isnan(got[:, 1]) if fast else np.ones(n, bool)
        assert keep.mean() > 0.97
        same = (got[keep] == ref[keep]) | (np.isnan(got[keep]) & np.isnan(ref[keep]))
        assert same.all(), f"{name} fast={fast}: {int((~same).sum())} values differ"


# ---------------------------------- certified numerators (policy Cert, DESIGN.md §5 L7)
U = 2.0 ** -53


def cert_rows(n, rng, near_ties):
    """Rows [F, eF, v, ev, z0, s, es] with SGI_MODE_EFT's magnitude relations (|eF| <= 3u|F|,
    |ev| <= u|v|, |es| <= 1.5u|s|) and spread exponents; with near_ties, es is re-chosen (exact
    rationals) so that the + root's exact dot product V = (F + eF) z0 + (v + ev)(s + es) lies
    within ~u^2 |v s| of a rounding boundary of X+ (a midpoint between adjacent doubles): the
    regime where the guard must fail or be right."""
    from fractions import Fraction as Fr
    import math
    F = rng.uniform(0.5, 1, n) * 2.0 ** rng.integers(-40, 10, n) * rng.choice([-1, 1], n)
    z0 = rng.uniform(-1, 1, n)
    v = rng.uniform(0.5, 1, n) * 2.0 ** rng.integers(-40, 10, n) * rng.choice([-1, 1], n)
    s = np.abs(F * z0 / v) * rng.uniform(0.01, 4, n)      # v s comparable to F z0: cancellations
    eF = F * rng.uniform(-3, 3, n) * U
    ev = v * rng.uniform(-1, 1, n) * U
    es = s * rng.uniform(-1, 1, n) * U
    if near_ties:
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
    return np.ascontiguousarray(np.stack([F, eF, v, ev, z0, s, es], axis=1))


@pytest.mark.parametrize("op", [11, 12, 14])
@pytest.mark.parametrize("near_ties", [False, True])
def test_certified_numerators_equal_compdot(op, near_ties):
    """Policy Cert's numerators either equal the paper's CompDot (oracle (a), bit for bit) or
    report failure (then the query is recomputed with the listing's sequence); near ties the
    guard must fire, so the test also checks that it does.  op 12 runs the two-lane (W2) type,
    op 14 the one-root form (the - root through negated s, es), each root certified alone."""
    lib = ctypes.CDLL(build_devtests())
    lib.sgi_devprim.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]
    rng = np.random.default_rng(11 + near_ties)
    n = 20_000 if near_ties else 400_000
    rows = cert_rows(n, rng, near_ties)
    F, eF, v, ev, z0, s, es = rows.T
    w = np.stack([z0, z0, s, s, es, es], axis=1)
    ref = np.empty((n, 2))
    for k, sg in enumerate((1.0, -1.0)):
        x = np.stack([F, eF, sg * v, sg * ev, sg * v, sg * ev], axis=1)
        ref[:, k] = oracle.prim("comp_dot", np.ascontiguousarray(np.hstack([x, w])), 6)[:, 0]
    din = torch.from_numpy(rows).cuda()
    dout = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    assert lib.sgi_devprim(op, 0, ctypes.c_void_p(din.data_ptr()), 7, n,
                           ctypes.c_void_p(dout.data_ptr()), 0) == 0
    got = dout.cpu().numpy()
    ok = ~np.isnan(got)
    same = (got[ok] == ref[ok])
    assert same.all(), f"{int((~same).sum())} certified numerators differ from CompDot"
    fired = (~ok).any(axis=1)
    if near_ties:
        assert fired.mean() > 0.2, f"guard fired on only {fired.mean():.3f} of near-tie rows"
    else:
        assert fired.mean() < 0.001


def cert_front_rows(n, rng, target):
    """Rows [nx, ex, ny, ey, nz, ez, z0] shaped like SGI_MODE_EFT's renormalised normal pairs
    (|e| <= u|n|) with z0 inside the circle's z-range.  target "S2" / "sigma": ey / ez re-chosen
    (exact rationals) so that nx^2 + ny^2 + 2(nx ex + ny ey) -- resp. that minus
    (|n|^2 + 2 n.e) z0^2 -- lies within ~u^2 of a rounding boundary of the listing's rounded
    |n_xy|^2 -- resp. s^2 -- where the certificate must fail or be right."""
    from fractions import Fraction as Fr
    import math
    n3 = rng.normal(size=(n, 3)) * 2.0 ** rng.integers(-30, 1, (n, 1))
    n3[:, 2] *= rng.uniform(0.5, 2.0, n)
    e3 = n3 * rng.uniform(-1, 1, (n, 3)) * U
    S = n3[:, 0] ** 2 + n3[:, 1] ** 2
    N = S + n3[:, 2] ** 2
    z0 = rng.uniform(-1, 1, n) * np.sqrt(S / N)
    if target is not None:
        for i in range(n):
            nx, ny, nz = (Fr(v) for v in n3[i])
            ex, ey, ez = (Fr(v) for v in e3[i])
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
                sig = S2 - (S2 + nz * nz + 2 * nz * ez) * z2
                h = float(sig)
                if h <= 0 or z2 == 0 or nz == 0:
                    continue
                m = Fr(h) + sgn * Fr(math.ulp(h)) / 2
                rest = S2 - (S2 + nz * nz) * z2
                new = float((rest - m) / (2 * nz * z2))
                if abs(new) <= U * abs(n3[i, 2]):
                    e3[i, 2] = new
    return np.ascontiguousarray(np.stack([n3[:, 0], e3[:, 0], n3[:, 1], e3[:, 1], n3[:, 2],
                                          e3[:, 2], z0], axis=1))


def listing_front(rows):
    """The listing's S2 and s^2 high part (AccuX lines 5-11) from oracle (a)'s operators."""
    nx, ex, ny, ey, nz, ez, z0 = rows.T
    S2 = oracle.prim("sum_of_squares_c", np.ascontiguousarray(np.stack([nx, ny, ex, ey], 1)), 2)
    S3 = oracle.prim("sum_of_squares_c",
                     np.ascontiguousarray(np.stack([nx, ny, nz, ex, ey, ez], 1)), 3)
    C = oracle.prim("two_prod", np.ascontiguousarray(np.stack([z0, z0], 1)))
    D = oracle.prim("comp_dot_c", np.ascontiguousarray(np.stack(
        [S3[:, 0], S3[:, 0], S3[:, 1], S3[:, 1], C[:, 0], C[:, 1], C[:, 0], C[:, 1]], 1)), 4)
    E = oracle.prim("two_sum", np.ascontiguousarray(np.stack([S2[:, 0], -D[:, 0]], 1)))
    e = (S2[:, 1] - D[:, 1]) + E[:, 1]
    sig = oracle.prim("fast_two_sum", np.ascontiguousarray(np.stack([E[:, 0], e], 1)))
    return S2[:, 0], sig[:, 0]


@pytest.mark.parametrize("target", [None, "S2", "sigma"])
def test_certified_front_equals_listing(target):
    """Policy Cert's |n_xy|^2 high part and s^2 high part either equal the listing's
    (SumOfSquaresC, CompDotC, TwoSum chain of AccuX lines 5-11 by oracle (a)'s operators) bit
    for bit or report failure; rows placed at rounding boundaries must make the certificate
    fire."""
    lib = ctypes.CDLL(build_devtests())
    lib.sgi_devprim.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]
    rng = np.random.default_rng({None: 21, "S2": 22, "sigma": 23}[target])
    n = 400_000 if target is None else 20_000
    rows = cert_front_rows(n, rng, target)
    S2, sh = listing_front(rows)
    din = torch.from_numpy(rows).cuda()
    dout = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    assert lib.sgi_devprim(13, 0, ctypes.c_void_p(din.data_ptr()), 7, n,
                           ctypes.c_void_p(dout.data_ptr()), 0) == 0
    got = dout.cpu().numpy()
    ok = ~np.isnan(got[:, 0])
    assert (got[ok, 0] == S2[ok]).all(), int((got[ok, 0] != S2[ok]).sum())
    assert (got[ok, 1] == sh[ok]).all(), int((got[ok, 1] != sh[ok]).sum())
    if target is None:
        assert ok.mean() > 0.999
    else:
        assert (~ok).mean() > 0.2, f"certificate fired on only {(~ok).mean():.3f} of the rows"
