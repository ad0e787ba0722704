"""GPU tests of the fused zonal-mean pass (sgi_zonal_intersect).

  * the candidate filter is conservative: every (edge, latitude) with a nonzero count under
    brute force (oracle (a) on ALL pairs) is a candidate;
  * every candidate's count and points equal oracle (a) on that pair (parity up to the sign of
    zero) — i.e. the fused head/tail split is the plain query;
  * candidates with count 0 sit within 2 * 2^-40 of the arc's z-range (oracle (b), shifted z0);
  * output order is edge-major, latitude ascending; the run is bitwise repeatable; cap
    truncation and count-only calls report the same total; large tables use the global path;
  * the full C4 workload (cubed sphere ne=1024 x 1,800 latitudes) gives the same nonzero pairs
    and values as the unfused kernel on the materialised pairs.
"""
import numpy as np
import pytest

import oracle
import sgi_inputs
from oracle import exact

torch = pytest.importorskip("torch")
import paper_2510_09892_b200 as sgi  # noqa: E402

pytestmark = pytest.mark.gpu
DELTA = 2.0 ** -40


def same(x, y):
    return (x == y) | (np.isnan(x) & np.isnan(y))


@pytest.fixture(scope="module", autouse=True)
def _build():
    sgi.build()


def run_zonal(va, vb, lat, mode="eft", cap=None):
    dva = torch.from_numpy(np.ascontiguousarray(va)).cuda()
    dvb = torch.from_numpy(np.ascontiguousarray(vb)).cuda()
    dl = torch.from_numpy(np.ascontiguousarray(lat)).cuda()
    out = sgi.zonal_intersect(dva, dvb, dl, mode=mode, cap=cap)
    torch.cuda.synchronize()
    m = min(out["cap"], int(out["total"].item()))
    return ({k: v[..., :m].cpu().numpy() for k, v in out.items() if k in ("edge", "lat", "count", "xyz")},
            int(out["total"].item()))


def brute_force(va, vb, lat, mode):
    """oracle (a) on every (edge, latitude) pair; returns counts [E, K] and points."""
    E, K = va.shape[1], len(lat)
    a = np.repeat(va, K, axis=1)
    b = np.repeat(vb, K, axis=1)
    z = np.tile(lat, E)
    out, cnt = oracle.intersect(mode, a, b, z, nthreads=16)
    return cnt.reshape(E, K), out.reshape(2, 3, E, K)


def check_against_brute(va, vb, lat, mode_name, omode):
    res, total = run_zonal(va, vb, lat, mode_name)
    cnt, pts = brute_force(va, vb, lat, omode)
    e, k = res["edge"], res["lat"]
    assert total == len(e)
    # order: edge-major, latitude ascending
    key = e.astype(np.int64) * len(lat) + k
    assert np.all(np.diff(key) > 0)
    # conservative: all nonzero pairs are candidates
    nz = np.argwhere(cnt != 0)
    cand = set(key.tolist())
    missing = [tuple(p) for p in nz if p[0] * len(lat) + p[1] not in cand]
    assert missing == [], missing[:5]
    # values equal the plain query
    assert np.array_equal(res["count"], cnt[e, k])
    assert same(res["xyz"], pts[:, :, e, k]).all()
    return res, cnt


def test_small_mesh_against_brute_force():
    va, vb = sgi_inputs.cubed_sphere_edges(16)
    lat = sgi_inputs.latitudes(1800)
    res, cnt = check_against_brute(va, vb, lat, "eft", oracle.MODE_EFT)
    zero = np.flatnonzero(res["count"] == 0)
    for j in zero[:200]:                      # margin candidates lie within 2*delta of the arc
        e, k = res["edge"][j], res["lat"][j]
        hits = [exact.exact_query(va[:, e], vb[:, e], lat[k] + s * 2 * DELTA).count
                for s in (-1.0, 1.0)]
        assert any(h not in (0,) for h in hits)


@pytest.mark.parametrize("mode,omode", [("eft", oracle.MODE_EFT), ("eft_literal", oracle.MODE_EFT_LITERAL),
                                        ("naive", oracle.MODE_NAIVE), ("yac", oracle.MODE_YAC),
                                        ("base", oracle.MODE_BASE),
                                        ("naive_kahan", oracle.MODE_NAIVE_KAHAN)])
def test_long_arcs_many_latitudes(mode, omode):
    """C1 arcs (long, up to pi) against 181 latitudes: edges spanning many latitudes, two-point
    pairs, dense redistribution of candidates across threads."""
    a, b, _ = sgi_inputs.generate_host(1, 700)
    lat = np.sin(np.radians(np.linspace(-90, 90, 183)[1:-1]))
    res, cnt = check_against_brute(a, b, lat, mode, omode)
    assert (res["count"] == 2).sum() > 0 and (np.bincount(res["edge"]) > 20).any()


def test_degenerate_and_special_edges():
    va = np.array([[1, 0, 0], [1, 0, 0], [0.6, 0, 0.8], [1, 0, 1], [1, 0, -1], [0, 0, 1]], float).T.copy()
    vb = np.array([[0, 1, 0], [0, 0, 1], [0.6, 0, 0.8], [-1, 0, 1], [-1, 0, -1], [1, 0, 0]], float).T.copy()
    lat = np.array([-0.75, -0.5, 0.0, 0.5, 0.75, 0.8, 1.0])
    check_against_brute(va, vb, lat, "eft", oracle.MODE_EFT)


@pytest.mark.parametrize("kind", ["wide", "near_unit"])
def test_non_unit_endpoints(kind):
    """The filter's heights z/|x| for endpoints off the unit sphere: scaled by 2^[-20, 20]
    ("wide"), or by 1 +- 2^-43 / 2^-46 / 2^-52 — either side of the filter's unit-norm shortcut
    (|x|^2 within 2^-44 of 1: z itself) — on C1 arcs against 181 latitudes."""
    rng = np.random.default_rng(44)
    a, b, _ = sgi_inputs.generate_host(1, 800)
    if kind == "wide":
        fa, fb = (2.0 ** rng.uniform(-20, 20, (2, a.shape[1])))
    else:
        eps = np.array([2.0 ** -43, 2.0 ** -46, 2.0 ** -52, 0.0])
        fa = 1 + rng.choice([-1, 1], a.shape[1]) * rng.choice(eps, a.shape[1])
        fb = 1 + rng.choice([-1, 1], a.shape[1]) * rng.choice(eps, a.shape[1])
    a, b = a * fa, b * fb
    lat = np.sin(np.radians(np.linspace(-90, 90, 183)[1:-1]))
    res, cnt = check_against_brute(a, b, lat, "eft", oracle.MODE_EFT)
    assert (cnt != 0).sum() > 1000


def test_table_with_clustered_and_out_of_range_entries():
    """The bucket index over z in [-1, 1]: entries outside it (clamped into the end buckets),
    many entries in one bucket (the binary-search fallback) and entries a few ulps apart."""
    a, b, _ = sgi_inputs.generate_host(1, 600)
    z = np.concatenate([[-3.0, -1.5, -1.0 - 2.0 ** -40], np.linspace(-1, 1, 97),
                        0.3 + np.arange(40) * 2.0 ** -20, 0.7 + np.arange(5) * 2.0 ** -50,
                        [1.0 + 2.0 ** -40, 2.0]])
    lat = np.unique(z)
    check_against_brute(a, b, lat, "eft", oracle.MODE_EFT)


def test_latitudes_at_the_filter_margins():
    """A table built from the edges' own critical heights — endpoint z (and one ulp either side)
    and apex heights of arcs whose extremum lies inside (and +-2 ulps) — so latitudes sit exactly
    where the filter's z-ranges end; no nonzero pair may be missed (C1 arcs and a small mesh)."""
    rng = np.random.default_rng(77)
    a, b, _ = sgi_inputs.generate_host(1, 400)
    va, vb = sgi_inputs.cubed_sphere_edges(8)
    va, vb = np.concatenate([a, va], axis=1), np.concatenate([b, vb], axis=1)
    n = np.cross(va.T, vb.T).T
    apex = np.sqrt(n[0] ** 2 + n[1] ** 2) / np.linalg.norm(n, axis=0)
    pick = rng.choice(va.shape[1], 600, replace=False)
    z = [va[2, pick] / np.linalg.norm(va[:, pick], axis=0), vb[2, pick[:300]]]
    z += [np.nextafter(z[0], 2.0), np.nextafter(z[0], -2.0)]
    ap = apex[pick[:400]] * rng.choice([-1.0, 1.0], 400)
    z += [ap, np.nextafter(np.nextafter(ap, 2.0), 2.0), np.nextafter(np.nextafter(ap, -2.0), -2.0)]
    lat = np.unique(np.clip(np.concatenate(z), -1.0, 1.0))
    assert 1000 < len(lat) <= 4096
    check_against_brute(va, vb, lat, "eft", oracle.MODE_EFT)


def test_special_edges_and_latitudes():
    """Edges between special vectors (poles, axis and equator points, negated, scaled by 2^+-60,
    one-ulp perturbed, degenerate and antipodal pairs) against a table of special latitudes and
    the edges' own endpoint heights (+-1 ulp): conservative filter and plain-query values."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "fz", os.path.join(os.path.dirname(__file__), "test_gpu_fuzz.py"))
    fz = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(fz)
    rng = np.random.default_rng(5)
    va, vb, z = fz.specials(rng, 3000)
    zs = np.concatenate([z, np.nextafter(z, 2.0), np.nextafter(z, -2.0),
                         [-1.0, 0.0, 1.0, 0.5, -0.5, 0.8, -0.8, np.sqrt(0.5)]])
    lat = np.unique(np.clip(zs[np.isfinite(zs)], -1.0, 1.0))
    lat = lat[lat != 0] if (lat == 0).sum() > 1 else lat        # (+0 and -0 compare equal)
    assert 10 < len(lat) <= 4096
    check_against_brute(np.ascontiguousarray(va), np.ascontiguousarray(vb), lat, "eft",
                        oracle.MODE_EFT)


@pytest.mark.parametrize("lo,hi", [(-16, -10), (-12, -5)])
def test_short_and_nearly_parallel_arcs(lo, hi):
    """Arcs 10^[lo, hi] rad long (down to a few ulps of the endpoints), some reversed into
    nearly antipodal pairs: the plain query's rounded containment on nearly parallel endpoints
    may report points far from the arc, and the filter must still hand it every such pair."""
    rng = np.random.default_rng(100 + lo)
    n = 1500
    m = rng.normal(size=(3, n)); m /= np.linalg.norm(m, axis=0)
    t = np.cross(m.T, rng.normal(size=(n, 3))).T; t /= np.linalg.norm(t, axis=0)
    L = 10.0 ** rng.uniform(lo, hi, n)
    va, vb = m - t * L / 2, m + t * L / 2
    va /= np.linalg.norm(va, axis=0); vb /= np.linalg.norm(vb, axis=0)
    flip = rng.random(n) < 0.2
    vb[:, flip] = -vb[:, flip]
    lat = np.sin(np.radians(np.linspace(-90, 90, 362)[1:-1]))
    check_against_brute(np.ascontiguousarray(va), np.ascontiguousarray(vb), lat, "eft",
                        oracle.MODE_EFT)


def test_repeatable_truncation_and_count_only():
    a, b, _ = sgi_inputs.generate_host(5, 20000)
    lat = sgi_inputs.latitudes(1800)
    r1, t1 = run_zonal(a, b, lat)
    r2, t2 = run_zonal(a, b, lat)
    assert t1 == t2 and all(np.array_equal(r1[k].view(np.uint8), r2[k].view(np.uint8)) for k in r1)
    r3, t3 = run_zonal(a, b, lat, cap=t1 // 3)
    assert t3 == t1 and len(r3["edge"]) == t1 // 3
    assert np.array_equal(r3["edge"], r1["edge"][:t1 // 3]) and same(r3["xyz"], r1["xyz"][:, :, :t1 // 3]).all()


def test_large_latitude_table_global_path():
    a, b, _ = sgi_inputs.generate_host(2, 1000)
    lat = np.sin(np.radians(-90 + (np.arange(10000) + 0.5) * 180 / 10000))
    check_against_brute(a, b, lat, "eft", oracle.MODE_EFT)


def test_empty_inputs():
    va = np.zeros((3, 0)); lat = sgi_inputs.latitudes(10)
    res, total = run_zonal(va, va, lat)
    assert total == 0
    a, b, _ = sgi_inputs.generate_host(1, 100)
    res, total = run_zonal(a, b, np.zeros(0))
    assert total == 0


def test_c4_full_size_against_unfused_path():
    va, vb = sgi_inputs.cubed_sphere_edges(1024)
    lat = sgi_inputs.latitudes(1800)
    res, total = run_zonal(va, vb, lat)
    pa, pb, pz, pe = sgi_inputs.c4_pairs(1024, 1800)
    da, db, dz = (torch.from_numpy(x).cuda() for x in (pa, pb, pz))
    out, cnt = sgi.intersect_arc_lat(da, db, dz, mode="eft")
    torch.cuda.synchronize()
    out, cnt = out.cpu().numpy(), cnt.cpu().numpy()
    k_of = np.searchsorted(lat, pz)
    nz_unfused = set((pe[cnt != 0] * 1800 + k_of[cnt != 0]).tolist())
    key = res["edge"] * 1800 + res["lat"]
    nzmask = res["count"] != 0
    assert set(key[nzmask].tolist()) == nz_unfused
    # values: fused pairs that the numpy pairing also produced must be bit-equal
    _, jf, ju = np.intersect1d(key, pe * 1800 + k_of, assume_unique=True, return_indices=True)
    assert np.array_equal(res["count"][jf], cnt[ju])
    assert same(res["xyz"][:, :, jf], out[:, :, ju]).all()
    assert total >= len(nz_unfused) and len(nz_unfused) > 5_900_000


@pytest.mark.parametrize("pad,shift", [(5, 1), (0, 1), (37, 0)])
def test_padded_and_unaligned_edge_planes(pad, shift):
    """Edge planes with ld_e > n_edges and a base only 8-byte aligned (a view one element into a
    buffer): same pairs and values as the packed call; the workspace stays 16-byte aligned."""
    a, b, _ = sgi_inputs.generate_host(2, 3001)
    lat = sgi_inputs.latitudes(500)
    ref, t_ref = run_zonal(a, b, lat)
    n = a.shape[1]
    ld = n + pad
    dl = torch.from_numpy(lat).cuda()

    def planes(x):
        buf = torch.full((3 * ld + shift,), float("nan"), dtype=torch.float64, device="cuda")
        v = buf[shift:].view(3, ld)
        v[:, :n] = torch.from_numpy(x).cuda()
        return v

    va, vb = planes(a), planes(b)
    assert va.data_ptr() % 16 == 8 * shift % 16
    out = sgi.zonal_intersect(va, vb, dl, mode="eft", n_edges=n)
    torch.cuda.synchronize()
    m = int(out["total"].item())
    assert m == t_ref
    assert np.array_equal(out["edge"][:m].cpu().numpy(), ref["edge"])
    assert np.array_equal(out["lat"][:m].cpu().numpy(), ref["lat"])
    assert np.array_equal(out["count"][:m].cpu().numpy(), ref["count"])
    assert same(out["xyz"][..., :m].cpu().numpy(), ref["xyz"]).all()
