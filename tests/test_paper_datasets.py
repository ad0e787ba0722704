"""The paper's primary and secondary accuracy datasets:
generator shapes, and the per-group accuracy the paper reports, with oracle (a) against oracle
(b) on the CPU.  The GPU path is bitwise equal to oracle (a) (tests/test_gpu_paper_datasets.py),
so these per-group numbers are the GPU's too.

Set SGI_REPORT_DIR to also write the per-group CSV reports there.
"""
import math
import os

import numpy as np
import pytest

import oracle
import sgi_inputs
from oracle import exact
import paper_accuracy as pa

MODES = {"eft": oracle.MODE_EFT, "eft_literal": oracle.MODE_EFT_LITERAL,
         "naive": oracle.MODE_NAIVE, "yac": oracle.MODE_YAC, "base": oracle.MODE_BASE,
         "naive_kahan": oracle.MODE_NAIVE_KAHAN}


def test_primary_bands_and_longitudes():
    """Both endpoints of arc i at latitudes in band i % 17 ("ensuring that their latitudes
    fell within the corresponding band"), longitudes spread over 0-360 degrees, z0 between."""
    n = 17 * 400
    a, b, z0 = sgi_inputs.generate_host(6, n)
    g = sgi_inputs.group_of(6, np.arange(n))
    edges = sgi_inputs.PRIMARY_BAND_EDGES
    for v in (a, b):
        r = np.linalg.norm(v, axis=0)
        assert np.all(np.abs(r - 1) < 4e-16)
        lat = np.degrees(np.arcsin(np.clip(v[2] / r, -1, 1)))
        lo, hi = np.array(edges)[g], np.array(edges)[g + 1]
        tol = 1e-9 * np.maximum(1.0, hi)           # float64 trig on both sides
        assert np.all(lat > lo - tol) and np.all(lat <= hi + tol)
        lon = np.degrees(np.arctan2(v[1], v[0])) % 360
        assert np.histogram(lon, bins=8, range=(0, 360))[0].min() > n / 8 * 0.8
    assert np.all(z0 >= np.minimum(a[2], b[2])) and np.all(z0 <= np.maximum(a[2], b[2]))


def test_secondary_shallow_arcs_near_the_top():
    """Endpoints in the latitude band (0, 1e-4 deg]; z0 = top of the circle - r, r in decade
    i % 13; both intersection points lie on the arc (exact count 2)."""
    n = 13 * 200
    a, b, z0 = sgi_inputs.generate_host(7, n)
    zband = math.sin(math.radians(1e-4))
    for v in (a, b):
        assert np.all(v[2] > 0) and np.all(v[2] <= zband * (1 + 1e-12))
        assert np.all(np.abs(np.linalg.norm(v, axis=0) - 1) < 4e-16)
    assert np.all(z0 > np.maximum(a[2], b[2]))
    # the offset below the circle's top, from an independent float64 evaluation of the top
    nrm = np.cross(a.T, b.T).T
    top = np.hypot(nrm[0], nrm[1]) / np.linalg.norm(nrm, axis=0)
    r = top - z0
    d = sgi_inputs.group_of(7, np.arange(n))
    lo = np.array([x[0] for x in sgi_inputs.SECONDARY_DECADES])[d]
    big = lo >= 1e-13                              # float64 top is only good to ~1e-16 abs
    assert np.all(r[big] > 0.9 * lo[big]) and np.all(r[big] < 10.1 * lo[big])
    counts = [exact.exact_query(a[:, i], b[:, i], z0[i]).count for i in range(0, n, 7)]
    assert set(counts) == {2}


@pytest.mark.parametrize("config,per_group", [(6, 120), (7, 120)])
def test_per_group_accuracy_matches_the_paper(config, per_group):
    ng = 17 if config == 6 else 13
    n = ng * per_group
    a, b, z0 = sgi_inputs.generate_host(config, n)
    idx = np.arange(n)
    ex = pa.exact_results(a, b, z0, idx)
    stats = {}
    for name, m in MODES.items():
        out, cnt = oracle.intersect(m, a, b, z0)
        stats[name] = pa.group_stats(config, idx, ex, out, cnt, z0)
    pa.check_paper_claims(config, stats)
    rdir = os.environ.get("SGI_REPORT_DIR")
    if rdir:
        pa.write_csv(os.path.join(rdir, f"paper_accuracy_c{config}_oracle_a.csv"), config, stats,
                     f"oracle (a), {per_group} arcs per group")
