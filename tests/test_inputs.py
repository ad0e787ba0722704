"""The seeded input generators (sgi_inputs): determinism, sharding and workload shapes."""
import numpy as np
import pytest

import sgi_inputs


@pytest.mark.parametrize("config", [1, 2, 3, 5])
def test_deterministic_and_shard_invariant(config):
    a, b, z = sgi_inputs.generate_host(config, 3000)
    a2, b2, z2 = sgi_inputs.generate_host(config, 3000)
    assert np.array_equal(a, a2) and np.array_equal(b, b2) and np.array_equal(z, z2)
    # any split of the global index range reproduces the same arcs (R-invariance, §8(e))
    for lo, hi in ((0, 1000), (1000, 1777), (1777, 3000)):
        sa, sb, sz = sgi_inputs.generate_host(config, hi - lo, offset=lo)
        assert np.array_equal(sa, a[:, lo:hi]) and np.array_equal(sz, z[lo:hi])
    # padded leading dimension leaves the tail untouched
    pa, pb, pz = sgi_inputs.generate_host(config, 100, ld=128)
    assert np.array_equal(pa[:, :100], a[:, :100]) and not pa[:, 100:].any()


def test_seed_changes_stream():
    a, _, _ = sgi_inputs.generate_host(1, 100, seed=0)
    a2, _, _ = sgi_inputs.generate_host(1, 100, seed=1)
    assert not np.array_equal(a, a2)


@pytest.mark.parametrize("config", [1, 2, 3, 5])
def test_unit_endpoints_and_z0_between(config):
    a, b, z = sgi_inputs.generate_host(config, 6000)
    for v in (a, b):
        r = np.sqrt((v * v).sum(0))
        assert np.all(np.abs(r - 1) < 4e-16)
    between = np.ones(len(z), bool)
    if config == 3:
        between[0::3] = False                      # near-tangent: z0 near the apex
    if config == 5:
        between[3::4] = False                      # free z0 in [-1, 1]
    lo, hi = np.minimum(a[2], b[2]), np.maximum(a[2], b[2])
    assert np.all((z[between] >= lo[between]) & (z[between] <= hi[between]))
    assert np.all(np.abs(z) <= 1)


def test_c2_arc_lengths():
    a, b, _ = sgi_inputs.generate_host(2, 20000)
    L = 2 * np.arcsin(np.linalg.norm(a - b, axis=0) / 2)
    assert L.min() > 0.99e-4 and L.max() < 1.01e-2
    # log-uniform: each decade holds about half of the arcs
    assert 0.45 < np.mean(L < 1e-3) < 0.55


def test_c3_classes():
    a, b, z = sgi_inputs.generate_host(3, 9000)
    # near-polar endpoints: |z| in [1 - 1e-10, 1)
    assert np.all(np.abs(a[2, 1::3]) >= 1 - 1.0000001e-10) and np.all(np.abs(a[2, 1::3]) < 1)
    # near-coincident endpoints: separation in [1e-12, 1e-7] rad (up to rounding of unit())
    sep = np.linalg.norm(a[:, 2::3] - b[:, 2::3], axis=0)
    assert sep.min() > 0.9e-12 and sep.max() < 1.1e-7
    # near-tangent: z0 within [1e-15, 1e-6] relative of the designed apex height
    L = np.linalg.norm(a[:, 0::3] - b[:, 0::3], axis=0)
    assert L.min() > 1.9e-2 and L.max() < 0.21
    assert np.all(np.sign(z[0::3][0::2]) >= 0) and np.all(np.sign(z[0::3][1::2]) <= 0)


def test_c4_mesh_structure():
    ne = 16
    va, vb = sgi_inputs.cubed_sphere_edges(ne)
    assert va.shape[1] == 12 * ne * ne                   # unique edges of the cubed sphere
    for v in (va, vb):
        assert np.all(np.abs(np.sqrt((v * v).sum(0)) - 1) < 4e-16)
    verts = np.unique(np.concatenate([va, vb], 1), axis=1)
    assert verts.shape[1] == 6 * ne * ne + 2             # Euler: V - E + F = 2
    a, b, z0, edge = sgi_inputs.c4_pairs(ne, 1800)
    lat = sgi_inputs.latitudes(1800)
    assert np.all(np.isin(z0, lat)) and np.all(np.diff(edge) >= 0)
    assert a.shape == (3, len(z0)) and len(z0) > 0
