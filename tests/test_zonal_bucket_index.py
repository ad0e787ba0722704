"""The fused zonal kernel's exact bucket index (csrc/sgi_zonal.cu bucket_of / build_buckets /
bucket_search, DESIGN.md §5 zonal) emulated on the CPU with the same float32 steps: the bucket
function is monotone, so both searches of x only need the entries of x's own bucket — checked
against numpy's searchsorted on tables with entries outside [-1, 1], dense clusters, entries one
ulp apart, and queries on and next to every entry."""
import numpy as np
import pytest

KB = 2048


def bucket_of(x):
    """floor((f32(x) + 1) * KB/2) in float32, clamped to [0, KB - 1] (NaN-free inputs)."""
    f = (np.asarray(x, np.float64).astype(np.float32) + np.float32(1.0)) * np.float32(KB // 2)
    f = np.minimum(np.maximum(f, np.float32(0.0)), np.float32(KB - 1))
    return f.astype(np.int64)


def build(tab):
    """bkt[b] = the first k with bucket(tab[k]) >= b, b = 0..KB."""
    bt = bucket_of(tab)
    return np.searchsorted(bt, np.arange(KB + 1), side="left")


def search(bkt, tab, x, upper):
    b = bucket_of(x)
    lo, hi = bkt[b], bkt[b + 1]
    side = "right" if upper else "left"
    return lo + np.array([np.searchsorted(tab[l:h], v, side=side) for l, h, v in zip(lo, hi, x)])


def tables(rng):
    yield np.sin(np.radians(-90 + (np.arange(1800) + 0.5) * 0.1))             # the C4 table
    yield np.sin(np.radians(np.linspace(-90, 90, 183)[1:-1]))
    z = np.concatenate([[-3.0, -1.5, -1.0 - 2.0 ** -40], np.linspace(-1, 1, 97),
                        0.3 + np.arange(40) * 2.0 ** -20, 0.7 + np.arange(5) * 2.0 ** -50,
                        [1.0 + 2.0 ** -40, 2.0]])
    yield np.unique(z)
    yield np.unique(rng.uniform(-1, 1, 4000))
    yield np.unique(np.concatenate([1 - 10.0 ** rng.uniform(-16, -1, 500),
                                    -1 + 10.0 ** rng.uniform(-16, -1, 500)]))


def test_bucket_function_is_monotone():
    rng = np.random.default_rng(3)
    x = np.sort(np.concatenate([rng.uniform(-2, 2, 200000), np.linspace(-1, 1, 4097),
                                np.nextafter(np.linspace(-1, 1, 4097), 2.0)]))
    assert np.all(np.diff(bucket_of(x)) >= 0)


@pytest.mark.parametrize("k", range(5))
def test_bucket_searches_equal_searchsorted(k):
    rng = np.random.default_rng(10 + k)
    tab = list(tables(rng))[k]
    assert np.all(np.diff(tab) > 0)
    bkt = build(tab)
    q = np.concatenate([tab, np.nextafter(tab, 3.0), np.nextafter(tab, -3.0),
                        rng.uniform(-1.2, 1.2, 20000), [-5.0, -1.0, 0.0, 1.0, 5.0]])
    for upper in (False, True):
        want = np.searchsorted(tab, q, side="right" if upper else "left")
        assert np.array_equal(search(bkt, tab, q, upper), want)
    # the kernel's unrolled case: most buckets of the C4 table hold at most two entries
    if k == 0:
        assert (np.diff(bkt) <= 2).mean() > 0.97
