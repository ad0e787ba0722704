"""GPU parity: the CUDA path (through the C ABI) against oracle (a) element by element and
against oracle (b) on samples, on every BASELINE.json config, plus edge cases.

Parity bar: counts bit-exact; points bitwise equal to oracle (a) up to the sign
of zero (IEEE ==, NaN == NaN); EFT points within err_u <= 3 of oracle (b) (Eq.BOUND,
P:897-913).  Sizes: C1 in full; C2, C3 in full (2^24, the bench's launch configuration);
C4 in full (~6.0 M pairs); C5 (2^30) on a deterministic sample of global indices generated on
the device in the bench's launch configuration.
"""
import numpy as np
import pytest

import oracle
import sgi_inputs
from oracle import exact

torch = pytest.importorskip("torch")
import paper_2510_09892_b200 as sgi  # noqa: E402

pytestmark = pytest.mark.gpu

MODES = [("eft", oracle.MODE_EFT), ("eft_literal", oracle.MODE_EFT_LITERAL),
         ("naive", oracle.MODE_NAIVE), ("yac", oracle.MODE_YAC), ("base", oracle.MODE_BASE),
         ("naive_kahan", oracle.MODE_NAIVE_KAHAN)]
NTHREADS = 16


def same(x, y):
    return (x == y) | (np.isnan(x) & np.isnan(y))


def expected_path(mode, n, entry=0):
    """The kernel a freshly allocated (256-B aligned, ld = n) batch must take."""
    if n < (1 << 19) or n % 2:
        return "ldg"
    return "tma_pair" if entry == 0 and mode in ("eft", "eft_literal") else "tma"


def run_gpu(a, b, z0, mode, n=None, path=None):
    """The device entry on copies of a, b, z0; `path` asserts which kernel the call launches."""
    da, db, dz = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (a, b, z0))
    ld = dz.shape[0]
    out = torch.empty((2, 3, ld), dtype=torch.float64, device="cuda")
    cnt = torch.empty(ld, dtype=torch.uint8, device="cuda")
    if path is not None:
        assert sgi.dispatch_path(da, db, dz, out, cnt, mode=mode, n=n) == path
    sgi.intersect_arc_lat(da, db, dz, mode=mode, n=n, out_xyz=out, out_count=cnt)
    torch.cuda.synchronize()
    return out.cpu().numpy(), cnt.cpu().numpy()


def assert_parity(got, gcnt, ref, rcnt, n=None):
    n = len(rcnt) if n is None else n
    assert np.array_equal(gcnt[:n], rcnt[:n]), int((gcnt[:n] != rcnt[:n]).sum())
    ok = same(got[..., :n], ref[..., :n])
    assert ok.all(), f"{int((~ok).sum())} coordinates differ"


@pytest.fixture(scope="module", autouse=True)
def _build():
    sgi.build()
    sgi_inputs.build(device=True)


# ------------------------------------------------------------------ device generator == host
@pytest.mark.parametrize("config", [1, 2, 3, 5, 6, 7])
def test_device_generator_matches_host(config):
    n = 100_003
    a, b, z = sgi_inputs.generate_host(config, n, offset=12345)
    da = torch.empty((3, n), dtype=torch.float64, device="cuda")
    db = torch.empty_like(da)
    dz = torch.empty(n, dtype=torch.float64, device="cuda")
    sgi_inputs.generate_device(config, n, da, db, dz, offset=12345)
    torch.cuda.synchronize()
    assert np.array_equal(da.cpu().numpy(), a)
    assert np.array_equal(db.cpu().numpy(), b)
    assert np.array_equal(dz.cpu().numpy(), z)


# ------------------------------------------------------------------------------ C1 in full
@pytest.mark.parametrize("mode,omode", MODES)
def test_c1_parity_all_modes(mode, omode):
    a, b, z0 = sgi_inputs.generate_host(1, sgi_inputs.CONFIG_SIZES[1])
    got, gcnt = run_gpu(a, b, z0, mode)
    ref, rcnt = oracle.intersect(omode, a, b, z0, nthreads=NTHREADS)
    assert_parity(got, gcnt, ref, rcnt)


def test_two_point_lane_mixes_on_the_pair_kernel():
    """The pair kernel computes a query's second root only where it stores one (§5): in scalar
    form when the other query of the thread has none, two-lane when both have two.  C3's
    near-tangent arcs give every mix at an even, TMA-sized n (~380 both-two, ~87,000 one-two
    lanes); all must equal oracle (a) bit for bit."""
    n = (1 << 19) + 2
    a, b, z0 = sgi_inputs.generate_host(3, n)
    got, gcnt = run_gpu(a, b, z0, "eft", path="tma_pair")
    ref, rcnt = oracle.intersect(oracle.MODE_EFT, a, b, z0, nthreads=NTHREADS)
    assert_parity(got, gcnt, ref, rcnt)
    c0, c1 = rcnt[0::2], rcnt[1::2]
    assert ((c0 == 2) & (c1 == 2)).sum() > 100                       # both lanes two-lane
    assert ((c0 == 2) & (c1 != 2)).sum() > 100 and ((c0 != 2) & (c1 == 2)).sum() > 100   # one lane


def test_c1_eft_against_exact_oracle():
    a, b, z0 = sgi_inputs.generate_host(1, sgi_inputs.CONFIG_SIZES[1])
    got, gcnt = run_gpu(a, b, z0, "eft")
    worst = 0.0
    for i in range(len(z0)):
        ex = exact.exact_query(a[:, i], b[:, i], z0[i])
        assert ex.count == gcnt[i]
        for k in range(ex.count if ex.count != exact.DEGENERATE else 0):
            worst = max(worst, exact.err_u((got[k, 0, i], got[k, 1, i]), ex.points[k], z0[i]))
    assert worst <= 3.0


# -------------------------------------------------------- C2, C3 at full size (2^24 each)
def _device_config(config, n):
    da = torch.empty((3, n), dtype=torch.float64, device="cuda")
    db = torch.empty_like(da)
    dz = torch.empty(n, dtype=torch.float64, device="cuda")
    sgi_inputs.generate_device(config, n, da, db, dz)
    return da, db, dz


@pytest.mark.parametrize("config", [2, 3])
@pytest.mark.parametrize("mode,omode", MODES)
def test_full_size_parity(config, mode, omode):
    n = sgi_inputs.CONFIG_SIZES[config]
    da, db, dz = _device_config(config, n)
    out, cnt = sgi.intersect_arc_lat(da, db, dz, mode=mode)
    assert sgi.dispatch_path(da, db, dz, out, cnt, mode=mode) == expected_path(mode, n)
    torch.cuda.synchronize()
    a, b, z0 = da.cpu().numpy(), db.cpu().numpy(), dz.cpu().numpy()
    ref, rcnt = oracle.intersect(omode, a, b, z0, nthreads=NTHREADS)
    assert_parity(out.cpu().numpy(), cnt.cpu().numpy(), ref, rcnt)


@pytest.mark.parametrize("config", [2, 3])
def test_full_size_eft_sampled_exact(config):
    n = sgi_inputs.CONFIG_SIZES[config]
    da, db, dz = _device_config(config, n)
    out, cnt = sgi.intersect_arc_lat(da, db, dz, mode="eft")
    torch.cuda.synchronize()
    idx = np.random.default_rng(config).choice(n, 1500, replace=False)
    a, b, z0 = da[:, idx].cpu().numpy(), db[:, idx].cpu().numpy(), dz[idx].cpu().numpy()
    got, gcnt = out[:, :, idx].cpu().numpy(), cnt[idx].cpu().numpy()
    worst, bad = 0.0, []
    for j in range(len(idx)):
        ex = exact.exact_query(a[:, j], b[:, j], z0[j])
        if ex.count != gcnt[j]:
            bad.append(min(ex.margins))          # endpoint-on-latitude ties (R7)
            continue
        for k in range(ex.count if ex.count != exact.DEGENERATE else 0):
            worst = max(worst, exact.err_u((got[k, 0, j], got[k, 1, j]), ex.points[k], z0[j]))
    assert worst <= 3.0
    # C2 has no endpoint-on-latitude ties: the counts are the exact ones.  C3's near-polar third
    # puts z0 on an endpoint's height to within rounding; there the rounded containment test may
    # differ from the exact count, only at margins below 4u (reading R7', sgi.h)
    if config == 2:
        assert bad == []
    else:
        assert all(m < 4 * 2.0 ** -53 for m in bad) and len(bad) <= 15


# ------------------------------------------------------------------------- C4 in full
def test_c4_full_parity():
    a, b, z0, _ = sgi_inputs.c4_pairs(1024, 1800)
    got, gcnt = run_gpu(a, b, z0, "eft")
    ref, rcnt = oracle.intersect(oracle.MODE_EFT, a, b, z0, nthreads=NTHREADS)
    assert_parity(got, gcnt, ref, rcnt)
    idx = np.random.default_rng(44).choice(len(z0), 1000, replace=False)
    for i in idx:
        ex = exact.exact_query(a[:, i], b[:, i], z0[i])
        assert ex.count == gcnt[i]
        for k in range(ex.count if ex.count != exact.DEGENERATE else 0):
            assert exact.err_u((got[k, 0, i], got[k, 1, i]), ex.points[k], z0[i]) <= 3.0


# ------------------------------------------------- C5 (2^30) sampled, generated on the device
def test_c5_full_size_sampled():
    n = sgi_inputs.CONFIG_SIZES[5]
    torch.cuda.empty_cache()              # the previous 2^30 test's blocks back to the driver
    free, _ = torch.cuda.mem_get_info()
    if free < n * 110:
        pytest.skip("needs ~113 GB free HBM")
    da, db, dz = _device_config(5, n)
    out, cnt = sgi.intersect_arc_lat(da, db, dz, mode="eft")
    assert sgi.dispatch_path(da, db, dz, out, cnt, mode="eft") == "tma_pair"
    hist = sgi.count_histogram(cnt)
    torch.cuda.synchronize()
    idx = np.unique(np.concatenate([np.arange(0, n, 4096),
                                    np.random.default_rng(5).choice(n, 4096), [n - 1]]))
    ti = torch.from_numpy(idx).cuda()
    got = out[:, :, ti].cpu().numpy()
    gcnt = cnt[ti].cpu().numpy()
    a, b, z0 = da[:, ti].cpu().numpy(), db[:, ti].cpu().numpy(), dz[ti].cpu().numpy()
    del da, db, dz, out, cnt
    ref, rcnt = oracle.intersect(oracle.MODE_EFT, a, b, z0, nthreads=NTHREADS)
    assert_parity(got, gcnt, ref, rcnt)
    # the sample really is what the host generator makes for those global indices
    for j in (0, len(idx) // 2, len(idx) - 1):
        ha, hb, hz = sgi_inputs.generate_host(5, 1, offset=int(idx[j]))
        assert np.array_equal(ha[:, 0], a[:, j]) and hz[0] == z0[j]
    h = hist.cpu().numpy()
    assert h[:4].sum() == n and h[4] == h[1] + 2 * h[2]
    assert h[0] > 0 and h[1] > 0 and h[2] > 0       # mixed 0/1/2 by construction (config 5)
    worst = 0.0
    for j in range(0, len(idx), 4):
        ex = exact.exact_query(a[:, j], b[:, j], z0[j])
        assert ex.count == gcnt[j]
        for k in range(ex.count if ex.count != exact.DEGENERATE else 0):
            worst = max(worst, exact.err_u((got[k, 0, j], got[k, 1, j]), ex.points[k], z0[j]))
    assert worst <= 3.0


def test_c5_full_size_every_query():
    """C5 in full: all 2^30 queries of the full-size launch (the bench's launch configuration,
    the TMA pair kernel with policy Cert) against oracle (a), bit for bit (up to the sign of zero),
    in host chunks of 2^25 queries — the north star's "bit-identical on all five configs"."""
    n = sgi_inputs.CONFIG_SIZES[5]
    torch.cuda.empty_cache()              # the previous 2^30 test's blocks back to the driver
    free, _ = torch.cuda.mem_get_info()
    if free < n * 110:
        pytest.skip("needs ~113 GB free HBM")
    da, db, dz = _device_config(5, n)
    out, cnt = sgi.intersect_arc_lat(da, db, dz, mode="eft")
    assert sgi.dispatch_path(da, db, dz, out, cnt, mode="eft") == "tma_pair"
    torch.cuda.synchronize()
    chunk = 1 << 25
    for off in range(0, n, chunk):
        m = min(chunk, n - off)
        a = da[:, off:off + m].contiguous().cpu().numpy()
        b = db[:, off:off + m].contiguous().cpu().numpy()
        z0 = dz[off:off + m].cpu().numpy()
        got = out[:, :, off:off + m].contiguous().cpu().numpy()
        gcnt = cnt[off:off + m].cpu().numpy()
        ref, rcnt = oracle.intersect(oracle.MODE_EFT, a, b, z0, nthreads=NTHREADS)
        assert np.array_equal(gcnt, rcnt), (off, int((gcnt != rcnt).sum()))
        ok = same(got, ref)
        assert ok.all(), (off, int((~ok).sum()))


# ---------------------------------------------------------------------------- edge cases
@pytest.mark.parametrize("n", [1, 31, 255, 257, 1000, 148 * 256 * 4 + 77])
def test_ragged_sizes_and_padding(n):
    ld = n + 13
    a, b, z0 = sgi_inputs.generate_host(5, n, ld=ld)
    a[:, n:] = 7.0; b[:, n:] = 7.0; z0[n:] = 0.5               # padding must not be read as data
    da, db, dz = (torch.from_numpy(x).cuda() for x in (a, b, z0))
    out = torch.full((2, 3, ld), -123.0, dtype=torch.float64, device="cuda")
    cnt = torch.full((ld,), 77, dtype=torch.uint8, device="cuda")
    sgi.intersect_arc_lat(da, db, dz, mode="eft", out_xyz=out, out_count=cnt, n=n)
    torch.cuda.synchronize()
    got, gcnt = out.cpu().numpy(), cnt.cpu().numpy()
    ref, rcnt = oracle.intersect(oracle.MODE_EFT, a, b, z0, n=n)
    assert_parity(got, gcnt, ref, rcnt, n=n)
    assert (got[..., n:] == -123.0).all() and (gcnt[n:] == 77).all()


def test_empty_batch_is_a_noop():
    z = torch.empty(0, dtype=torch.float64, device="cuda")
    out, cnt = sgi.intersect_arc_lat(torch.empty((3, 0), dtype=torch.float64, device="cuda"),
                                     torch.empty((3, 0), dtype=torch.float64, device="cuda"), z)
    assert out.shape == (2, 3, 0) and cnt.shape == (0,)


def degenerate_and_special():
    """Hand-made edge inputs: degenerate arcs, exact zeros, poles, huge/tiny scales, NaN."""
    rows = [
        ((1, 0, 0), (0, 0, 1), 0.5), ((1, 0, 0), (0, 0, 1), 0.0), ((1, 0, 0), (0, 0, 1), 1.0),
        ((1, 0, 0), (0, 0, 1), 1.0000000000000009), ((1, 0, 0), (0, 1, 0), 0.0),
        ((1, 0, 0), (0, 1, 0), 0.5), ((0.6, 0, 0.8), (0.6, 0, 0.8), 0.5),
        ((1, 0, 0), (-1, 0, 0), 0.0), ((0, 0, 0), (1, 0, 0), 0.3), ((0, 0, 1), (0, 0, -1), 0.0),
        ((1, 0, 1), (-1, 0, 1), 0.75), ((1, 0, -1), (-1, 0, -1), -0.75),
        ((2.0 ** 150, 0, 2.0 ** 150), (-(2.0 ** 150), 0, 2.0 ** 150), 0.75),
        ((2.0 ** -150, 0, 2.0 ** -150), (-(2.0 ** -150), 0, 2.0 ** -150), 0.75),
        ((1, 0, 0), (0, 0, 1), float("nan")), ((float("nan"), 0, 0), (0, 0, 1), 0.5),
        ((0, 0, 1), (1, 0, 0), -0.0), ((1, 1e-300, 0), (1, -1e-300, 0), 0.0),
        ((0.3, 0.4, 0.5), (0.3, 0.4, 0.5000000000000001), 0.5),
        # an equatorial arc (n_xy = 0) at subnormal latitudes: not the equator, count 0
        ((0.6, 0.8, 0.0), (0.8, -0.6, 0.0), 5e-324), ((0.6, 0.8, 0.0), (0.8, -0.6, 0.0), -1e-323),
        ((0.6, 0.8, 0.0), (0.8, -0.6, 0.0), 2.0 ** -1050),
    ]
    a = np.array([r[0] for r in rows], float).T.copy()
    b = np.array([r[1] for r in rows], float).T.copy()
    z = np.array([r[2] for r in rows], float)
    return a, b, z


@pytest.mark.parametrize("mode,omode", MODES)
def test_edge_inputs(mode, omode):
    a, b, z0 = degenerate_and_special()
    got, gcnt = run_gpu(a, b, z0, mode)
    ref, rcnt = oracle.intersect(omode, a, b, z0)
    assert_parity(got, gcnt, ref, rcnt)
    assert gcnt[4] == 0xFF and gcnt[6] == 0xFF and gcnt[7] == 0xFF and gcnt[8] == 0xFF
    assert gcnt[14] == 0 and gcnt[15] == 0                     # NaN inputs: no points


@pytest.mark.parametrize("mode,omode", MODES)
@pytest.mark.parametrize("stride", [997, 2])
def test_special_rows_on_the_tma_path(mode, omode, stride):
    """The special rows (meridian arcs whose zero numerators fail the division guard, poles,
    degenerate and NaN inputs, extreme scales) spread through a batch large enough for the
    TMA-staged kernel (even ld, a ragged tail of 322 queries past the last whole tile), at odd
    and even positions: in the EFT modes each half of a thread's query pair takes the Exact
    recompute on its own (stride 997), or both do (stride 2)."""
    n = (1 << 19) + 322
    a, b, z0 = sgi_inputs.generate_host(1, n)
    sa, sb, sz = degenerate_and_special()
    k = sz.shape[0]
    idx = np.arange(5, n, stride)
    a[:, idx] = sa[:, idx % k]
    b[:, idx] = sb[:, idx % k]
    z0[idx] = sz[idx % k]
    got, gcnt = run_gpu(a, b, z0, mode, path=expected_path(mode, n))
    ref, rcnt = oracle.intersect(omode, a, b, z0, nthreads=NTHREADS)
    assert_parity(got, gcnt, ref, rcnt)


def test_output_layout_and_canonical_nan():
    a, b, z0 = sgi_inputs.generate_host(5, 4096)
    got, gcnt = run_gpu(a, b, z0, "eft")
    bits = got.view(np.uint64)
    for k in range(2):
        used = (gcnt != 0xFF) & (gcnt > k)
        assert np.array_equal(got[k, 2, used], z0[used])                   # P_z = z0 bitwise
        assert (bits[k, :, ~used] == 0x7FF8000000000000).all()            # canonical qNaN


def test_power_of_two_scaling_gpu():
    a, b, z0 = sgi_inputs.generate_host(3, 30000)
    base, bc = run_gpu(a, b, z0, "eft")
    for k in (-30, 30):
        got, gc = run_gpu(a * 2.0 ** k, b, z0, "eft")
        assert np.array_equal(gc, bc) and same(got, base).all()


# --------------------------------------------------------- host entry, streams, determinism
@pytest.mark.parametrize("mode", ["eft", "naive"])
def test_host_entry_matches_device_entry(mode):
    n = 1_000_003
    a, b, z0 = sgi_inputs.generate_host(5, n)
    dev, dcnt = run_gpu(a, b, z0, mode)
    pa, pb, pz = (torch.from_numpy(x).pin_memory() for x in (a, b, z0))
    out = torch.empty((2, 3, n), dtype=torch.float64).pin_memory()
    cnt = torch.empty(n, dtype=torch.uint8).pin_memory()
    work = torch.empty(sgi.host_workspace_bytes(100_000), dtype=torch.uint8, device="cuda")
    sgi.intersect_arc_lat_host(pa, pb, pz, mode=mode, out_xyz=out, out_count=cnt, work=work)
    assert np.array_equal(cnt.numpy(), dcnt) and same(out.numpy(), dev).all()
    # pageable numpy buffers work too
    o2, c2 = sgi.intersect_arc_lat_host(a, b, z0, mode=mode, work=work)
    assert np.array_equal(c2, dcnt) and same(o2, dev).all()


def test_host_entry_with_tma_sized_chunks():
    """The e2e configuration: chunks of >= 2^19 queries (so every chunk runs the TMA-staged
    kernel on the workspace's padded planes) and a ragged last chunk; equal to the device call."""
    n = (1 << 23) + 5
    a, b, z0 = sgi_inputs.generate_host(5, n)
    dev, dcnt = run_gpu(a, b, z0, "eft")
    pa, pb, pz = (torch.from_numpy(x).pin_memory() for x in (a, b, z0))
    out = torch.empty((2, 3, n), dtype=torch.float64).pin_memory()
    cnt = torch.empty(n, dtype=torch.uint8).pin_memory()
    work = torch.empty(sgi.host_workspace_bytes(1 << 21), dtype=torch.uint8, device="cuda")
    sgi.intersect_arc_lat_host(pa, pb, pz, mode="eft", out_xyz=out, out_count=cnt, work=work)
    assert np.array_equal(cnt.numpy(), dcnt) and same(out.numpy(), dev).all()


def test_side_stream_and_repeatability():
    n = 1 << 20
    da, db, dz = _device_config(5, n)
    out1, cnt1 = sgi.intersect_arc_lat(da, db, dz, mode="eft")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        out2, cnt2 = sgi.intersect_arc_lat(da, db, dz, mode="eft", stream=s)
    torch.cuda.synchronize()
    assert torch.equal(cnt1, cnt2)
    assert torch.equal(out1.view(torch.int64), out2.view(torch.int64))   # bitwise


def test_sharding_is_rank_invariant():
    """R = 1, 2, 4, 8 shards (generated by global index) concatenate to the R = 1 result."""
    n = 1 << 20
    da, db, dz = _device_config(5, n)
    ref, rcnt = sgi.intersect_arc_lat(da, db, dz, mode="eft")
    hist_ref = sgi.count_histogram(rcnt)
    for R in (2, 4, 8):
        hist = torch.zeros(5, dtype=torch.int64, device="cuda")
        for r in range(R):
            lo, hi = r * n // R, (r + 1) * n // R
            m = hi - lo
            sa = torch.empty((3, m), dtype=torch.float64, device="cuda")
            sb = torch.empty_like(sa)
            sz = torch.empty(m, dtype=torch.float64, device="cuda")
            sgi_inputs.generate_device(5, m, sa, sb, sz, offset=lo)
            o, c = sgi.intersect_arc_lat(sa, sb, sz, mode="eft")
            sgi.count_histogram(c, hist=hist)
            assert torch.equal(c, rcnt[lo:hi])
            assert torch.equal(o.view(torch.int64), ref[:, :, lo:hi].contiguous().view(torch.int64))
        assert torch.equal(hist, hist_ref)


def test_bench_strong_split_dry_run():
    """bench.py's own strong-scaling path on one device, R = 1, 2, 4, 8 ranks run one after the
    other: dist.shard_strong slices, device generation at the slice offset (bench.device_arcs),
    the EFT kernel, the histogram, the chunked K5 statistics against naive
    (bench.ref_mode_chunks) and the accuracy sample indices (dist.sample_indices); the per-rank
    results combined as reduce_after_step / reduce_accuracy combine them (SUM of histograms
    and counts, MAX of statistics) equal the R = 1 results.  This is the 1/2/4/8-GPU run's
    data path without the NCCL transport."""
    import bench
    from paper_2510_09892_b200 import dist as sdist
    n = (1 << 22) + 6                       # C5 layout, a ragged split
    stream = torch.cuda.current_stream()
    results = {}
    for R in (1, 2, 4, 8):
        hist = torch.zeros(5, dtype=torch.int64, device="cuda")
        stats = torch.zeros(2, dtype=torch.float64, device="cuda")
        counts = torch.zeros(2, dtype=torch.int64, device="cuda")
        sample = []
        for r in range(R):
            off, m = sdist.shard_strong(r, R, n)
            a = torch.empty((3, m), dtype=torch.float64, device="cuda")
            b = torch.empty_like(a)
            z0 = torch.empty(m, dtype=torch.float64, device="cuda")
            bench.device_arcs(5, m, a, b, z0, offset=off)
            out = torch.empty((2, 3, m), dtype=torch.float64, device="cuda")
            cnt = torch.empty(m, dtype=torch.uint8, device="cuda")
            sgi.intersect_arc_lat(a, b, z0, mode="eft", out_xyz=out, out_count=cnt)
            h = sgi.count_histogram(cnt)
            st, ct = bench.ref_mode_chunks(a, b, z0, m, out, cnt, "naive", stream, sgi,
                                           chunk=1 << 20)
            hist += h
            stats = torch.maximum(stats, st)
            counts += ct
            idx = sdist.sample_indices(n, 2000, off, m)
            ti = torch.from_numpy(idx).cuda()
            sample.append((out.index_select(-1, ti).cpu(), cnt.index_select(0, ti).cpu()))
        t = torch.zeros(1, dtype=torch.float64, device="cuda")
        sdist.reduce_after_step(t, hist, stats, counts)     # no process group: identity
        results[R] = (hist.cpu(), stats.cpu(), counts.cpu(),
                      torch.cat([o for o, _ in sample], -1), torch.cat([c for _, c in sample]))
    h1, s1, c1, o1, k1 = results[1]
    assert h1[:4].sum() == n and h1[0] > 0 and h1[1] > 0 and h1[2] > 0
    for R in (2, 4, 8):
        h, st, ct, o, k = results[R]
        assert torch.equal(h, h1) and torch.equal(ct, c1) and torch.equal(st, s1), R
        assert torch.equal(k, k1) and torch.equal(o.view(torch.int64), o1.view(torch.int64)), R


def test_histogram_matches_bincount():
    a, b, z0 = sgi_inputs.generate_host(5, 200_000)
    da, db, dz = (torch.from_numpy(x).cuda() for x in (a, b, z0))
    _, cnt = sgi.intersect_arc_lat(da, db, dz, mode="eft")
    hist = sgi.count_histogram(cnt).cpu().numpy()
    c = cnt.cpu().numpy()
    assert hist.tolist() == [int((c == 0).sum()), int((c == 1).sum()), int((c == 2).sum()),
                             int((c == 0xFF).sum()), int((c == 1).sum() + 2 * (c == 2).sum())]


# ------------------------------------------------------------- K5 output statistics (§8(e))
def test_output_stats_kernel():
    """sgi_output_stats against numpy on C3 (ill-conditioned: naive and EFT differ a lot):
    max ||P|-1|/u (x87 extended precision on the host), Pz == z0, count mismatches and the
    max EFT-vs-naive distance."""
    n = 150_000
    a, b, z0 = sgi_inputs.generate_host(3, n)
    da, db, dz = (torch.from_numpy(x).cuda() for x in (a, b, z0))
    o1, c1 = sgi.intersect_arc_lat(da, db, dz, mode="eft")
    o2, c2 = sgi.intersect_arc_lat(da, db, dz, mode="naive")
    st, ct = sgi.output_stats(o1, c1, dz, ref_xyz=o2, ref_count=c2)
    st0, ct0 = sgi.output_stats(o1, c1, dz)
    torch.cuda.synchronize()
    O1, C1, O2, C2 = o1.cpu().numpy(), c1.cpu().numpy(), o2.cpu().numpy(), c2.cpu().numpy()
    U = 2.0 ** -53
    dev, rdev = 0.0, 0.0
    for k in range(2):
        m = (C1 == 1) | (C1 == 2) if k == 0 else (C1 == 2)
        p = O1[k][:, m].astype(np.longdouble)
        nrm = (p[0] * p[0] + p[1] * p[1] + p[2] * p[2]) - 1
        dev = max(dev, float(np.abs(nrm).max() / 2 / U))
        assert np.array_equal(O1[k][2, m].view(np.int64), z0[m].view(np.int64))
        same = m & (C1 == C2)
        d = np.hypot(O1[k][0, same] - O2[k][0, same], O1[k][1, same] - O2[k][1, same]) / U
        rdev = max(rdev, float(d.max()))
    s = st.cpu().numpy()
    assert abs(s[0] - dev) <= 0.02 + 1e-3 * dev, (s[0], dev)
    assert 0 < s[0] <= 4.0                     # |P~| within a few u of 1
    assert s[1] == pytest.approx(rdev, rel=1e-12)
    assert ct.cpu().tolist() == [0, int((C1 != C2).sum())]
    assert ct0.cpu().tolist() == [0, 0] and st0.cpu().numpy()[1] == 0


# ------------------------------------------------------- double-word points (§8(f4), R11)
@pytest.mark.parametrize("config,n", [(1, 10_000), (3, 30_000), (6, 17 * 1000), (7, 13 * 1000),
                                      (2, (1 << 19) + 334), (3, (1 << 19) + 1000)])
@pytest.mark.parametrize("mode,omode", [("eft", oracle.MODE_EFT),
                                        ("eft_literal", oracle.MODE_EFT_LITERAL)])
def test_double_word_parity(config, n, mode, omode):
    """Small batches run the grid-stride kernel, n >= 2^19 the TMA-staged one (with a tail)."""
    a, b, z0 = sgi_inputs.generate_host(config, n)
    da, db, dz = (torch.from_numpy(x).cuda() for x in (a, b, z0))
    out, lo, cnt = sgi.intersect_arc_lat_dw(da, db, dz, mode=mode)
    assert sgi.dispatch_path(da, db, dz, out, cnt, mode=mode, entry=1) == expected_path(mode, n, 1)
    plain, pcnt = sgi.intersect_arc_lat(da, db, dz, mode=mode)
    torch.cuda.synchronize()
    ref, rlo, rcnt = oracle.intersect_dw(omode, a, b, z0, nthreads=NTHREADS)
    assert np.array_equal(cnt.cpu().numpy(), rcnt)
    assert same(out.cpu().numpy(), ref).all()
    assert same(lo.cpu().numpy(), rlo).all()
    assert same(plain.cpu().numpy(), out.cpu().numpy()).all()      # hi part = the plain result
    assert np.array_equal(pcnt.cpu().numpy(), rcnt)


@pytest.mark.parametrize("mode,omode", [("eft", oracle.MODE_EFT),
                                        ("eft_literal", oracle.MODE_EFT_LITERAL)])
@pytest.mark.parametrize("n", [20_000, (1 << 19) + 78])
def test_double_word_special_rows(mode, omode, n):
    """Double-word outputs with the special rows spread through the batch: the grid-stride
    kernel (small n) and the TMA-staged one, both through their Exact recomputes."""
    a, b, z0 = sgi_inputs.generate_host(1, n)
    sa, sb, sz = degenerate_and_special()
    idx = np.arange(3, n, 101)
    a[:, idx] = sa[:, idx % sz.shape[0]]
    b[:, idx] = sb[:, idx % sz.shape[0]]
    z0[idx] = sz[idx % sz.shape[0]]
    da, db, dz = (torch.from_numpy(x).cuda() for x in (a, b, z0))
    out, lo, cnt = sgi.intersect_arc_lat_dw(da, db, dz, mode=mode)
    assert sgi.dispatch_path(da, db, dz, out, cnt, mode=mode, entry=1) == expected_path(mode, n, 1)
    torch.cuda.synchronize()
    ref, rlo, rcnt = oracle.intersect_dw(omode, a, b, z0, nthreads=NTHREADS)
    assert np.array_equal(cnt.cpu().numpy(), rcnt)
    assert same(out.cpu().numpy(), ref).all()
    assert same(lo.cpu().numpy(), rlo).all()


def test_double_word_rejects_plain_modes():
    z = torch.zeros(8, dtype=torch.float64, device="cuda")
    v = torch.zeros((3, 8), dtype=torch.float64, device="cuda")
    with pytest.raises(sgi.SGIError):
        sgi.intersect_arc_lat_dw(v, v, z, mode="naive")


@pytest.mark.parametrize("n", [70_001, 600_001, 600_002])
@pytest.mark.parametrize("shift_in,shift_out", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("mode,omode", [("eft", oracle.MODE_EFT),
                                        ("eft_literal", oracle.MODE_EFT_LITERAL),
                                        ("naive", oracle.MODE_NAIVE)])
def test_alignment_paths(n, shift_in, shift_out, mode, omode):
    """Small batches, an odd ld and 8-B (not 16-B) aligned inputs take the LDG kernel; large
    aligned batches with an even ld the TMA kernel, two-query (EFT modes, 16-B aligned outputs)
    or one-query (8-B aligned outputs, or the other modes); every path gives the oracle's
    results, and the test asserts which kernel ran."""
    a, b, z0 = sgi_inputs.generate_host(5, n)
    def shifted(x, k):
        flat = torch.empty(x.size + k, dtype=torch.float64, device="cuda")
        v = flat[k:].view(x.shape)
        v.copy_(torch.from_numpy(x))
        return v
    da, db, dz = shifted(a, shift_in), shifted(b, shift_in), shifted(z0, shift_in)
    ob = torch.empty(6 * n + shift_out, dtype=torch.float64, device="cuda")
    out = ob[shift_out:].view(2, 3, n)
    cb = torch.empty(n + shift_out, dtype=torch.uint8, device="cuda")
    cnt = cb[shift_out:]
    if n < (1 << 19) or n % 2 or shift_in:
        want = "ldg"
    elif mode in ("eft", "eft_literal") and not shift_out:
        want = "tma_pair"
    else:
        want = "tma"
    assert sgi.dispatch_path(da, db, dz, out, cnt, mode=mode) == want
    sgi.intersect_arc_lat(da, db, dz, mode=mode, out_xyz=out, out_count=cnt)
    torch.cuda.synchronize()
    ref, rcnt = oracle.intersect(omode, a, b, z0, nthreads=NTHREADS)
    assert_parity(out.cpu().numpy(), cnt.cpu().numpy(), ref, rcnt)


@pytest.mark.parametrize("mode", ["eft", "eft_literal"])
def test_paths_agree_bitwise(mode):
    """The same queries through the TMA pair kernel, the one-query TMA kernel and the LDG kernel
    give identical outputs bit for bit (the result does not depend on lane width or tiling,
    SPEC S:298), special rows included."""
    n = (1 << 19) + 2 * 1024 + 10
    a, b, z0 = sgi_inputs.generate_host(5, n)
    sa, sb, sz = degenerate_and_special()
    idx = np.arange(7, n, 131)
    a[:, idx] = sa[:, idx % sz.shape[0]]
    b[:, idx] = sb[:, idx % sz.shape[0]]
    z0[idx] = sz[idx % sz.shape[0]]
    da, db, dz = (torch.from_numpy(x).cuda() for x in (a, b, z0))
    res = {}
    for path, shift in (("tma_pair", 0), ("tma", 1)):
        ob = torch.empty(6 * n + shift, dtype=torch.float64, device="cuda")
        out = ob[shift:].view(2, 3, n)
        cb = torch.empty(n + shift, dtype=torch.uint8, device="cuda")
        cnt = cb[shift:]
        assert sgi.dispatch_path(da, db, dz, out, cnt, mode=mode) == path
        sgi.intersect_arc_lat(da, db, dz, mode=mode, out_xyz=out, out_count=cnt)
        res[path] = (out.clone(), cnt.clone())
    # odd ld: the LDG kernel on the same data (padded planes)
    pa = torch.zeros((3, n + 1), dtype=torch.float64, device="cuda"); pa[:, :n] = da
    pb = torch.zeros((3, n + 1), dtype=torch.float64, device="cuda"); pb[:, :n] = db
    pz = torch.zeros(n + 1, dtype=torch.float64, device="cuda"); pz[:n] = dz
    out = torch.empty((2, 3, n + 1), dtype=torch.float64, device="cuda")
    cnt = torch.empty(n + 1, dtype=torch.uint8, device="cuda")
    assert sgi.dispatch_path(pa, pb, pz, out, cnt, mode=mode, n=n) == "ldg"
    sgi.intersect_arc_lat(pa, pb, pz, mode=mode, out_xyz=out, out_count=cnt, n=n)
    res["ldg"] = (out[:, :, :n].contiguous(), cnt[:n].clone())
    torch.cuda.synchronize()
    ref_o, ref_c = res["tma_pair"]
    for k in ("tma", "ldg"):
        o, c = res[k]
        assert torch.equal(c, ref_c), k
        assert torch.equal(o.view(torch.int64), ref_o.view(torch.int64)), k
