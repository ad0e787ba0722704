"""The kernels under a debug build (-DSGI_DEBUG_CHECKS=1): device asserts on every shared-memory
queue, table and tile index, and shared scratch poisoned at kernel start — the stand-in for
compute-sanitizer memcheck / initcheck, which this GPU pool does not run
(profiles/r02/r02h_compute_sanitizer_unavailable.log).  Every path must run without a device
assert and give exactly the release library's outputs: the TMA pair kernel with its deferred
recompute queue, the one-query TMA kernel, the LDG kernel, the fused zonal pass, the three-launch
zonal pass (count-only call and a latitude table too large for shared memory)."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2510_09892_b200 as sgi  # noqa: E402
import sgi_inputs  # noqa: E402
from paper_2510_09892_b200._build import build_debug  # noqa: E402

pytestmark = pytest.mark.gpu
vp, i64 = ctypes.c_void_p, ctypes.c_int64


@pytest.fixture(scope="module")
def dbg():
    L = ctypes.CDLL(build_debug())
    L.sgi_intersect_arc_lat.argtypes = [vp, vp, vp, i64, i64, vp, vp, ctypes.c_int, vp]
    L.sgi_zonal_intersect.argtypes = [vp, vp, i64, i64, vp, ctypes.c_int32, i64, vp, vp, vp,
                                      vp, vp, vp, ctypes.c_size_t, ctypes.c_int, vp]
    L.sgi_zonal_workspace_bytes.restype = ctypes.c_size_t
    L.sgi_zonal_workspace_bytes.argtypes = [i64]
    return L


def _special_batch(n):
    a, b, z0 = sgi_inputs.generate_host(5, n)
    # meridian (zero numerators), pole tangent, degenerate, NaN rows: certificates fail, the
    # deferred queue runs
    rows = [((1, 0, 0), (0, 0, 1), 0.5), ((1, 0, 0), (0, 0, 1), 1.0), ((1, 0, 0), (-1, 0, 0), 0.0),
            ((1, 0, 0), (0, 0, 1), float("nan")), ((1, 0, 1), (-1, 0, 1), 0.75)]
    idx = np.arange(3, n, 97)
    for j, i in enumerate(idx):
        ra, rb, rz = rows[j % len(rows)]
        a[:, i], b[:, i], z0[i] = ra, rb, rz
    return a, b, z0


@pytest.mark.parametrize("mode", ["eft", "naive"])
@pytest.mark.parametrize("n,shift", [((1 << 20) + 2, 0), ((1 << 20) + 2, 1), (100_001, 0)])
def test_batch_kernels_under_checks(dbg, mode, n, shift):
    a, b, z0 = _special_batch(n)
    da, db, dz = (torch.from_numpy(x).cuda() for x in (a, b, z0))
    ob = torch.empty(6 * n + shift, dtype=torch.float64, device="cuda")
    out = ob[shift:].view(2, 3, n)
    cb = torch.empty(n + shift, dtype=torch.uint8, device="cuda")
    cnt = cb[shift:]
    rc = dbg.sgi_intersect_arc_lat(da.data_ptr(), db.data_ptr(), dz.data_ptr(), n, n,
                                   out.data_ptr(), cnt.data_ptr(), sgi.MODES[mode], None)
    assert rc == 0
    torch.cuda.synchronize()                       # a device assert would surface here
    ref, rcnt = sgi.intersect_arc_lat(da, db, dz, mode=mode)
    torch.cuda.synchronize()
    assert torch.equal(cnt, rcnt)
    assert torch.equal(out.view(torch.int64), ref.view(torch.int64))


def _zonal(L, va, vb, lat, cap, mode=1):
    ne = va.shape[1]
    work = torch.empty(max(int(L.sgi_zonal_workspace_bytes(ne)), 8), dtype=torch.uint8,
                       device="cuda")
    total = torch.zeros(1, dtype=torch.int64, device="cuda")
    o = {"edge": torch.empty(max(cap, 1), dtype=torch.int64, device="cuda"),
         "lat": torch.empty(max(cap, 1), dtype=torch.int32, device="cuda"),
         "count": torch.empty(max(cap, 1), dtype=torch.uint8, device="cuda"),
         "xyz": torch.empty((2, 3, max(cap, 1)), dtype=torch.float64, device="cuda")}
    rc = L.sgi_zonal_intersect(va.data_ptr(), vb.data_ptr(), ne, ne, lat.data_ptr(), lat.shape[0],
                               cap, o["edge"].data_ptr(), o["lat"].data_ptr(),
                               o["count"].data_ptr(), o["xyz"].data_ptr(), total.data_ptr(),
                               work.data_ptr(), work.numel(), mode, None)
    assert rc == 0
    torch.cuda.synchronize()
    return o, int(total.item())


@pytest.mark.parametrize("ne,nlat", [(32, 180), (64, 1800), (16, 5000)])
def test_zonal_under_checks(dbg, ne, nlat):
    va, vb = sgi_inputs.cubed_sphere_edges(ne)
    dva, dvb = torch.from_numpy(va).cuda(), torch.from_numpy(vb).cuda()
    lat = torch.from_numpy(sgi_inputs.latitudes(nlat)).cuda()
    ref = sgi.zonal_intersect(dva, dvb, lat, mode="eft")
    torch.cuda.synchronize()
    cap = ref["cap"]
    _, tot0 = _zonal(dbg, dva, dvb, lat, 0)           # count-only: the three-launch filter/scan
    assert tot0 == cap
    got, tot = _zonal(dbg, dva, dvb, lat, cap)
    assert tot == cap
    for k in ("edge", "lat", "count"):
        assert torch.equal(got[k][:cap], ref[k][:cap]), k
    assert torch.equal(got["xyz"][..., :cap].contiguous().view(torch.int64),
                       ref["xyz"][..., :cap].contiguous().view(torch.int64))
