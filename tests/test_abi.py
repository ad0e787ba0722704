"""The C ABI (include/sgi.h) without a GPU: the library loads, exports every declared symbol,
and rejects invalid arguments before touching CUDA."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2510_09892_b200 as sgi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    sgi.build()
    return sgi.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sgi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sgi_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    assert declared_symbols() == sorted([
        "sgi_intersect_arc_lat", "sgi_intersect_arc_lat_host", "sgi_host_workspace_bytes",
        "sgi_count_histogram", "sgi_status_str", "sgi_last_error", "sgi_abi_version",
        "sgi_zonal_intersect", "sgi_zonal_workspace_bytes", "sgi_intersect_trace",
        "sgi_trace_fields", "sgi_output_stats", "sgi_intersect_arc_lat_dw", "sgi_dispatch_path"])


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_no_torch_in_signatures():
    src = open(os.path.join(ROOT, "include", "sgi.h")).read()
    assert "torch" not in src.lower().replace("pytorch", "") and "at::" not in src


def test_version_and_status_strings(lib):
    assert sgi.abi_version() == 1
    assert [sgi.status_str(c) for c in (0, 1, 2)] == ["SGI_OK", "SGI_E_INVALID", "SGI_E_CUDA"]


def test_workspace_bytes(lib):
    assert sgi.host_workspace_bytes(0) == 0
    assert sgi.host_workspace_bytes(1) == 3 * (13 * 256 + 256)
    assert sgi.host_workspace_bytes(1 << 20) == 3 * (13 * (8 << 20) + (1 << 20))


def _call(lib, a, b, z, n, ld, out, cnt, mode):
    return lib.sgi_intersect_arc_lat(a, b, z, n, ld, out, cnt, mode, None)


def test_invalid_arguments_rejected_without_launch(lib):
    n = 64
    a = np.zeros((3, n)); b = np.zeros((3, n)); z = np.zeros(n)
    out = np.zeros((2, 3, n)); cnt = np.zeros(n, np.uint8)
    P = lambda x: x.ctypes.data  # noqa: E731
    assert _call(lib, P(a), P(b), P(z), -1, n, P(out), P(cnt), 1) == sgi.SGI_E_INVALID
    assert _call(lib, P(a), P(b), P(z), n, n - 1, P(out), P(cnt), 1) == sgi.SGI_E_INVALID
    assert _call(lib, P(a), P(b), P(z), n, n, P(out), P(cnt), 6) == sgi.SGI_E_INVALID
    assert _call(lib, P(a), P(b), P(z), n, n, P(out), P(cnt), -1) == sgi.SGI_E_INVALID
    assert _call(lib, None, P(b), P(z), n, n, P(out), P(cnt), 1) == sgi.SGI_E_INVALID
    assert "null" in sgi.last_error()
    # outputs aliasing inputs
    assert _call(lib, P(a), P(b), P(z), n, n, P(a), P(cnt), 1) == sgi.SGI_E_INVALID
    assert "overlap" in sgi.last_error()
    assert _call(lib, P(a), P(b), P(z), n, n, P(out), P(out), 1) == sgi.SGI_E_INVALID
    # n == 0 is a no-op, even with null pointers
    assert _call(lib, None, None, None, 0, 0, None, None, 1) == sgi.SGI_OK
    assert lib.sgi_count_histogram(None, -1, None, None) == sgi.SGI_E_INVALID
    assert lib.sgi_count_histogram(None, 0, None, None) == sgi.SGI_OK


def test_zonal_validates_arguments(lib):
    tot = np.zeros(1, np.uint64)
    assert lib.sgi_zonal_intersect(None, None, -1, 0, None, 0, 0, None, None, None, None,
                                   tot.ctypes.data, None, 0, 1, None) == sgi.SGI_E_INVALID
    e = np.zeros((3, 8)); lat = np.zeros(4)
    assert lib.sgi_zonal_intersect(e.ctypes.data, e.ctypes.data, 8, 8, lat.ctypes.data, 4, 0,
                                   None, None, None, None, tot.ctypes.data, None, 0, 1,
                                   None) == sgi.SGI_E_INVALID          # no workspace
    assert lib.sgi_zonal_intersect(e.ctypes.data, e.ctypes.data, 8, 8, lat.ctypes.data, 4, 0,
                                   None, None, None, None, tot.ctypes.data, 0x10008, 1 << 20, 1,
                                   None) == sgi.SGI_E_INVALID          # workspace not 16-B aligned
    assert sgi.zonal_workspace_bytes(0) == 8                       # the tile-sum terminator
    assert sgi.zonal_workspace_bytes(1000) == 1000 * 8 + (2 + 1) * 8   # 512-edge tiles
    assert sgi.zonal_workspace_bytes(-1) == 0


def test_host_entry_validates_workspace(lib):
    n = 16
    a = np.zeros((3, n)); b = np.zeros((3, n)); z = np.zeros(n)
    out = np.zeros((2, 3, n)); cnt = np.zeros(n, np.uint8)
    P = lambda x: x.ctypes.data  # noqa: E731
    rc = lib.sgi_intersect_arc_lat_host(P(a), P(b), P(z), n, n, P(out), P(cnt), 1, None, 0, None)
    assert rc == sgi.SGI_E_INVALID


def test_dispatch_path_rules(lib):
    """The kernel choice (no device access): LDG below 2^19 queries, for an odd ld or inputs not
    16-B aligned; the TMA pair kernel in the EFT modes with 16-B aligned outputs; the one-query
    TMA kernel otherwise; the double-word entry never pairs."""
    D = lib.sgi_dispatch_path
    n = 1 << 20
    base = 1 << 40                                   # fake, well separated 256-B aligned bases
    a, b, z, out, cnt = (base + k * (1 << 34) for k in range(5))
    eft, lit, naive = 1, 2, 0
    assert D(a, b, z, n, n, out, cnt, eft, 0) == 3
    assert D(a, b, z, n, n, out, cnt, lit, 0) == 3
    assert D(a, b, z, n, n, out, cnt, naive, 0) == 2
    assert D(a, b, z, n, n, out + 8, cnt, eft, 0) == 2        # 8-B aligned outputs: one query
    assert D(a, b, z, n, n, out, cnt + 1, eft, 0) == 2        # odd count base: one query
    assert D(a + 8, b, z, n, n, out, cnt, eft, 0) == 1        # 8-B aligned inputs: LDG
    assert D(a, b, z, n - 1, n - 1, out, cnt, eft, 0) == 1    # odd ld: LDG
    assert D(a, b, z, n - 1, n, out, cnt, eft, 0) == 3        # odd n, even ld: TMA + tail
    assert D(a, b, z, (1 << 19) - 2, 1 << 19, out, cnt, eft, 0) == 1   # small batch
    assert D(a, b, z, n, n, out, cnt, eft, 1) == 2            # double-word: one query / thread
    assert D(a, b, z, n, n, out, cnt, naive, 1) == 0          # double-word needs an EFT mode
    assert D(a, b, z, 0, 0, out, cnt, eft, 0) == 0
    assert D(a, b, z, n, n, a, cnt, eft, 0) == 0              # aliasing: rejected
    assert D(a, b, z, n, n - 2, out, cnt, eft, 0) == 0        # ld < n: rejected


def test_host_binding_validates_host_arrays():
    """The host-buffer binding checks dtype, shape and contiguity before any pointer reaches C
    (a wrong array would make the 2D copies read or write past the host buffers)."""
    n = 64
    a = np.zeros((3, n)); b = np.zeros((3, n)); z = np.zeros(n)
    bad = [dict(a=a.astype(np.float32)), dict(a=np.zeros((n, 3))), dict(b=np.zeros((3, 2 * n))[:, ::2]),
           dict(out_xyz=np.zeros((2, 3, n), np.float32)), dict(out_count=np.zeros(n, np.int32)),
           dict(z0=np.zeros(n + 1), a=np.zeros((3, n + 1)), b=np.zeros((3, n)))]
    for kw in bad:
        args = dict(a=a, b=b, z0=z)
        args.update(kw)
        with pytest.raises(ValueError):
            sgi.intersect_arc_lat_host(args.pop("a"), args.pop("b"), args.pop("z0"), **args)
    with pytest.raises(ValueError):
        sgi.intersect_arc_lat_host(a, b, z, n=n + 1)


def test_product_package_does_not_import_oracle():
    """The product path never routes through the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2510_09892_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "eft_oracle" not in text, f


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(sgi, "_lib", None)
    monkeypatch.setattr(sgi, "LIB_PATH", str(tmp_path / "libsgi.so"))
    with pytest.raises(sgi.SGIError):
        sgi.abi_version()
