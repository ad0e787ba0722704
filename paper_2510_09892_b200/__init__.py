"""paper_2510_09892_b200 — B200-native batched arc/latitude intersections (arXiv 2510.09892).

Thin ctypes binding over the C ABI of ``libsgi.so`` (include/sgi.h): argument marshalling only;
every step of the path runs in the CUDA kernels of ``csrc/``.  There is no CPU fallback: if the
library is missing or no CUDA device is present, calls raise.

Public API (same names as the C ABI):
    intersect_arc_lat(a, b, z0, mode="eft", out_xyz=None, out_count=None, n=None, stream=None)
    intersect_arc_lat_host(a, b, z0, mode="eft", out_xyz=None, out_count=None, work=None, ...)
    count_histogram(out_count, n=None, hist=None, stream=None)
    zonal_intersect(va, vb, lat_z0, mode="eft", cap=None, stream=None)
    intersect_trace(a, b, z0, mode="eft", n=None, stream=None)   (Appendix-A intermediates)
    output_stats(out_xyz, out_count, z0, ref_xyz=None, ref_count=None)  (K5 invariants)
    intersect_arc_lat_dw(a, b, z0, mode="eft")                   (double-word points)
    host_workspace_bytes(chunk), abi_version(), status_str(code), last_error()
Layout: a[3, ld], b[3, ld], z0[ld] float64; out_xyz[2, 3, ld] float64; out_count[ld] uint8.
"""
from __future__ import annotations

import ctypes
import os

from ._build import LIB_PATH, build  # noqa: F401

MODES = {"naive": 0, "eft": 1, "eft_literal": 2, "yac": 3, "base": 4, "naive_kahan": 5}
# sgi_intersect_trace field order (include/sgi.h SGI_TRACE_*)
TRACE_FIELDS = ("nx", "ex", "ny", "ey", "nz", "ez", "S2", "s2", "S3", "s3", "C", "eC", "D", "eD",
                "sh", "sl", "s", "es", "Fx", "eFx", "Fy", "eFy", "Xp", "Yp", "Xm", "Ym",
                "Ppx", "Ppy", "Pmx", "Pmy",
                "Xp_p", "Xp_s", "Yp_p", "Yp_s", "Xm_p", "Xm_s", "Ym_p", "Ym_s")
DEGENERATE = 0xFF
SGI_OK, SGI_E_INVALID, SGI_E_CUDA = 0, 1, 2
# sgi_dispatch_path results (include/sgi.h SGI_PATH_*)
PATHS = {0: "none", 1: "ldg", 2: "tma", 3: "tma_pair"}

_lib = None


class SGIError(RuntimeError):
    pass


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SGIError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                           "g.build()'` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        L.sgi_intersect_arc_lat.restype = ctypes.c_int
        L.sgi_intersect_arc_lat.argtypes = [vp, vp, vp, i64, i64, vp, vp, ctypes.c_int, vp]
        L.sgi_intersect_arc_lat_host.restype = ctypes.c_int
        L.sgi_intersect_arc_lat_host.argtypes = [vp, vp, vp, i64, i64, vp, vp, ctypes.c_int, vp,
                                                 ctypes.c_size_t, vp]
        L.sgi_host_workspace_bytes.restype = ctypes.c_size_t
        L.sgi_host_workspace_bytes.argtypes = [i64]
        L.sgi_count_histogram.restype = ctypes.c_int
        L.sgi_count_histogram.argtypes = [vp, i64, vp, vp]
        L.sgi_zonal_intersect.restype = ctypes.c_int
        L.sgi_zonal_intersect.argtypes = [vp, vp, i64, i64, vp, ctypes.c_int32, i64, vp, vp, vp,
                                          vp, vp, vp, ctypes.c_size_t, ctypes.c_int, vp]
        L.sgi_zonal_workspace_bytes.restype = ctypes.c_size_t
        L.sgi_zonal_workspace_bytes.argtypes = [i64]
        L.sgi_intersect_arc_lat_dw.restype = ctypes.c_int
        L.sgi_intersect_arc_lat_dw.argtypes = [vp, vp, vp, i64, i64, vp, vp, vp, ctypes.c_int, vp]
        L.sgi_output_stats.restype = ctypes.c_int
        L.sgi_output_stats.argtypes = [vp, vp, vp, i64, i64, vp, vp, vp, vp, vp]
        L.sgi_intersect_trace.restype = ctypes.c_int
        L.sgi_intersect_trace.argtypes = [vp, vp, vp, i64, i64, vp, vp, ctypes.c_int, vp]
        L.sgi_trace_fields.restype = ctypes.c_int
        L.sgi_trace_fields.argtypes = []
        L.sgi_status_str.restype = ctypes.c_char_p
        L.sgi_status_str.argtypes = [ctypes.c_int]
        L.sgi_last_error.restype = ctypes.c_char_p
        L.sgi_last_error.argtypes = []
        L.sgi_abi_version.restype = ctypes.c_int
        L.sgi_abi_version.argtypes = []
        L.sgi_dispatch_path.restype = ctypes.c_int
        L.sgi_dispatch_path.argtypes = [vp, vp, vp, i64, i64, vp, vp, ctypes.c_int, ctypes.c_int]
        _lib = L
    return _lib


def lib():
    """The loaded libsgi.so (ctypes.CDLL)."""
    return _load()


def abi_version() -> int:
    return _load().sgi_abi_version()


def status_str(code: int) -> str:
    return _load().sgi_status_str(code).decode()


def last_error() -> str:
    return _load().sgi_last_error().decode()


def _check(rc: int, what: str) -> None:
    if rc != SGI_OK:
        raise SGIError(f"{what}: {status_str(rc)}: {last_error()}")


def _mode(mode) -> int:
    return MODES[mode] if isinstance(mode, str) else int(mode)


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _cuda_f64(t, shape, name):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
            and t.is_contiguous() and tuple(t.shape) == shape):
        raise ValueError(f"{name} must be a contiguous CUDA float64 tensor of shape {shape}")


def _cuda_u8(t, name, shape=None):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.uint8
            and t.is_contiguous() and t.dim() == 1 and (shape is None or tuple(t.shape) == shape)):
        raise ValueError(f"{name} must be a contiguous 1-D CUDA uint8 tensor"
                         + (f" of shape {shape}" if shape else ""))


def intersect_arc_lat(a, b, z0, mode="eft", out_xyz=None, out_count=None, n=None, stream=None):
    """Device entry: torch CUDA tensors a[3, ld], b[3, ld], z0[ld] -> (out_xyz[2,3,ld], out_count[ld]).

    Enqueued on `stream` (torch.cuda.Stream, default: current); does not synchronise."""
    import torch
    ld = z0.shape[0]
    n = ld if n is None else n
    _cuda_f64(a, (3, ld), "a")
    _cuda_f64(b, (3, ld), "b")
    _cuda_f64(z0, (ld,), "z0")
    if out_xyz is None:
        out_xyz = torch.empty((2, 3, ld), dtype=torch.float64, device=z0.device)
    if out_count is None:
        out_count = torch.empty(ld, dtype=torch.uint8, device=z0.device)
    _cuda_f64(out_xyz, (2, 3, ld), "out_xyz")
    _cuda_u8(out_count, "out_count", (ld,))
    rc = _load().sgi_intersect_arc_lat(a.data_ptr(), b.data_ptr(), z0.data_ptr(), n, ld,
                                       out_xyz.data_ptr(), out_count.data_ptr(), _mode(mode),
                                       _stream_ptr(stream))
    _check(rc, "sgi_intersect_arc_lat")
    return out_xyz, out_count


def intersect_arc_lat_dw(a, b, z0, mode="eft", n=None, stream=None):
    """Double-word points (sgi_intersect_arc_lat_dw): -> (out_xyz[2,3,ld], out_lo[2,2,ld],
    out_count[ld]); P ~ out_xyz + out_lo for x and y."""
    import torch
    ld = z0.shape[0]
    n = ld if n is None else n
    _cuda_f64(a, (3, ld), "a")
    _cuda_f64(b, (3, ld), "b")
    _cuda_f64(z0, (ld,), "z0")
    out = torch.empty((2, 3, ld), dtype=torch.float64, device=z0.device)
    lo = torch.empty((2, 2, ld), dtype=torch.float64, device=z0.device)
    cnt = torch.empty(ld, dtype=torch.uint8, device=z0.device)
    rc = _load().sgi_intersect_arc_lat_dw(a.data_ptr(), b.data_ptr(), z0.data_ptr(), n, ld,
                                          out.data_ptr(), lo.data_ptr(), cnt.data_ptr(),
                                          _mode(mode), _stream_ptr(stream))
    _check(rc, "sgi_intersect_arc_lat_dw")
    return out, lo, cnt


def output_stats(out_xyz, out_count, z0, ref_xyz=None, ref_count=None, n=None, stats=None,
                 counts=None, stream=None):
    """sgi_output_stats: (stats float64[2] = [max ||P|-1|/u, max |P - Pref|/u], counts int64[2] =
    [points with Pz != z0, count mismatches vs ref]) as CUDA tensors (accumulated if given)."""
    import torch
    ld = z0.shape[0]
    n = ld if n is None else n
    _cuda_f64(z0, (ld,), "z0")
    _cuda_f64(out_xyz, (2, 3, ld), "out_xyz")
    _cuda_u8(out_count, "out_count", (ld,))
    if (ref_xyz is None) != (ref_count is None):
        raise ValueError("give both ref_xyz and ref_count, or neither")
    if ref_xyz is not None:
        _cuda_f64(ref_xyz, (2, 3, ld), "ref_xyz")
        _cuda_u8(ref_count, "ref_count", (ld,))
    dev = z0.device
    if stats is None:
        stats = torch.zeros(2, dtype=torch.float64, device=dev)
    if counts is None:
        counts = torch.zeros(2, dtype=torch.int64, device=dev)
    rc = _load().sgi_output_stats(out_xyz.data_ptr(), out_count.data_ptr(), z0.data_ptr(), n, ld,
                                  None if ref_xyz is None else ref_xyz.data_ptr(),
                                  None if ref_count is None else ref_count.data_ptr(),
                                  stats.data_ptr(), counts.data_ptr(), _stream_ptr(stream))
    _check(rc, "sgi_output_stats")
    return stats, counts


def intersect_trace(a, b, z0, mode="eft", n=None, stream=None):
    """Appendix-A instrumentation (sgi_intersect_trace): every intermediate of each query ->
    (trace[len(TRACE_FIELDS), ld] float64 CUDA tensor, out_count[ld] uint8)."""
    import torch
    ld = z0.shape[0]
    n = ld if n is None else n
    _cuda_f64(a, (3, ld), "a")
    _cuda_f64(b, (3, ld), "b")
    _cuda_f64(z0, (ld,), "z0")
    L = _load()
    assert L.sgi_trace_fields() == len(TRACE_FIELDS)
    trace = torch.zeros((len(TRACE_FIELDS), ld), dtype=torch.float64, device=z0.device)
    cnt = torch.empty(ld, dtype=torch.uint8, device=z0.device)
    rc = L.sgi_intersect_trace(a.data_ptr(), b.data_ptr(), z0.data_ptr(), n, ld, trace.data_ptr(),
                               cnt.data_ptr(), _mode(mode), _stream_ptr(stream))
    _check(rc, "sgi_intersect_trace")
    return trace, cnt


def dispatch_path(a, b, z0, out_xyz, out_count, mode="eft", n=None, entry=0) -> str:
    """Which kernel sgi_intersect_arc_lat (entry 0) or sgi_intersect_arc_lat_dw (entry 1) launches
    for these tensors: "ldg", "tma" (one query per thread) or "tma_pair" (two per thread)."""
    ld = z0.shape[0]
    n = ld if n is None else n
    return PATHS[_load().sgi_dispatch_path(a.data_ptr(), b.data_ptr(), z0.data_ptr(), n, ld,
                                           out_xyz.data_ptr(), out_count.data_ptr(), _mode(mode),
                                           entry)]


def _host_array(x, shape, dtype):
    """Host buffer check for the host-buffer entry: C-contiguous numpy array or CPU tensor of
    exactly this shape and dtype (the C side reads/writes ld-pitched planes through it)."""
    import numpy as np
    import torch
    if isinstance(x, torch.Tensor):
        tdt = {np.float64: torch.float64, np.uint8: torch.uint8}[dtype]
        ok = (x.device.type == "cpu" and x.dtype == tdt and x.is_contiguous()
              and tuple(x.shape) == shape)
        return ok and x.data_ptr()
    if isinstance(x, np.ndarray):
        ok = x.dtype == dtype and x.flags.c_contiguous and x.shape == shape
        return ok and x.ctypes.data
    return False


def host_workspace_bytes(chunk: int) -> int:
    return int(_load().sgi_host_workspace_bytes(chunk))


def intersect_arc_lat_host(a, b, z0, mode="eft", out_xyz=None, out_count=None, work=None,
                           n=None, stream=None):
    """Host-buffer entry (end to end): numpy or CPU torch arrays in, host arrays out.

    `work` is a CUDA uint8 tensor used as the device workspace (default: a 64 Mi-arc chunk
    buffer is allocated).  Pinned host memory lets the chunked copies overlap the kernels."""
    import numpy as np
    import torch

    ld = z0.shape[0]
    n = ld if n is None else n
    if not 0 <= n <= ld:
        raise ValueError(f"need 0 <= n <= ld, got n={n}, ld={ld}")
    if out_xyz is None:
        out_xyz = np.empty((2, 3, ld), np.float64)
    if out_count is None:
        out_count = np.empty(ld, np.uint8)
    ptrs = []
    for x, shape, dt, name in ((a, (3, ld), np.float64, "a"), (b, (3, ld), np.float64, "b"),
                               (z0, (ld,), np.float64, "z0"),
                               (out_xyz, (2, 3, ld), np.float64, "out_xyz"),
                               (out_count, (ld,), np.uint8, "out_count")):
        p = _host_array(x, shape, dt)
        if p is False:
            raise ValueError(f"{name} must be a C-contiguous host {np.dtype(dt).name} array "
                             f"(numpy or CPU tensor) of shape {shape}")
        ptrs.append(p)
    if work is None:
        work = torch.empty(host_workspace_bytes(min(max(n, 1), 1 << 22)), dtype=torch.uint8,
                           device="cuda")
    if not (isinstance(work, torch.Tensor) and work.is_cuda and work.is_contiguous()):
        raise ValueError("work must be a contiguous CUDA tensor")
    rc = _load().sgi_intersect_arc_lat_host(*ptrs[:3], n, ld, *ptrs[3:], _mode(mode),
                                            work.data_ptr(), work.numel() * work.element_size(),
                                            _stream_ptr(stream))
    _check(rc, "sgi_intersect_arc_lat_host")
    return out_xyz, out_count


def count_histogram(out_count, n=None, hist=None, stream=None):
    """Device histogram [#0, #1, #2, #degenerate, #points] (int64 CUDA tensor, accumulated)."""
    import torch
    _cuda_u8(out_count, "out_count")
    n = out_count.shape[0] if n is None else n
    if not 0 <= n <= out_count.shape[0]:
        raise ValueError(f"n={n} outside out_count's length {out_count.shape[0]}")
    if hist is None:
        hist = torch.zeros(5, dtype=torch.int64, device=out_count.device)
    if not (hist.is_cuda and hist.dtype == torch.int64 and hist.is_contiguous()
            and tuple(hist.shape) == (5,)):
        raise ValueError("hist must be a contiguous CUDA int64 tensor of shape (5,)")
    rc = _load().sgi_count_histogram(out_count.data_ptr(), n, hist.data_ptr(), _stream_ptr(stream))
    _check(rc, "sgi_count_histogram")
    return hist


def zonal_workspace_bytes(n_edges: int) -> int:
    return int(_load().sgi_zonal_workspace_bytes(n_edges))


def zonal_intersect(va, vb, lat_z0, mode="eft", cap=None, n_edges=None, stream=None, work=None):
    """Fused zonal-mean pass (sgi_zonal_intersect): CUDA float64 edges va[3, ld], vb[3, ld] and a
    strictly increasing latitude table lat_z0[K] -> dict(edge int64, lat int32, count uint8,
    xyz float64 [2, 3, m]) over the m candidate pairs, edge-major, latitude ascending.

    With cap=None a count-only call sizes the outputs first (one synchronisation)."""
    import torch
    ld = va.shape[1]
    n_edges = ld if n_edges is None else n_edges
    _cuda_f64(va, (3, ld), "va")
    _cuda_f64(vb, (3, ld), "vb")
    _cuda_f64(lat_z0, (lat_z0.shape[0],), "lat_z0")
    dev = va.device
    L = _load()
    if work is None:
        work = torch.empty(max(zonal_workspace_bytes(n_edges), 8), dtype=torch.uint8, device=dev)
    total = torch.zeros(1, dtype=torch.int64, device=dev)
    sp = _stream_ptr(stream)
    if cap is None:
        rc = L.sgi_zonal_intersect(va.data_ptr(), vb.data_ptr(), n_edges, ld, lat_z0.data_ptr(),
                                   lat_z0.shape[0], 0, None, None, None, None, total.data_ptr(),
                                   work.data_ptr(), work.numel(), _mode(mode), sp)
        _check(rc, "sgi_zonal_intersect (count)")
        (torch.cuda.current_stream() if stream is None else stream).synchronize()
        cap = int(total.item())
    cap_alloc = max(cap, 1)
    out = {"edge": torch.empty(cap_alloc, dtype=torch.int64, device=dev),
           "lat": torch.empty(cap_alloc, dtype=torch.int32, device=dev),
           "count": torch.empty(cap_alloc, dtype=torch.uint8, device=dev),
           "xyz": torch.empty((2, 3, cap_alloc), dtype=torch.float64, device=dev)}
    rc = L.sgi_zonal_intersect(va.data_ptr(), vb.data_ptr(), n_edges, ld, lat_z0.data_ptr(),
                               lat_z0.shape[0], cap, out["edge"].data_ptr(), out["lat"].data_ptr(),
                               out["count"].data_ptr(), out["xyz"].data_ptr(), total.data_ptr(),
                               work.data_ptr(), work.numel(), _mode(mode), sp)
    _check(rc, "sgi_zonal_intersect")
    out["total"] = total
    out["cap"] = cap
    return out
