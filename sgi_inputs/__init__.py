"""sgi_inputs — seeded synthetic workloads for the arc/latitude intersection path.

A module of its own (see gen.h): it builds inputs only and holds none of the method's
arithmetic.  Both the oracles (tests, cpu_baseline) and the CUDA path (tests, bench) consume
its output.  Layout everywhere is SoA: ``a[3, ld]``, ``b[3, ld]``, ``z0[ld]`` float64.

Configs (BASELINE.json ``configs``, recipe in DESIGN.md §3):
  1  C1  10,000 arcs, endpoints uniform on the sphere, z0 between endpoint z   (seed 0)
  2  C2  2^24 short arcs, length log-uniform in [1e-4, 1e-2] rad               (seed 2)
  3  C3  2^24 ill-conditioned arcs: near-tangent / near-polar / near-coincident (seed 3)
  4  C4  cubed-sphere ne=1024 edges x 1,800 latitudes, zonal-mean pairing      (numpy, host)
  5  C5  2^30 mixed arcs, sharded by global index                              (seed 5)
  6  the paper's primary accuracy dataset: 17 latitude bands, arc i in band i % 17 (seed 6)
  7  the paper's secondary dataset: 13 decades of the offset r, arc i in decade
     i % 13                                                                     (seed 7)
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
HOST_LIB = os.path.join(_HERE, "libsgi_gen_host.so")
DEV_LIB = os.path.join(_HERE, "libsgi_gen_dev.so")

CONFIG_SIZES = {1: 10_000, 2: 1 << 24, 3: 1 << 24, 5: 1 << 30, 6: 17 << 16, 7: 13 << 16}
CONFIG_SEEDS = {1: 0, 2: 2, 3: 3, 4: 4, 5: 5, 6: 6, 7: 7}
C3_CLASSES = ("near-tangent", "near-polar", "near-coincident")
# gen.h gen_band_edge(): latitude band edges in degrees of the primary dataset (SPEC S:506's
# default schedule; the paper does not print its own), and the secondary dataset's r decades
PRIMARY_BAND_EDGES = (0.0, 1e-4, 1e-3, 1e-2, 0.1, 1.0, 11.0, 21.0, 31.0, 41.0, 51.0, 61.0, 71.0,
                      81.0, 89.0, 89.9, 89.99, 89.999)
SECONDARY_DECADES = tuple((10.0 ** (d - 15), 10.0 ** (d - 14)) for d in range(13))


def group_of(config: int, index):
    """Band (config 6) or r decade (config 7) of global arc index (scalar or array)."""
    if config == 6:
        return index % (len(PRIMARY_BAND_EDGES) - 1)
    if config == 7:
        return index % len(SECONDARY_DECADES)
    raise ValueError(f"config {config} has no groups")


def group_label(config: int, g: int) -> str:
    if config == 6:
        return f"lat ({PRIMARY_BAND_EDGES[g]:g}, {PRIMARY_BAND_EDGES[g + 1]:g}] deg"
    lo, hi = SECONDARY_DECADES[g]
    return f"r [{lo:.0e}, {hi:.0e})"


def _newer(target: str, *sources: str) -> bool:
    return os.path.exists(target) and all(
        os.path.getmtime(target) >= os.path.getmtime(s) for s in sources)


def build(device: bool = True) -> None:
    """Compile the host (gcc) and device (nvcc, sm_100a) builds of gen.h in-tree."""
    hdr = os.path.join(_HERE, "gen.h")
    src = os.path.join(_HERE, "gen_host.c")
    if not _newer(HOST_LIB, hdr, src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-fast-math", "-fopenmp", "-o", HOST_LIB, src, "-lm"])
    if device:
        dsrc = os.path.join(_HERE, "gen_device.cu")
        if not _newer(DEV_LIB, hdr, dsrc):
            subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                                   "-fmad=false", "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
                                   "-o", DEV_LIB, dsrc])


_host = None
_dev = None


def _host_lib():
    global _host
    if _host is None:
        if not os.path.exists(HOST_LIB):
            build(device=False)
        lib = ctypes.CDLL(HOST_LIB)
        lib.sgi_gen_host.restype = ctypes.c_int
        lib.sgi_gen_host.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p]
        _host = lib
    return _host


def _dev_lib():
    global _dev
    if _dev is None:
        if not os.path.exists(DEV_LIB):
            raise RuntimeError(f"{DEV_LIB} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(DEV_LIB)
        lib.sgi_gen_device.restype = ctypes.c_int
        lib.sgi_gen_device.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _dev = lib
    return _dev


def generate_host(config: int, n: int, offset: int = 0, seed: int | None = None,
                  ld: int | None = None):
    """Arcs [offset, offset+n) of `config` (1, 2, 3, 5, 6 or 7) on the host.

    Returns (a, b, z0) as float64 arrays of shapes (3, ld), (3, ld), (ld,); columns >= n are 0.
    """
    if seed is None:
        seed = CONFIG_SEEDS[config]
    ld = n if ld is None else ld
    a = np.zeros((3, ld), np.float64)
    b = np.zeros((3, ld), np.float64)
    z0 = np.zeros(ld, np.float64)
    rc = _host_lib().sgi_gen_host(config, seed, offset, n, ld, a.ctypes.data, b.ctypes.data,
                                  z0.ctypes.data)
    if rc != 0:
        raise ValueError(f"sgi_gen_host rejected config={config} n={n} ld={ld} offset={offset}")
    return a, b, z0


def generate_device(config: int, n: int, a, b, z0, offset: int = 0, seed: int | None = None,
                    stream=None) -> None:
    """Fill caller-owned CUDA tensors a[3, ld], b[3, ld], z0[ld] (float64, contiguous) with arcs
    [offset, offset+n) of `config` on `stream` (a torch.cuda.Stream or None = current)."""
    import torch
    if seed is None:
        seed = CONFIG_SEEDS[config]
    ld = z0.shape[0]
    for t, shape in ((a, (3, ld)), (b, (3, ld)), (z0, (ld,))):
        if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous() or tuple(t.shape) != shape:
            raise ValueError("generate_device expects contiguous CUDA float64 a[3,ld], b[3,ld], z0[ld]")
    if stream is None:
        stream = torch.cuda.current_stream()
    rc = _dev_lib().sgi_gen_device(config, seed, offset, n, ld, a.data_ptr(), b.data_ptr(),
                                   z0.data_ptr(), ctypes.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"sgi_gen_device failed rc={rc}")


# ----------------------------------------------------------------------------- C4 (host, numpy)
def latitudes(nlat: int = 1800) -> np.ndarray:
    """z0_k = RN(sin(phi_k)), phi_k = -90 + (k + 1/2) * 180/nlat degrees (cell-centred)."""
    return np.array([math.sin(math.radians(-90.0 + (k + 0.5) * 180.0 / nlat))
                     for k in range(nlat)], np.float64)


def _cube_tan(ne: int) -> np.ndarray:
    """Equiangular coordinate t(k) = tan(-pi/4 + k*pi/(2 ne)), exactly antisymmetric, t(0) = -1."""
    t = np.array([math.tan(-math.pi / 4 + k * math.pi / (2 * ne)) for k in range(ne + 1)])
    t[0], t[ne] = -1.0, 1.0
    for k in range(ne // 2 + 1):
        t[ne - k] = -t[k]
    if ne % 2 == 0:
        t[ne // 2] = 0.0
    return t


def cubed_sphere_edges(ne: int = 1024):
    """Unique great-circle edges of the equiangular gnomonic cubed sphere.

    Vertices live on the integer cube lattice {0..ne}^3 surface; their coordinates are
    unit((t(X), t(Y), t(Z))), computed once per lattice vertex so shared seam vertices are
    bit-identical.  Returns (va, vb) float64 arrays of shape (3, E), oriented low -> high id.
    """
    t = _cube_tan(ne)
    m = ne + 1
    i, j = np.meshgrid(np.arange(m, dtype=np.int64), np.arange(m, dtype=np.int64), indexing="ij")
    i, j = i.ravel(), j.ravel()
    ids = []
    for axis in range(3):
        for side in (0, ne):
            lat = [None, None, None]
            lat[axis] = np.full_like(i, side)
            o1, o2 = [c for c in range(3) if c != axis]
            lat[o1], lat[o2] = i, j
            lid = (lat[0] * m + lat[1]) * m + lat[2]
            grid = lid.reshape(m, m)
            # edges along both in-face directions
            ids.append(np.stack([grid[:-1, :].ravel(), grid[1:, :].ravel()]))
            ids.append(np.stack([grid[:, :-1].ravel(), grid[:, 1:].ravel()]))
    e = np.concatenate(ids, axis=1)
    lo, hi = np.minimum(e[0], e[1]), np.maximum(e[0], e[1])
    key = np.unique(lo * (m ** 3) + hi)
    lo, hi = key // (m ** 3), key % (m ** 3)

    def coords(lid):
        X, rem = np.divmod(lid, m * m)
        Y, Z = np.divmod(rem, m)
        v = np.stack([t[X], t[Y], t[Z]])
        r = np.sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2])
        return v / r

    return coords(lo), coords(hi)


def c4_pairs(ne: int = 1024, nlat: int = 1800):
    """C4 zonal-mean workload: each edge paired with the latitudes its z-range spans.

    The z-range is [min(za, zb), max(za, zb)], widened to the great circle's apex (antapex)
    height when that extremum lies strictly inside the edge.  This is workload construction
    in plain float64, not the method: a pair whose latitude grazes the range may come out
    with count 0, which the oracles decide.  Returns (a, b, z0, edge_index) SoA arrays.
    """
    va, vb = cubed_sphere_edges(ne)
    z0 = latitudes(nlat)
    za, zb = va[2], vb[2]
    zlo, zhi = np.minimum(za, zb), np.maximum(za, zb)
    nrm = np.cross(va.T, vb.T).T
    nxy = np.sqrt(nrm[0] ** 2 + nrm[1] ** 2)
    nn = np.sqrt(nxy ** 2 + nrm[2] ** 2)
    ok = nxy > 0
    h = np.where(ok, nxy / np.where(nn > 0, nn, 1.0), 0.0)      # apex height of the circle
    # apex direction (e_z - (e_z.n)n)/|..| lies inside the edge iff both endpoint cross tests agree
    apx = np.stack([-nrm[0] * nrm[2], -nrm[1] * nrm[2], nxy ** 2])
    g1 = np.einsum("ij,ij->j", np.cross(va.T, apx.T).T, nrm)
    g2 = np.einsum("ij,ij->j", np.cross(apx.T, vb.T).T, nrm)
    zhi = np.where(ok & (g1 > 0) & (g2 > 0), np.maximum(zhi, h), zhi)
    g1 = np.einsum("ij,ij->j", np.cross(va.T, -apx.T).T, nrm)
    g2 = np.einsum("ij,ij->j", np.cross(-apx.T, vb.T).T, nrm)
    zlo = np.where(ok & (g1 > 0) & (g2 > 0), np.minimum(zlo, -h), zlo)
    klo = np.searchsorted(z0, zlo, side="left")
    khi = np.searchsorted(z0, zhi, side="right")
    cnt = khi - klo
    edge = np.repeat(np.arange(va.shape[1], dtype=np.int64), cnt)
    start = np.repeat(klo - np.cumsum(cnt) + cnt, cnt)
    k = start + np.arange(edge.shape[0], dtype=np.int64)
    return (np.ascontiguousarray(va[:, edge]), np.ascontiguousarray(vb[:, edge]),
            np.ascontiguousarray(z0[k]), edge)
