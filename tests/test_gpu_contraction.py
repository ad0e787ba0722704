"""Contraction-proof arithmetic (P:1095-1099 compile with -ffp-contract=off): every
operation of the path is an explicit round-to-nearest intrinsic, so building libsgi.so with
-fmad=true (nvcc free to fuse a*b+c) must give bit-identical outputs in every mode."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import sgi_inputs

torch = pytest.importorskip("torch")
import paper_2510_09892_b200 as sgi  # noqa: E402
from paper_2510_09892_b200._build import NVCC_FLAGS, PKG, ROOT  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fmad_lib(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("fmad") / "libsgi_fmad.so")
    flags = [f for f in NVCC_FLAGS if f not in ("-fmad=false", "-Xptxas", "-v")] + ["-fmad=true"]
    src = [os.path.join(PKG, "csrc", f) for f in ("sgi_capi.cu", "sgi_zonal.cu")]
    r = subprocess.run(["nvcc", *flags, "-I", os.path.join(ROOT, "include"), "-o", out, *src],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    L = ctypes.CDLL(out)
    L.sgi_intersect_arc_lat.restype = ctypes.c_int
    L.sgi_intersect_arc_lat.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] * 2 + \
        [ctypes.c_void_p] * 2 + [ctypes.c_int, ctypes.c_void_p]
    return L


@pytest.mark.parametrize("config", [2, 3, 5])
def test_fmad_true_build_is_bit_identical(fmad_lib, config):
    n = 1 << 20
    a = torch.empty((3, n), dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    z0 = torch.empty(n, dtype=torch.float64, device="cuda")
    sgi_inputs.generate_device(config, n, a, b, z0)
    for mode in sgi.MODES:
        ref, rcnt = sgi.intersect_arc_lat(a, b, z0, mode=mode)
        out = torch.empty_like(ref)
        cnt = torch.empty_like(rcnt)
        rc = fmad_lib.sgi_intersect_arc_lat(a.data_ptr(), b.data_ptr(), z0.data_ptr(), n, n,
                                            out.data_ptr(), cnt.data_ptr(), sgi.MODES[mode], None)
        assert rc == 0
        torch.cuda.synchronize()
        assert torch.equal(cnt, rcnt), mode
        assert np.array_equal(out.cpu().numpy().view(np.int64), ref.cpu().numpy().view(np.int64)), mode
