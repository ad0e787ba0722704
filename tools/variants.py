"""Build and time launch-shape variants of libsgi.so (tools, not product).

    python tools/variants.py build            # here: nvcc each variant into build/variants/
    python tools/variants.py time [--n N]     # on the GPU: time every variant, check bitwise
                                              # equality with the default library's output
Variant knobs are the SGI_* macros of csrc/sgi_capi.cu.
"""
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "variants")

VARIANTS = {
    "base": {},
    "t128": {"SGI_THREADS": 128},
    "t160": {"SGI_THREADS": 160},
    "t192": {"SGI_THREADS": 192},
    "minb3": {"SGI_MINB": 3},
    "t128_minb6": {"SGI_THREADS": 128, "SGI_MINB": 6},
    "knuth": {"SGI_TS_KNUTH": 1},
    "knuth_minb3": {"SGI_TS_KNUTH": 1, "SGI_MINB": 3},
    "grid8": {"SGI_GRID_MULT": 8},
    "t128_grid8": {"SGI_THREADS": 128, "SGI_GRID_MULT": 8},
    "ilp2_minb1": {"SGI_ILP": 2, "SGI_MINB": 1},
}


def build():
    from paper_2510_09892_b200._build import NVCC_FLAGS
    os.makedirs(OUT, exist_ok=True)
    src = os.path.join(ROOT, "paper_2510_09892_b200", "csrc", "sgi_capi.cu")
    for name, defs in VARIANTS.items():
        d = [f"-D{k}={v}" for k, v in defs.items()]
        lib = os.path.join(OUT, f"libsgi_{name}.so")
        r = subprocess.run(["nvcc", *NVCC_FLAGS, *d, "-I", os.path.join(ROOT, "include"), "-o",
                            lib, src], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        regs = [l.strip() for l in r.stderr.splitlines() if "registers" in l or "spill" in l]
        print(name, regs[:6])


def time_all(n):
    import torch
    import sgi_inputs
    dev = torch.device("cuda", 0)
    a = torch.empty((3, n), dtype=torch.float64, device=dev)
    b = torch.empty_like(a)
    z0 = torch.empty(n, dtype=torch.float64, device=dev)
    sgi_inputs.generate_device(2, n, a, b, z0)
    ref = {}
    rows = []
    for name in VARIANTS:
        L = ctypes.CDLL(os.path.join(OUT, f"libsgi_{name}.so"))
        f = L.sgi_intersect_arc_lat
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] * 2 + [ctypes.c_void_p] * 2 + \
            [ctypes.c_int, ctypes.c_void_p]
        for mode in (1, 0, 2):
            out = torch.empty((2, 3, n), dtype=torch.float64, device=dev)
            cnt = torch.empty(n, dtype=torch.uint8, device=dev)
            st = torch.cuda.current_stream()
            call = lambda: f(a.data_ptr(), b.data_ptr(), z0.data_ptr(), n, n, out.data_ptr(),
                             cnt.data_ptr(), mode, ctypes.c_void_p(st.cuda_stream))
            for _ in range(5):
                assert call() == 0
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 50
            e0.record()
            for _ in range(reps):
                call()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            key = mode
            if key not in ref:
                ref[key] = (out.clone(), cnt.clone())
            same = torch.equal(cnt, ref[key][1]) and torch.equal(
                out.view(torch.int64), ref[key][0].view(torch.int64))
            rows.append({"variant": name, "mode": mode, "ms": round(ms, 4),
                         "Garcs_s": round(n / ms / 1e6, 2), "bitwise_same_as_base": same})
            print(json.dumps(rows[-1]), flush=True)
    return rows


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        n = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 24
        rows = time_all(n)
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", "variants.json"), "w") as fh:
            json.dump(rows, fh, indent=1)
