"""Build and time launch-shape variants of the fused zonal pass (tools, not product).
    python tools/zonal_variants.py build      # here
    python tools/zonal_variants.py time       # on the GPU: C4 mesh x 1,800 latitudes
Knobs: SGI_ZONAL_THREADS (tile = 2x edges), SGI_ZONAL_FILTER_MINB, SGI_ZONAL_FILTER_PREFETCH (0/1/2),
SGI_ZONAL_WTHREADS (emit CTA size), SGI_ZONAL_EMIT_W2 (two queries per lane), SGI_ZONAL_FUSED (one
launch), SGI_ZONAL_FT (fused kernel's CTA size; tile = 4x edges), SGI_ZONAL_STATIC, SGI_ZONAL_PARK."""
import ctypes
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "zvariants")
VARIANTS = {
    "fused": {},
    "count_fallbacks": {"SGI_ZONAL_COUNT_FALLBACKS": 1},
    "count_reasons": {"SGI_ZONAL_COUNT_FALLBACKS": 1, "SGI_CERT_DEBUG_REASONS": 1},
    "zero_div_off": {"SGI_CERT_ZERO_DIV": 0},
    "two_barriers": {"SGI_ZONAL_ONE_BARRIER": 0},
    "no_l2_prefetch": {"SGI_ZONAL_L2_PREFETCH": 0},
    "consec_filter": {"SGI_ZONAL_CONSEC_FILTER": 1},
    "fallback_fast": {"SGI_ZONAL_FALLBACK_FAST": 1},
    "both_roots": {"SGI_CERT_ONE_ROOT": 0},
    "branch_two": {"SGI_ZONAL_DEFER_TWO": 0},
    "rsqrt_z": {"SGI_ZONAL_UNIT_Z": 0},
    "bracket_bkt": {"SGI_ZONAL_EXACT_BKT": 0},
    "late_tk": {"SGI_ZONAL_EARLY_TK": 0},
    "prev": None,                    # a library built by hand (e.g. the previous commit), not rebuilt
    "tk_before_queries": {"SGI_ZONAL_EARLY_TK": 2},
    "loop_top_tma": {"SGI_ZONAL_EARLY_TMA": 0},
    "no_lb_pref": {"SGI_ZONAL_LB_PREFETCH": 0},
    "late_tk_no_lb_pref": {"SGI_ZONAL_EARLY_TK": 0, "SGI_ZONAL_LB_PREFETCH": 0},
    "ft128": {"SGI_ZONAL_FT": 128},
    "ft128_minb5": {"SGI_ZONAL_FT": 128, "SGI_ZONAL_MINB": 5},
    "ft256_minb3": {"SGI_ZONAL_MINB": 3},
    "fused_park": {"SGI_ZONAL_PARK": 1},
    "fused_lb8": {"SGI_ZONAL_LB": 8},
    "fused_lb2": {"SGI_ZONAL_LB": 2},
    "b4096": {"SGI_ZONAL_BUCKETS": 4096},
    "b1024": {"SGI_ZONAL_BUCKETS": 1024},
    "fused_lb4": {"SGI_ZONAL_LB": 4},
    "fused_lb16": {"SGI_ZONAL_LB": 16},
    "ws7": {"SGI_ZONAL_WS": 1},
    "three_launch": {"SGI_ZONAL_FUSED": 0},
}
if os.environ.get("SGI_VARIANTS"):
    VARIANTS = {k: v for k, v in VARIANTS.items() if k in os.environ["SGI_VARIANTS"].split(",")}


def build():
    from paper_2510_09892_b200._build import NVCC_FLAGS
    os.makedirs(OUT, exist_ok=True)
    srcs = [os.path.join(ROOT, "paper_2510_09892_b200", "csrc", f) for f in ("sgi_capi.cu", "sgi_zonal.cu")]
    for name, defs in VARIANTS.items():
        if defs is None:
            continue
        d = [f"-D{k}={v}" for k, v in defs.items()]
        lib = os.path.join(OUT, f"libsgi_{name}.so")
        flags = [f for f in NVCC_FLAGS if f not in ("-Xptxas", "-v")]
        r = subprocess.run(["nvcc", *flags, *d, "-I", os.path.join(ROOT, "include"), "-o", lib,
                            *srcs], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        print(name, "ok")


def time_all(rounds=5, reps=10):
    import torch
    import sgi_inputs
    va, vb = sgi_inputs.cubed_sphere_edges(1024)
    lat = sgi_inputs.latitudes(1800)
    dva, dvb = torch.from_numpy(va).cuda(), torch.from_numpy(vb).cuda()
    dl = torch.from_numpy(lat).cuda()
    ne = va.shape[1]
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    libs = {}
    for name in VARIANTS:
        L = ctypes.CDLL(os.path.join(OUT, f"libsgi_{name}.so"))
        L.sgi_zonal_intersect.restype = ctypes.c_int
        L.sgi_zonal_intersect.argtypes = [vp, vp, i64, i64, vp, ctypes.c_int32, i64, vp, vp, vp,
                                          vp, vp, vp, ctypes.c_size_t, ctypes.c_int, vp]
        L.sgi_zonal_workspace_bytes.restype = ctypes.c_size_t
        L.sgi_zonal_workspace_bytes.argtypes = [i64]
        libs[name] = L
    cap = 6_100_000
    outs = {"edge": torch.empty(cap, dtype=torch.int64, device="cuda"),
            "lat": torch.empty(cap, dtype=torch.int32, device="cuda"),
            "count": torch.empty(cap, dtype=torch.uint8, device="cuda"),
            "xyz": torch.empty((2, 3, cap), dtype=torch.float64, device="cuda")}
    total = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    times = {n: [] for n in VARIANTS}
    ref = None
    same = {}
    for r in range(rounds):
        for name, L in libs.items():
            work = torch.empty(L.sgi_zonal_workspace_bytes(ne), dtype=torch.uint8, device="cuda")
            call = lambda: L.sgi_zonal_intersect(  # noqa: E731
                dva.data_ptr(), dvb.data_ptr(), ne, ne, dl.data_ptr(), len(lat), cap,
                outs["edge"].data_ptr(), outs["lat"].data_ptr(), outs["count"].data_ptr(),
                outs["xyz"].data_ptr(), total.data_ptr(), work.data_ptr(), work.numel(), 1,
                ctypes.c_void_p(st.cuda_stream))
            for _ in range(2):
                assert call() == 0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                call()
            e1.record()
            torch.cuda.synchronize()
            times[name].append(e0.elapsed_time(e1) / reps)
            if r == 0:
                m = int(total.item())
                cur = (outs["edge"][:m].clone(), outs["xyz"][..., :m].clone())
                if ref is None:
                    ref = cur
                same[name] = torch.equal(cur[0], ref[0]) and torch.equal(
                    cur[1].view(torch.int64), ref[1].view(torch.int64))
    for name in VARIANTS:
        print(json.dumps({"variant": name, "ms_median": round(statistics.median(times[name]), 4),
                          "ms_min": round(min(times[name]), 4), "same_as_first": same[name]}))


if __name__ == "__main__":
    build() if sys.argv[1] == "build" else time_all()
