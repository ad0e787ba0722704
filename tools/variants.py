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
    "dbg_fallbacks": {"SGI_DBG_CLOCK": 1},
    "stages2": {"SGI_EFT_STAGES": 2},
    "ldg_only": {"SGI_USE_TMA": 0},
    "ts_knuth": {"SGI_TS_KNUTH": 1},
    "eft_t384": {"SGI_EFT_THREADS": 384},
    "eft_t640": {"SGI_EFT_THREADS": 640, "SGI_EFT_STAGES": 2},
    "one_query": {"SGI_EFT_PAIR": 0},
    "prev": None,                    # a library built by hand (e.g. the previous commit), not rebuilt
    "both_roots": {"SGI_CERT_ONE_ROOT": 0},
    "same_bits": {"SGI_CERT_SAME_BITS": 1},
    "zero_div_all": {"SGI_CERT_ZERO_DIV_ALL": 1},
    "small_s2_50": {"SGI_CERT_SMALL_S2": "0x1p50"},
    "small_s2_70": {"SGI_CERT_SMALL_S2": "0x1p70"},
    "small_s2_80": {"SGI_CERT_SMALL_S2": "0x1p80"},
    "count_reasons": {"SGI_CERT_DEBUG_REASONS": 1, "SGI_DBG_CLOCK": 1},
    "tiny_guard": {"SGI_CERT_TINY_GUARD": 1},
    "hiword_z0": {"SGI_EXACT_ZERO_TESTS": 0},
    "w2_second": {"SGI_CERT_SCALAR_SECOND": 0},
    "one_query_t768": {"SGI_EFT_PAIR": 0, "SGI_EFT_THREADS": 768, "SGI_EFT_STAGES": 2},
}
if os.environ.get("SGI_VARIANTS"):
    VARIANTS = {k: v for k, v in VARIANTS.items() if k in os.environ["SGI_VARIANTS"].split(",")}


def build():
    from paper_2510_09892_b200._build import NVCC_FLAGS
    os.makedirs(OUT, exist_ok=True)
    src = os.path.join(ROOT, "paper_2510_09892_b200", "csrc", "sgi_capi.cu")
    for name, defs in VARIANTS.items():
        if defs is None:
            continue
        flags = list(NVCC_FLAGS)
        if defs.get("FMAD"):                       # contraction allowed (the intrinsics must not care)
            flags = [f for f in flags if f != "-fmad=false"] + ["-fmad=true"]
        d = [f"-D{k}={v}" for k, v in defs.items() if k != "FMAD"]
        lib = os.path.join(OUT, f"libsgi_{name}.so")
        r = subprocess.run(["nvcc", *flags, *d, "-I", os.path.join(ROOT, "include"), "-o",
                            lib, src], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        regs = [l.strip() for l in r.stderr.splitlines() if "registers" in l or "spill" in l]
        print(name, regs[:6])


def time_all(n, rounds=7, reps=20, config=2):
    """Interleaved timing: every round times every (variant, mode) once, so clock drift hits
    all variants alike; reports the median over rounds and the SM clock seen (NVML)."""
    import statistics
    import torch
    import sgi_inputs
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        clock = lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)  # noqa: E731
    except Exception:
        clock = lambda: -1  # noqa: E731
    dev = torch.device("cuda", 0)
    a = torch.empty((3, n), dtype=torch.float64, device=dev)
    b = torch.empty_like(a)
    z0 = torch.empty(n, dtype=torch.float64, device=dev)
    sgi_inputs.generate_device(config, n, a, b, z0, seed=config)
    out = torch.empty((2, 3, n), dtype=torch.float64, device=dev)
    cnt = torch.empty(n, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    fns, libs = {}, {}
    for name in VARIANTS:
        L = ctypes.CDLL(os.path.join(OUT, f"libsgi_{name}.so"))
        libs[name] = L
        f = L.sgi_intersect_arc_lat
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] * 2 + [ctypes.c_void_p] * 2 + \
            [ctypes.c_int, ctypes.c_void_p]
        fns[name] = f
    modes = tuple(int(m) for m in os.environ.get("SGI_VARIANT_MODES", "1").split(","))
    times = {(v, m): [] for v in VARIANTS for m in modes}
    eff = {(v, m): [] for v in VARIANTS for m in modes}
    clocks = []
    ref = {}
    same = {}
    for r in range(rounds):
        for name, f in fns.items():
            for mode in modes:
                call = lambda: f(a.data_ptr(), b.data_ptr(), z0.data_ptr(), n, n, out.data_ptr(),  # noqa: E731
                                 cnt.data_ptr(), mode, ctypes.c_void_p(st.cuda_stream))
                for _ in range(3):
                    assert call() == 0
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    call()
                e1.record()
                torch.cuda.synchronize()
                clocks.append(clock())
                times[(name, mode)].append(e0.elapsed_time(e1) / reps)
                if hasattr(libs[name], "sgi_dbg_fallbacks") and r == 0:
                    libs[name].sgi_dbg_fallbacks.restype = ctypes.c_ulonglong
                    fb = libs[name].sgi_dbg_fallbacks()
                    print(json.dumps({"variant": name, "config": config,
                                      "exact_recomputations_per_launch": fb / (reps + 3)}))
                if hasattr(libs[name], "sgi_dbg_clock"):
                    buf = (ctypes.c_longlong * 2)()
                    libs[name].sgi_dbg_clock(buf)
                    if buf[1] > 0:
                        eff[(name, mode)].append(buf[0] / buf[1] * 1e3)
                if r == 0:
                    if mode not in ref:
                        ref[mode] = (out.clone(), cnt.clone())
                    same[(name, mode)] = torch.equal(cnt, ref[mode][1]) and torch.equal(
                        out.view(torch.int64), ref[mode][0].view(torch.int64))
    rows = []
    for (name, mode), ts in times.items():
        med = statistics.median(ts)
        rows.append({"variant": name, "mode": mode, "ms_median": round(med, 4),
                     "ms_min": round(min(ts), 4), "Garcs_s": round(n / med / 1e6, 2),
                     "bitwise_same_as_base": same[(name, mode)],
                     "cta0_clock_mhz": round(statistics.median(eff[(name, mode)]), 1)
                     if eff[(name, mode)] else None})
        print(json.dumps(rows[-1]), flush=True)
    print(json.dumps({"sm_clock_mhz_min": min(clocks), "sm_clock_mhz_median":
                      statistics.median(clocks), "sm_clock_mhz_max": max(clocks)}))
    return rows


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[2] == "--n" else 1 << 24
        cfg = int(sys.argv[sys.argv.index("--config") + 1]) if "--config" in sys.argv else 2
        rows = time_all(n, config=cfg)
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", "variants.json"), "w") as fh:
            json.dump(rows, fh, indent=1)
