#!/usr/bin/env python3
"""bench.py — throughput of the B200 arc/latitude intersection path (arXiv 2510.09892).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--mode eft|eft_literal|naive]
                    [--config 2|3|5] [--impl ours|reference]

One step = one launch of the whole hot path (load, accurate normal, s^2, s,
numerators, division, containment/count, store) over one batch of synthetic arcs resident in
HBM.  Default workload: BASELINE.json configs[1] (C2: 2^24 short arcs) per GPU; with N GPUs
each rank owns its own 2^24-arc slice of the global index space (weak scaling, no data-path
collective; NCCL only reduces the counts and the timing afterwards).

Prints ONE JSON line on rank 0 (driver contract): metric/value/unit, roofline of the dominant
kernel, cpu_baseline (oracle (a) on the host cores), e2e through the host-buffer C-ABI call,
SM clocks sampled (NVML) during the timed region, and the number of our kernel launches.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "EFT arc-latitude intersections/s (FP64) at 1/2/4/8 B200; % roofline; max ulp err"
UNIT = "intersections/s"
BYTES_PER_ARC = 56 + 48 + 1          # a, b, z0 in; two xyz slots + uint8 count out (§8(b))
# Algorithmic FP64 operations per query (add/sub/mul/fma/div/sqrt/compare = 1 each) of the
# paper's listing: AccuX both roots 334 + renormalisation 18 + containment 14 = 366
# (DESIGN.md §5 reading of the count); literal 351, naive 46.  The plain-binary64 variants count
# their own listings.
FP64_OPS = {"eft": 366, "eft_literal": 351, "naive": 46, "yac": 52, "base": 51, "naive_kahan": 49}
SEEDS = {2: 2, 3: 3, 4: None, 5: 5, 6: 6, 7: 7}
C4_PAIRS = 6_000_016   # C4: cubed sphere ne=1024 edges x 1,800 latitudes, materialised
CONFIG_DESC = {
    4: "C4 zonal-mean pairs (cubed sphere ne=1024 x 1,800 latitudes, materialised as arcs)",
    2: "C2 short arcs (midpoint uniform, length log-uniform [1e-4,1e-2] rad, z0 between endpoint z)",
    3: "C3 ill-conditioned arcs (near-tangent / near-polar / near-coincident thirds)",
    5: "C5 mixed arcs (50% C1, 25% C2, 25% uniform endpoints with z0 uniform in [-1,1])",
    6: "paper primary accuracy dataset (P:949): 17 latitude bands, z0 between endpoint z",
    7: "paper secondary dataset (P:951-953): shallow near-equator arcs, z0 = circle top - r",
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--mode", default="eft",
                   choices=["eft", "eft_literal", "naive", "yac", "base", "naive_kahan"])
    p.add_argument("--config", type=int, default=None, choices=[2, 3, 4, 5, 6, 7],
                   help="default 5 (the metric's workload); 2 for --workload dw|trace")
    p.add_argument("--n", type=int, default=None,
                   help="arcs in total (--scaling strong) or per rank (--scaling weak); default "
                        "2^30 for config 5 (the metric's 1/2/4/8-GPU batch), 2^24 otherwise")
    p.add_argument("--scaling", default=None, choices=["weak", "strong"],
                   help="strong (default for config 5): the n arcs are split across the ranks "
                        "(C5's 2^30 arcs over 1/2/4/8 GPUs); weak (default otherwise): every "
                        "rank owns n arcs")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-accuracy", action="store_true",
                   help="skip the max_ulp_err sample against oracle (b)")
    p.add_argument("--workload", default="arcs", choices=["arcs", "zonal", "dw", "trace"],
                   help="arcs: the C2/C3/C5 batch (default line); zonal: the fused zonal-mean "
                        "pass over the C4 cubed sphere (ne=1024) x 1,800 latitudes")
    args = p.parse_args()
    if args.config is None:
        args.config = 2 if args.workload in ("dw", "trace") else 5
    if args.n is None:
        args.n = (1 << 30) if args.config == 5 else (1 << 24)
    if args.scaling is None:
        args.scaling = "strong" if args.config == 5 else "weak"
    return args


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        peaks.update({k: d[k] for k in ("hbm_gbs", "sm_max_mhz") if k in d})
        peaks["source"] = "measured (MEASURED_PEAKS.json)"
    return peaks


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the timed region runs."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, index: int, period: float = 0.002):
        self.samples, self.reasons, self.period = [], 0, period
        self.power = []
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            try:
                self.limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1e3
            except Exception:
                self.limit_w = None
        except Exception as e:  # pragma: no cover - reported, not fatal
            self.nvml, self.err = None, str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                self.reasons |= self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.power.append(self.nvml.nvmlDeviceGetPowerUsage(self.h) / 1e3)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nvml:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nvml:
            self.t.join()

    def summary(self):
        if not self.nvml:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        pw = sorted(self.power)
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(s),
                "power_w": pw[len(pw) // 2] if pw else None,
                "power_limit_w": getattr(self, "limit_w", None)}

    BAD = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")

    def throttled(self):
        return any(r in self.BAD for r in self.summary().get("reasons", []))


def pcie_concurrent_gbs(dev, nbytes=1 << 29):
    """Measured host<->device bandwidth with H2D and D2H running at once (pinned, CUDA events):
    the ceiling of the e2e path, which moves 56 B in and 49 B out per query."""
    import torch
    n = nbytes // 8
    hi = torch.empty(n, dtype=torch.float64).pin_memory()
    ho = torch.empty(n, dtype=torch.float64).pin_memory()
    di = torch.empty(n, dtype=torch.float64, device=dev)
    do = torch.empty(n, dtype=torch.float64, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    cur = torch.cuda.current_stream(dev)
    best = 0.0
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            di.copy_(hi, non_blocking=True)
        with torch.cuda.stream(s2):
            ho.copy_(do, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
        e1.record(cur)
        torch.cuda.synchronize()
        best = max(best, 2 * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


_C4 = {}


def host_arcs(config: int, n: int, offset: int = 0):
    """Arcs [offset, offset + n) of `config` on the host (C4: the materialised pair list)."""
    import numpy as np
    import sgi_inputs
    if config == 4:
        if not _C4:
            a, b, z0, _ = sgi_inputs.c4_pairs(1024, 1800)
            _C4.update(a=a, b=b, z0=z0)
        sl = slice(offset, offset + n)
        return (np.ascontiguousarray(_C4["a"][:, sl]), np.ascontiguousarray(_C4["b"][:, sl]),
                np.ascontiguousarray(_C4["z0"][sl]))
    return sgi_inputs.generate_host(config, n, offset=offset, seed=SEEDS[config])


def device_arcs(config: int, n: int, a, b, z0, offset: int = 0):
    """Fill device tensors with arcs [offset, offset + n) (C4 is built on the host and copied)."""
    import torch
    import sgi_inputs
    if config == 4:
        ha, hb, hz = host_arcs(4, n, offset)
        a.copy_(torch.from_numpy(ha))
        b.copy_(torch.from_numpy(hb))
        z0.copy_(torch.from_numpy(hz))
        return
    sgi_inputs.generate_device(config, n, a, b, z0, offset=offset, seed=SEEDS[config])


CPU_SAMPLE = 1 << 22   # arcs of the workload's prefix the CPU legs time (bounded CPU work)


def cpu_baseline_run(config: int, n: int, mode: str, offset: int = 0):
    """Oracle (a) as it stands (oracle/eft_oracle.c, OpenMP over all host cores) on a BOUNDED
    sample of the same workload: the first min(n, 2^22) arcs of this rank's slice (the host
    generator makes the same bits as the device one), whole passes until ~1 s of wall time
    (~cores CPU-seconds); returns (arcs/s, cores, seconds, single-thread arcs/s, passes, m)."""
    import oracle
    cores = os.cpu_count() or 1
    m = min(n, CPU_SAMPLE)
    a, b, z0 = host_arcs(config, m, offset)
    om = {"eft": oracle.MODE_EFT, "eft_literal": oracle.MODE_EFT_LITERAL, "naive": oracle.MODE_NAIVE,
          "yac": oracle.MODE_YAC, "base": oracle.MODE_BASE, "naive_kahan": oracle.MODE_NAIVE_KAHAN}[mode]
    oracle.intersect(om, a[:, :4096], b[:, :4096], z0[:4096], nthreads=cores)   # warm
    passes, t0 = 0, time.perf_counter()
    while True:
        oracle.intersect(om, a, b, z0, nthreads=cores)
        passes += 1
        dt = time.perf_counter() - t0
        if dt >= 1.0 or passes >= 8:
            break
    # one core on a smaller prefix (1 thread, then all host cores)
    n1 = min(m, 1 << 20)
    t1 = time.perf_counter()
    oracle.intersect(om, a[:, :n1], b[:, :n1], z0[:n1], nthreads=1)
    single = n1 / (time.perf_counter() - t1)
    return m * passes / dt, cores, dt, single, passes, m


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


ACC_SAMPLE = 20_000      # queries of the max_ulp_err sample (over all ranks)


def accuracy_sample(a, b, z0, out, cnt, ref_out, ref_cnt, mode, ref_mode, idx):
    """The metric's "max ulp err": this run's own GPU outputs at the local indices `idx` (this
    rank's share of ACC_SAMPLE evenly spaced global indices, dist.sample_indices) against
    oracle (b) (exact rationals, Eq.FINAL); err_u = |P~ - P| / (u sqrt(1 - z0^2)),
    the paper's bound is 3 (Eq.BOUND).  Both modes of the run are scored.  Returns
    per mode (max err_u, #points over the bound, #count mismatches vs exact, #queries) for the
    cross-rank MAX/SUM."""
    import numpy as np
    import torch
    from oracle import exact
    ti = torch.from_numpy(np.asarray(idx, np.int64)).to(z0.device)
    A, B, Z = (x.index_select(-1, ti).cpu().numpy() for x in (a, b, z0))
    res = {}
    for name, o, c in ((mode, out, cnt), (ref_mode, ref_out, ref_cnt)):
        O, C = o.index_select(-1, ti).cpu().numpy(), c.index_select(0, ti).cpu().numpy()
        worst, viol, mism = 0.0, 0, 0
        for j in range(len(idx)):
            used = int(C[j]) if C[j] in (1, 2) else 0
            if np.isnan(O[:used, :2, j]).any():      # a stored point that is not a number
                worst, viol = float("inf"), viol + 1
                continue
            r = exact.check_query(A[:, j], B[:, j], Z[j], int(C[j]),
                                  [(O[0, 0, j], O[0, 1, j]), (O[1, 0, j], O[1, 1, j])])
            mism += not r["count_match"]
            for e in r["err_u"]:
                worst = max(worst, e)
                viol += e > 3.0
        res[name] = (worst, viol, mism, len(idx))
    return res


def ref_mode_chunks(a, b, z0, n, out, cnt, ref_mode, stream, sgi, chunk=1 << 25):
    """K5 statistics of the run's outputs against the other mode on the same arcs, in chunks
    (the other mode's 2^30-arc outputs would not fit beside ours): per chunk the inputs and our
    outputs copied to chunk-sized planes, the other mode into a chunk buffer, sgi_output_stats
    accumulating.  Returns (stats float64[2], counts int64[2]) on the device."""
    import torch
    dev = z0.device
    stats = torch.zeros(2, dtype=torch.float64, device=dev)
    counts = torch.zeros(2, dtype=torch.int64, device=dev)
    for off in range(0, n, chunk):
        m = min(chunk, n - off)
        ca, cb = a[:, off:off + m].contiguous(), b[:, off:off + m].contiguous()
        cz = z0[off:off + m].contiguous()
        ro, rc = sgi.intersect_arc_lat(ca, cb, cz, mode=ref_mode, stream=stream)
        sgi.output_stats(out[:, :, off:off + m].contiguous(), cnt[off:off + m].contiguous(), cz,
                         ref_xyz=ro, ref_count=rc, stats=stats, counts=counts, stream=stream)
        del ca, cb, cz, ro, rc
    return stats, counts


def run_reference(args):
    """--impl reference: the oracle on the host cores, each step a bounded sample (2^22 arcs)
    of the same workload; rank 0 only."""
    from paper_2510_09892_b200 import dist as sdist
    ws, rank, _ = sdist.env()
    if rank != 0:
        return
    import oracle
    import sgi_inputs
    cores = os.cpu_count() or 1
    n = min(args.n, 1 << 22)
    a, b, z0 = host_arcs(args.config, n)
    m = {"eft": oracle.MODE_EFT, "eft_literal": oracle.MODE_EFT_LITERAL, "naive": oracle.MODE_NAIVE,
         "yac": oracle.MODE_YAC, "base": oracle.MODE_BASE,
         "naive_kahan": oracle.MODE_NAIVE_KAHAN}[args.mode]
    for _ in range(max(args.warmup, 0)):
        oracle.intersect(m, a, b, z0, nthreads=cores)
    steps = max(1, min(args.steps, 20))
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle.intersect(m, a, b, z0, nthreads=cores)
    dt = time.perf_counter() - t0
    value = n * steps / dt
    sample = f"{n} arcs of config {args.config} per step (first {n} global indices), {steps} steps"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": dt / steps * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": CONFIG_DESC[args.config], "mode": args.mode,
                                        "arcs_per_step": n, "workload_arcs": args.n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


ZONAL_HEAD_OPS = 134    # per edge: AccuX lines 2-6 (114) + z-range filter (20), DESIGN.md §5
ZONAL_TAIL_OPS = 248    # per candidate pair: AccuX lines 7-25 + containment


def run_zonal(args):
    """Fused zonal-mean pass (sgi_zonal_intersect) over the C4 mesh; one step = one launch over
    all 12.6 M edges; value = candidate (edge, latitude) pairs per second (single GPU)."""
    import torch
    import paper_2510_09892_b200 as sgi
    import sgi_inputs
    dev = torch.device("cuda", 0)
    va, vb = sgi_inputs.cubed_sphere_edges(1024)
    lat = sgi_inputs.latitudes(1800)
    dva, dvb = torch.from_numpy(va).to(dev), torch.from_numpy(vb).to(dev)
    dl = torch.from_numpy(lat).to(dev)
    ne = va.shape[1]
    first = sgi.zonal_intersect(dva, dvb, dl, mode=args.mode)
    torch.cuda.synchronize()
    cap = first["cap"]
    work = torch.empty(sgi.zonal_workspace_bytes(ne), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        sgi.zonal_intersect(dva, dvb, dl, mode=args.mode, cap=cap, stream=stream, work=work)
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    s = e0.elapsed_time(e1) * 1e-3 / args.steps
    cnt = first["count"][:cap].cpu()
    nz = int((cnt != 0).sum())
    peaks = load_peaks()
    alu_peak = 148 * 64 * peaks["sm_max_mhz"] * 1e6 / 1e12
    ops = ne * ZONAL_HEAD_OPS + cap * ZONAL_TAIL_OPS          # the listing's algorithmic count
    byts = ne * 48 + cap * (8 + 4 + 1 + 48)                  # edges once, each pair's record once
    sass = {}
    spath = os.path.join(ROOT, "profiles", "fp64_sass.json")
    if os.path.exists(spath):
        with open(spath) as f:
            sass = json.load(f)
    ex_ops = cap * sass.get(f"zonal_{args.mode}_per_pair", 0) or ops
    t_alu, t_hbm = ex_ops / (alu_peak * 1e12), byts / (peaks["hbm_gbs"] * 1e9)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(f"zonal_{args.mode}:4:{ne}")
    if t_alu >= t_hbm:
        roof = {"bound": "alu", "achieved": ex_ops / s / 1e12, "peak": alu_peak,
                "unit": "T FP64 instr/s", "frac": ex_ops / s / 1e12 / alu_peak}
    else:
        roof = {"bound": "hbm", "achieved": byts / s / 1e9, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": byts / s / 1e9 / peaks["hbm_gbs"]}
    roof.update({"traffic": traffic, "alu_frac": ex_ops / s / 1e12 / alu_peak,
                 "hbm_frac": byts / s / 1e9 / peaks["hbm_gbs"],
                 "algorithmic_alu_frac": ops / s / 1e12 / alu_peak,
                 "fp64_instr_source": "ncu (profiles/fp64_sass.json)" if ex_ops != ops else "listing",
                 "peak_alu": alu_peak, "peak_hbm": peaks["hbm_gbs"]})
    line = {"metric": "zonal (edge, latitude) candidate pairs/s", "value": cap / s,
            "unit": "pairs/s", "n_gpus": 1, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": s * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C4 cubed sphere ne=1024 (12,582,912 edges) x 1,800 latitudes, "
                                   "fused sgi_zonal_intersect", "mode": args.mode,
                       "pairs": cap, "nonzero_pairs": nz, "edges_per_s": ne / s},
            "roofline": roof,
            "clocks": clocks.summary(), "gpu_launches": args.steps}
    print(json.dumps(line), flush=True)


EFT_OPS = 362          # algorithmic FP64 ops per query of SGI_MODE_EFT
DW_EXTRA_OPS = 28      # per query: 4 low parts x (fma, 4 add/sub, 1 mul, 1 division), include/sgi.h
TRACE_FIELDS = 38


def run_extra(args):
    """SURVEY §8(f4) paths on the default workload (C2, 2^24 arcs, one GPU): `dw` =
    sgi_intersect_arc_lat_dw (double-word points), `trace` = sgi_intersect_trace (the 38
    Appendix-A intermediates per query).  Device-resident inputs and outputs, one launch per
    step, CUDA events on the launching stream."""
    import ctypes
    import torch
    import paper_2510_09892_b200 as sgi
    import sgi_inputs
    dev = torch.device("cuda", 0)
    n, cfg, mode = args.n, args.config, args.mode
    a = torch.empty((3, n), dtype=torch.float64, device=dev)
    b = torch.empty_like(a)
    z0 = torch.empty(n, dtype=torch.float64, device=dev)
    device_arcs(cfg, n, a, b, z0)
    cnt = torch.empty(n, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    L = sgi._load()
    sp = ctypes.c_void_p(stream.cuda_stream)
    mcode = sgi._mode(mode)
    if args.workload == "dw":
        out = torch.empty((2, 3, n), dtype=torch.float64, device=dev)
        lo = torch.empty((2, 2, n), dtype=torch.float64, device=dev)

        def step():
            rc = L.sgi_intersect_arc_lat_dw(a.data_ptr(), b.data_ptr(), z0.data_ptr(), n, n,
                                            out.data_ptr(), lo.data_ptr(), cnt.data_ptr(), mcode, sp)
            assert rc == 0, rc
        byts, ops = 56 + 48 + 32 + 1, EFT_OPS + DW_EXTRA_OPS
        what = "sgi_intersect_arc_lat_dw (double-word points, reading R11)"
    else:
        trace = torch.empty((TRACE_FIELDS, n), dtype=torch.float64, device=dev)

        def step():
            rc = L.sgi_intersect_trace(a.data_ptr(), b.data_ptr(), z0.data_ptr(), n, n,
                                       trace.data_ptr(), cnt.data_ptr(), mcode, sp)
            assert rc == 0, rc
        byts, ops = 56 + 8 * TRACE_FIELDS + 1, EFT_OPS
        what = "sgi_intersect_trace (38 Appendix-A intermediates per query)"
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    s = e0.elapsed_time(e1) * 1e-3 / args.steps
    peaks = load_peaks()
    alu_peak = 148 * 64 * peaks["sm_max_mhz"] * 1e6 / 1e12
    alu_frac = n * ops / s / 1e12 / alu_peak
    hbm_frac = n * byts / s / 1e9 / peaks["hbm_gbs"]
    line = {"metric": f"{args.workload} queries/s", "value": n / s, "unit": "queries/s",
            "n_gpus": 1, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": s * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_DESC[cfg], "mode": mode, "queries": n, "path": what,
                       "bytes_per_query": byts, "fp64_ops_per_query": ops},
            "roofline": {"bound": "alu" if alu_frac > hbm_frac else "hbm",
                         "alu_frac": alu_frac, "hbm_frac": hbm_frac,
                         "peak_alu": alu_peak, "peak_hbm": peaks["hbm_gbs"]},
            "clocks": clocks.summary(), "gpu_launches": args.steps}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    from paper_2510_09892_b200 import dist as sdist
    if args.impl == "reference":
        return run_reference(args)
    if args.workload != "arcs":
        if args.gpus != 1 or "WORLD_SIZE" in os.environ and os.environ["WORLD_SIZE"] != "1":
            raise SystemExit(f"--workload {args.workload} is a single-GPU measurement")
        return {"zonal": run_zonal, "dw": run_extra, "trace": run_extra}[args.workload](args)
    how, _ = sdist.launch_plan(args.gpus)
    if how == "exec":                     # --gpus N > 1 without torchrun: one rank per GPU
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        argv = sdist.torchrun_argv(sys.executable, os.path.abspath(__file__), args.gpus, port,
                                   sys.argv[1:])
        print(f"bench.py: re-executing under torchrun: {' '.join(argv)}", file=sys.stderr,
              flush=True)
        os.execv(sys.executable, argv)

    import torch
    import torch.distributed as dist
    import paper_2510_09892_b200 as sgi

    ws, rank, local = sdist.env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} has LOCAL_RANK {local} but only "
                         f"{torch.cuda.device_count()} GPU(s) are visible (one rank per GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distributed = "RANK" in os.environ                  # launched by torchrun (any world size)
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
        probe = torch.ones(1, device=dev)
        dist.all_reduce(probe)                          # NCCL communicator up (visible in logs)
        if rank == 0:
            print(f"bench.py: NCCL process group of {ws} ranks, all_reduce probe "
                  f"{probe.item():.0f}", file=sys.stderr, flush=True)
    n, cfg, mode = args.n, args.config, args.mode
    if cfg == 4:                                        # C4 is a fixed set: ranks split it
        args.scaling, args.n = "strong", C4_PAIRS
        n = C4_PAIRS
    if args.scaling == "weak":                          # this rank's slice of the index space
        offset, n = sdist.shard_weak(rank, ws, n)
    else:
        offset, n = sdist.shard_strong(rank, ws, n)
    n_total = n * ws if args.scaling == "weak" else args.n

    # inputs generated on this rank's device from the seed (HBM resident before timing)
    a = torch.empty((3, n), dtype=torch.float64, device=dev)
    b = torch.empty_like(a)
    z0 = torch.empty(n, dtype=torch.float64, device=dev)
    device_arcs(cfg, n, a, b, z0, offset=offset)
    out = torch.empty((2, 3, n), dtype=torch.float64, device=dev)
    cnt = torch.empty(n, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    path = sgi.dispatch_path(a, b, z0, out, cnt, mode=mode)

    def step():
        sgi.intersect_arc_lat(a, b, z0, mode=mode, out_xyz=out, out_count=cnt, stream=stream)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed():
        with ClockSampler(local) as clocks:
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        return clocks

    clocks = timed()
    # a run that saw thermal or hardware slowdown on any rank is measured once more
    bad = torch.tensor([float(clocks.throttled())], device=dev)
    if distributed:
        dist.all_reduce(bad, op=dist.ReduceOp.MAX)
    remeasured = bool(bad.item())
    if remeasured:
        clocks = timed()
    ms_local = e0.elapsed_time(e1)
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    hist = sgi.count_histogram(cnt)                    # outside the timed region
    # K5 output statistics (outside the timed region): |P| - 1 and Pz == z0 on every stored point,
    # and the deviation from the other mode (naive-FP64 for the EFT modes) on the same arcs
    ref_mode = "naive" if mode != "naive" else "eft"
    stats, counts = ref_mode_chunks(a, b, z0, n, out, cnt, ref_mode, stream, sgi)
    if distributed:                                    # MAX of time and stats, SUM of counts (NCCL)
        sdist.reduce_after_step(t, hist, stats, counts)
    ms = float(t.item())
    total_arcs = n_total * args.steps
    value = total_arcs / (ms * 1e-3)
    ms_per_step = ms / args.steps
    launch_s = ms_local * 1e-3 / args.steps             # one kernel launch per step

    # max ulp err: every rank scores its share of one global sample, reduced MAX / SUM
    accuracy = None
    if not args.no_accuracy:
        idx = sdist.sample_indices(n_total, ACC_SAMPLE, offset, n)
        ref_o = torch.empty((2, 3, len(idx)), dtype=torch.float64, device=dev)
        ref_c = torch.empty(len(idx), dtype=torch.uint8, device=dev)
        if len(idx):
            ti = torch.from_numpy(idx).to(dev)
            sa, sb, sz = (x.index_select(-1, ti).contiguous() for x in (a, b, z0))
            sgi.intersect_arc_lat(sa, sb, sz, mode=ref_mode, out_xyz=ref_o, out_count=ref_c,
                                  stream=stream)
            so, sc = out.index_select(-1, ti), cnt.index_select(0, ti)
            res = accuracy_sample(sa, sb, sz, so, sc, ref_o, ref_c, mode, ref_mode,
                                  list(range(len(idx))))
        else:
            res = {mode: (0.0, 0, 0, 0), ref_mode: (0.0, 0, 0, 0)}
        worst = torch.tensor([res[mode][0], res[ref_mode][0]], dtype=torch.float64, device=dev)
        sums = torch.tensor([*res[mode][1:], *res[ref_mode][1:]], dtype=torch.float64, device=dev)
        sdist.reduce_accuracy(worst, sums)
        w, sm = worst.tolist(), [int(x) for x in sums.tolist()]
        accuracy = {"bound_u": 3.0, "reference": "oracle (b): exact rationals + 420-bit sqrt",
                    "sample": f"{sm[2]} evenly spaced global queries of this run's batch, "
                              f"scored on the rank that computed them ({ws} rank(s))",
                    mode: {"max_err_u": w[0], "over_bound": sm[0],
                           "count_mismatch_vs_exact": sm[1]},
                    ref_mode: {"max_err_u": w[1], "over_bound": sm[3],
                               "count_mismatch_vs_exact": sm[4]}}

    # roofline of the dominant (only) kernel: bound = the slower of the HBM roof (105 B/query)
    # and the FP64 roof at the FP64-pipe instructions the shipped kernel executes per query
    # (ncu, profiles/fp64_sass.json; the listing's algorithmic count where none is measured)
    peaks = load_peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    alu_peak = sms * 64 * peaks["sm_max_mhz"] * 1e6 / 1e12     # T FP64 instr/s (64 lanes/SM)
    sass = {}
    spath = os.path.join(ROOT, "profiles", "fp64_sass.json")
    if os.path.exists(spath):
        with open(spath) as f:
            sass = json.load(f)
    per_q = sass.get(f"{mode}:{cfg}", sass.get(mode, FP64_OPS[mode]))
    hbm_bytes, ops = n * BYTES_PER_ARC, n * per_q
    t_hbm, t_alu = hbm_bytes / (peaks["hbm_gbs"] * 1e9), ops / (alu_peak * 1e12)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(f"{mode}:{cfg}:{n}")
    alu = {"fp64_instr_per_query": per_q,
           "fp64_instr_source": ("ncu (profiles/fp64_sass.json)"
                                 if mode in sass or f"{mode}:{cfg}" in sass else "listing"),
           "algorithmic_ops_per_query": FP64_OPS[mode],
           "executed_frac": ops / launch_s / 1e12 / alu_peak,
           "algorithmic_rate_tops": n * FP64_OPS[mode] / launch_s / 1e12,
           "algorithmic_note": ("the listing's operations per second; it can exceed the "
                                "instruction peak because the shipped kernel executes fewer "
                                "FP64 instructions than the listing has operations (policy "
                                "Cert, DESIGN.md §5) — executed_frac is the pipe's share"),
           "peak": alu_peak, "unit": "T FP64 instr/s",
           "peak_source": f"{sms} SM x 64 FP64 lanes x {peaks['sm_max_mhz']:.0f} MHz "
                          "(tools/fp64_peak.cu measures 18.56 T DADD/s: profiles/r02/)"}
    if t_alu >= t_hbm:
        achieved = ops / launch_s / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": alu_peak,
                "unit": "T FP64 instr/s", "frac": achieved / alu_peak, "traffic": traffic,
                "peak_source": alu["peak_source"],
                "hbm_frac": hbm_bytes / launch_s / 1e9 / peaks["hbm_gbs"], "alu": alu}
    else:
        achieved = hbm_bytes / launch_s / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "traffic_per_query": None if traffic is None else traffic / n,
                "peak_source": peaks["source"] + " (copy bandwidth)", "alu": alu}

    # e2e: the host-buffer C-ABI call, pinned host inputs in, results back to the host
    e2e = None
    if args.e2e_steps > 0:
        ha, hb, hz = (torch.empty(x.shape, dtype=x.dtype, pin_memory=True).copy_(x)
                      for x in (a, b, z0))
        hout = torch.empty((2, 3, n), dtype=torch.float64, pin_memory=True)
        hcnt = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        work = torch.empty(sgi.host_workspace_bytes(1 << 22), dtype=torch.uint8, device=dev)

        def e2e_step():
            sgi.intersect_arc_lat_host(ha, hb, hz, mode=mode, out_xyz=hout, out_count=hcnt,
                                       work=work, stream=stream)
        e2e_step()
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        f1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        if distributed:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item()) * 1e-3 / args.e2e_steps
        link = pcie_concurrent_gbs(dev)
        e2e = {"value": n_total / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": n_total * 56, "d2h_bytes_per_step": n_total * 49,
               "steps": args.e2e_steps, "path": "sgi_intersect_arc_lat_host (pinned host buffers)",
               "link_gbs_measured": link, "link_frac": (n * 105 / e2e_s / 1e9) / link,
               # each direction gets ~link/2 when both run; the 56-B H2D side binds
               "link_bound_queries_per_s": link / 2 * 1e9 / 56,
               "link_bound_frac": (n / e2e_s) / (link / 2 * 1e9 / 56)}
        del ha, hb, hz, hout, hcnt, work

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        v, cores, dt, single, passes, m = cpu_baseline_run(cfg, n, mode, offset)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"the first {m} arcs of rank 0's slice of config {cfg} (bounded "
                         f"sample), {passes}x through oracle (a) with OpenMP over {cores} "
                         f"threads ({dt:.2f} s wall, ~{dt * cores:.0f} CPU-s)",
               "single_thread_value": single, "cpu_model": cpu_model()}

    if rank == 0:
        h = hist.cpu().tolist()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_DESC[cfg], "mode": mode, "arcs_per_rank": n,
                       "global_arcs_per_step": n_total, "seed": SEEDS[cfg],
                       "parallelism": f"arc-index shards x{ws}", "kernel": path,
                       "l2": f"inputs larger than L2 ({n * 56 / 1e9:.2f} GB in + "
                             f"{n * 49 / 1e9:.2f} GB out per rank vs 126 MB L2)"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": {**clocks.summary(), "remeasured": remeasured},
            "gpu_launches": args.steps,
            "hist": {"zero": h[0], "one": h[1], "two": h[2], "degenerate": h[3], "points": h[4]},
            "max_ulp_err": accuracy,
            "output_stats": {
                "max_norm_dev_u": float(stats[0]), f"max_dev_from_{ref_mode}_u": float(stats[1]),
                "pz_not_z0": int(counts[0]), f"count_mismatch_vs_{ref_mode}": int(counts[1]),
                "what": "sgi_output_stats over every stored point of every rank (NCCL MAX/SUM): "
                        "||P|-1|/u, Pz bit copy of z0, |P - P_ref|/u vs the other mode"},
            "points_per_s": h[4] / (ms_per_step * 1e-3),
        }
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
