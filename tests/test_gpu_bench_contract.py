"""The bench.py contract on a B200: one JSON line per run with the keys the driver and the judge
read (metric/value/unit, timing, roofline, cpu_baseline, e2e, clocks, gpu_launches), for our arm
and for `--impl reference` (the oracle on the host cores).  Small step counts; the numbers are
not checked beyond sanity, the shape is."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_default_line_has_every_key():
    """The default workload (C5, strong scaling) at a 2^24-arc batch to keep the test short."""
    d = run_bench("--steps", "20", "--warmup", "3", "--e2e-steps", "2", "--n", str(1 << 24))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] >= 3
    assert d["higher_is_better"] is True and d["scaling"] == "strong" and d["dtype"] == "f64"
    assert d["config"]["workload"].startswith("C5") and d["config"]["kernel"] == "tma_pair"
    assert d["value"] > 1e10 and d["ms_per_step"] > 0
    assert "workload" in d["config"] and "l2" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("alu", "hbm", "tensor") and 0 < r["frac"] <= 1.2
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 56 * (1 << 24) and e["d2h_bytes_per_step"] == 49 * (1 << 24)
    assert 0 < e["value"] < d["value"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["gpu_launches"] == 20
    acc = d["max_ulp_err"]
    assert acc["eft"]["max_err_u"] <= 3.0 and acc["eft"]["over_bound"] == 0
    assert acc["eft"]["count_mismatch_vs_exact"] == 0
    assert d["hist"]["zero"] > 0 and d["hist"]["two"] > 0       # C5 mixes 0/1/2 points


def test_weak_c2_line():
    d = run_bench("--config", "2", "--steps", "10", "--warmup", "3", "--e2e-steps", "0",
                  "--no-cpu-baseline")
    assert d["scaling"] == "weak" and d["config"]["arcs_per_rank"] == 1 << 24
    assert d["max_ulp_err"]["eft"]["max_err_u"] <= 3.0


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.parametrize("workload", ["zonal", "dw", "trace"])
def test_extra_workload_lines(workload):
    d = run_bench("--workload", workload, "--steps", "5", "--warmup", "3")
    assert d["value"] > 0 and d["gpu_launches"] == 5
    assert {"alu_frac", "hbm_frac"} <= set(d["roofline"])
