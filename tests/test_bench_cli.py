"""bench.py's command line without a GPU: the defaults name the metric's workload (C5, 2^30 arcs
split across the ranks), and the single-GPU workloads refuse --gpus > 1."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _parse(*argv):
    import bench
    old = sys.argv
    sys.argv = ["bench.py", *argv]
    try:
        return bench.parse()
    finally:
        sys.argv = old


def test_defaults_are_the_metric_workload():
    a = _parse()
    assert (a.config, a.n, a.scaling, a.gpus, a.mode) == (5, 1 << 30, "strong", 1, "eft")
    b = _parse("--config", "2")
    assert (b.n, b.scaling) == (1 << 24, "weak")
    c = _parse("--config", "5", "--scaling", "weak", "--n", "1000")
    assert (c.n, c.scaling) == (1000, "weak")


def test_single_gpu_workloads_refuse_more_gpus():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "zonal",
                        "--gpus", "2"], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "single-GPU" in r.stderr
