"""GPU path on the paper's primary and secondary accuracy datasets
(SURVEY §8(f1)): bitwise parity with oracle (a) in every mode at 2^14 arcs per group, generated
on the device, and the per-group accuracy against oracle (b) on a deterministic sample, with the
paper's reported shapes asserted (tests/paper_accuracy.py).  The per-group CSV reports go to
$SGI_REPORT_DIR (default gpurun_out/)."""
import os

import numpy as np
import pytest

import oracle
import paper_accuracy as pa
import sgi_inputs

torch = pytest.importorskip("torch")
import paper_2510_09892_b200 as sgi  # noqa: E402

pytestmark = pytest.mark.gpu

MODES = {"eft": oracle.MODE_EFT, "eft_literal": oracle.MODE_EFT_LITERAL,
         "naive": oracle.MODE_NAIVE, "yac": oracle.MODE_YAC, "base": oracle.MODE_BASE,
         "naive_kahan": oracle.MODE_NAIVE_KAHAN}
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def same(x, y):
    return (x == y) | (np.isnan(x) & np.isnan(y))


@pytest.mark.parametrize("config", [6, 7])
def test_paper_dataset_parity_and_accuracy(config):
    ng = 17 if config == 6 else 13
    n = ng << 14
    da = torch.empty((3, n), dtype=torch.float64, device="cuda")
    db = torch.empty_like(da)
    dz = torch.empty(n, dtype=torch.float64, device="cuda")
    sgi_inputs.generate_device(config, n, da, db, dz)
    a, b, z0 = (t.cpu().numpy() for t in (da, db, dz))
    sample = np.arange(0, n, 8)
    ex = pa.exact_results(a, b, z0, sample)
    stats = {}
    for name, m in MODES.items():
        out, cnt = sgi.intersect_arc_lat(da, db, dz, mode=name)
        torch.cuda.synchronize()
        got, gcnt = out.cpu().numpy(), cnt.cpu().numpy()
        ref, rcnt = oracle.intersect(m, a, b, z0, nthreads=16)
        assert np.array_equal(gcnt, rcnt), f"{name}: {int((gcnt != rcnt).sum())} counts differ"
        ok = same(got, ref)
        assert ok.all(), f"{name}: {int((~ok).sum())} coordinates differ"
        stats[name] = pa.group_stats(config, sample, ex, got, gcnt, z0)
    pa.check_paper_claims(config, stats)
    rdir = os.environ.get("SGI_REPORT_DIR", os.path.join(ROOT, "gpurun_out"))
    pa.write_csv(os.path.join(rdir, f"paper_accuracy_c{config}_gpu.csv"), config, stats,
                 f"CUDA path (libsgi.so), {n} arcs generated on the device, oracle (b) on every "
                 f"8th ({len(sample)})")
