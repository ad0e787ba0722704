"""Appendix-A intermediate errors on the primary dataset, oracle (a)
against exact arithmetic.  The paper: "All intermediate results of AccuX exhibit relative errors
below u until the final steps where the numerator and denominator are each rounded to a single
working-precision value ... and then divided.  After these roundings, the relative error
stabilizes close to u".  The GPU trace kernel is bitwise equal to oracle (a)'s trace
(tests/test_gpu_trace.py), so this table is the GPU's too.  SGI_REPORT_DIR: write the CSV."""
import os

import numpy as np

import appendix_a as aa
import oracle
import sgi_inputs
from helpers import U


def test_appendix_a_accux_below_u_until_the_final_roundings():
    n = 17 * 60
    a, b, z0 = sgi_inputs.generate_host(6, n)
    exacts = [aa.exact_values(a[:, i], b[:, i], z0[i]) for i in range(n)]
    tables = {}
    for name, m in (("eft", oracle.MODE_EFT), ("eft_literal", oracle.MODE_EFT_LITERAL),
                    ("naive", oracle.MODE_NAIVE)):
        traces = [oracle.trace(m, a[:, i], b[:, i], z0[i])[1] for i in range(n)]
        tables[name] = aa.mean_table(traces, exacts)
    eft, naive = tables["eft"], tables["naive"]
    pairs = [lab for lab, hi, lo, _ in aa.ITEMS if lo]
    rounded = ["fl(numerator)", "fl(|n_xy|^2)", "p_x"]
    for lab in pairs:
        assert eft[lab][0] < U, (lab, eft[lab])
    for lab in rounded:
        assert U / 16 <= eft[lab][0] <= 2 * U, (lab, eft[lab])
    # the pairs carry ~u^2-level errors, far below binary64's own rounding of the same values
    assert eft["s"][0] < 1e-3 * naive["s"][0]
    assert eft["p_x"][0] < naive["p_x"][0]
    rdir = os.environ.get("SGI_REPORT_DIR")
    if rdir:
        aa.write_csv(os.path.join(rdir, "appendix_a_oracle_a.csv"), tables,
                     f"oracle (a), primary dataset (config 6), {n} queries")
