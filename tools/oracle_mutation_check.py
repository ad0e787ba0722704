"""Mutation check of the oracle pins (tools, not product): apply plausible transcription
mistakes to oracle/eft_oracle.c one at a time and confirm the -m "not gpu" oracle tests catch
each.  Restores the source afterwards.  Run from the repo root:
    python tools/oracle_mutation_check.py
"""
import os, shutil, subprocess, sys

ORIG = '/tmp/eft_oracle_orig.c'
shutil.copy('oracle/eft_oracle.c', ORIG)
muts = [
 ("drop es", "double w[6] = {z0, z0, s.hi, s.hi, s.lo, s.lo};", "double w[6] = {z0, z0, s.hi, s.hi, 0.0, 0.0};"),
 ("printed r1+r2", "double err = ds.lo + (p1.lo - p2.lo);", "double err = ds.lo + (p1.lo + p2.lo);"),
 ("drop eD", "double e = (S2.lo - D.lo) + E.lo;", "double e = S2.lo + E.lo;"),
 ("drop eFx3", "double eFx = (Fx1.lo + eFx2) + eFx3;", "double eFx = (Fx1.lo + eFx2);"),
 ("y sign root2", "double ym[6] = {Fy1.hi, eFy, nx.hi, nx.lo, nx.hi, nx.lo};", "double ym[6] = {Fy1.hi, eFy, nx.hi, -nx.lo, nx.hi, nx.lo};"),
 ("drop s2 in sosc", "double R = fma(2.0, Rstar, Ss.lo);", "double R = 2.0 * Rstar;"),
 ("cross transposed", "pair ny = accu_dop(x1[2], x1[0], x2[2], x2[0]);", "pair ny = accu_dop(x1[0], x1[2], x2[0], x2[2]);"),
 ("sqrt no h", "double t = r + h;", "double t = r;"),
 ("containment >", "int inp = (A1 >= B1) && (A2 <= B2);", "int inp = (A1 > B1) && (A2 <= B2);"),
 ("order flip", "const double* first = g1 >= 0.0 ? t.Pp : t.Pm;", "const double* first = g1 >= 0.0 ? t.Pm : t.Pp;"),
 # double-word low part (reading R11), caught by test_oracle_dw.py's first-order bound
 ("dw drop hi*s2", "double r = (t + dl) + (hi * s2);", "double r = (t + dl);"),
 ("dw drop dl", "double r = (t + dl) + (hi * s2);", "double r = t + (hi * s2);"),
 ("dw sign of s2", "double r = (t + dl) + (hi * s2);", "double r = (t + dl) - (hi * s2);"),
 ("dw drop sigma", "double dl = (num_pair[0] - X) + num_pair[1];", "double dl = (num_pair[0] - X);"),
]
TESTS = ['tests/test_oracle_accux.py', 'tests/test_oracle_eft_ops.py', 'tests/test_oracle_dw.py']
for name, old, new in muts:
    src = open(ORIG).read()
    assert old in src, name
    open('oracle/eft_oracle.c','w').write(src.replace(old, new))
    r = subprocess.run([sys.executable, '-m', 'pytest', *TESTS, '-x', '-q'], capture_output=True, text=True)
    print(f"{name:20s} -> {'CAUGHT' if r.returncode else 'MISSED'}  {r.stdout.strip().splitlines()[-1]}")
shutil.copy(ORIG, 'oracle/eft_oracle.c')
os.utime('oracle/eft_oracle.c')
