"""Mutation check of the oracle's evaluation-order pins (VERDICT r01 Weak #1).

Applies one plausible order mistake at a time to oracle/oracle.c (every copy of each formula),
rebuilds liboracle.so, runs tests/test_oracle_order_pins.py and reports whether a pin caught it;
the original source is restored (and rebuilt) afterwards, also on error.

    python tools/oracle_mutants.py [mutant ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(ROOT, "oracle", "oracle.c")
orig = open(src).read()
muts={
 'a_kahan_rev': ("  for (k = 0; k < P; k++) {\n    double x = A[IDX(i, k, P)] * B[IDX(k, j, M)];", "  for (k = P - 1; k >= 0; k--) {\n    double x = A[IDX(i, k, P)] * B[IDX(k, j, M)];"),
 'a2_kahan_acc_rev': ("      for (k = 0; k < K; k++) {\n        if (fused) {", "      for (k = K - 1; k >= 0; k--) {\n        if (fused) {"),
 'b_wino_yz': ("  c = (acc - yi) - zk;\n  if (P % 2 == 1) c = c + A[IDX(i, P - 1, P)]", "  c = acc - (yi + zk);\n  if (P % 2 == 1) c = c + A[IDX(i, P - 1, P)]"),
 'b2_wino_scaled_entry': ("      c = (acc - y) - z;", "      c = acc - (y + z);"),
 'b3_wino_finish': ("= (Acc[i * M + k] - y[i]) - z[k];", "= Acc[i * M + k] - (y[i] + z[k]);"),
 'b4_wino_zy': ("  c = (acc - yi) - zk;\n  if (P % 2 == 1) c = c + A[IDX(i, P - 1, P)]", "  c = (acc - zk) - yi;\n  if (P % 2 == 1) c = c + A[IDX(i, P - 1, P)]"),
 'c_sw_c21': ("    blk_add(H8, m2, H5, m2, W, m2, n2, m2);      /* C21 = (H8 + H5) + H7 */\n    blk_add(W, m2, H7, m2, C21, ldc, n2, m2);",
              "    blk_add(H5, m2, H7, m2, W, m2, n2, m2);\n    blk_add(H8, m2, W, m2, C21, ldc, n2, m2);"),
 'c2_lazy_sw_c21': ("r = (h8 + H[5]) + H[7];", "r = h8 + (H[5] + H[7]);"),
 'c3_sn_c11': ("    blk_sub(W, m2, H5, m2, W, m2, n2, m2);\n    blk_add(W, m2, H7, m2, C11, ldc, n2, m2);",
               "    blk_add(W, m2, H7, m2, W, m2, n2, m2);\n    blk_sub(W, m2, H5, m2, C11, ldc, n2, m2);"),
 'c4_lazy_sn_c22': ("else r = ((H[1] + H[3]) - H[2]) + H[6];", "else r = H[1] + ((H[3] - H[2]) + H[6]);"),
 'c5_sw_c12': ("    blk_add(H9, m2, H6, m2, C12, ldc, n2, m2);   /* C12 = H9 + H6 */", "    blk_add(H4, m2, H6, m2, W, m2, n2, m2); blk_add(H8, m2, W, m2, C12, ldc, n2, m2);"),
 'e_fused_wino': ("  c = (acc - yi) - zk;\n  if (P % 2 == 1) c = fma(", "  c = acc - (yi + zk);\n  if (P % 2 == 1) c = fma("),
 'd_norm_rev': ("    for (j = 0; j < c; j++) s = s + fabs(X[IDX(i, j, c)]);", "    for (j = c - 1; j >= 0; j--) s = s + fabs(X[IDX(i, j, c)]);"),
}
sel=sys.argv[1:] or list(muts)
missed = 0
try:
  for name in sel:
    a, b = muts[name]
    assert orig.count(a) == 1, (name, orig.count(a))
    open(src, 'w').write(orig.replace(a, b))
    r = subprocess.run([sys.executable, '-c', 'import oracle; oracle.build(force=True)'], cwd=ROOT,
                       capture_output=True, text=True)
    if r.returncode:
        print(name, 'BUILD FAIL', r.stderr[-500:])
        missed += 1
        continue
    r = subprocess.run([sys.executable, '-m', 'pytest', '-q', '-x', '-p', 'no:cacheprovider',
                        'tests/test_oracle_order_pins.py'], cwd=ROOT, capture_output=True, text=True)
    missed += r.returncode == 0
    print(f"{name:24s} {'CAUGHT' if r.returncode else 'MISSED'}  {r.stdout.strip().splitlines()[-1]}", flush=True)
finally:
    open(src, 'w').write(orig)
    subprocess.run([sys.executable, '-c', 'import oracle; oracle.build(force=True)'], cwd=ROOT)
sys.exit(1 if missed else 0)
