"""One small multiply per class family under compute-sanitizer (tools/sanitize.sh): reduced
c2 (3D27 20^3), c3b (Graph500 R-MAT s12), c4b (smoothed Galerkin 16^3), forced warp / ESC /
CTA-hash / long classes, the long-row bucket path and the bitmap multi-tile path, both
strategies, fp64 and fp32.  Every result is checked against the oracle (structure exact)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import gen  # noqa: E402
import oracle  # noqa: E402
import paper_1504_05022_b200 as sg  # noqa: E402
from util import run_gpu  # noqa: E402


def check(A, B, flags, fp32=False, what=""):
    g = run_gpu(A, B, flags=flags, fp32=fp32)
    R = oracle.spgemm(A, B, fp32=fp32)
    assert np.array_equal(g["rp"], R.rp) and np.array_equal(g["ci"], R.ci), what
    print("ok", what, flush=True)


cases = [("c2 3d27 20^3", gen.stencil("3d27", 20), None),
         ("c3b rmat s12", gen.rmat(12, 16, (0.57, 0.19, 0.19, 0.05), mode="real"), None)]
A4, P4, R4 = gen.amg_levels("3d7", 16, 1)[0]
for name, A, B in cases:
    for fl in (0, sg.FLAG_PRECISE):
        check(A, A, fl, what="%s flags=%d" % (name, fl))
for fl in (0, sg.FLAG_PRECISE):
    check(A4, P4, fl, what="c4b AP flags=%d" % fl)
us = [2, 7, 30, 100, 700, 1500, 3000, 6000, 9000]
for tier in (7, 10, 12, 13, 16, 17, 18, 19, 20):
    A, B = gen.forced_u_pair(us, n=12000, seed=tier, mode="real", dup=0.5)
    sg.set_debug(tier, 256 if tier == 20 else 0, 40 if tier == 20 else 0)
    for fl in (0, sg.FLAG_PRECISE):
        check(A, B, fl, what="forced tier %d flags=%d" % (tier, fl))
    check(A, B, sg.FLAG_PRECISE, fp32=True, what="forced tier %d fp32" % tier)
sg.set_debug(-1, 0, 40)
sg.set_debug_long_tile(8192)
B = gen.random_rows(500, 400_000, np.full(500, 64), seed=31, mode="real")
A = gen.random_rows(20, 500, np.array([3, 20, 100, 300] * 5), seed=32, mode="real")
for fl in (0, sg.FLAG_PRECISE):
    check(A, B, fl, what="long multi-tile / bucket flags=%d" % fl)
sg.set_debug_long_bucket(1)
check(A, B, sg.FLAG_PRECISE, what="long bucket path (all long rows)")
sg.set_debug_long_bucket(0)
sg.set_debug_long_tile(0)
sg.set_debug(-1, 0, 0)
# window class: word-format and column-format structure rows (precise), k_bw_one rows and its
# overflow rows (> 56 granules: the two-walk fallback) in the hybrid strategy
n = 60_000
rows, cols = [], []
for r in range(200):
    base = (r * 97) % (n - 3000)
    for k in range(3):
        rows += [r] * 8
        cols += list(range(base + 1000 * k + (r % 32), base + 1000 * k + (r % 32) + 8))
for r in range(200, 400):
    rows += [r] * 16
    cols += list(20_000 + (r - 200) + 128 * np.arange(16))
Bw = gen.with_values(gen.from_coo(np.array(rows), np.array(cols), (400, n)), "real", 81)
ar, ac = [], []
for i in range(96):
    js = (np.arange(i, i + 6) % 200 if i % 3 == 0 else
          200 + (i * 3) % 60 + np.array([0, 60, 120]) if i % 3 == 1 else
          200 + (i * 3) % 40 + np.array([0, 30, 60, 90, 120]))
    ar += [i] * len(js)
    ac += list(js)
Aw = gen.with_values(gen.from_coo(np.array(ar), np.array(ac), (96, 400)), "real", 82)
for fl in (0, sg.FLAG_PRECISE):
    check(Aw, Bw, fl, what="window word/column/overflow rows flags=%d" % fl)
    check(Aw, Bw, fl, fp32=True, what="window rows fp32 flags=%d" % fl)
print("SANITIZE_RUN_DONE")
