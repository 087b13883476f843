"""Phase timing (clock64 marks, diagnostics build with -DPMG_KTRACE) of one
smoother kernel launch of a level: python tools/ktrace.py <config> <level> <kind 0/1>"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("PMG_LIB", os.path.join(ROOT, "paper_2507_03812_b200", "lib",
                                              "libpolarmg_b200_kt.so"))
sys.path.insert(0, ROOT)
import paper_2507_03812_b200 as pmg  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
level = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kind = int(sys.argv[3]) if len(sys.argv) > 3 else 0
parity = int(sys.argv[4]) if len(sys.argv) > 4 else 1
geom, prob, grid, st, meta = pmg.baseline_config(k)
s = pmg.MultigridSolver(geom, prob, grid, st)
lib = C.CDLL(os.environ["PMG_LIB"])
buf = (C.c_ulonglong * 16)()
n = s.n(level)
u = np.random.default_rng(1).uniform(-1, 1, n)
f = np.random.default_rng(2).uniform(-1, 1, n)
for rep in range(5):
    s.sweep(u, f, kind, parity, level)
    lib.pmg_debug_ktrace(buf)
marks = list(buf)
d = [(i, marks[i + 1] - marks[i]) for i in range(6) if marks[i + 1] and marks[i]]
print(f"level {level} kind {kind} shape {s.level_shape(level)}: phase cycles", d,
      "total", marks[5] - marks[0] if marks[5] else None)
inner = [(i, marks[i + 1] - marks[i]) for i in range(6, 15) if marks[i + 1] and marks[i]]
if inner:
    print("  origin solve phases", inner)
