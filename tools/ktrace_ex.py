"""Exact-order (reference_order) line solves: clock64 phase marks and wave
counts of block (0,0) of one sweep launch per level (diagnostics build
-DPMG_KTRACE).  python tools/ktrace_ex.py <config> [levels]"""
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
nlev = int(sys.argv[2]) if len(sys.argv) > 2 else 3
geom, prob, grid, st, meta = pmg.baseline_config(k, reference_order=True)
s = pmg.MultigridSolver(geom, prob, grid, st)
lib = C.CDLL(os.environ["PMG_LIB"])
buf = (C.c_ulonglong * 32)()
for level in range(min(nlev, s.num_levels() - 1)):
    n = s.n(level)
    rng = np.random.default_rng(1)
    # a smooth-ish iterate: the exact solution of a random rhs after a few sweeps
    u = rng.uniform(-1, 1, n)
    f = rng.uniform(-1, 1, n)
    for kind, parity in ((0, 0), (0, 1), (1, 0), (1, 1)):
        for rep in range(3):
            for i in range(32):
                buf[i] = 0
            lib.pmg_debug_ktrace_reset()
            s.sweep(u, f, kind, parity, level)
            lib.pmg_debug_ktrace(buf)
        m = list(buf)
        ph = [m[i + 1] - m[i] if m[i + 1] and m[i] else None for i in range(5)]
        line = (f"L{level} {s.level_shape(level)} {'circle' if kind == 0 else 'radial'} p{parity}: "
                f"phases {ph} total {m[5] - m[0] if m[5] and m[0] else None}")
        if kind == 0 and parity == 0:
            inner = [m[i + 1] - m[i] if m[i + 1] and m[i] else None for i in range(6, 11)]
            line += f" | origin phases {inner} waves fwd {m[28]} bwd {m[29]}"
        else:
            line += f" | waves fwd {m[30] % 1000} bwd {m[30] // 1000}"
        print(line)
