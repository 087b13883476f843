"""Per-phase clock64 marks of the one-block tail's smoothing on the 8/16/32-angle
levels (diagnostics build -DPMG_KTRACE): python tools/ktrace_tail.py [config] [V|W]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("PMG_LIB", os.path.join(ROOT, "paper_2507_03812_b200", "lib",
                                              "libpolarmg_b200_kt.so"))
os.environ.setdefault("PMG_MID_NODES", "0")
sys.path.insert(0, ROOT)
import paper_2507_03812_b200 as pmg  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cyc = sys.argv[2] if len(sys.argv) > 2 else "W"
geom, prob, grid, st, meta = pmg.baseline_config(k, cycle=cyc)
s = pmg.MultigridSolver(geom, prob, grid, st)
s.seeded_rhs(7)
s.solve()
lib = C.CDLL(os.environ["PMG_LIB"])
buf = (C.c_ulonglong * 32)()
lib.pmg_debug_ktrace(buf)
for slot, nt in enumerate((8, 16, 32)):
    m = list(buf)[16 + 5 * slot: 21 + 5 * slot]
    if all(m):
        print(f"n_theta={nt}: circle0 {m[1]-m[0]}  circle1 {m[2]-m[1]}  radial0 {m[3]-m[2]}  "
              f"radial1 {m[4]-m[3]} cycles")
b = list(buf)
print("n_theta=16 circle1 warp line solve:", b[1] - b[0], "cycles; phase start -> solve start:",
      b[0] - b[16 + 5 * 1 + 1])
