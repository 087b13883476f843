"""Per-op timing of the single-block coarse tail (PMG_TAIL_TRACE=1).

usage: python tools/tail_trace.py [config k] [V|W|F]"""
import os, sys
os.environ["PMG_TAIL_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_03812_b200 as pmg

k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cyc = sys.argv[2] if len(sys.argv) > 2 else "V"
geom, prob, grid, st, meta = pmg.baseline_config(k, cycle=cyc)
s = pmg.MultigridSolver(geom, prob, grid, st)
s.seeded_rhs(7)
for _ in range(2):
    s.solve()
