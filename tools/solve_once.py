"""One warm solve of a baseline config (for ncu launch lists).

usage: python tools/solve_once.py [k] [V|W|F] [solves]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_03812_b200 as pmg

k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cyc = sys.argv[2] if len(sys.argv) > 2 else "V"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 2
geom, prob, grid, st, meta = pmg.baseline_config(k, cycle=cyc)
B = meta["n_sections"]
s = pmg.MultigridSolver(geom, prob, grid, st, n_sections=B,
                        alpha_scales=pmg.section_scales(B) if B > 1 else None)
s.seeded_rhs(20240611)
for _ in range(n):
    r = s.solve()
print("iterations", r.iterations)
