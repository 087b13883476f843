"""Runs a few c1 solves with the single-block coarse tail (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_03812_b200 as pmg
geom, prob, grid, st, _ = pmg.baseline_config(1)
st.max_iterations = 2
s = pmg.MultigridSolver(geom, prob, grid, st)
s.seeded_rhs(20240611)
s.solve()
print("ok")
