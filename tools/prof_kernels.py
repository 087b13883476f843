"""Runs the hot kernels of one BASELINE config on the finest level a few
times (for ncu captures; numbers printed here are not bench values)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_03812_b200 as pmg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--kinds", default="residual,circle,radial")
ap.add_argument("--solve", action="store_true")
a = ap.parse_args()
geom, prob, grid, st, meta = pmg.baseline_config(a.config)
s = pmg.MultigridSolver(geom, prob, grid, st, n_sections=1)
n = s.n(0)
rng = np.random.default_rng(1)
s.residual(rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), 0)
for k in a.kinds.split(","):
    ms = s.time_kernel(k, 0, a.reps, True)
    print(f"{k}: {ms:.4f} ms/launch")
if a.solve:
    s.seeded_rhs(20240611)
    r = s.solve()
    print("solve", r.iterations, r.solve_seconds)
