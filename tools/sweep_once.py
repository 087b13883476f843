"""One smoother sweep of a level (for ncu captures): python tools/sweep_once.py <config>
<level> <kind 0 circle|1 radial> <parity> [fast]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_03812_b200 as pmg  # noqa: E402

k, level, kind, parity = (int(x) for x in sys.argv[1:5])
fast = len(sys.argv) > 5 and sys.argv[5] == "fast"
geom, prob, grid, st, meta = pmg.baseline_config(k, reference_order=not fast)
B = meta["n_sections"]
s = pmg.MultigridSolver(geom, prob, grid, st, n_sections=B,
                        alpha_scales=pmg.section_scales(B) if B > 1 else None)
n = s.n(level) * B
rng = np.random.default_rng(1)
u, f = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
for _ in range(3):
    s.sweep(u, f, kind, parity, level)
