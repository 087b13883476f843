"""Phase times of the thread-per-line radial sweep (PMG_TPL_TRACE=1):
python tools/tpl_trace.py [config] [level]"""
import ctypes as C
import os
import sys

import numpy as np

os.environ["PMG_TPL_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2507_03812_b200 as pmg  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
level = int(sys.argv[2]) if len(sys.argv) > 2 else 0
geom, prob, grid, st, meta = pmg.baseline_config(k)
B = meta["n_sections"]
s = pmg.MultigridSolver(geom, prob, grid, st, n_sections=B,
                        alpha_scales=pmg.section_scales(B) if B > 1 else None)
lib = pmg.load_library()
n = s.n(level) * B
rng = np.random.default_rng(1)
u, f = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
buf = (C.c_ulonglong * 8)()
for rep in range(3):
    lib.pmg_debug_tpl_trace(buf)
    s.sweep(u, f, 1, 0, level)
    lib.pmg_debug_tpl_trace(buf)
    m = list(buf)
    c = max(m[4], 1)
    print(f"level {level} {s.level_shape(level)} G={os.environ.get('PMG_TPL_G', 'auto')} "
          f"nopf={os.environ.get('PMG_TPL_NOPF', '0')}: CTAs {m[4]} "
          f"gather {m[0] / c / 1e3:.1f} us fwd {m[1] / c / 1e3:.1f} us bwd {m[2] / c / 1e3:.1f} us "
          f"store {m[3] / c / 1e3:.1f} us  total {sum(m[:4]) / c / 1e3:.1f} us per CTA")
