python - <<PY
import sys, numpy as np
sys.path.insert(0,'.')
import paper_2507_03812_b200 as pmg
geom, prob, grid, st, meta = pmg.baseline_config(3)
s = pmg.MultigridSolver(geom, prob, grid, st, n_sections=256, alpha_scales=pmg.section_scales(256))
s.seeded_rhs(20240611)
print('radial B+W ms', round(s.time_kernel('radial',0,20,True),4), 'circle', round(s.time_kernel('circle',0,20,True),4))
PY
timeout 600 python -m pytest tests/test_gpu_configs.py::test_config3_all_sections -q -m gpu 2>&1 | tail -1
