import sys; sys.path.insert(0,'.')
import paper_2507_03812_b200 as pmg
for k in (0,1):
    geom, prob, grid, st, _ = pmg.baseline_config(k)
    s = pmg.MultigridSolver(geom, prob, grid, st)
    s.seeded_rhs(20240611)
    s.profile(True)
    try:
        r = s.solve(); print(k, "ok", r.iterations)
    except Exception as e:
        print(k, "ERR", e)
