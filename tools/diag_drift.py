"""Ring profile of |u_gpu - u_ref| after a full solve (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.oracle import RefSolver, config_case, canonical_to_node, SEED
import paper_2507_03812_b200 as pmg
k = int(sys.argv[1]); cyc = sys.argv[2] if len(sys.argv) > 2 else "V"
ref = RefSolver(config_case(k, cycle=cyc))
_, f = ref.seeded_rhs(SEED)
out = ref.solve(f)
geom, prob, grid, st, _ = pmg.baseline_config(k, cycle=cyc)
g = pmg.MultigridSolver(geom, prob, grid, st)
g.set_rhs(f); rep = g.solve(); u = g.solution()
nr, nt, sp = ref.levels[0]
perm = canonical_to_node(sp, nr, nt)
d = np.abs(u - out["u"])[perm].reshape(nr, nt)
scale = np.abs(out["u"]).max()
prof = d.max(axis=1) / scale
print("iters", out["iterations"], rep.iterations, "relmax", prof.max(), "at ring", prof.argmax(), "split", sp)
for s in [0,1,2,3,4,5,8,16,32,64,128,sp-1,sp,sp+1,nr//2,nr-2]:
    if s < nr: print(f"ring {s}: {prof[s]:.3e}")
# per-cycle history diff
h = np.array(rep.residual_norms); hr = out["residual_norms"]
print("hist rel diff", np.abs(h[:len(hr)] - hr[:len(h)]) / h[0])
