"""Sweep-level parity of the line kernels at the sizes the roofline numbers
come from (config 2: 4097x4096, config 4: 8193x8192), against the compiled
reference's own smoother (`smoother.cpp:95-142,184-205` via oracle/_ref).

At these sizes the circle rings (n_theta >= 2048) run on thread-block
clusters (k_circle_cl: DSMEM / st.async carry exchange) and the radial spokes
of more than 1024 nodes on k_radial_cl, so these are the only direct checks of
the cluster line kernels.  The finest two levels of each config are swept:
4097x4096 and 2049x2048 (config 2), 8193x8192 and 4097x4096 (config 4).

Benched mode (reference_order): every sweep and the smoothing step bitwise.
Fast line scans: within 1e-12 relative max-norm per sweep.
"""
import numpy as np
import pytest

from conftest import have_ref
from oracle.oracle import RefSolver, config_case
import paper_2507_03812_b200 as pmg

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")]


def relmax(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.fixture(scope="module", params=[2, 4], ids=["c2_4097", "c4_8193"])
def ref(request):
    r = RefSolver(config_case(request.param, max_iterations=0))
    r.k = request.param
    yield r
    r.__del__()


@pytest.mark.parametrize("ro", [True, False], ids=["reforder", "fast"])
def test_large_sweeps(ref, ro):
    geom, prob, grid, st, _ = pmg.baseline_config(ref.k, reference_order=ro)
    gpu = pmg.MultigridSolver(geom, prob, grid, st)
    try:
        assert gpu.level_shape(0) == ref.levels[0]
        for l in (0, 1):
            n = ref.n(l)
            rng = np.random.default_rng(900 + 10 * ref.k + l)
            u = rng.uniform(-1, 1, n)
            f = rng.uniform(-1, 1, n)
            for kind in (0, 1):  # circle, radial
                for parity in (0, 1):  # black, white
                    a = gpu.sweep(u, f, kind, parity, l)
                    b = ref.sweep(u, f, kind, parity, l)
                    if ro:
                        assert np.array_equal(a, b), (l, kind, parity, relmax(a, b))
                    else:
                        assert relmax(a, b) < 1e-12, (l, kind, parity, relmax(a, b))
            a = gpu.smooth(u, f, l)
            b = ref.smooth(u, f, l)
            if ro:
                assert np.array_equal(a, b), (l, relmax(a, b))
            else:
                assert relmax(a, b) < 1e-12, (l, relmax(a, b))
            r_gpu = gpu.residual(u, f, l)
            assert np.array_equal(r_gpu, ref.residual(u, f, l, "Take"))
    finally:
        gpu.close()
