"""GPU path against the committed golden fixtures (generated from the
compiled reference; needs no oracle/_ref at run time)."""
import glob
import os

import numpy as np
import pytest

import paper_2507_03812_b200 as pmg

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
import importlib.util

_spec = importlib.util.spec_from_file_location("mg", os.path.join(HERE, "golden", "make_golden.py"))
_mg = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_mg)
GOLDEN = sorted(os.path.join(HERE, "golden", f"{k}.npz") for k in _mg.CASES)
PROBLEM_GOLDEN = sorted(os.path.join(HERE, "golden", f"{k}.npz") for k in _mg.PROBLEM_CASES)


def gpu_for(name, reference_order=True):
    c = _mg.CASES[name] if name in _mg.CASES else _mg.PROBLEM_CASES[name]
    geom = pmg.GeometryMap(c.geometry, c.kappa_eps, c.delta_e)
    prob = pmg.ProblemCase("Zoni" if c.alpha_coeff else "Poisson",
                           "InverseAlpha" if c.beta_coeff else "Zero", c.rmax, c.alpha_jump,
                           c.delta_r, c.alpha_scale, solution="Polar" if c.solution else "None")
    grid = (pmg.PolarGrid.uniform(c.R0, c.rmax, c.a, c.b) if c.grid_mode == 0 else
            pmg.PolarGrid.build(c.R0, c.rmax, c.a, c.b, c.aniso, c.divide_by_2))
    st = pmg.MultigridSettings(stencil_mode=c.stencil_mode,
                               boundary_mode=["AcrossOrigin", "InteriorDirichlet"][c.boundary_mode],
                               cycle=c.cycle, relative_tolerance=c.rel_tol,
                               max_iterations=c.max_iterations, fmg=bool(c.fmg),
                               fmg_iterations=c.fmg_iterations, fmg_cycle=c.fmg_cycle,
                               extrapolation=bool(c.extrapolation),
                               reference_order=reference_order)
    return c, pmg.MultigridSolver(geom, prob, grid, st)


@pytest.mark.parametrize("reference_order", [True, False], ids=["reforder", "fast"])
@pytest.mark.parametrize("path", PROBLEM_GOLDEN, ids=[os.path.basename(p)[:-4] for p in PROBLEM_GOLDEN])
def test_gpu_problem_against_golden(path, reference_order):
    """Manufactured RHS (bitwise), FMG start and the reference's solve() outputs."""
    g = np.load(path)
    c, s = gpu_for(os.path.basename(path)[:-4], reference_order)
    if not c.fmg and not c.extrapolation:
        s.assemble_rhs()
        assert np.array_equal(s.get_rhs(), g["rhs_l0"])
    rep = s.solve()
    if c.fmg and not c.extrapolation:  # the FMG start assembled the finest RHS itself
        assert np.array_equal(s.get_rhs(), g["rhs_l0"])
    assert rep.iterations == int(g["solve_iterations"])
    assert rep.fine_cycles_total == int(g["fine_cycles_total"])
    u = s.solution()
    err = np.abs(u - g["solve_u"]).max() / np.abs(g["solve_u"]).max()
    if reference_order and c.stencil_mode == "Take":
        assert err == 0.0
        np.testing.assert_allclose([rep.exact_error_weighted, rep.exact_error_infinity],
                                   g["exact_errors"], rtol=1e-12)
    else:
        assert err <= (1e-10 if reference_order else 1e-8)
        np.testing.assert_allclose([rep.exact_error_weighted, rep.exact_error_infinity],
                                   g["exact_errors"], rtol=1e-6)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_gpu_against_golden(path):
    g = np.load(path)
    c, s = gpu_for(os.path.basename(path)[:-4])
    assert [s.level_shape(l) for l in range(s.num_levels())] == [tuple(x) for x in g["levels"]]
    u, f = g["u_in"], g["f_in"]
    assert np.array_equal(s.apply(u, 0), g["apply_take"]) or c.stencil_mode == "Give"
    if c.stencil_mode == "Take":
        assert np.array_equal(s.residual(u, f, 0), g["residual"])
        assert np.array_equal(s.smooth(u, f, 0), g["smooth"])
    else:  # Give: the reference scatters in a different summation order
        np.testing.assert_allclose(s.apply(u, 0), g["apply_give"], rtol=0,
                                   atol=1e-13 * np.abs(g["apply_give"]).max())
    assert np.array_equal(s.restrict(u, 0), g["restrict"])
    assert np.array_equal(s.prolongate(g["coarse_in"], u, 0, add=True), g["prolongate_add"])
    assert np.array_equal(s.coarse_solve(g["coarse_f"]), g["coarse_solve"])
    us = s.seeded_rhs(20240611, return_ustar=True)
    assert np.array_equal(us, g["seeded_ustar"])
    assert np.array_equal(s.get_rhs(), g["seeded_f"])
    rep = s.solve()
    assert rep.iterations == int(g["solve_iterations"])
    err = np.abs(s.solution() - g["solve_u"]).max() / np.abs(g["solve_u"]).max()
    if c.stencil_mode == "Take":
        assert err == 0.0
    else:
        assert err < 1e-10
