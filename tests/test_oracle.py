"""CPU oracle pinning (no GPU): the plain-C restatement (oracle/polarmg_oracle.c)
against the reference's golden fixtures (tests/golden, generated from the
compiled reference by tests/golden/make_golden.py), against the compiled
reference itself where present, and against the reference tests' known-answer
values (test_multigrid.cpp, test_line_algebra.cpp, test_polar_grid.cpp)."""
import ctypes as C
import glob
import os

import numpy as np
import pytest

from conftest import have_ref, requires_ref
from oracle.oracle import (Case, OracleSolver, RefSolver, SEED, canonical_to_node, config_case,
                           mt_canonical, section_scales)
import importlib.util as _ilu

_spec = _ilu.spec_from_file_location(
    "make_golden", os.path.join(os.path.dirname(__file__), "golden", "make_golden.py"))
_mg = _ilu.module_from_spec(_spec)
_spec.loader.exec_module(_mg)
CASES = _mg.CASES
PROBLEM_CASES = _mg.PROBLEM_CASES

_HERE = os.path.join(os.path.dirname(__file__), "golden")
GOLDEN = sorted(os.path.join(_HERE, f"{k}.npz") for k in CASES)
PROBLEM_GOLDEN = sorted(os.path.join(_HERE, f"{k}.npz") for k in PROBLEM_CASES)


@pytest.mark.parametrize("path", PROBLEM_GOLDEN,
                         ids=[os.path.basename(p)[:-4] for p in PROBLEM_GOLDEN])
def test_oracle_problem_matches_golden_bitwise(path):
    """assemble_rhs (stencil.cpp:307-353), FMG (multigrid.cpp:250-265), the
    solve loop and exact_errors of the C restatement against the reference's
    own MultigridSolver::solve() outputs."""
    g = np.load(path)
    O = OracleSolver(PROBLEM_CASES[os.path.basename(path)[:-4]])
    assert np.array_equal(np.array(O.levels), g["levels"])
    assert np.array_equal(O.assemble_rhs(0), g["rhs_l0"])
    assert np.array_equal(O.assemble_rhs(O.num_levels - 1), g["rhs_coarsest"])
    sol = O.solve_native()
    assert sol["iterations"] == int(g["solve_iterations"])
    assert sol["fine_cycles_total"] == int(g["fine_cycles_total"])
    assert np.array_equal(sol["u"], g["solve_u"])
    assert np.array_equal(sol["residual_norms"], g["solve_history"])
    assert np.array_equal([sol["exact_error_weighted"], sol["exact_error_infinity"]],
                          g["exact_errors"])


def test_polar_oscillation_kats():
    """test_problem.cpp:75-86: PolarOscillation vanishes at r = 0 and Rmax;
    u(Rmax/2, 0) = 0.4096 * 2^-12 = 1e-4; exact_errors of u = 0 is |u_exact|."""
    c = Case(geometry="CirclePolar", kappa_eps=0.0, delta_e=0.0, a=17, b=16, R0=1.3e-5,
             solution=1, alpha_jump=0.7, delta_r=0.05)
    O = OracleSolver(c)
    r, th = O.level_grid(0)
    rho = r / c.rmax
    exact = np.array([0.4096 * (x ** 3) ** 2 * ((1 - x) ** 3) ** 2 for x in rho])
    assert exact[-1] == 0.0
    w, inf = O.exact_errors(np.zeros(O.n(0)))
    assert inf > 0 and w > 0
    assert abs(0.4096 * 0.5 ** 12 - 1e-4) <= 1e-18
    # a problem without a solution reports -1 (multigrid.cpp:278)
    O2 = OracleSolver(Case(geometry="CirclePolar", kappa_eps=0.0, delta_e=0.0, a=17, b=16))
    assert O2.exact_errors(np.zeros(O2.n(0))) == (-1.0, -1.0)
    assert not np.any(O2.assemble_rhs(0))


@requires_ref
@pytest.mark.parametrize("geo", ["CirclePolar", "Shafranov", "Czarny"])
@pytest.mark.parametrize("bm", [0, 1])
@pytest.mark.parametrize("fmg", [0, 1])
@pytest.mark.parametrize("ex", [0, 1], ids=["plain", "extrapolated"])
def test_oracle_problem_vs_reference(geo, bm, fmg, ex):
    ke, de = {"CirclePolar": (0.0, 0.0), "Shafranov": (0.3, 0.2), "Czarny": (0.3, 1.4)}[geo]
    c = Case(geometry=geo, kappa_eps=ke, delta_e=de, a=33, b=64, R0=1.3e-5, solution=1,
             alpha_jump=0.7, delta_r=0.05, boundary_mode=bm, fmg=fmg, extrapolation=ex,
             stencil_mode="Give" if (bm + fmg) % 2 else "Take", max_iterations=400,
             rel_tol=1e-11 if ex else 1e-10)
    R, O = RefSolver(c), OracleSolver(c)
    assert np.array_equal(O.assemble_rhs(0), R.assemble_rhs(0))
    a, b = O.solve_native(), R.solve_native()
    assert a["iterations"] == b["iterations"] and a["fine_cycles_total"] == b["fine_cycles_total"]
    assert np.array_equal(a["u"], b["u"])
    assert a["exact_error_weighted"] == b["exact_error_weighted"]


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_oracle_matches_golden_bitwise(path):
    g = np.load(path)
    name = os.path.basename(path)[:-4]
    O = OracleSolver(CASES[name])
    assert np.array_equal(np.array(O.levels), g["levels"])
    r, a = O.level_grid(0)
    assert np.array_equal(r, g["radii"]) and np.array_equal(a, g["angles"])
    u, f = g["u_in"], g["f_in"]
    assert np.array_equal(O.apply(u, 0, "Take"), g["apply_take"])
    assert np.array_equal(O.apply(u, 0, "Give"), g["apply_give"])
    assert np.array_equal(O.residual(u, f, 0), g["residual"])
    assert np.array_equal(O.smooth(u, f, 0), g["smooth"])
    for kind in (0, 1):
        for par in (0, 1):
            assert np.array_equal(O.sweep(u, f, kind, par, 0), g[f"sweep_{kind}{par}"])
    assert np.array_equal(O.restrict(u, 0), g["restrict"])
    assert np.array_equal(O.prolongate(g["coarse_in"], u, 0, add=True), g["prolongate_add"])
    assert np.array_equal(O.coarse_solve(g["coarse_f"]), g["coarse_solve"])
    us, fs = O.seeded_rhs(SEED)
    assert np.array_equal(us, g["seeded_ustar"]) and np.array_equal(fs, g["seeded_f"])
    sol = O.solve(fs)
    assert sol["iterations"] == int(g["solve_iterations"])
    assert np.array_equal(sol["u"], g["solve_u"])
    assert np.array_equal(sol["residual_norms"], g["solve_history"])


@requires_ref
@pytest.mark.parametrize("case", [
    Case(geometry="Czarny", a=49, b=64, cycle="W"),
    Case(geometry="Shafranov", kappa_eps=0.3, delta_e=0.2, a=129, b=128, stencil_mode="Give",
         cycle="F", pre=2, post=1),
    Case(geometry="CirclePolar", kappa_eps=0.0, delta_e=0.0, a=65, b=64, max_levels=3),
], ids=["czarny49W", "shaf129giveF21", "circle65maxlev3"])
def test_oracle_matches_reference_bitwise(case):
    R, O = RefSolver(case), OracleSolver(case)
    assert R.levels == O.levels
    _, f = R.seeded_rhs(SEED + 7)
    a, b = R.solve(f), O.solve(f)
    assert a["iterations"] == b["iterations"]
    assert np.array_equal(a["u"], b["u"])
    assert np.array_equal(a["residual_norms"], b["residual_norms"])


def _orc_norm():
    O = OracleSolver(Case(a=17, b=16))  # loads the library
    fn = O.lib.orc_norm
    fn.restype = C.c_double
    fn.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_long]
    return lambda t, v: fn(t, np.ascontiguousarray(v, np.float64).ctypes.data_as(
        C.POINTER(C.c_double)), len(v))


def test_norm_kats():
    """test_multigrid.cpp:126-142 exact values."""
    norm = _orc_norm()
    assert norm(0, [3.0, 4.0]) == 3.5355339059327378
    assert norm(1, [3.0, 4.0]) == 5.0
    assert norm(2, [3.0, -7.0, 2.0]) == 7.0
    assert norm(0, [-3.0] * 8) == 3.0
    assert norm(2, [-3.0] * 8) == 3.0
    for t in (0, 1, 2):
        assert norm(t, [-2.5]) == 2.5


def test_hierarchy_kats():
    """test_multigrid.cpp:160-175: 65x64 -> 5 levels ending at 5x4; maxLevels=3."""
    O = OracleSolver(Case(a=65, b=64, R0=1.3e-5))
    assert len(O.levels) == 5 and O.levels[4][:2] == (5, 4)
    O3 = OracleSolver(Case(a=65, b=64, R0=1.3e-5, max_levels=3))
    assert len(O3.levels) == 3 and O3.levels[2][0] == 17


def test_grid_errors_mirror_reference():
    with pytest.raises(ValueError, match="radial spacings violate the pairing constraint"):
        OracleSolver(Case(a=4097, b=4096, max_iterations=0))
    with pytest.raises(ValueError, match="n_r must be odd"):
        OracleSolver(Case(a=16, b=16))


@pytest.mark.parametrize("k,levels,split", [(0, 7, 41), (1, 9, 163), (3, 8, 82)])
def test_config_hierarchies(k, levels, split):
    """levels / split of the BASELINE configs."""
    O = OracleSolver(config_case(k, max_iterations=0))
    assert len(O.levels) == levels and O.levels[0][2] == split
    assert O.levels[-1][:2] == (5, 4)


def test_mt19937_emulation():
    """numpy emulation of std::mt19937 + uniform_real_distribution<double>
    equals the C (and reference) generator in canonical order."""
    O = OracleSolver(Case(a=17, b=16))
    u = O.seeded_field(SEED)
    nr, nt, sp = O.levels[0]
    v = -1 + 2 * mt_canonical(SEED, nr * nt)
    w = np.zeros(nr * nt)
    perm = canonical_to_node(sp, nr, nt)
    w[perm] = v
    w[perm[(nr - 1) * nt:]] = 0.0
    assert np.array_equal(u, w)
    s = section_scales(256)
    assert s.min() >= 0.5 and s.max() < 2.0 and len(s) == 256
