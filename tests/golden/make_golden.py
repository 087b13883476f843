"""Generates the golden fixtures of tests/golden/*.npz from the compiled,
unmodified reference (oracle/_ref/libpolarmg_ref.so, built from
/root/reference by oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py [--all]   (missing fixtures only, or all)

Every array is in the reference's NodeIndexing order.  Inputs are seeded
(numpy default_rng / std::mt19937 seeds noted per key).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Case, RefSolver, SEED  # noqa: E402

CASES = {
    # name: Case
    "czarny_33x32_take_V": Case(geometry="Czarny", kappa_eps=0.3, delta_e=1.4, a=33, b=32),
    "shafranov_65x64_give_V": Case(geometry="Shafranov", kappa_eps=0.3, delta_e=0.2, a=65, b=64,
                                   stencil_mode="Give"),
    "circle_33x64_give_W": Case(geometry="CirclePolar", kappa_eps=0.0, delta_e=0.0, beta_coeff=0,
                                a=33, b=64, stencil_mode="Give", cycle="W"),
    "czarny_aniso_F": Case(geometry="Czarny", kappa_eps=0.3, delta_e=1.4, grid_mode=1, a=4, b=4,
                           aniso=1, divide_by_2=1, R0=0.01, cycle="F"),
    "shafranov_interior_dirichlet": Case(geometry="Shafranov", kappa_eps=0.3, delta_e=0.2, a=33,
                                         b=32, boundary_mode=1, R0=0.013),
}


# the reference's verification problem (testsup::polar_case + make_map,
# proj/tests/support.hpp:43-58; grids of acceptance.cpp:85,237)
POLAR = dict(solution=1, R0=1.3e-5, alpha_jump=0.7, delta_r=0.05, max_iterations=150)
PROBLEM_CASES = {
    "problem_czarny_49x64_V": Case(geometry="Czarny", kappa_eps=0.3, delta_e=1.4, a=49, b=64,
                                   **POLAR),
    "problem_shafranov_interior_fmgF": Case(geometry="Shafranov", kappa_eps=0.3, delta_e=0.2,
                                            a=49, b=64, boundary_mode=1, fmg=1, **POLAR),
    "problem_czarny_97x128_give_fmgV": Case(geometry="Czarny", kappa_eps=0.3, delta_e=1.4, a=97,
                                            b=128, stencil_mode="Give", fmg=1, fmg_cycle="V",
                                            fmg_iterations=1, rel_tol=1e-8, **POLAR),
    "problem_czarny_49x64_extrapolated": Case(geometry="Czarny", kappa_eps=0.3, delta_e=1.4, a=49,
                                              b=64, extrapolation=1, rel_tol=1e-11,
                                              **dict(POLAR, max_iterations=400)),
}


def make_problem(name, c):
    R = RefSolver(c)
    out = {"levels": np.array(R.levels, dtype=np.int64)}
    out["rhs_l0"] = R.assemble_rhs(0)
    out["rhs_coarsest"] = R.assemble_rhs(R.num_levels - 1)
    sol = R.solve_native()  # the reference's own MultigridSolver::solve()
    out["solve_u"] = sol["u"]
    out["solve_history"] = sol["residual_norms"]
    out["solve_iterations"] = np.array(sol["iterations"])
    out["fine_cycles_total"] = np.array(sol["fine_cycles_total"])
    out["exact_errors"] = np.array([sol["exact_error_weighted"], sol["exact_error_infinity"]])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, R.levels[0], sol["iterations"], "cycles", sol["fine_cycles_total"], "fine")


def make(name, c):
    R = RefSolver(c)
    out = {"levels": np.array(R.levels, dtype=np.int64)}
    r, a = R.level_grid(0)
    out["radii"], out["angles"] = r, a
    rng = np.random.default_rng(1234)
    n0 = R.n(0)
    u = rng.uniform(-1, 1, n0)
    f = rng.uniform(-1, 1, n0)
    out["u_in"], out["f_in"] = u, f
    out["apply_take"] = R.apply(u, 0, "Take")
    out["apply_give"] = R.apply(u, 0, "Give")
    out["residual"] = R.residual(u, f, 0)
    out["smooth"] = R.smooth(u, f, 0)
    for kind in (0, 1):
        for par in (0, 1):
            out[f"sweep_{kind}{par}"] = R.sweep(u, f, kind, par, 0)
    out["restrict"] = R.restrict(u, 0)
    cu = rng.uniform(-1, 1, R.n(1))
    out["coarse_in"] = cu
    out["prolongate_add"] = R.prolongate(cu, u, 0, add=True)
    fc = rng.uniform(-1, 1, R.n(R.num_levels - 1))
    out["coarse_f"] = fc
    out["coarse_solve"] = R.coarse_solve(fc)
    ustar, fs = R.seeded_rhs(SEED)  # std::mt19937(20240611)
    out["seeded_ustar"], out["seeded_f"] = ustar, fs
    sol = R.solve(fs)
    out["solve_u"] = sol["u"]
    out["solve_history"] = sol["residual_norms"]
    out["solve_iterations"] = np.array(sol["iterations"])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, R.levels[0], sol["iterations"], "cycles")


if __name__ == "__main__":
    for name, c in CASES.items():
        if not os.path.exists(os.path.join(HERE, f"{name}.npz")) or "--all" in sys.argv:
            make(name, c)
    for name, c in PROBLEM_CASES.items():
        if not os.path.exists(os.path.join(HERE, f"{name}.npz")) or "--all" in sys.argv:
            make_problem(name, c)
