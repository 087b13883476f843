// polarmg_b200.hpp -- RAII mirror of polarmg::MultigridSolver
// (reference core/include/polarmg/multigrid.hpp:86-151) over the C ABI of
// include/polarmg_b200.h.  This is the binding a polarmg maintainer would add
// to switch the solve path to the B200 library: construct it from the
// reference's own GeometryMap / ProblemCase / PolarGrid / MultigridSettings,
// call solve(), read solution().  Compiled and run against the reference
// headers and a reference MultigridSolver by tests/binding_demo.cpp.
#pragma once
#include <stdexcept>
#include <string>
#include <vector>
#include "polarmg/multigrid.hpp"   // reference types
#include "polarmg_b200.h"           // this repo: include/polarmg_b200.h

namespace polarmg_b200 {

inline void check(int rc) {
    if (rc == PMG_OK || rc == PMG_ENOTCONV) return;
    if (rc == PMG_EINVAL) throw std::invalid_argument(pmg_last_error());
    throw std::runtime_error(pmg_last_error());
}

class MultigridSolver {
  public:
    MultigridSolver(const polarmg::GeometryMap& g, const polarmg::ProblemCase& p,
                    const polarmg::PolarGrid& grid, const polarmg::MultigridSettings& s,
                    int device = 0) {
        pmg_geometry G{static_cast<int>(g.kind()), g.kappa_eps(), g.delta_e(), g.x0(), g.y0()};
        pmg_problem P{static_cast<int>(p.alpha_coeff()), static_cast<int>(p.beta_coeff()),
                      p.rmax(), p.alpha_jump(), p.delta_r(), 1.0,
                      p.has_solution() ? 1 : 0};  // PolarOscillation is the only solution
        pmg_grid R{};  // explicit radii/angles: bitwise the same grid
        R.mode = 2;
        R.radii = grid.radii().data();   R.n_r = grid.n_r();
        R.angles = grid.angles().data(); R.n_theta = grid.n_theta();
        pmg_settings S;
        pmg_default_settings(&S);
        S.stencil_mode = static_cast<int>(s.stencil_mode);
        S.boundary_mode = static_cast<int>(s.boundary_mode);
        S.max_levels = s.max_levels;
        S.pre_smoothing = s.pre_smoothing;
        S.post_smoothing = s.post_smoothing;
        S.cycle = static_cast<int>(s.cycle);
        S.norm_type = static_cast<int>(s.norm_type);
        S.max_iterations = s.max_iterations;
        S.absolute_tolerance = s.absolute_tolerance;
        S.relative_tolerance = s.relative_tolerance;
        S.extrapolation = s.extrapolation ? 1 : 0;
        S.fmg = s.fmg ? 1 : 0;
        S.fmg_iterations = s.fmg_iterations;
        S.fmg_cycle = static_cast<int>(s.fmg_cycle);
        check(pmg_create(&G, &P, &R, &S, device, nullptr, &h_));
        assemble_ = p.has_solution();
        int nr, nt, sp;
        check(pmg_level_info(h_, 0, &nr, &nt, &sp));
        u_.resize(static_cast<size_t>(nr) * nt);
    }
    ~MultigridSolver() { pmg_destroy(h_); }
    MultigridSolver(const MultigridSolver&) = delete;
    MultigridSolver& operator=(const MultigridSolver&) = delete;

    // any other f (NodeIndexing order); disables the per-solve assembly
    void set_rhs(const std::vector<double>& f) {
        check(pmg_set_rhs(h_, f.data(), PMG_LAYOUT_NODE));
        assemble_ = false;
    }

    polarmg::ConvergenceReport solve() {
        if (assemble_) check(pmg_assemble_rhs(h_));  // as multigrid.cpp:309 does
        pmg_report r{};
        std::vector<double> hist(1 + 10000);
        check(pmg_solve(h_, &r, hist.data(), static_cast<int>(hist.size())));
        polarmg::ConvergenceReport rep;
        rep.converged = r.converged != 0;
        rep.iterations = r.iterations;
        rep.fine_cycles_total = r.fine_cycles_total;
        rep.residual_norms.assign(hist.begin(), hist.begin() + r.num_residuals);
        rep.reduction_factor_mean = r.reduction_factor_mean;
        rep.setup_seconds = r.setup_seconds;
        rep.solve_seconds = r.solve_seconds;
        rep.exact_error_weighted = r.exact_error_weighted;
        rep.exact_error_infinity = r.exact_error_infinity;
        check(pmg_get_solution(h_, u_.data(), PMG_LAYOUT_NODE));
        return rep;
    }
    const std::vector<double>& solution() const { return u_; }

  private:
    pmg_handle h_ = nullptr;
    std::vector<double> u_;
    bool assemble_ = false;
};

}  // namespace polarmg_b200
