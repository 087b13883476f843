// Drop-in check of the C++ binding (include/polarmg_b200.hpp): the same
// reference objects (polarmg::GeometryMap / ProblemCase / PolarGrid /
// MultigridSettings) drive the reference's own polarmg::MultigridSolver
// (multigrid.hpp:86-151, linked from oracle/_ref/libpolarmg_ref.so) and the
// B200 library through the binding; the solves must agree bit for bit
// (reference_order is the library default).
//
// TEST INFRASTRUCTURE: built by `make -C oracle binding` into
// oracle/_ref/binding_demo, run by tests/test_binding.py (-m gpu).
#include <cstdio>
#include <cstring>
#include <memory>

#include "polarmg_b200.hpp"

using namespace polarmg;

static int run(const char* name, GeometryKind kind, double ke, double de, int nr, int nt,
               StencilMode mode, CycleType cyc, bool fmg, bool extrap) {
    GeometryMap g(kind, ke, de);
    ProblemCase p(AlphaCoeff::Zoni, BetaCoeff::InverseAlpha,
                  std::make_shared<PolarOscillation>(1.3), 1.3, 0.5, 0.1);
    PolarGrid grid = PolarGrid::uniform(1.3e-5, 1.3, nr, nt);
    MultigridSettings s;
    s.stencil_mode = mode;
    s.cycle = cyc;
    s.fmg = fmg;
    s.extrapolation = extrap;
    s.relative_tolerance = 1e-10;
    s.max_iterations = 300;
    s.max_threads = 1;

    MultigridSolver ref(g, p, grid, s);
    const ConvergenceReport rr = ref.solve();
    polarmg_b200::MultigridSolver gpu(g, p, grid, s, 0);
    const ConvergenceReport rg = gpu.solve();

    const std::vector<double>& a = ref.solution();
    const std::vector<double>& b = gpu.solution();
    double dmax = 0.0, amax = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        dmax = std::max(dmax, std::abs(a[i] - b[i]));
        amax = std::max(amax, std::abs(a[i]));
    }
    // equal values everywhere (what numpy.array_equal checks in the Python
    // parity tests); bit patterns that differ with equal values can only be
    // signed zeros, which are counted and reported
    bool bitwise = a.size() == b.size();
    size_t zeros = 0;
    for (size_t i = 0; bitwise && i < a.size(); ++i) {
        if (!(a[i] == b[i])) {
            bitwise = false;
            std::printf("  first mismatch at %zu: ref %.17g b200 %.17g\n", i, a[i], b[i]);
        } else if (std::memcmp(&a[i], &b[i], 8) != 0) {
            ++zeros;
        }
    }
    if (zeros) std::printf("  %zu nodes differ in the sign of zero\n", zeros);
    const bool same = rr.converged == rg.converged && rr.iterations == rg.iterations &&
                      rr.fine_cycles_total == rg.fine_cycles_total;
    // Give accumulates the smoother rhs by a gather (the reference scatters):
    // 1e-10, everything else bitwise
    const bool ok = same && (mode == StencilMode::Take ? bitwise : dmax <= 1e-10 * amax);
    if (!same) std::printf("  converged ref %d b200 %d\n", (int)rr.converged, (int)rg.converged);
    std::printf("%-28s ref %3d cycles (%d fine)  b200 %3d cycles (%d fine)  relmax %.3e  "
                "err_w ref %.6e b200 %.6e  %s\n",
                name, rr.iterations, rr.fine_cycles_total, rg.iterations, rg.fine_cycles_total,
                amax > 0 ? dmax / amax : dmax, rr.exact_error_weighted, rg.exact_error_weighted,
                ok ? (bitwise ? "BITWISE" : "OK") : "FAIL");
    return ok ? 0 : 1;
}

int main() {
    int bad = 0;
    try {
        bad += run("czarny65 Take V", GeometryKind::Czarny, 0.3, 1.4, 65, 64, StencilMode::Take,
                   CycleType::V, false, false);
        bad += run("shafranov129 Take W", GeometryKind::Shafranov, 0.3, 0.2, 129, 128,
                   StencilMode::Take, CycleType::W, false, false);
        bad += run("circle65 Give V", GeometryKind::CirclePolar, 0.0, 0.0, 65, 64,
                   StencilMode::Give, CycleType::V, false, false);
        bad += run("czarny97 Take FMG+extrap", GeometryKind::Czarny, 0.3, 1.4, 97, 128,
                   StencilMode::Take, CycleType::V, true, true);
    } catch (const std::exception& e) {
        std::printf("exception: %s\n", e.what());
        return 2;
    }
    std::printf(bad ? "binding_demo: %d FAILED\n" : "binding_demo: all ok\n", bad);
    return bad ? 1 : 0;
}
