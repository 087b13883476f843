// Host polar grid (see pmg_grid.hpp).  Restates reference polar_grid.cpp.
#include "pmg_grid.hpp"

#include <algorithm>
#include <cmath>

namespace pmg {

namespace {

constexpr double kTwoPi = 2.0 * 3.141592653589793;

bool paired(const std::vector<double>& sp, double tol) {  // polar_grid.cpp:18-26
    if (sp.empty()) return true;
    const double scale = *std::max_element(sp.begin(), sp.end());
    for (std::size_t i = 0; i + 1 < sp.size(); i += 2)
        if (std::abs(sp[i] - sp[i + 1]) > tol * scale) return false;
    return true;
}

void invalid(const char* msg) { throw std::invalid_argument(msg); }

}  // namespace

HostGrid make_grid(std::vector<double> radii, std::vector<double> angles, double tol) {
    HostGrid g;
    g.r = std::move(radii);
    g.th = std::move(angles);
    const int nr = g.nr(), nt = g.nt();
    g.h.assign(nr > 1 ? nr - 1 : 0, 0.0);
    for (int i = 0; i + 1 < nr; ++i) g.h[i] = g.r[i + 1] - g.r[i];
    g.k.assign(nt, 0.0);
    for (int j = 0; j + 1 < nt; ++j) g.k[j] = g.th[j + 1] - g.th[j];
    if (nt > 0) g.k[nt - 1] = kTwoPi - g.th[nt - 1];

    // validate(), polar_grid.cpp:69-97
    if (nr < 3 || nt < 2) invalid("grid too small: need at least 3 radii and 2 angles");
    if (g.r[0] <= 0.0)
        invalid("invertible mapping requires r_1 > 0 (inner radius must be positive)");
    for (int i = 0; i + 1 < nr; ++i)
        if (g.r[i + 1] <= g.r[i]) invalid("radii must be strictly increasing");
    if (g.th[0] != 0.0) invalid("angles must start at 0");
    for (int j = 0; j + 1 < nt; ++j)
        if (g.th[j + 1] <= g.th[j]) invalid("angles must be strictly increasing");
    if (g.th[nt - 1] >= kTwoPi) invalid("angles must lie in [0, 2pi)");
    if (nr % 2 != 1) invalid("n_r must be odd (pairing constraint)");
    if (nt % 2 != 0) invalid("n_theta must be even (pairing constraint)");
    if (!paired(g.h, tol)) invalid("radial spacings violate the pairing constraint");
    if (!paired(g.k, tol)) invalid("angular spacings violate the pairing constraint");
    double sum = 0.0;
    for (double kk : g.k) sum += kk;
    if (std::abs(sum - kTwoPi) > 1e-14 * kTwoPi) invalid("angular spacings must sum to 2pi");

    g.uniform_angles = true;
    const double k0 = g.k[0];
    for (double kk : g.k)
        if (std::abs(kk - k0) > tol * k0) {
            g.uniform_angles = false;
            break;
        }
    int split = nr;  // numbering default when undefined (polar_grid.cpp:66)
    if (g.uniform_angles) {  // compute_smoother_split, polar_grid.cpp:30-40, clamp :63-65
        for (int i = 0; i < nr; ++i) {
            const double hh = g.h[std::min<std::size_t>(i, g.h.size() - 1)];
            if (g.r[i] * k0 > hh) {
                split = i;
                break;
            }
        }
        split = std::clamp(split, 1, nr);
    }
    g.split = split;
    return g;
}

HostGrid uniform_grid(double R0, double Rmax, int nr, int nt, double tol) {
    if (R0 <= 0.0)
        invalid("invertible mapping requires r_1 > 0 (inner radius must be positive)");
    if (Rmax <= R0) invalid("Rmax must exceed R0");
    if (nr < 3 || nt < 2) invalid("grid too small");
    std::vector<double> radii(nr);
    const double h = (Rmax - R0) / (nr - 1);
    for (int i = 0; i < nr; ++i) radii[i] = R0 + i * h;
    radii.back() = Rmax;
    std::vector<double> angles(nt);
    const double k = kTwoPi / nt;
    for (int j = 0; j < nt; ++j) angles[j] = j * k;
    return make_grid(std::move(radii), std::move(angles), tol);
}

static HostGrid refine_global(const HostGrid& g, double tol) {  // polar_grid.cpp:209-225
    std::vector<double> radii;
    radii.reserve(2 * g.nr() - 1);
    for (int i = 0; i + 1 < g.nr(); ++i) {
        radii.push_back(g.r[i]);
        radii.push_back(0.5 * (g.r[i] + g.r[i + 1]));
    }
    radii.push_back(g.r.back());
    std::vector<double> angles;
    angles.reserve(2 * g.nt());
    for (int j = 0; j < g.nt(); ++j) {
        angles.push_back(g.th[j]);
        const double next = j + 1 < g.nt() ? g.th[j + 1] : kTwoPi;
        angles.push_back(0.5 * (g.th[j] + next));
    }
    return make_grid(std::move(radii), std::move(angles), tol);
}

HostGrid build_grid(double R0, double Rmax, int nr_exp, int nt_exp, int aniso, int divide_by_2,
                    double tol) {
    if (R0 <= 0.0) invalid("invertible mapping requires r_1 > 0 (set R0 > 0)");
    if (Rmax <= R0) invalid("Rmax must exceed R0");
    if (nr_exp < 2 || nr_exp > 24) invalid("nr_exp out of range [2, 24]");
    if (nt_exp < 2 || nt_exp > 24) invalid("ntheta_exp out of range [2, 24]");
    if (aniso < 0) invalid("anisotropic_factor must be >= 0");
    if (divide_by_2 < 0) invalid("divideBy2 must be >= 0");
    HostGrid g = uniform_grid(R0, Rmax, (1 << nr_exp) + 1, 1 << nt_exp, tol);
    const double lo = 0.6 * Rmax, hi = 0.8 * Rmax;
    for (int round = 0; round < aniso; ++round) {
        const std::vector<double>& r = g.r;
        std::vector<double> refined;
        refined.reserve(r.size() * 2);
        for (std::size_t p = 0; 2 * p + 2 < r.size(); ++p) {
            const double left = r[2 * p], mid = r[2 * p + 1], right = r[2 * p + 2];
            refined.push_back(left);
            if (left >= lo && right <= hi) {
                refined.push_back(0.5 * (left + mid));
                refined.push_back(mid);
                refined.push_back(0.5 * (mid + right));
            } else {
                refined.push_back(mid);
            }
        }
        refined.push_back(r.back());
        g = make_grid(std::move(refined), g.th, tol);
    }
    for (int d = 0; d < divide_by_2; ++d) g = refine_global(g, tol);
    return g;
}

bool can_coarsen(const HostGrid& g, double tol) {
    const int cnr = (g.nr() + 1) / 2, cnt = g.nt() / 2;
    if (cnr % 2 != 1 || cnt % 2 != 0) return false;
    if (cnr < 5 || cnt < 4) return false;
    std::vector<double> ch(cnr - 1);
    for (int m = 0; m + 1 < cnr; ++m) ch[m] = g.r[2 * m + 2] - g.r[2 * m];
    return paired(ch, tol);
}

HostGrid coarsen(const HostGrid& g, double tol) {
    if (!can_coarsen(g, tol)) throw std::runtime_error("cannot coarsen this grid");
    std::vector<double> radii, angles;
    for (int i = 0; i < g.nr(); i += 2) radii.push_back(g.r[i]);
    for (int j = 0; j < g.nt(); j += 2) angles.push_back(g.th[j]);
    return make_grid(std::move(radii), std::move(angles), tol);
}

}  // namespace pmg
