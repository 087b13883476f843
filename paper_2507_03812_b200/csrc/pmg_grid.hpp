// Host-side polar grid of the B200 solve path: construction, validation and
// the coarsening chain, restating reference polar_grid.cpp so that radii,
// angles and the circle/radial split are bitwise identical to the reference
// (which the GPU operator and the parity tests rely on).
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

namespace pmg {

struct HostGrid {
    std::vector<double> r, th, h, k;  // radii, angles, radial / angular spacings
    int split = 0;                    // first radially smoothed ring
    bool uniform_angles = false;
    int nr() const { return static_cast<int>(r.size()); }
    int nt() const { return static_cast<int>(th.size()); }
    long n() const { return static_cast<long>(nr()) * nt(); }
    int idx(int s, int t) const {
        return s < split ? s * nt() + t : split * nt() + t * (nr() - split) + (s - split);
    }
};

// PolarGrid(radii, angles) with validation (polar_grid.cpp:42-97).  `tol`
// replaces the hard-coded 1e-12 of polar_grid.cpp:23,57,194.
HostGrid make_grid(std::vector<double> radii, std::vector<double> angles, double tol);
// PolarGrid::uniform (polar_grid.cpp:99-113)
HostGrid uniform_grid(double R0, double Rmax, int nr, int nt, double tol);
// build_grid (polar_grid.cpp:131-178)
HostGrid build_grid(double R0, double Rmax, int nr_exp, int nt_exp, int aniso, int divide_by_2,
                    double tol);
// can_coarsen / coarsen (polar_grid.cpp:180-207)
bool can_coarsen(const HostGrid& g, double tol);
HostGrid coarsen(const HostGrid& g, double tol);

}  // namespace pmg
