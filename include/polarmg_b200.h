/*
 * polarmg_b200 -- C ABI of the B200-native GMGPolar multigrid solve path.
 *
 * Drop-in boundary for the reference's C++ class API
 *   polarmg::MultigridSolver (reference proj/core/include/polarmg/multigrid.hpp:86-151)
 * and its internal operator seams (stencil.hpp:108-113, smoother.hpp:51-53,
 * interpolation.hpp:27-36, line_algebra.hpp:90-91).  Plain pointers and sizes
 * only; no C++ or torch types cross this boundary.  No exceptions cross it
 * either: every entry point returns a status and records a thread-local
 * message retrievable with pmg_last_error() whose text mirrors the
 * reference's exception messages (config.cpp:150-183, polar_grid.cpp:69-97,
 * line_algebra.cpp:24-33).
 *
 * Ownership: a handle owns all device memory of its level hierarchy (one
 * device, one stream).  The caller owns host buffers.  A handle is not
 * thread-safe; distinct handles may be driven from distinct host threads.
 *
 * Vector layouts (argument `layout`):
 *   PMG_LAYOUT_NODE      reference NodeIndexing order (polar_grid.hpp:17-37):
 *                        rings 0..split-1 ring-major, rings split..n_r-1
 *                        spoke-major.  This is also the device layout.
 *   PMG_LAYOUT_CANONICAL s * n_theta + t for every node.
 * Batched handles (pmg_create_batch) hold n_sections independent problems
 * that share one grid; every vector argument is then n_sections contiguous
 * per-section vectors.
 */
#ifndef POLARMG_B200_H
#define POLARMG_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (extend runner.hpp:17-19 exit codes) */
#define PMG_OK 0
#define PMG_EINVAL 1      /* invalid argument / configuration (std::invalid_argument) */
#define PMG_ERUNTIME 2    /* numerical / runtime failure (std::runtime_error) */
#define PMG_ECUDA 3       /* CUDA error */
#define PMG_ENOTCONV 4    /* solve ended without meeting a tolerance */

#define PMG_LAYOUT_NODE 0
#define PMG_LAYOUT_CANONICAL 1

typedef struct pmg_solver* pmg_handle;

/* GeometryMap(kind, kappa_eps, delta_e, x0, y0)  -- geometry.hpp:35-77 */
typedef struct {
    int kind;          /* 0 CirclePolar, 1 Shafranov, 2 Czarny */
    double kappa_eps;  /* Shafranov kappa / Czarny epsilon */
    double delta_e;    /* Shafranov delta / Czarny e */
    double x0, y0;     /* map offsets (do not enter the operator) */
} pmg_geometry;

/* ProblemCase(alpha_coeff, beta_coeff, -, rmax, alpha_jump, delta_r) -- problem.hpp:47-94
 * alpha(r) = alpha_scale * exp(-tanh((r/rmax - alpha_jump)/delta_r)) (Zoni) or 1;
 * beta(r) = 0 or 1/alpha(r).  alpha_scale = 1 is the reference; batched
 * handles take one scale per section (config 3). */
typedef struct {
    int alpha_coeff;   /* 0 Poisson, 1 Zoni */
    int beta_coeff;    /* 0 Zero, 1 InverseAlpha */
    double rmax;
    double alpha_jump;
    double delta_r;
    double alpha_scale;
    int solution;      /* manufactured solution: 0 None (f = 0, u_D = 0), 1 PolarOscillation
                          (problem.cpp:48-72; make_problem, problem.cpp:150-156) */
} pmg_problem;

/* Grid construction -- polar_grid.cpp:99-178.
 * mode 0: PolarGrid::uniform(R0, Rmax, n_r, n_theta)
 * mode 1: build_grid({R0, Rmax, nr_exp, ntheta_exp, anisotropic_factor, divideBy2})
 * mode 2: explicit radii[n_r] / angles[n_theta] (PolarGrid(radii, angles))
 * pair_tolerance: relative tolerance of the pairing/uniformity checks; the
 * reference hard-codes 1e-12 (polar_grid.cpp:23,57,194); 8193x8192 needs a
 * roundoff-scaled value (documented deviation). */
typedef struct {
    int mode;
    double R0, Rmax;
    int n_r, n_theta;              /* mode 0 */
    int nr_exp, ntheta_exp;        /* mode 1 */
    int anisotropic_factor, divide_by_2;
    const double* radii;           /* mode 2 */
    const double* angles;          /* mode 2 */
    double pair_tolerance;         /* <= 0 selects 1e-12 */
} pmg_grid;

/* MultigridSettings -- multigrid.hpp:32-51 */
typedef struct {
    int stencil_mode;      /* 0 Take, 1 Give */
    int boundary_mode;     /* 0 AcrossOrigin, 1 InteriorDirichlet */
    int cache_profile;     /* accepted; alpha/beta tables are always device-resident */
    int cache_geometry;    /* Give + 1 => coefficient arrays stored (Take forces it) */
    int max_levels;        /* 0 = coarsen as far as possible */
    int pre_smoothing, post_smoothing;
    int cycle;             /* 0 V, 1 W, 2 F */
    int extrapolation;     /* 1: implicit extrapolation (multigrid.cpp:159-168,224-248); pmg_solve
                              then assembles the manufactured RHS of levels 0 and 1 (like the
                              reference's solve()) instead of using the RHS set by pmg_set_rhs */
    int fmg;               /* 1: full-multigrid start (multigrid.cpp:250-265); pmg_solve then
                              assembles the manufactured RHS of every level (like the
                              reference's solve()) instead of using the current f */
    int fmg_iterations, fmg_cycle;  /* cycles per FMG level (>= 1); 0 V, 1 W, 2 F */
    int norm_type;         /* 0 weighted-l2, 1 euclidean, 2 infinity */
    int max_iterations;
    double absolute_tolerance;  /* <= 0 disables */
    double relative_tolerance;  /* <= 0 disables */
    int max_threads;       /* accepted for API compatibility (host threads unused) */
    int verbose;
    /* extension: 1 (default) = every line solve reproduces the reference's
     * sequential substitution bit for bit (computed in parallel by speculation
     * and verification), so solves are bitwise identical to the
     * reference CPU solver; 0 = chunked parallel line scans (faster, results
     * differ from the reference at the problem's roundoff floor). */
    int reference_order;
} pmg_settings;

/* ConvergenceReport -- multigrid.hpp:55-68 (per section for batches) */
typedef struct {
    int converged;
    int iterations;
    int fine_cycles_total;
    int num_residuals;           /* iterations + 1 */
    double reduction_factor_mean;
    double initial_residual, final_residual;
    double setup_seconds;        /* host wall time of pmg_create */
    double solve_seconds;        /* device time (CUDA events) of the solve window */
    size_t device_bytes;         /* all device allocations of the handle */
    double exact_error_weighted; /* exact_errors() (multigrid.cpp:277-296); -1 without a */
    double exact_error_infinity; /* manufactured solution */
} pmg_report;

const char* pmg_last_error(void);
const char* pmg_version(void);

/* fills the reference defaults of MultigridSettings (multigrid.hpp:32-51) */
void pmg_default_settings(pmg_settings* s);

/* MultigridSolver(geometry, problem, grid, settings) -- multigrid.cpp:61-124.
 * device: CUDA ordinal; stream: cudaStream_t (NULL = handle-owned stream). */
int pmg_create(const pmg_geometry* geom, const pmg_problem* prob, const pmg_grid* grid,
               const pmg_settings* settings, int device, void* stream, pmg_handle* out);
/* n_sections problems on one grid, section i with alpha scaled by alpha_scales[i]. */
int pmg_create_batch(const pmg_geometry* geom, const pmg_problem* prob, const pmg_grid* grid,
                     const pmg_settings* settings, int n_sections, const double* alpha_scales,
                     int device, void* stream, pmg_handle* out);
int pmg_destroy(pmg_handle h);

/* host-only (no device needed): the level chain the solver would build --
 * build_grid/uniform + can_coarsen/coarsen (polar_grid.cpp:99-207,
 * multigrid.cpp:81-87).  Arrays receive min(levels, capacity) entries. */
int pmg_grid_hierarchy(const pmg_grid* grid, int max_levels, int capacity, int* levels,
                       int* n_r, int* n_theta, int* split);

/* hierarchy inspection -- multigrid.hpp:99-108 */
int pmg_num_levels(pmg_handle h, int* levels);
int pmg_num_sections(pmg_handle h, int* sections);
int pmg_level_info(pmg_handle h, int level, int* n_r, int* n_theta, int* split);
int pmg_level_grid(pmg_handle h, int level, double* radii, double* angles);

/* right-hand side of the finest level (new: the reference re-assembles its
 * manufactured RHS in solve(), multigrid.cpp:306-317).  f_host holds
 * n_sections * n_r * n_theta doubles in `layout`. */
int pmg_set_rhs(pmg_handle h, const double* f_host, int layout);
/* copy of the current finest-level RHS (all sections) */
int pmg_get_rhs(pmg_handle h, double* f_host, int layout);
/* same from device memory (already in NODE layout) */
int pmg_set_rhs_device(pmg_handle h, const void* f_device);
/* seeded synthetic RHS: u* ~ U(-1,1) from std::mt19937(seed + section),
 * canonical order, outer ring zeroed; f = A_take u* computed on the device.
 * If ustar_host is non-NULL it receives u* (layout). */
int pmg_seeded_rhs(pmg_handle h, unsigned seed, double* ustar_host, int layout);

/* f = the manufactured RHS of the finest level: DiscreteOperator::assemble_rhs
 * (stencil.cpp:307-353: rhs_f of problem.cpp:108-148 scaled by |det DF| and the
 * node weight, Dirichlet rows u_D, lifting of Dirichlet couplings), computed on
 * the device bitwise equal to the reference.  pmg_assemble_rhs + pmg_solve is
 * the reference's MultigridSolver::solve() (multigrid.cpp:309-316).
 * PMG_ERUNTIME carries the reference's "rhs_f lost accuracy" / "singular
 * Jacobian" messages. */
int pmg_assemble_rhs(pmg_handle h);
/* exact_errors() of the current finest-level u against the manufactured
 * solution (multigrid.cpp:277-296), one value per section; -1 without one. */
int pmg_exact_errors(pmg_handle h, double* weighted, double* infinity);

/* MultigridSolver::solve() with the current RHS.  reports: one per section.
 * history (optional): n_sections * history_cap doubles of residual norms. */
int pmg_solve(pmg_handle h, pmg_report* reports, double* history, int history_cap);
/* solution() of the finest level (all sections) */
int pmg_get_solution(pmg_handle h, double* u_host, int layout);
/* device pointer of the finest-level solution (NODE layout) */
int pmg_solution_device(pmg_handle h, const void** u_device);

/* ---- operator seams (host buffers, NODE layout, per level, all sections) ---- */
/* DiscreteOperator::apply / residual -- stencil.hpp:108-113 */
int pmg_apply(pmg_handle h, int level, const double* u, double* y);
int pmg_residual(pmg_handle h, int level, const double* u, const double* f, double* r);
/* Smoother::smooth (all four sweeps) -- smoother.hpp:51-53; u in/out */
int pmg_smooth(pmg_handle h, int level, double* u, const double* f);
/* one coloured sweep: kind 0 circle, 1 radial; parity 0 black, 1 white */
int pmg_sweep(pmg_handle h, int level, int kind, int parity, double* u, const double* f);
/* restrict_transpose(fine=level) -- interpolation.hpp:34-36 */
int pmg_restrict(pmg_handle h, int level, const double* fine, double* coarse);
/* prolongate(_add)(fine=level) -- interpolation.hpp:27-32 */
int pmg_prolongate(pmg_handle h, int level, const double* coarse, double* fine, int add);
/* coarsest SparseDirectFactor::solve -- multigrid.cpp:183-187 */
int pmg_coarse_solve(pmg_handle h, const double* f, double* u);
/* weighted-l2 / euclidean / infinity norm of n doubles (compute_norm, multigrid.cpp:48-59), on device */
int pmg_norm(pmg_handle h, int type, const double* v_host, long n, double* out);

/* ---- measurement helpers ---- */
/* number of kernels this handle has launched so far (graph replays counted per node) */
int pmg_launch_count(pmg_handle h, long long* count);
/* times `reps` back-to-back launches of one kernel class on level `level` with
 * CUDA events on the handle stream; kind: 0 residual, 1 circle sweep (B+W),
 * 2 radial sweep (B+W), 3 smoothing step, 4 restrict, 5 prolongate-add.
 * flush_l2 != 0 writes a >L2 buffer between repetitions (not timed). */
int pmg_time_kernel(pmg_handle h, int kind, int level, int reps, int flush_l2, double* ms_per_call);
/* per-kernel-class device time (ms) and launch count accumulated while
 * profiling is enabled (CUDA events around each launch; slows the solve). */
int pmg_profile_enable(pmg_handle h, int on);
int pmg_profile_read(pmg_handle h, int kind, double* total_ms, long long* launches);

#ifdef __cplusplus
}
#endif
#endif /* POLARMG_B200_H */
