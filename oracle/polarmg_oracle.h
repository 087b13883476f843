/* TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference polarmg
 * multigrid solve path (see polarmg_oracle.c).  Same extern ABI as the
 * reference shim ref_shim.cpp, with prefix orc_.  Never linked into the
 * product. */
#ifndef POLARMG_ORACLE_H
#define POLARMG_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
int orc_create(int geom_kind, double kappa_eps, double delta_e, int alpha_coeff,
               int beta_coeff, double rmax, double alpha_jump, double delta_r,
               double alpha_scale, int grid_mode, double R0, int a, int b,
               int aniso, int divide_by_2, double pair_tol, int stencil_mode,
               int boundary_mode, int max_levels, int pre, int post, int cycle,
               int norm_type, int max_iterations, double abs_tol,
               double rel_tol, int threads, void** out);
void orc_destroy(void* h);
int orc_num_levels(void* h);
int orc_level_info(void* h, int level, int* nr, int* nt, int* split);
int orc_level_grid(void* h, int level, double* radii, double* angles);
int orc_level_coeffs(void* h, int level, double* arr, double* art, double* att,
                     double* det, double* alpha, double* beta);
int orc_row(void* h, int level, int s, int t, int* cols, double* vals, int* count);
int orc_apply(void* h, int level, int mode, const double* u, double* y);
int orc_residual(void* h, int level, int mode, const double* u, const double* f,
                 double* r);
int orc_smooth(void* h, int level, double* u, const double* f);
int orc_sweep(void* h, int level, int kind, int parity, double* u, const double* f);
int orc_restrict(void* h, int fine_level, const double* fine, double* coarse);
int orc_prolongate(void* h, int fine_level, const double* coarse, double* fine, int add);
int orc_coarse_solve(void* h, const double* f, double* u);
int orc_seeded_field(void* h, unsigned seed, double* u);
int orc_solve(void* h, const double* f, double* u_out, double* history,
              int* iterations, int* converged, double* mean_reduction,
              double* seconds);
double orc_norm(int type, const double* v, long n);
/* extras for the next orc_create on this thread: manufactured solution
 * (0 None, 1 PolarOscillation), FMG settings (multigrid.hpp:42-45) and
 * implicit extrapolation (multigrid.hpp:41) */
int orc_set_extra(int solution, int fmg, int fmg_iterations, int fmg_cycle, int extrapolation);
int orc_solve_native(void* h, double* u_out, double* history, int* iterations,
                     int* fine_cycles, int* converged, double* mean_reduction,
                     double* err_weighted, double* err_inf);
int orc_assemble_rhs(void* h, int level, double* b);
int orc_exact_errors(void* h, const double* u, double* w, double* inf);

#ifdef __cplusplus
}
#endif
#endif
