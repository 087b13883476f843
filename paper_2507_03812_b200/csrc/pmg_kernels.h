// Host launchers of the B200 multigrid kernels (pmg_kernels.cu, pmg_setup.cu).
#pragma once

#include <cuda_runtime.h>

#include "pmg_common.cuh"

namespace pmg {

// first kernel-launch error since the last call, else cudaGetLastError()
cudaError_t last_error();

// Envelope LDL^T of the across-origin ring in antipodally interleaved order
// (reference smoother.cpp:33-49, line_algebra.cpp:122-255).  Rows < n-2
// have bandwidth <= 2; the two closing rows are dense (Moebius ladder).
struct OriginFactor {
    const double* band1;  // [B][n] L(i,i-1)
    const double* band2;  // [B][n] L(i,i-2)
    const double* row1;   // [B][n] L(n-2,k), k in [fc1, n-2)
    const double* row2;   // [B][n] L(n-1,k), k in [fc2, n-1)
    const double* D;      // [B][n] LDL^T diagonal
    int fc1, fc2;
    const double* inv;    // [B][n][n] dense inverse, column-major (rings of <= 32 nodes, the
                          // one-block tail), or null
};

// Generic envelope factor with identity ordering (coarsest level).
struct EnvFactor {
    const int* fc;      // [n] first column per row
    const long* ro;     // [n+1] row offsets into L
    const double* L;    // [B][nnz]
    const double* D;    // [B][n]
    const double* inv;  // [B][n][n] A^-1 column-major (coarse tail, n <= 64) or null
    long nnz;
    int n;
};

struct Weights {  // transfer weights of a fine level (interpolation.cpp:19-36)
    const double* rwb;  // [nr] radial_weight_below(sf) (odd sf)
    const double* rwa;  // [nr] radial_weight_above(sf)
    const double* awb;  // [nt] angular_weight_below(tf) (odd tf)
    const double* awa;  // [nt] angular_weight_above(tf)
};

// Device description of one level for the single-launch coarse cycle.
struct CoarseLevel {
    LevelView v;
    double *u, *f, *res;
    const double *cl, *cm, *corner;  // circle factors [B][split*nt], corner [B][split]
    const double *rl, *rm;           // radial factors [B][nt*len]
    const double* rows;              // assembled rows [B][10][n] (launch_rows)
    const double* cz;                // Sherman-Morrison vectors [B][split*nt] (exact mode)
    OriginFactor of;
    Weights w;  // this level as the fine level of a transfer
    int exact;  // reference-order (bitwise) line solves
};

enum CoarseOp {
    OP_SMOOTH = 0,
    OP_RESIDUAL = 1,
    OP_RESTRICT = 2,
    OP_PROLONG = 3,
    OP_COARSE = 4,
    OP_TAIL = 5  // cluster kernel: run the resident tail program of cycle type (op >> 8)
};

// Level descriptors of the coarse tail passed BY VALUE (constant bank):
// lv[i] describes level first + i.
constexpr int kMaxCoarse = 12;
// One array of one level copied into shared memory (resident tail).
struct CopyDesc {
    const void* src;  // global base of section 0
    long stride;      // bytes between sections (0: shared by all sections)
    int bytes;        // bytes to copy
    int dst;          // byte offset in dynamic shared memory
};
// Shared-memory image of the tail's level table: the host writes it with
// shared-memory offsets (+8, 0 = null) in every pointer field and a bit mask of
// the pointer words; the block copies it in and rebases the marked words.
struct TailImage {
    CoarseLevel lv[kMaxCoarse];
    EnvFactor env;
};
static_assert(sizeof(TailImage) % 8 == 0, "TailImage is copied as 8-byte words");

struct CoarseParams {
    CoarseLevel lv[kMaxCoarse];
    EnvFactor env;
    int first;
    // resident mode: every pointer above holds (shared-memory byte offset + 8),
    // 0 = null; the block copies `ncopy` arrays in, runs, and writes the top
    // level's u back to `top_u_global`
    int resident;
    int kw;  // rows per lane of the warp line solves (1, 2, 4, 8)
    int ncopy;
    int smem_bytes;
    const CopyDesc* copies;
    const unsigned long long* image;  // TailImage words
    const unsigned* image_mask;       // bit i: word i is a pointer
    double* top_u_global;
    // diagnostics (PMG_TAIL_TRACE): %globaltimer of block 0 at entry, after
    // staging and after every op; null = off
    unsigned long long* trace;
};

// Levels between the level kernels and the resident tail, run by one
// thread-block cluster per section (global memory, L2-resident).
constexpr int kMaxMid = 8;
struct MidParams {
    CoarseLevel lv[kMaxMid + 1];  // lv[i] = level first + i (global pointers); lv[nmid] = tail top
    int kw[kMaxMid];              // rows per lane of level first + i
    int first, nmid;
    int cl;                       // cluster size
    const int* tprog[3];          // resident tail programs per cycle type
    int tlen[3];
    CoarseParams tail;
    unsigned long long* trace;  // PMG_TAIL_TRACE: %globaltimer per op (cluster 0, rank 0)
};
#ifdef PMG_KTRACE
void read_ktrace(unsigned long long* out);  // diagnostics build only
void reset_ktrace();                       // diagnostics build only
#endif
void launch_mid_cycle(const MidParams& mp, const int* prog, int nops, int B, const int* active,
                      cudaStream_t st);
// largest cluster size <= want (power of 2) that can be scheduled, 0 if none
int mid_cluster_size(size_t smem, int want);

// Runs an op program (op | level << 8) over the coarse levels, one block per
// section.
void launch_coarse_cycle(const CoarseParams& cp, const int* prog, int nops, int B, bool onfly,
                         const int* active, cudaStream_t st);

// kernel classes for launch accounting / profiling
enum KernelKind {
    KK_RESIDUAL = 0,
    KK_CIRCLE = 1,
    KK_RADIAL = 2,
    KK_SMOOTH = 3,
    KK_RESTRICT = 4,
    KK_PROLONG = 5,
    KK_COARSE = 6,
    KK_NORM = 7,
    KK_OTHER = 8,
    KK_COUNT = 9
};

// y = A u (mode 0) or r = f - A u (mode 1); when partials != nullptr also
// writes per-block sum of squares (norm_type 0/1) or max |r| (norm_type 2)
// into partials[b * gridDim.x + block].  Returns the number of partial blocks.
int launch_apply(const LevelView& L, bool onfly, int mode, const double* u, const double* f,
                 double* out, double* partials, int norm_type, const int* active,
                 cudaStream_t st);
int apply_blocks(const LevelView& L);
int apply_launches(const LevelView& L);  // kernels one launch_apply issues

// serial: line solves in the reference's sequential operation order (bitwise
// reproduction of the reference); otherwise chunked parallel scans.
// exact_rings: circle rings s <= exact_rings use the exact-order solve even
// when serial is false (the ill-conditioned innermost rings).
void launch_circle(const LevelView& L, bool onfly, double* u, const double* f, const double* cil,
                   const double* cm, const double* corner, const double* cz,
                   const OriginFactor& of, int parity, bool serial, int exact_rings,
                   const int* active, cudaStream_t st);
// kernels one launch_circle (kind 0) / launch_radial (kind 1) issues
int line_launches(const LevelView& L, bool serial, bool onfly, int exact_rings, int kind,
                  int parity);
void launch_radial(const LevelView& L, bool onfly, double* u, const double* f, const double* ril,
                   const double* rm, int parity, bool serial, const int* active,
                   cudaStream_t st);

// Fused smoothing step (all four zebra sweeps of one level in ONE launch) for
// levels whose lines run one CTA each.  Lines are claimed through a ticket
// counter in a host-built order (fused_order) in which every line comes after
// the lines it must wait for; a CTA waits on the epoch-stamped completion
// flags of those lines, solves its line and stamps its own flag.
struct FuseCtl {
    unsigned* ctl;     // [0] ticket, [1] done, [2] epoch (starts at 1)
    unsigned* flags;   // [B][split + nt] completion epochs of rings, then spokes
};
bool fused_ok(const LevelView& L, bool serial, int exact_rings);
// claim order of the B*(split+nt) lines (codes b*(split+nt) + c; c < split:
// ring c, else spoke c - split)
void fused_order(int split, int nt, int B, int* out);
int radial_wave_cluster(const LevelView& L, bool serial, bool onfly);
void radial_wave_order(int nt, int C, int* out);
// both colours of a clustered radial sweep in one launch (flags [nt * C])
void launch_radial_wave(const LevelView& L, double* u, const double* f, const double* ril,
                        const double* rm, const FuseCtl& fc, const int* order, cudaStream_t st);
void launch_smooth_fused(const LevelView& L, bool onfly, double* u, const double* f,
                         const double* cil, const double* cm, const double* corner,
                         const double* cz, const OriginFactor& of, const double* ril,
                         const double* rm, int exact_rings, bool serial, const FuseCtl& fc,
                         const int* order, const int* active, cudaStream_t st);

// mask: zero the coarse Dirichlet rows (mask_dirichlet_rows, multigrid.cpp:146-153)
void launch_restrict(const LevelView& F, const LevelView& C, const Weights& w, const double* fr,
                     double* cf, double* cu_zero, bool mask, const int* active, cudaStream_t st);
void launch_prolong(const LevelView& F, const LevelView& C, const Weights& w, const double* cu,
                    double* fu, bool add, const int* active, cudaStream_t st);
void launch_coarse(const LevelView& L, const EnvFactor& E, const double* f, double* u,
                   const int* active, cudaStream_t st);

// per-section norm from partial block values
void launch_norm_final(const double* partials, int nblk, int B, long n, int norm_type,
                       double* norms, cudaStream_t st);
// sum of squares / max partials of an arbitrary vector set [B][n]
int launch_norm_partials(const double* v, long n, int B, int norm_type, double* partials,
                         cudaStream_t st);

// convergence bookkeeping after a residual norm (multigrid.cpp:321-340)
struct ConvState {
    double* r0;         // [B]
    double* hist;       // [B][cap]
    int* active;        // [B]
    int* iters;         // [B]
    int* converged;     // [B]
    int* remaining;     // [1]
    int* count;         // [B] norms taken so far (the iteration index)
    int cap;
};
void launch_check(const double* norms, ConvState cs, int B, int max_it, double rel_tol,
                  double abs_tol, cudaStream_t st);
// norm + convergence check in one launch (launch_norm_final + launch_check)
void launch_norm_check(const double* partials, int nblk, int B, long n, int norm_type,
                       double* norms, ConvState cs, int max_it, double rel_tol, double abs_tol,
                       cudaStream_t st);

void launch_fill(double* p, long n, double v, cudaStream_t st);
// warp-per-line radial sweep (pmg_radial_warp.cu); false: not applicable
bool launch_radial_warp(const LevelView& L, bool onfly, double* u, const double* f,
                        const double* ril, const double* rm, int parity, bool serial,
                        const int* active, cudaStream_t st);
// whether a batch of lines_total lines of n nodes runs on the warp-per-line kernels
bool warp_batch_ok(int n, long lines_total);
// warp-per-line circle sweep of rings s_first, s_first + 2, ... (nl rings, not the origin ring)
bool launch_circle_warp(const LevelView& L, double* u, const double* f, const double* cil,
                        const double* cm, const double* corner, const double* cz, int s_first,
                        int nl, bool serial, const int* active, cudaStream_t st);
// thread-per-line radial sweep (pmg_tpl.cu); false: not applicable to this level / batch
bool launch_radial_tpl(const LevelView& L, bool onfly, double* u, const double* f,
                       const double* ril, const double* rm, int parity, const int* active,
                       cudaStream_t st);
void launch_loop_cond(cudaGraphConditionalHandle h, const int* remaining, cudaStream_t st);
void launch_set_active(int* active, int* count, int* conv, int* remaining, int B,
                       cudaStream_t st);
void launch_flush(double* buf, long n, cudaStream_t st);

// ---- setup (pmg_setup.cu) ----
// coefficient arrays [B][n]; returns via *bad (device int) when |det| < 1e-14
void launch_coeffs(const LevelView& L, double* arr, double* art, double* att, double* det,
                   int* bad, cudaStream_t st);
// circle-line cyclic factors of rings [0, split) (ring 0 skipped when across-origin)
void launch_factor_circle(const LevelView& L, bool onfly, double* cil, double* cm,
                          double* corner, int* bad, cudaStream_t st);
// z = T^{-1}(e_1 + e_n) of every circle line, exact reference order
void launch_circle_z(const LevelView& L, const double* cil, const double* cm, double* cz,
                     cudaStream_t st);
void launch_factor_radial(const LevelView& L, bool onfly, double* ril, double* rm, int* bad,
                          cudaStream_t st);
// ---- manufactured problem (problem.cpp:48-148, stencil.cpp:297-353) ----
// Host-computed transcendental tables (std::exp/tanh/sin/cos, the reference's
// own libm values) at the shifted points of rhs_f's difference stencils; all
// arithmetic on them runs on the device in the reference's operation order.
struct RhsTables {
    const double* th;     // [nt] angles
    const double* aR;     // [B][nr][8] alpha(r -/+ k e), k = 2,1,1,2; e = er, er/2
    const double* sT;     // [nt][8] sin(theta -/+ k e), e = et, et/2
    const double* cT;     // [nt][8] cos(...)
    const double* s11;    // [nt][8] sin(11 (theta -/+ k e))
    const double* c11;    // [nt][8] cos(11 (theta -/+ k e))
    const double* s11_0;  // [nt] sin(11 theta)
    const double* c11_0;  // [nt] cos(11 theta)
    double rmax;          // ProblemCase / PolarOscillation rmax
    int sol;              // 1: PolarOscillation, 0: none (f = 0, u_D = 0)
};
// f = assemble_rhs of the level (raw RHS, Dirichlet rows, lifting); *bad:
// 1 singular Jacobian, 2 Richardson check failed, 3 r <= 0
void launch_assemble_rhs(const LevelView& L, const RhsTables& T, double* f, int* bad,
                         cudaStream_t st);
// set_dirichlet_rows (multigrid.cpp:133-143)
void launch_set_dirichlet(const LevelView& L, const RhsTables& T, double* u, cudaStream_t st);
// per-block partial sums of e^2 and max |e|, e = u - u_exact (multigrid.cpp:277-296);
// partials [B][nblk][2]; returns nblk
int launch_exact_errors(const LevelView& L, const RhsTables& T, const double* u,
                        double* partials, int cap, cudaStream_t st);

// ---- implicit extrapolation (pmg_extrap.cu) ----
// g = 3/4 f (f on Dirichlet rows): RHS of the extrapolated line sweeps
void launch_ex_fhat(const LevelView& L, const double* f, double* g, const int* active,
                    cudaStream_t st);
// extrapolated_pointwise + extrapolated_origin_pairs (smoother.cpp:400-503)
void launch_ex_pointwise(const LevelView& L, bool onfly, double* u, const double* f,
                         const int* active, cudaStream_t st);
// inject (interpolation.cpp:145-154)
void launch_inject(const LevelView& F, const LevelView& C, const double* fu, double* cu,
                   const int* active, cudaStream_t st);
// extrapolated_residual combination (multigrid.cpp:231-247); out holds A0 u0
void launch_ex_residual(const LevelView& F, const LevelView& C, const double* u0,
                        const double* f0, const double* a1, double* out, const int* active,
                        cudaStream_t st);
// build_extrapolated_rhs up to set_dirichlet_rows (multigrid.cpp:159-167)
void launch_ex_rhs(const LevelView& F, const LevelView& C, double* f0, const double* f1,
                   cudaStream_t st);

// assembled rows [B][10][n] of a coarse-tail level (see k_rows)
void launch_rows(const LevelView& L, bool onfly, double* rows, cudaStream_t st);
// f = A u on the finest level for seeded RHS (same as launch_apply mode 0)

}  // namespace pmg
