// Implicit extrapolation on the finest level:
//   extrapolated smoother   smoother.cpp:83-91, 400-503
//   extrapolated residual   multigrid.cpp:224-248
//   extrapolated RHS        multigrid.cpp:159-168
//   injection               interpolation.cpp:145-165
// Every node update evaluates the reference's expressions in the reference's
// order (no FMA contraction), so results are bitwise identical.  The
// fine-only pointwise phases have no intra-phase dependencies (their
// neighbours are coarse nodes or nodes of the preceding line sweeps), so they
// run one thread per node; the circle part precedes the radial part
// (smoother.cpp:407-465) through launch order.
#include <cuda_runtime.h>

#include <type_traits>

#include "pmg_common.cuh"
#include "pmg_kernels.h"

namespace pmg {
namespace {

// 3/4 f on non-Dirichlet rows, f on Dirichlet rows: the right-hand side the
// extrapolated line sweeps gather (take_rhs_circle/radial with extrapolated,
// smoother.cpp:162-205)
__global__ void k_ex_fhat(LevelView L, const double* __restrict__ f, double* __restrict__ g,
                          const int* __restrict__ active) {
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= L.n) return;
    int s, t;
    L.node(p, s, t);
    const long o = (long)b * L.n + p;
    g[o] = L.dir(s) ? f[o] : 0.75 * f[o];
}

// u_p = (3/4 fhat_p - sum_{c != p} A_pc u_c) / A_pp with the eliminated row
// in build_row order (stencil.cpp:44-137)
template <bool ONFLY>
__device__ __forceinline__ void point_update(const LevelView& L, double* __restrict__ U,
                                             const double* __restrict__ F, long off, int b,
                                             int s, int t) {
    const int p = L.idx(s, t);
    if (L.dir(s)) {
        U[p] = F[p];
        return;
    }
    using CF = std::conditional_t<ONFLY, CoefOnTheFly, CoefArrays>;
    const CF cf{&L, b};
    (void)off;
    const Row R = make_row(L, cf, s, t);
    const Nbr q = neighbours(L, s, t, p);
    double acc = 0.75 * F[p];
    if (R.has_sm) acc -= R.sm * U[q.pSM];
    if (R.has_sp) acc -= R.sp * U[q.pSP];
    acc -= R.tm * U[q.pTM];
    acc -= R.tp * U[q.pTP];
    if (R.has_sm) {
        acc -= R.mm * U[q.pSMTM];
        acc -= R.mp * U[q.pSMTP];
    }
    if (R.has_sp) {
        acc -= R.pm * U[q.pSPTM];
        acc -= R.pp * U[q.pSPTP];
    }
    if (R.origin) acc -= R.ph * U[R.t2];
    U[p] = acc / R.d;
}

// fine-only nodes (odd t) of even circle rings (smoother.cpp:407-435)
template <bool ONFLY>
__global__ void k_ex_point_circle(LevelView L, double* __restrict__ u,
                                  const double* __restrict__ f, const int* __restrict__ active) {
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int nt_odd = L.nt / 2;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int rings = (L.split + 1) / 2;
    if (i >= rings * nt_odd) return;
    const int s = 2 * (i / nt_odd), t = 2 * (i % nt_odd) + 1;
    if (s == 0 && L.boundary == 0) return;  // joint antipodal phase
    const long off = (long)b * L.n;
    point_update<ONFLY>(L, u + off, f + off, off, b, s, t);
}

// fine-only nodes (odd rings) of even spokes (smoother.cpp:437-464)
template <bool ONFLY>
__global__ void k_ex_point_radial(LevelView L, double* __restrict__ u,
                                  const double* __restrict__ f, const int* __restrict__ active) {
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int N = L.nr - 1;
    const int s0 = L.split % 2 == 0 ? L.split + 1 : L.split;
    const int per = s0 <= N ? (N - s0) / 2 + 1 : 0;
    const int spokes = (L.nt + 1) / 2;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= spokes * per) return;
    const int t = 2 * (i / per), s = s0 + 2 * (i % per);
    const long off = (long)b * L.n;
    point_update<ONFLY>(L, u + off, f + off, off, b, s, t);
}

// antipodal fine-only pairs (t, t + n_theta/2), t odd < n_theta/2, of the
// across-origin ring: 2x2 solves (smoother.cpp:467-503)
template <bool ONFLY>
__global__ void k_ex_origin_pairs(LevelView L, double* __restrict__ u,
                                  const double* __restrict__ f, const int* __restrict__ active) {
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int half = L.nt / 2;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= half / 2) return;
    const int t = 2 * i + 1, t2 = t + half;
    const long off = (long)b * L.n;
    double* U = u + off;
    const double* F = f + off;
    using CF = std::conditional_t<ONFLY, CoefOnTheFly, CoefArrays>;
    const CF cf{&L, b};
    const int p = L.idx(0, t), qn = L.idx(0, t2);
    // row (0, ta): diagonal -> self, phantom column -> partner, rest to b
    const auto row_sys = [&](int ta, int self, int partner, double& a_self, double& a_part,
                             double& rhs) {
        const Row R = make_row(L, cf, 0, ta);
        const Nbr q = neighbours(L, 0, ta, self);
        a_self = 1.0;
        a_part = 0.0;
        rhs = 0.75 * F[self];
        const auto sub = [&](int col, double v) {
            if (col == self)
                a_self = v;
            else if (col == partner)
                a_part = v;
            else
                rhs -= v * U[col];
        };
        sub(self, R.d);
        if (R.has_sm) sub(q.pSM, R.sm);
        if (R.has_sp) sub(q.pSP, R.sp);
        sub(q.pTM, R.tm);
        sub(q.pTP, R.tp);
        if (R.has_sm) {
            sub(q.pSMTM, R.mm);
            sub(q.pSMTP, R.mp);
        }
        if (R.has_sp) {
            sub(q.pSPTM, R.pm);
            sub(q.pSPTP, R.pp);
        }
        if (R.origin) sub(R.t2, R.ph);
    };
    double a11, a12, a21, a22, b1, b2;
    row_sys(t, p, qn, a11, a12, b1);
    row_sys(t2, qn, p, a22, a21, b2);
    const double det = a11 * a22 - a12 * a21;
    U[p] = (b1 * a22 - a12 * b2) / det;
    U[qn] = (a11 * b2 - a21 * b1) / det;
}

// inject (interpolation.cpp:145-154): cu(sc,tc) = fu(2sc,2tc)
__global__ void k_inject(LevelView F, LevelView C, const double* __restrict__ fu,
                         double* __restrict__ cu, const int* __restrict__ active) {
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int pc = blockIdx.x * blockDim.x + threadIdx.x;
    if (pc >= C.n) return;
    int sc, tc;
    C.node(pc, sc, tc);
    cu[(long)b * C.n + pc] = fu[(long)b * F.n + F.idx(2 * sc, 2 * tc)];
}

// extrapolated_residual (multigrid.cpp:224-248) given out = A0 u0 and
// a1 = A1 (I u0): out = f0 - 4/3 out; out(2sc,2tc) += a1 * (1/3);
// Dirichlet rows out = f0 - u0
__global__ void k_ex_residual(LevelView F, LevelView C, const double* __restrict__ u0,
                              const double* __restrict__ f0, const double* __restrict__ a1,
                              double* __restrict__ out, const int* __restrict__ active) {
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= F.n) return;
    int s, t;
    F.node(p, s, t);
    const long o = (long)b * F.n + p;
    double v = f0[o] - (4.0 / 3.0) * out[o];
    if (!(s & 1) && !(t & 1)) v += a1[(long)b * C.n + C.idx(s >> 1, t >> 1)] * (1.0 / 3.0);
    if (F.dir(s)) v = f0[o] - u0[o];
    out[o] = v;
}

// build_extrapolated_rhs (multigrid.cpp:159-168) up to set_dirichlet_rows:
// f0 = f0 * 4/3; f0(2sc,2tc) += -f1 / 3
__global__ void k_ex_rhs(LevelView F, LevelView C, double* __restrict__ f0,
                         const double* __restrict__ f1) {
    const int b = blockIdx.y;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= F.n) return;
    int s, t;
    F.node(p, s, t);
    const long o = (long)b * F.n + p;
    double v = f0[o] * (4.0 / 3.0);
    if (!(s & 1) && !(t & 1)) v += -f1[(long)b * C.n + C.idx(s >> 1, t >> 1)] / 3.0;
    f0[o] = v;
}

inline dim3 grid_for(long n, int B) { return dim3((unsigned)((n + 127) / 128), B); }

}  // namespace

void launch_ex_fhat(const LevelView& L, const double* f, double* g, const int* active,
                    cudaStream_t st) {
    k_ex_fhat<<<grid_for(L.n, L.B), 128, 0, st>>>(L, f, g, active);
}

void launch_ex_pointwise(const LevelView& L, bool onfly, double* u, const double* f,
                         const int* active, cudaStream_t st) {
    const long nc = (long)((L.split + 1) / 2) * (L.nt / 2);
    const int N = L.nr - 1;
    const int s0 = L.split % 2 == 0 ? L.split + 1 : L.split;
    const long nrad = L.split < L.nr ? (long)((L.nt + 1) / 2) * (s0 <= N ? (N - s0) / 2 + 1 : 0)
                                     : 0;
    if (onfly) {
        if (nc > 0) k_ex_point_circle<true><<<grid_for(nc, L.B), 128, 0, st>>>(L, u, f, active);
        if (nrad > 0) k_ex_point_radial<true><<<grid_for(nrad, L.B), 128, 0, st>>>(L, u, f, active);
        if (L.boundary == 0 && L.nt / 4 > 0)
            k_ex_origin_pairs<true><<<grid_for(L.nt / 4, L.B), 128, 0, st>>>(L, u, f, active);
    } else {
        if (nc > 0) k_ex_point_circle<false><<<grid_for(nc, L.B), 128, 0, st>>>(L, u, f, active);
        if (nrad > 0)
            k_ex_point_radial<false><<<grid_for(nrad, L.B), 128, 0, st>>>(L, u, f, active);
        if (L.boundary == 0 && L.nt / 4 > 0)
            k_ex_origin_pairs<false><<<grid_for(L.nt / 4, L.B), 128, 0, st>>>(L, u, f, active);
    }
}

void launch_inject(const LevelView& F, const LevelView& C, const double* fu, double* cu,
                   const int* active, cudaStream_t st) {
    k_inject<<<grid_for(C.n, C.B), 128, 0, st>>>(F, C, fu, cu, active);
}

void launch_ex_residual(const LevelView& F, const LevelView& C, const double* u0,
                        const double* f0, const double* a1, double* out, const int* active,
                        cudaStream_t st) {
    k_ex_residual<<<grid_for(F.n, F.B), 128, 0, st>>>(F, C, u0, f0, a1, out, active);
}

void launch_ex_rhs(const LevelView& F, const LevelView& C, double* f0, const double* f1,
                   cudaStream_t st) {
    k_ex_rhs<<<grid_for(F.n, F.B), 128, 0, st>>>(F, C, f0, f1);
}

}  // namespace pmg
