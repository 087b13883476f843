// Setup kernels of the B200 solve path (not timed by the metric): node
// coefficients (level_cache.cpp:44-58) and the line factorizations of the
// zebra smoother (smoother.cpp:50-62, stencil.cpp:375-409,
// line_algebra.cpp:10-96), one thread per (section, line).
#include <algorithm>

#include "pmg_kernels.h"

namespace pmg {

namespace {

__global__ void k_coeffs(LevelView L, double* arr, double* art, double* att, double* det,
                         int* bad) {
    const int b = blockIdx.y;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= L.n) return;
    int s, t;
    L.node(p, s, t);
    bool ok = true;
    const Coef c = transform(L.geo, L.alpha[(long)b * L.nr + s], L.r[s], L.sn[t], L.cs[t], &ok);
    const long q = (long)b * L.n + p;
    arr[q] = c.arr;
    art[q] = c.art;
    att[q] = c.att;
    det[q] = c.det;
    if (!ok) atomicExch(bad, 1);
}

template <class CFT>
__device__ void factor_circle_line(const LevelView& L, const CFT& cf, int s, double* il, double* m,
                                   double* corner_out, int* bad) {
    const int nt = L.nt;
    if (L.dir(s)) {  // identity cyclic line (Dirichlet ring)
        for (int t = 0; t < nt; ++t) {
            il[t] = 1.0;
            m[t] = 0.0;
        }
        *corner_out = 0.0;
        return;
    }
    // corner = A((s,nt-1),(s,0)); core T = A - corners, T00 -= c, Tnn -= c
    const double corner = make_row(L, cf, s, nt - 1).tp;
    *corner_out = corner;
    double lprev = 0.0, offprev = 0.0;
    for (int t = 0; t < nt; ++t) {
        const Row R = make_row(L, cf, s, t);
        double d = R.d;
        if (t == 0 || t == nt - 1) d -= corner;
        double l;
        if (t == 0) {
            if (d <= 0.0) {
                atomicCAS(bad, 0, 2);
                return;
            }
            l = sqrt(d);
        } else {
            const double mm = offprev / lprev;
            const double piv = d - mm * mm;
            if (piv <= 0.0) {
                atomicCAS(bad, 0, 2);
                return;
            }
            m[t - 1] = mm;
            l = sqrt(piv);
        }
        il[t] = l;  // L diagonal (the kernels divide by it or take 1/l)
        lprev = l;
        offprev = R.tp;  // A((s,t),(s,t+1)) for t < nt-1
    }
    m[nt - 1] = 0.0;
}

template <bool ONFLY>
__global__ void k_factor_circle(LevelView L, double* cil, double* cm, double* corner, int* bad) {
    const int b = blockIdx.y;
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= L.split) return;
    if (s == 0 && L.boundary == 0) return;  // across-origin ring: envelope factor (host)
    const long o = (long)b * L.split * L.nt + (long)s * L.nt;
    if (ONFLY) {
        CoefOnTheFly cf{&L, b};
        factor_circle_line(L, cf, s, cil + o, cm + o, corner + (long)b * L.split + s, bad);
    } else {
        CoefArrays cf{&L, b};
        factor_circle_line(L, cf, s, cil + o, cm + o, corner + (long)b * L.split + s, bad);
    }
}

template <bool ONFLY>
__global__ void k_factor_radial(LevelView L, double* ril, double* rm, int* bad) {
    const int b = blockIdx.y;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= L.nt) return;
    const long o = ((long)b * L.nt + t) * L.len;
    double* il = ril + o;
    double* m = rm + o;
    double lprev = 0.0, offprev = 0.0;
    for (int i = 0; i < L.len; ++i) {
        const int s = L.split + i;
        Row R;
        if (ONFLY) {
            CoefOnTheFly cf{&L, b};
            R = make_row(L, cf, s, t);
        } else {
            CoefArrays cf{&L, b};
            R = make_row(L, cf, s, t);
        }
        const double d = R.d;
        double l;
        if (i == 0) {
            if (d <= 0.0) {
                atomicCAS(bad, 0, 3);
                return;
            }
            l = sqrt(d);
        } else {
            const double mm = offprev / lprev;
            const double piv = d - mm * mm;
            if (piv <= 0.0) {
                atomicCAS(bad, 0, 3);
                return;
            }
            m[i - 1] = mm;
            l = sqrt(piv);
        }
        il[i] = l;
        lprev = l;
        offprev = R.has_sp ? R.sp : 0.0;  // A((s,t),(s+1,t)); 0 next to the Dirichlet ring
    }
    m[L.len - 1] = 0.0;
}

__device__ __forceinline__ double xdiv_s(double a, double l, double r) {
    const double q0 = a * r;
    const double e = fma(-l, q0, a);
    return fma(e, r, q0);
}

// z = T^{-1}(e_1 + e_n) by the exact sequential substitution of
// line_algebra.cpp:42-62 (same bits as the reference's per-solve recompute)
__global__ void k_circle_z(LevelView L, const double* cl, const double* cm, double* cz) {
    const int b = blockIdx.y;
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= L.split) return;
    const int n = L.nt;
    const long o = (long)b * L.split * n + (long)s * n;
    const double* l = cl + o;
    const double* m = cm + o;
    double* z = cz + o;
    double y = xdiv_s(1.0, l[0], __drcp_rn(l[0]));
    z[0] = y;
    for (int i = 1; i < n; ++i) {
        y = xdiv_s((i == n - 1 ? 1.0 : 0.0) - m[i - 1] * y, l[i], __drcp_rn(l[i]));
        z[i] = y;
    }
    y = xdiv_s(y, l[n - 1], __drcp_rn(l[n - 1]));
    z[n - 1] = y;
    for (int i = n - 2; i >= 0; --i) {
        y = xdiv_s(z[i] - m[i] * y, l[i], __drcp_rn(l[i]));
        z[i] = y;
    }
}

// Assembled stencil rows of a coarse-tail level: rows[b][k][p], k = d, sm,
// sp, tm, tp, mm, mp, pm, pp, ph (make_row, stencil.cpp:44-137), couplings
// the row does not have stored as 0 so the tail evaluates every row with the
// same 10 multiply-adds.
template <bool ONFLY>
__global__ void k_rows(LevelView L, double* __restrict__ rows) {
    const int b = blockIdx.y;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= L.n) return;
    int s, t;
    L.node(p, s, t);
    const long off = (long)b * L.n;
    const CoefAt<ONFLY> cf{&L, off, b};
    const Nbr q = neighbours(L, s, t, p);
    const Row R = make_row_fast(L, cf, s, t, p, q);
    double* o = rows + (long)b * 10 * L.n + p;
    const long n = L.n;
    o[0] = R.d;
    o[1 * n] = R.has_sm ? R.sm : 0.0;
    o[2 * n] = R.has_sp ? R.sp : 0.0;
    o[3 * n] = R.ident ? 0.0 : R.tm;
    o[4 * n] = R.ident ? 0.0 : R.tp;
    o[5 * n] = R.has_sm ? R.mm : 0.0;
    o[6 * n] = R.has_sm ? R.mp : 0.0;
    o[7 * n] = R.has_sp ? R.pm : 0.0;
    o[8 * n] = R.has_sp ? R.pp : 0.0;
    o[9 * n] = R.origin ? R.ph : 0.0;
}

// ------------------------------------------------- manufactured problem
// PolarOscillation (problem.cpp:48-72); c11 = cos(11 theta), s11 = sin(11 theta)
__device__ __forceinline__ double sol_u(double rmax, double r, double c11) {
    const double rho = r / rmax;
    const double a = rho * rho * rho;
    const double omr = 1.0 - rho;
    const double b = omr * omr * omr;
    return 0.4096 * (a * a) * (b * b) * c11;
}
__device__ __forceinline__ double sol_ur(double rmax, double r, double c11) {
    const double rho = r / rmax;
    const double rho5 = rho * rho * rho * rho * rho;
    const double omr = 1.0 - rho;
    const double omr5 = omr * omr * omr * omr * omr;
    return 0.4096 * 6.0 * rho5 * omr5 * (1.0 - 2.0 * rho) * c11 / rmax;
}
__device__ __forceinline__ double sol_ut(double rmax, double r, double s11) {
    const double rho = r / rmax;
    const double a = rho * rho * rho;
    const double omr = 1.0 - rho;
    const double b = omr * omr * omr;
    return -11.0 * 0.4096 * (a * a) * (b * b) * s11;
}

__device__ __forceinline__ void flag(int* bad, int code) { atomicCAS(bad, 0, code); }

// assemble_rhs_raw + assemble_rhs (stencil.cpp:307-353) with rhs_f
// (problem.cpp:108-148) restated: one thread per node.
__global__ void k_assemble_rhs(LevelView L, RhsTables T, double* __restrict__ f,
                               int* __restrict__ bad) {
    const int b = blockIdx.y;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= L.n) return;
    int s, t;
    L.node(p, s, t);
    const int nr = L.nr, N = nr - 1;
    const double r = L.r[s];
    const double as = L.alpha[(long)b * nr + s], bs = L.beta[(long)b * nr + s];
    bool ok = true;
    const Coef cP = transform(L.geo, as, r, L.sn[t], L.cs[t], &ok);
    if (!ok) flag(bad, 1);
    const double det_abs = cP.det;
    double fv = 0.0;
    if (T.sol) {
        if (!(r > 0.0)) flag(bad, 3);
        const double rmax = T.rmax;
        const double a1 = 1e-4 * rmax, a2 = r / 3.0;
        const double er = a2 < a1 ? a2 : a1;
        const double et = 1e-4 * (2.0 * 3.141592653589793);
        const double bu = bs * sol_u(rmax, r, T.c11_0[t]);
        const double sn = L.sn[t], cs = L.cs[t], c0 = T.c11_0[t], s0 = T.s11_0[t];
        const double* aR = T.aR + ((long)b * nr + s) * 8;
        double fs[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const double scale = k == 0 ? 1.0 : 0.5;
            const double e = er * scale, fe = et * scale;
            const double xs[4] = {r - 2.0 * e, r - e, r + e, r + 2.0 * e};
            double g[4], q[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                bool o1 = true, o2 = true;
                const Coef cr = transform(L.geo, aR[4 * k + j], xs[j], sn, cs, &o1);
                g[j] = 2.0 * cr.arr * sol_ur(rmax, xs[j], c0) + cr.art * sol_ut(rmax, xs[j], s0);
                const int ti = t * 8 + 4 * k + j;
                const Coef ct = transform(L.geo, as, r, T.sT[ti], T.cT[ti], &o2);
                q[j] = ct.art * sol_ur(rmax, r, T.c11[ti]) + 2.0 * ct.att * sol_ut(rmax, r, T.s11[ti]);
                if (!o1 || !o2) flag(bad, 1);
            }
            const double d_r = (g[0] - 8.0 * g[1] + 8.0 * g[2] - g[3]) / (12.0 * e);
            const double d_t = (q[0] - 8.0 * q[1] + 8.0 * q[2] - q[3]) / (12.0 * fe);
            fs[k] = (-d_r - d_t) / det_abs + bu;
        }
        if (fabs(fs[0] - fs[1]) > 1e-7) flag(bad, 2);
        fv = (16.0 * fs[1] - fs[0]) / 15.0;
    }
    // node_weight (stencil.cpp:297-305)
    const int tm = L.tminus(t), tp = L.tplus(t);
    const double hm = s > 0 ? L.h[s - 1] : 0.0;
    const double hp = s < N ? L.h[s] : 0.0;
    const double km = L.k[tm], kp = L.k[t];
    double bv = fv * det_abs * (0.5 * (hm + hp) * 0.5 * (km + kp));
    const auto du = [&](int ss, int tt) {
        return T.sol ? sol_u(T.rmax, L.r[ss], T.c11_0[tt]) : 0.0;
    };
    if (L.dir(s)) {
        bv = du(s, t);
    } else {
        const bool dm = s > 0 && L.dir(s - 1), dp = s < N && L.dir(s + 1);
        if (dm || dp) {  // lifting: the un-eliminated row's Dirichlet columns in
                         // build_row<false> order (stencil.cpp:97-136)
            const auto cf = [&](int ss, int tt) {
                return transform(L.geo, L.alpha[(long)b * nr + ss], L.r[ss], L.sn[tt], L.cs[tt],
                                 nullptr);
            };
            const double kbar = 0.5 * (km + kp);
            const Coef cTM = cf(s, tm), cTP = cf(s, tp);
            const Coef z = {0.0, 0.0, 0.0, 0.0};
            const Coef cSM = s > 0 ? cf(s - 1, t) : z;
            const Coef cSP = s < N ? cf(s + 1, t) : z;
            if (dm) bv -= (-(kbar / hm) * (cP.arr + cSM.arr)) * du(s - 1, t);
            if (dp) bv -= (-(kbar / hp) * (cP.arr + cSP.arr)) * du(s + 1, t);
            if (dm) {
                bv -= (-(cTM.art + cSM.art) * 0.25) * du(s - 1, tm);
                bv -= ((cSM.art + cTP.art) * 0.25) * du(s - 1, tp);
            }
            if (dp) {
                bv -= ((cTM.art + cSP.art) * 0.25) * du(s + 1, tm);
                bv -= (-(cSP.art + cTP.art) * 0.25) * du(s + 1, tp);
            }
        }
    }
    f[(long)b * L.n + p] = bv;
}

__global__ void k_set_dirichlet(LevelView L, RhsTables T, double* __restrict__ u) {
    const int b = blockIdx.y;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= L.nt) return;
    double* U = u + (long)b * L.n;
    const int N = L.nr - 1;
    U[L.idx(N, t)] = T.sol ? sol_u(T.rmax, L.r[N], T.c11_0[t]) : 0.0;
    if (L.boundary == 1) U[L.idx(0, t)] = T.sol ? sol_u(T.rmax, L.r[0], T.c11_0[t]) : 0.0;
}

__global__ void __launch_bounds__(256) k_exact_err(LevelView L, RhsTables T,
                                                   const double* __restrict__ u,
                                                   double* __restrict__ partials) {
    const int b = blockIdx.y;
    double acc = 0.0, mx = 0.0;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < L.n; p += gridDim.x * blockDim.x) {
        int s, t;
        L.node(p, s, t);
        const double e = u[(long)b * L.n + p] - sol_u(T.rmax, L.r[s], T.c11_0[t]);
        acc += e * e;
        mx = fmax(mx, fabs(e));
    }
    __shared__ double ra[8], rm[8];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        acc += __shfl_down_sync(0xffffffffu, acc, d);
        mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, d));
    }
    if ((threadIdx.x & 31) == 0) {
        ra[threadIdx.x >> 5] = acc;
        rm[threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, m = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a += ra[w];
            m = fmax(m, rm[w]);
        }
        partials[((long)b * gridDim.x + blockIdx.x) * 2] = a;
        partials[((long)b * gridDim.x + blockIdx.x) * 2 + 1] = m;
    }
}

}  // namespace

void launch_circle_z(const LevelView& L, const double* cil, const double* cm, double* cz,
                     cudaStream_t st) {
    if (L.split <= 0) return;
    k_circle_z<<<dim3((L.split + 63) / 64, L.B), 64, 0, st>>>(L, cil, cm, cz);
}

void launch_coeffs(const LevelView& L, double* arr, double* art, double* att, double* det,
                   int* bad, cudaStream_t st) {
    k_coeffs<<<dim3((L.n + 255) / 256, L.B), 256, 0, st>>>(L, arr, art, att, det, bad);
}

void launch_factor_circle(const LevelView& L, bool onfly, double* cil, double* cm,
                          double* corner, int* bad, cudaStream_t st) {
    if (L.split <= 0) return;
    dim3 grid((L.split + 63) / 64, L.B);
    if (onfly)
        k_factor_circle<true><<<grid, 64, 0, st>>>(L, cil, cm, corner, bad);
    else
        k_factor_circle<false><<<grid, 64, 0, st>>>(L, cil, cm, corner, bad);
}

void launch_assemble_rhs(const LevelView& L, const RhsTables& T, double* f, int* bad,
                         cudaStream_t st) {
    k_assemble_rhs<<<dim3((L.n + 127) / 128, L.B), 128, 0, st>>>(L, T, f, bad);
}

void launch_set_dirichlet(const LevelView& L, const RhsTables& T, double* u, cudaStream_t st) {
    k_set_dirichlet<<<dim3((L.nt + 127) / 128, L.B), 128, 0, st>>>(L, T, u);
}

int launch_exact_errors(const LevelView& L, const RhsTables& T, const double* u,
                        double* partials, int cap, cudaStream_t st) {
    const int nb = std::max(1, std::min(cap, (L.n + 255) / 256));
    k_exact_err<<<dim3(nb, L.B), 256, 0, st>>>(L, T, u, partials);
    return nb;
}

void launch_rows(const LevelView& L, bool onfly, double* rows, cudaStream_t st) {
    dim3 grid((L.n + 127) / 128, L.B);
    if (onfly)
        k_rows<true><<<grid, 128, 0, st>>>(L, rows);
    else
        k_rows<false><<<grid, 128, 0, st>>>(L, rows);
}

void launch_factor_radial(const LevelView& L, bool onfly, double* ril, double* rm, int* bad,
                          cudaStream_t st) {
    if (L.len <= 0) return;
    dim3 grid((L.nt + 63) / 64, L.B);
    if (onfly)
        k_factor_radial<true><<<grid, 64, 0, st>>>(L, ril, rm, bad);
    else
        k_factor_radial<false><<<grid, 64, 0, st>>>(L, ril, rm, bad);
}

}  // namespace pmg
