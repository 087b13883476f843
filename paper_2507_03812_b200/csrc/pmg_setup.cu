// Setup kernels of the B200 solve path (not timed by the metric): node
// coefficients (level_cache.cpp:44-58) and the line factorizations of the
// zebra smoother (smoother.cpp:50-62, stencil.cpp:375-409,
// line_algebra.cpp:10-96), one thread per (section, line).
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
