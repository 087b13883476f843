// Shared host/device definitions of the B200 multigrid solve path.
//
// Everything here is __host__ __device__ so that the host-side setup (origin
// ring / coarsest factorizations) and the device kernels evaluate the SAME
// expressions in the SAME order.  The library is compiled with
// --fmad=false and IEEE div/sqrt, and the host compiler does not contract
// (x86-64 without -mfma), so geometry coefficients, operator rows and grid
// transfers are bitwise identical to the reference polarmg CPU code.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#define PMG_HD __host__ __device__ __forceinline__

namespace pmg {

// ---------------------------------------------------------------- geometry
// reference geometry.hpp:7-77, geometry.cpp:52-108
struct Geo {
    int kind;       // 0 CirclePolar, 1 Shafranov, 2 Czarny
    double ke;      // kappa (Shafranov) / epsilon (Czarny)
    double de;      // delta (Shafranov) / e (Czarny)
    double xi;      // Czarny 1/sqrt(1 - eps^2/4), else 1
};

struct Coef {
    double arr, art, att, det;
};

// TransformCoefficients of the logical-coordinate operator; *ok = false when
// |det DF| < 1e-14 (reference throws "singular Jacobian").
PMG_HD Coef transform(const Geo& G, double alpha, double r, double s, double c, bool* ok) {
    double xr, xt, yr, yt;
    if (G.kind == 0) {
        xr = c;
        xt = -r * s;
        yr = s;
        yt = r * c;
    } else if (G.kind == 1) {
        const double kap = G.ke, del = G.de;
        xr = (1.0 - kap) * c - 2.0 * del * r;
        xt = -(1.0 - kap) * r * s;
        yr = (1.0 + kap) * s;
        yt = (1.0 + kap) * r * c;
    } else {
        const double eps = G.ke, e = G.de;
        const double root = sqrt(1.0 + eps * (eps + 2.0 * r * c));
        const double denom = 2.0 - root;
        xr = -c / root;
        xt = r * s / root;
        yr = e * G.xi * s * (denom + r * eps * c / root) / (denom * denom);
        yt = e * G.xi * r * (c * denom - eps * r * s * s / root) / (denom * denom);
    }
    const double det = xr * yt - xt * yr;
    if (ok) *ok = !(fabs(det) < 1e-14);
    const double da = fabs(det);
    Coef o;
    o.arr = 0.5 * alpha * (xt * xt + yt * yt) / da;
    o.att = 0.5 * alpha * (xr * xr + yr * yr) / da;
    o.art = -alpha * (xr * xt + yr * yt) / da;
    o.det = da;
    return o;
}

// ------------------------------------------------------------- level view
// Device-side description of one level (all pointers device memory; the
// per-section arrays are [B][...] with the stated strides).
struct LevelView {
    int nr, nt, split, len;  // len = nr - split (radial line length)
    int n;                   // nr * nt
    int B;                   // sections
    int boundary;            // 0 AcrossOrigin, 1 InteriorDirichlet
    double r0;               // inner radius
    const double* r;         // [nr]
    const double* h;         // [nr-1] radial spacings
    const double* k;         // [nt] angular spacings (wrap at nt-1)
    const double* sn;        // [nt] sin(theta)
    const double* cs;        // [nt] cos(theta)
    const double* alpha;     // [B][nr]
    const double* beta;      // [B][nr]
    const double* arr;       // [B][n] node coefficients, NODE layout (Take)
    const double* art;
    const double* att;
    const double* det;
    const double* rh;        // [nr-1] RN(1/h_s)  (exact reciprocals for xdiv)
    const double* rk;        // [nt]   RN(1/k_t)
    const double* rows;      // [B][10][n] assembled rows (latency-bound levels) or null
    Geo geo;

    // reference NodeIndexing (polar_grid.hpp:24-27)
    PMG_HD int idx(int s, int t) const {
        return s < split ? s * nt + t : split * nt + t * len + (s - split);
    }
    PMG_HD void node(int p, int& s, int& t) const {
        const int cn = split * nt;
        if (p < cn) {
            s = p / nt;
            t = p - s * nt;
        } else {
            const int z = p - cn;
            t = z / len;
            s = split + (z - t * len);
        }
    }
    PMG_HD bool dir(int s) const { return s == nr - 1 || (s == 0 && boundary == 1); }
    PMG_HD int tminus(int t) const { return t == 0 ? nt - 1 : t - 1; }
    PMG_HD int tplus(int t) const { return t + 1 == nt ? 0 : t + 1; }
};

// Coefficient providers: Take reads the cached arrays (level_cache.cpp:44-58),
// Give evaluates them on the fly (level_cache.cpp:61-67) -- same values.
struct CoefArrays {
    const LevelView* L;
    int b;
    PMG_HD Coef operator()(int s, int t) const {
        const long p = (long)b * L->n + L->idx(s, t);
        Coef c;
        c.arr = L->arr[p];
        c.art = L->art[p];
        c.att = L->att[p];
        c.det = L->det[p];
        return c;
    }
};

struct CoefOnTheFly {
    const LevelView* L;
    int b;
    PMG_HD Coef operator()(int s, int t) const {
        return transform(L->geo, L->alpha[(long)b * L->nr + s], L->r[s], L->sn[t], L->cs[t],
                         nullptr);
    }
};

// ---------------------------------------------------------------- stencil
// One row of the eliminated 9-point (+ phantom) operator, reference
// stencil.cpp:44-137.  Entries: diagonal d; radial sm (s-1,t), sp (s+1,t);
// angular tm (s,t-1), tp (s,t+1); corners mm (s-1,t-1), mp (s-1,t+1),
// pm (s+1,t-1), pp (s+1,t+1); phantom ph (0,t2).  Couplings to Dirichlet
// rings are dropped (has_sm/has_sp false).  Dirichlet rows are identity.
struct Row {
    double d, sm, sp, tm, tp, mm, mp, pm, pp, ph;
    int t2;
    bool ident, has_sm, has_sp, origin;
};

template <class CF>
PMG_HD Row make_row(const LevelView& L, const CF& cf, int s, int t) {
    Row R;
    R.sm = R.sp = R.tm = R.tp = R.mm = R.mp = R.pm = R.pp = R.ph = 0.0;
    R.t2 = -1;
    R.has_sm = R.has_sp = R.origin = false;
    const int N = L.nr - 1;
    if (L.dir(s)) {
        R.ident = true;
        R.d = 1.0;
        return R;
    }
    R.ident = false;
    const int tm = L.tminus(t), tp = L.tplus(t);
    const double km = L.k[tm], kp = L.k[t];
    const double hm = s > 0 ? L.h[s - 1] : 0.0;
    const double hp = s < N ? L.h[s] : 0.0;
    const double kbar = 0.5 * (km + kp);
    const double hbar = 0.5 * (hm + hp);
    const Coef cP = cf(s, t), cTM = cf(s, tm), cTP = cf(s, tp);
    Coef cSM = {0.0, 0.0, 0.0, 0.0}, cSP = {0.0, 0.0, 0.0, 0.0};
    if (s > 0) cSM = cf(s - 1, t);
    if (s < N) cSP = cf(s + 1, t);
    const bool origin = s == 0 && L.boundary == 0;
    double diag = 0.0;
    if (s > 0) diag += (kbar / hm) * (cP.arr + cSM.arr);
    if (s < N) diag += (kbar / hp) * (cP.arr + cSP.arr);
    diag += (hbar / km) * (cP.att + cTM.att);
    diag += (hbar / kp) * (cP.att + cTP.att);
    diag += L.beta[(long)cf.b * L.nr + s] * cP.det * hbar * kbar;
    if (origin) {
        const int t2 = t + L.nt / 2 >= L.nt ? t + L.nt / 2 - L.nt : t + L.nt / 2;
        const int tlo = t < t2 ? t : t2;
        const int thi = t < t2 ? t2 : t;
        const double klo = 0.5 * (L.k[L.tminus(tlo)] + L.k[tlo]);
        const double khi = 0.5 * (L.k[L.tminus(thi)] + L.k[thi]);
        const double omega = (klo + khi) / (4.0 * L.r0);
        const double w = omega * (cf(0, tlo).arr + cf(0, thi).arr);
        diag += w;
        R.ph = -w;
        R.t2 = t2;
        R.origin = true;
    }
    R.d = diag;
    R.has_sm = s > 0 && !L.dir(s - 1);
    R.has_sp = s < N && !L.dir(s + 1);
    if (R.has_sm) R.sm = -(kbar / hm) * (cP.arr + cSM.arr);
    if (R.has_sp) R.sp = -(kbar / hp) * (cP.arr + cSP.arr);
    double south = -(hbar / km) * (cP.att + cTM.att);
    double north = -(hbar / kp) * (cP.att + cTP.att);
    if (s == 0) {
        south += (cP.art - cTM.art) * 0.25;
        north += (cTP.art - cP.art) * 0.25;
    } else if (s == N) {
        south += (cTM.art - cP.art) * 0.25;
        north += (cP.art - cTP.art) * 0.25;
    }
    R.tm = south;
    R.tp = north;
    if (R.has_sm) {
        R.mm = -(cTM.art + cSM.art) * 0.25;
        R.mp = (cSM.art + cTP.art) * 0.25;
    }
    if (R.has_sp) {
        R.pm = (cTM.art + cSP.art) * 0.25;
        R.pp = -(cSP.art + cTP.art) * 0.25;
    }
    return R;
}

// Correctly rounded a / b from r = RN(1/b) (Markstein): q0 = RN(a r) is within
// one ulp of a/b, e = a - b q0 is exact with an FMA, and RN(q0 + e r) = RN(a/b)
// for normal operands.  Used for the h/k quotients of the stencil so they stay
// bitwise identical to the reference's divisions at 3 dependent FP64 ops.
PMG_HD double xdiv(double a, double b, double r) {
    const double q0 = a * r;
    const double e = fma(-b, q0, a);
    return fma(e, r, q0);
}

// Flat NODE-layout offsets of the 8 neighbours of (s,t) (valid where the
// neighbour exists).  Interior radial rows (split < s < n_r-1) are spoke-major
// (+-1 along s, +-len across spokes), interior circle rows (0 < s < split-1)
// ring-major; the interface rows use the general NodeIndexing.
struct Nbr {
    int tm, tp;          // angular neighbour indices (wrapped)
    int pTM, pTP;        // (s,t-1), (s,t+1)
    int pSM, pSP;        // (s-1,t), (s+1,t)
    int pSMTM, pSMTP;    // (s-1,t-1), (s-1,t+1)
    int pSPTM, pSPTP;    // (s+1,t-1), (s+1,t+1)
};

PMG_HD Nbr neighbours(const LevelView& L, int s, int t, int p) {
    Nbr q;
    q.tm = L.tminus(t);
    q.tp = L.tplus(t);
    const int N = L.nr - 1;
    if (s > L.split && s < N) {
        q.pTM = p + (q.tm - t) * L.len;
        q.pTP = p + (q.tp - t) * L.len;
        q.pSM = p - 1;
        q.pSP = p + 1;
        q.pSMTM = q.pTM - 1;
        q.pSMTP = q.pTP - 1;
        q.pSPTM = q.pTM + 1;
        q.pSPTP = q.pTP + 1;
    } else if (s > 0 && s + 1 < L.split) {
        q.pTM = p + (q.tm - t);
        q.pTP = p + (q.tp - t);
        q.pSM = p - L.nt;
        q.pSP = p + L.nt;
        q.pSMTM = q.pTM - L.nt;
        q.pSMTP = q.pTP - L.nt;
        q.pSPTM = q.pTM + L.nt;
        q.pSPTP = q.pTP + L.nt;
    } else {
        q.pTM = L.idx(s, q.tm);
        q.pTP = L.idx(s, q.tp);
        q.pSM = s > 0 ? L.idx(s - 1, t) : p;
        q.pSP = s < N ? L.idx(s + 1, t) : p;
        q.pSMTM = s > 0 ? L.idx(s - 1, q.tm) : p;
        q.pSMTP = s > 0 ? L.idx(s - 1, q.tp) : p;
        q.pSPTM = s < N ? L.idx(s + 1, q.tm) : p;
        q.pSPTP = s < N ? L.idx(s + 1, q.tp) : p;
    }
    return q;
}

// Take-mode coefficient reads by flat index; Give evaluates them at (s,t).
template <bool ONFLY>
struct CoefAt;
template <>
struct CoefAt<false> {
    const LevelView* L;
    long off;
    int b;
    __device__ __forceinline__ Coef operator()(int s, int t, int p) const {
        (void)s;
        (void)t;
        Coef c;
        c.arr = L->arr[off + p];
        c.art = L->art[off + p];
        c.att = L->att[off + p];
        c.det = L->det[off + p];
        return c;
    }
};
template <>
struct CoefAt<true> {
    const LevelView* L;
    long off;
    int b;
    __device__ __forceinline__ Coef operator()(int s, int t, int p) const {
        (void)p;
        return transform(L->geo, L->alpha[(long)b * L->nr + s], L->r[s], L->sn[t], L->cs[t],
                         nullptr);
    }
};

// make_row with precomputed neighbour offsets and Markstein quotients: the
// same values as make_row (bitwise); fields a caller does not use are
// eliminated by the compiler after inlining.
// Row of (s,t) from the coefficients of the node and its four neighbours
// (no loads; the origin-ring phantom weight needs arr of the antipodal node,
// passed in arrAnti).  Same expressions and order as make_row
// (stencil.cpp:44-137); h/k quotients by Markstein division.
__host__ __device__ __forceinline__ Row row_from(const LevelView& L, int b, int s, int t, int tm,
                                                 const Coef& cP, const Coef& cTM,
                                                 const Coef& cTP, const Coef& cSM,
                                                 const Coef& cSP, double arrAnti) {
    Row R;
    R.sm = R.sp = R.tm = R.tp = R.mm = R.mp = R.pm = R.pp = R.ph = 0.0;
    R.t2 = -1;
    R.has_sm = R.has_sp = R.origin = false;
    const int N = L.nr - 1;
    if (L.dir(s)) {
        R.ident = true;
        R.d = 1.0;
        return R;
    }
    R.ident = false;
    const double km = L.k[tm], kp = L.k[t];
    const double hm = s > 0 ? L.h[s - 1] : 0.0;
    const double hp = s < N ? L.h[s] : 0.0;
    const double kbar = 0.5 * (km + kp);
    const double hbar = 0.5 * (hm + hp);
    const double qkm = s > 0 ? xdiv(kbar, hm, L.rh[s - 1]) : 0.0;  // kbar / hm
    const double qkp = s < N ? xdiv(kbar, hp, L.rh[s]) : 0.0;      // kbar / hp
    const double qhm = xdiv(hbar, km, L.rk[tm]);                   // hbar / km
    const double qhp = xdiv(hbar, kp, L.rk[t]);                    // hbar / kp
    double diag = 0.0;
    if (s > 0) diag += qkm * (cP.arr + cSM.arr);
    if (s < N) diag += qkp * (cP.arr + cSP.arr);
    diag += qhm * (cP.att + cTM.att);
    diag += qhp * (cP.att + cTP.att);
    diag += L.beta[(long)b * L.nr + s] * cP.det * hbar * kbar;
    if (s == 0 && L.boundary == 0) {
        const int t2 = t + L.nt / 2 >= L.nt ? t + L.nt / 2 - L.nt : t + L.nt / 2;
        const int tlo = t < t2 ? t : t2;
        const int thi = t < t2 ? t2 : t;
        const double klo = 0.5 * (L.k[L.tminus(tlo)] + L.k[tlo]);
        const double khi = 0.5 * (L.k[L.tminus(thi)] + L.k[thi]);
        const double omega = (klo + khi) / (4.0 * L.r0);
        const double alo = t < t2 ? cP.arr : arrAnti, ahi = t < t2 ? arrAnti : cP.arr;
        const double w = omega * (alo + ahi);
        diag += w;
        R.ph = -w;
        R.t2 = t2;
        R.origin = true;
    }
    R.d = diag;
    R.has_sm = s > 0 && !L.dir(s - 1);
    R.has_sp = s < N && !L.dir(s + 1);
    if (R.has_sm) R.sm = -qkm * (cP.arr + cSM.arr);
    if (R.has_sp) R.sp = -qkp * (cP.arr + cSP.arr);
    double south = -qhm * (cP.att + cTM.att);
    double north = -qhp * (cP.att + cTP.att);
    if (s == 0) {
        south += (cP.art - cTM.art) * 0.25;
        north += (cTP.art - cP.art) * 0.25;
    } else if (s == N) {
        south += (cTM.art - cP.art) * 0.25;
        north += (cP.art - cTP.art) * 0.25;
    }
    R.tm = south;
    R.tp = north;
    if (R.has_sm) {
        R.mm = -(cTM.art + cSM.art) * 0.25;
        R.mp = (cSM.art + cTP.art) * 0.25;
    }
    if (R.has_sp) {
        R.pm = (cTM.art + cSP.art) * 0.25;
        R.pp = -(cSP.art + cTP.art) * 0.25;
    }
    return R;
}

// make_row with precomputed neighbour offsets: loads then row_from.
template <class CF>
__device__ __forceinline__ Row make_row_fast(const LevelView& L, const CF& cf, int s, int t, int p,
                                             const Nbr& q) {
    const int N = L.nr - 1;
    if (L.dir(s)) {
        Row R;
        R.sm = R.sp = R.tm = R.tp = R.mm = R.mp = R.pm = R.pp = R.ph = 0.0;
        R.t2 = -1;
        R.has_sm = R.has_sp = R.origin = false;
        R.ident = true;
        R.d = 1.0;
        return R;
    }
    const Coef z = {0.0, 0.0, 0.0, 0.0};
    const Coef cP = cf(s, t, p), cTM = cf(s, q.tm, q.pTM), cTP = cf(s, q.tp, q.pTP);
    const Coef cSM = s > 0 ? cf(s - 1, t, q.pSM) : z;
    const Coef cSP = s < N ? cf(s + 1, t, q.pSP) : z;
    double anti = 0.0;
    if (s == 0 && L.boundary == 0) {
        const int t2 = t + L.nt / 2 >= L.nt ? t + L.nt / 2 - L.nt : t + L.nt / 2;
        anti = cf(0, t2, t2).arr;  // ring 0 is ring-major: flat index t2
    }
    return row_from(L, cf.b, s, t, q.tm, cP, cTM, cTP, cSM, cSP, anti);
}

}  // namespace pmg
