// Hot kernels of the B200 multigrid solve path (sm_100a, FP64).
//
// Data layout: every per-node array is in the reference NodeIndexing order
// (polar_grid.hpp:17-37): the circle region ring-major (theta contiguous),
// the radial region spoke-major (r contiguous).  Each smoother line is
// therefore one contiguous HBM segment: a line is staged into shared memory
// with coalesced loads, solved on chip by a chunked affine scan (one chunk of
// K rows per thread, block-wide scan of the chunk carries) and written back
// once -- the forward/backward intermediates never touch HBM.
//
// All arrays carry a leading section dimension [B][...]; blockIdx.y is the
// section, and sections whose `active` flag is 0 (converged) are skipped.
#include <mutex>
#include <set>
#include <utility>

#include "pmg_kernels.h"

namespace pmg {

namespace {

constexpr unsigned FULL = 0xffffffffu;
// The across-origin ring is solved in the reference's exact substitution
// order (origin_solve_exact) in reference_order mode and for rings of at most
// this length; longer rings use the parallel 2x2-map scan (origin_solve).
#ifndef PMG_ORIGIN_SCAN_MIN
#define PMG_ORIGIN_SCAN_MIN 0
#endif

__device__ __forceinline__ int P(int i) { return i + (i >> 4); }  // bank-conflict padding
__host__ __device__ __forceinline__ int padded(int n) { return n + (n >> 4) + 1; }

template <bool ONFLY>
struct CF;
template <>
struct CF<false> {
    using T = CoefArrays;
};
template <>
struct CF<true> {
    using T = CoefOnTheFly;
};

// ------------------------------------------------------------- block scan
// Scan of affine chunk maps y_out = A*y_in + B[v] (v < NV, common A) over the
// threads of a block, in thread order (FWD) or reverse thread order.  Returns
// in yin the value entering each thread's chunk (composition of all earlier
// chunks applied to 0).
template <int NV, bool FWD>
__device__ __forceinline__ void block_scan(double A, double (&B)[NV], double (&yin)[NV],
                                           double* scr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double Ao = FWD ? __shfl_up_sync(FULL, A, d) : __shfl_down_sync(FULL, A, d);
        double Bo[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v)
            Bo[v] = FWD ? __shfl_up_sync(FULL, B[v], d) : __shfl_down_sync(FULL, B[v], d);
        if (FWD ? (lane >= d) : (lane + d < 32)) {
#pragma unroll
            for (int v = 0; v < NV; ++v) B[v] = A * Bo[v] + B[v];
            A = A * Ao;
        }
    }
    if (lane == (FWD ? 31 : 0)) {
        scr[warp * (NV + 1)] = A;
#pragma unroll
        for (int v = 0; v < NV; ++v) scr[warp * (NV + 1) + 1 + v] = B[v];
    }
    __syncthreads();
    if (warp == 0) {
        const int pos = lane;
        const int wi = FWD ? pos : nw - 1 - pos;
        double a = 1.0, bb[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) bb[v] = 0.0;
        if (pos < nw) {
            a = scr[wi * (NV + 1)];
#pragma unroll
            for (int v = 0; v < NV; ++v) bb[v] = scr[wi * (NV + 1) + 1 + v];
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double ao = __shfl_up_sync(FULL, a, d);
            double bo[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) bo[v] = __shfl_up_sync(FULL, bb[v], d);
            if (pos >= d) {
#pragma unroll
                for (int v = 0; v < NV; ++v) bb[v] = a * bo[v] + bb[v];
                a = a * ao;
            }
        }
        if (pos < nw) {
            scr[wi * (NV + 1)] = a;
#pragma unroll
            for (int v = 0; v < NV; ++v) scr[wi * (NV + 1) + 1 + v] = bb[v];
        }
    }
    __syncthreads();
    const int pw = FWD ? warp - 1 : warp + 1;
    double pB[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) pB[v] = (pw >= 0 && pw < nw) ? scr[pw * (NV + 1) + 1 + v] : 0.0;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const double full = A * pB[v] + B[v];
        const double prev =
            FWD ? __shfl_up_sync(FULL, full, 1) : __shfl_down_sync(FULL, full, 1);
        yin[v] = lane == (FWD ? 0 : 31) ? pB[v] : prev;
    }
    __syncthreads();
}

// ----------------------------------------------------------- line solve
// Solves L L^T x = y on one line held in shared memory (Y: rhs in, x out;
// IL = 1/l, M = m, padded indexing), reference line_algebra.cpp:42-62; with
// CYC the Sherman-Morrison cyclic correction of line_algebra.cpp:98-120
// (z = T^{-1}(e_1 + e_n) is carried as a second right-hand side through the
// same scans instead of being stored).  Thread tid owns rows [tid*K, tid*K+K).
template <int K, bool CYC>
__device__ __forceinline__ void line_solve(double* Y, const double* IL, const double* M, int n,
                                           double corner, double* scr) {
    constexpr int NV = CYC ? 2 : 1;
    const int j0 = threadIdx.x * K;
    double y[K], z[CYC ? K : 1];
    // forward: chunk composite of y_j = a_j y_{j-1} + b_j il_j, a_j = -m_{j-1} il_j
    double A = 1.0, Bv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) Bv[v] = 0.0;
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const int j = j0 + q;
        if (j < n) {
            const double il = IL[P(j)];
            const double a = j > 0 ? -(M[P(j - 1)] * il) : 0.0;
            const double b = Y[P(j)];
            y[q] = b;
            Bv[0] = a * Bv[0] + b * il;
            if (CYC) Bv[NV - 1] = a * Bv[NV - 1] + ((j == 0 || j == n - 1) ? il : 0.0);
            A = a * A;
        }
    }
    double yin[NV];
    block_scan<NV, true>(A, Bv, yin, scr);
    {
        double yp = yin[0], zp = yin[NV - 1];
#pragma unroll
        for (int q = 0; q < K; ++q) {
            const int j = j0 + q;
            if (j < n) {
                const double il = IL[P(j)];
                const double mp = j > 0 ? M[P(j - 1)] : 0.0;
                yp = (y[q] - mp * yp) * il;
                y[q] = yp;
                if (CYC) {
                    zp = (((j == 0 || j == n - 1) ? 1.0 : 0.0) - mp * zp) * il;
                    z[q] = zp;
                }
            }
        }
    }
    // backward: x_j = g_j x_{j+1} + y_j il_j, g_j = -m_j il_j
    double G = 1.0, Dv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) Dv[v] = 0.0;
#pragma unroll
    for (int q = K - 1; q >= 0; --q) {
        const int j = j0 + q;
        if (j < n) {
            const double il = IL[P(j)];
            const double g = j < n - 1 ? -(M[P(j)] * il) : 0.0;
            Dv[0] = g * Dv[0] + y[q] * il;
            if (CYC) Dv[NV - 1] = g * Dv[NV - 1] + z[CYC ? q : 0] * il;
            G = g * G;
        }
    }
    double xin[NV];
    block_scan<NV, false>(G, Dv, xin, scr);
    {
        double xp = xin[0], zp = xin[NV - 1];
#pragma unroll
        for (int q = K - 1; q >= 0; --q) {
            const int j = j0 + q;
            if (j < n) {
                const double il = IL[P(j)];
                const double mj = j < n - 1 ? M[P(j)] : 0.0;
                xp = (y[q] - mj * xp) * il;
                y[q] = xp;
                if (CYC) {
                    zp = (z[CYC ? q : 0] - mj * zp) * il;
                    z[CYC ? q : 0] = zp;
                }
            }
        }
    }
    if (CYC) {
        // tau = c (x_0 + x_{n-1}) / (1 + c (z_0 + z_{n-1}))
#pragma unroll
        for (int q = 0; q < K; ++q) {
            const int j = j0 + q;
            if (j == 0) {
                scr[0] = y[q];
                scr[1] = z[CYC ? q : 0];
            }
            if (j == n - 1) {
                scr[2] = y[q];
                scr[3] = z[CYC ? q : 0];
            }
        }
        __syncthreads();
        const double tau = corner * (scr[0] + scr[2]) / (1.0 + corner * (scr[1] + scr[3]));
#pragma unroll
        for (int q = 0; q < K; ++q) y[q] -= tau * z[CYC ? q : 0];
    }
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const int j = j0 + q;
        if (j < n) Y[P(j)] = y[q];
    }
    __syncthreads();
}

// Scan of affine maps on 2-vectors, v_out = M v_in + c (M 2x2 row-major),
// over the threads of a block in thread order (FWD) or reverse order; returns
// the state entering each thread's chunk (earlier maps applied to v = 0).
struct Map2 {
    double m00, m01, m10, m11, c0, c1;
};
__device__ __forceinline__ Map2 compose2(const Map2& l, const Map2& e) {  // l after e
    Map2 r;
    r.m00 = l.m00 * e.m00 + l.m01 * e.m10;
    r.m01 = l.m00 * e.m01 + l.m01 * e.m11;
    r.m10 = l.m10 * e.m00 + l.m11 * e.m10;
    r.m11 = l.m10 * e.m01 + l.m11 * e.m11;
    r.c0 = l.m00 * e.c0 + l.m01 * e.c1 + l.c0;
    r.c1 = l.m10 * e.c0 + l.m11 * e.c1 + l.c1;
    return r;
}
__device__ __forceinline__ Map2 shfl2(const Map2& a, int d, bool up) {
    Map2 r;
    r.m00 = up ? __shfl_up_sync(FULL, a.m00, d) : __shfl_down_sync(FULL, a.m00, d);
    r.m01 = up ? __shfl_up_sync(FULL, a.m01, d) : __shfl_down_sync(FULL, a.m01, d);
    r.m10 = up ? __shfl_up_sync(FULL, a.m10, d) : __shfl_down_sync(FULL, a.m10, d);
    r.m11 = up ? __shfl_up_sync(FULL, a.m11, d) : __shfl_down_sync(FULL, a.m11, d);
    r.c0 = up ? __shfl_up_sync(FULL, a.c0, d) : __shfl_down_sync(FULL, a.c0, d);
    r.c1 = up ? __shfl_up_sync(FULL, a.c1, d) : __shfl_down_sync(FULL, a.c1, d);
    return r;
}
template <bool FWD>
__device__ __forceinline__ void block_scan2(Map2 a, double& in0, double& in1, double* scr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const Map2 o = shfl2(a, d, FWD);
        if (FWD ? (lane >= d) : (lane + d < 32)) a = compose2(a, o);
    }
    Map2* ws = reinterpret_cast<Map2*>(scr);
    if (lane == (FWD ? 31 : 0)) ws[warp] = a;
    __syncthreads();
    if (warp == 0) {
        const int wi = FWD ? lane : nw - 1 - lane;
        Map2 w = {1.0, 0.0, 0.0, 1.0, 0.0, 0.0};
        if (lane < nw) w = ws[wi];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const Map2 o = shfl2(w, d, true);
            if (lane >= d) w = compose2(w, o);
        }
        if (lane < nw) ws[wi] = w;
    }
    __syncthreads();
    const int pw = FWD ? warp - 1 : warp + 1;
    double p0 = 0.0, p1 = 0.0;
    if (pw >= 0 && pw < nw) {
        p0 = ws[pw].c0;
        p1 = ws[pw].c1;
    }
    const double f0 = a.m00 * p0 + a.m01 * p1 + a.c0;
    const double f1 = a.m10 * p0 + a.m11 * p1 + a.c1;
    const double q0 = FWD ? __shfl_up_sync(FULL, f0, 1) : __shfl_down_sync(FULL, f0, 1);
    const double q1 = FWD ? __shfl_up_sync(FULL, f1, 1) : __shfl_down_sync(FULL, f1, 1);
    const bool first = lane == (FWD ? 0 : 31);
    in0 = first ? p0 : q0;
    in1 = first ? p1 : q1;
    __syncthreads();
}

__device__ __forceinline__ double block_sum(double v, double* scr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(FULL, v, d);
    if (lane == 0) scr[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += scr[w];
    __syncthreads();
    return t;
}

// Parallel solve of the across-origin ring with its envelope LDL^T factor in
// antipodally interleaved order (reference line_algebra.cpp:211-255,
// smoother.cpp:42-46): rows i < n-2 carry L(i,i-1), L(i,i-2) only, the two
// closing rows are dense.  Forward and backward substitutions of the band
// are 2nd-order linear recurrences, solved as chunked scans of 2x2 affine
// maps; the dense rows are block reductions.  X: padded smem workspace.
template <int K>
__device__ void origin_solve(double* Y, double* X, const OriginFactor& of, int b, int n,
                             double* scr) {
    const long o = (long)b * n;
    const double* b1 = of.band1 + o;
    const double* b2 = of.band2 + o;
    const double* r1 = of.row1 + o;
    const double* r2 = of.row2 + o;
    const double* D = of.D + o;
    const int h = n / 2, nb = n - 2, T = blockDim.x;
    const int j0 = threadIdx.x * K;
    for (int k = threadIdx.x; k < n; k += T) X[P(k)] = Y[P((k & 1) ? h + (k >> 1) : (k >> 1))];
    __syncthreads();
    // forward band: z_i = x_i - L(i,i-2) z_{i-2} - L(i,i-1) z_{i-1}; state (z_{i-1}, z_i)
    Map2 m = {1.0, 0.0, 0.0, 1.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const int i = j0 + q;
        if (i < nb) {
            const double l1 = i >= 1 ? b1[i] : 0.0, l2 = i >= 2 ? b2[i] : 0.0;
            const Map2 mi = {0.0, 1.0, -l2, -l1, 0.0, X[P(i)]};
            m = compose2(mi, m);
        }
    }
    double zm2, zm1;
    block_scan2<true>(m, zm2, zm1, scr);
    double s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const int i = j0 + q;
        if (i < nb) {
            double sum = X[P(i)];
            if (i >= 2) sum -= b2[i] * zm2;
            if (i >= 1) sum -= b1[i] * zm1;
            X[P(i)] = sum;
            zm2 = zm1;
            zm1 = sum;
            if (i >= of.fc1) s1 += r1[i] * sum;
            if (i >= of.fc2) s2 += r2[i] * sum;
        }
    }
    s1 = block_sum(s1, scr);
    s2 = block_sum(s2, scr + 32);
    if (threadIdx.x == 0) {  // dense closing rows, then their diagonal scaling
        const double zn2 = X[P(n - 2)] - s1;
        double zn1 = X[P(n - 1)] - s2;
        if (n - 2 >= of.fc2) zn1 -= r2[n - 2] * zn2;
        const double xn1 = zn1 / D[n - 1];
        double xn2 = zn2 / D[n - 2];
        if (n - 2 >= of.fc2) xn2 -= r2[n - 2] * xn1;
        X[P(n - 1)] = xn1;
        X[P(n - 2)] = xn2;
    }
    __syncthreads();
    const double xn1 = X[P(n - 1)], xn2 = X[P(n - 2)];
    // backward band: x_k = g_k - L(k+2,k) x_{k+2} - L(k+1,k) x_{k+1},
    // g_k = w_k - L(n-1,k) x_{n-1} - L(n-2,k) x_{n-2}; state (x_{k+1}, x_{k+2})
    Map2 g = {1.0, 0.0, 0.0, 1.0, 0.0, 0.0};
#pragma unroll
    for (int q = K - 1; q >= 0; --q) {
        const int k = j0 + q;
        if (k < nb) {
            double gk = X[P(k)] / D[k];
            if (k >= of.fc2) gk -= r2[k] * xn1;
            if (k >= of.fc1) gk -= r1[k] * xn2;
            X[P(k)] = gk;
            const double l1 = k + 1 < nb ? b1[k + 1] : 0.0;
            const double l2 = k + 2 < nb ? b2[k + 2] : 0.0;
            const Map2 mk = {-l1, -l2, 1.0, 0.0, gk, 0.0};
            g = compose2(mk, g);
        }
    }
    double xp1, xp2;
    block_scan2<false>(g, xp1, xp2, scr);
#pragma unroll
    for (int q = K - 1; q >= 0; --q) {
        const int k = j0 + q;
        if (k < nb) {
            double x = X[P(k)];
            if (k + 2 < nb) x -= b2[k + 2] * xp2;
            if (k + 1 < nb) x -= b1[k + 1] * xp1;
            X[P(k)] = x;
            xp2 = xp1;
            xp1 = x;
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < n; k += T) Y[P((k & 1) ? h + (k >> 1) : (k >> 1))] = X[P(k)];
    __syncthreads();
}

// Correctly rounded a / l given r = RN(1/l) (Markstein): q0 = RN(a r) is
// within 1 ulp, e = a - l q0 is exact (FMA), RN(q0 + e r) = RN(a / l).  The
// reciprocal is off the dependency chain, so a sequential substitution costs
// 3 dependent FP64 ops per division instead of a full IEEE division.
__device__ __forceinline__ double xdiv(double a, double l, double r) {
    const double q0 = a * r;
    const double e = fma(-l, q0, a);
    return fma(e, r, q0);
}

// Sequential L L^T solve in the reference's exact operation order
// (tridiag_solve, line_algebra.cpp:42-62) -- bitwise identical results.
// Run by ONE thread on shared memory; Ld holds the raw L diagonal.
__device__ void tri_solve_exact(double* Y, const double* Ld, const double* M, int n) {
    double l = Ld[P(0)];
    double y = xdiv(Y[P(0)], l, __drcp_rn(l));
    Y[P(0)] = y;
#pragma unroll 4
    for (int i = 1; i < n; ++i) {
        const double li = Ld[P(i)];
        const double ri = __drcp_rn(li);
        y = xdiv(Y[P(i)] - M[P(i - 1)] * y, li, ri);
        Y[P(i)] = y;
    }
    l = Ld[P(n - 1)];
    y = xdiv(y, l, __drcp_rn(l));
    Y[P(n - 1)] = y;
#pragma unroll 4
    for (int i = n - 2; i >= 0; --i) {
        const double li = Ld[P(i)];
        const double ri = __drcp_rn(li);
        y = xdiv(Y[P(i)] - M[P(i)] * y, li, ri);
        Y[P(i)] = y;
    }
}

// Cyclic (Sherman-Morrison) solve in the reference's exact order
// (cyclic_tridiag_solve, line_algebra.cpp:98-120).  z = T^{-1}(e_1 + e_n) is
// rhs-independent; it was computed at setup by the same exact sequence
// (k_circle_z), so reading it equals recomputing it bit for bit.
__device__ void cyc_solve_exact(double* Y, const double* Ld, const double* M, int n, double c,
                                const double* __restrict__ z, double* scr) {
    if (threadIdx.x == 0) {
        tri_solve_exact(Y, Ld, M, n);
        scr[0] = c * (Y[P(0)] + Y[P(n - 1)]) / (1.0 + c * (z[0] + z[n - 1]));
    }
    __syncthreads();
    const double tau = scr[0];
    for (int i = threadIdx.x; i < n; i += blockDim.x) Y[P(i)] -= tau * z[i];
    __syncthreads();
}

// Across-origin ring solve in the reference's exact operation order
// (line_algebra.cpp:211-255 with the interleaved permutation of
// smoother.cpp:42-46) -- bitwise identical to the reference.  Only the two
// true recurrence chains (band forward / band backward) run on one thread;
// the band factors are staged in shared memory, the diagonal scaling and the
// dense-row column updates of the backward substitution are per element and
// run on all threads (same per-element operation order as the reference).
// Y: rhs in NATURAL order (padded) in, solution out.
__device__ __forceinline__ int operm(int k, int h) { return (k & 1) ? h + (k >> 1) : (k >> 1); }

__device__ void origin_solve_exact(double* Y, double* B1, double* B2, const OriginFactor& of,
                                   int b, int n) {
    const long o = (long)b * n;
    const double* __restrict__ r1 = of.row1 + o;
    const double* __restrict__ r2 = of.row2 + o;
    const double* __restrict__ D = of.D + o;
    const int h = n / 2, nb = n - 2, T = blockDim.x;
    for (int i = threadIdx.x; i < n; i += T) {
        B1[P(i)] = of.band1[o + i];
        B2[P(i)] = of.band2[o + i];
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        // forward: band rows, with the two dense-row sums accumulated in the
        // reference's k order as the z_k become available.  Warp 0 runs the
        // chain redundantly on all lanes; for each group of 32 rows every lane
        // preloads its row's operands (rhs, band and dense-row coefficients)
        // into registers and the chain consumes them through shuffles, so no
        // memory access sits on the dependency chain.
        const int lane = threadIdx.x;
        const int fc1 = of.fc1, fc2 = of.fc2;
        double zm2 = 0.0, zm1 = 0.0;
        double s1 = Y[P(operm(n - 2, h))], s2 = Y[P(operm(n - 1, h))];
        for (int g = 0; g < nb; g += 32) {
            const int i_l = g + lane;
            const bool ok = i_l < nb;
            const double y_l = ok ? Y[P(operm(i_l, h))] : 0.0;
            const double b1_l = ok ? B1[P(i_l)] : 0.0, b2_l = ok ? B2[P(i_l)] : 0.0;
            const double a1_l = ok ? r1[i_l] : 0.0, a2_l = ok ? r2[i_l] : 0.0;
            const int cnt = nb - g < 32 ? nb - g : 32;
            double res = 0.0;
            for (int j = 0; j < cnt; ++j) {
                const int i = g + j;
                const double yv = __shfl_sync(FULL, y_l, j);
                const double l1 = __shfl_sync(FULL, b1_l, j), l2 = __shfl_sync(FULL, b2_l, j);
                const double a1 = __shfl_sync(FULL, a1_l, j), a2 = __shfl_sync(FULL, a2_l, j);
                double sum = yv;
                if (i >= 2) sum -= l2 * zm2;
                if (i >= 1) sum -= l1 * zm1;
                zm2 = zm1;
                zm1 = sum;
                if (i >= fc1) s1 -= a1 * sum;
                if (i >= fc2) s2 -= a2 * sum;
                if (lane == j) res = sum;
            }
            if (ok) Y[P(operm(i_l, h))] = res;
        }
        if (lane == 0) {
            if (n - 2 >= fc2) s2 -= r2[n - 2] * s1;
            Y[P(operm(n - 2, h))] = s1;
            Y[P(operm(n - 1, h))] = s2;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += T) Y[P(operm(i, h))] /= D[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        const double xn1 = Y[P(operm(n - 1, h))];
        if (n - 2 >= of.fc2) Y[P(operm(n - 2, h))] -= r2[n - 2] * xn1;
    }
    __syncthreads();
    {
        const double xn1 = Y[P(operm(n - 1, h))], xn2 = Y[P(operm(n - 2, h))];
        for (int k = threadIdx.x; k < nb; k += T) {
            double x = Y[P(operm(k, h))];
            if (k >= of.fc2) x -= r2[k] * xn1;
            if (k >= of.fc1) x -= r1[k] * xn2;
            Y[P(operm(k, h))] = x;
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        // band backward: row i updates x_{i-2} then x_{i-1}; x_k is final once
        // rows k+2 and k+1 have been applied.  Same register/shuffle scheme.
        const int lane = threadIdx.x;
        double xp1 = 0.0, xp2 = 0.0;  // x_{k+1}, x_{k+2}
        for (int g = nb - 1; g >= 0; g -= 32) {
            const int k_l = g - lane;  // lane j handles row g - j
            const bool ok = k_l >= 0;
            const double x_l = ok ? Y[P(operm(k_l, h))] : 0.0;
            const double c2_l = (ok && k_l + 2 < nb) ? B2[P(k_l + 2)] : 0.0;
            const double c1_l = (ok && k_l + 1 < nb) ? B1[P(k_l + 1)] : 0.0;
            const int cnt = g + 1 < 32 ? g + 1 : 32;
            double res = 0.0;
            for (int j = 0; j < cnt; ++j) {
                const int k = g - j;
                double x = __shfl_sync(FULL, x_l, j);
                const double l2 = __shfl_sync(FULL, c2_l, j), l1 = __shfl_sync(FULL, c1_l, j);
                if (k + 2 < nb) x -= l2 * xp2;
                if (k + 1 < nb) x -= l1 * xp1;
                xp2 = xp1;
                xp1 = x;
                if (lane == j) res = x;
            }
            if (ok) Y[P(operm(k_l, h))] = res;
        }
    }
    __syncthreads();
}

// Serial envelope solve of the across-origin ring (reference
// line_algebra.cpp:211-255 with permutation smoother.cpp:42-46); run by one
// thread on the shared-memory rhs.
__device__ void origin_solve_serial(double* Y, double* X, const OriginFactor& of, int b, int n) {
    const long o = (long)b * n;
    const double* b1 = of.band1 + o;
    const double* b2 = of.band2 + o;
    const double* r1 = of.row1 + o;
    const double* r2 = of.row2 + o;
    const double* D = of.D + o;
    const int h = n / 2;
    for (int k = 0; k < n; ++k) X[k] = Y[P((k & 1) ? h + (k >> 1) : (k >> 1))];
    for (int i = 0; i < n - 2; ++i) {
        double sum = X[i];
        if (i >= 2) sum -= b2[i] * X[i - 2];
        if (i >= 1) sum -= b1[i] * X[i - 1];
        X[i] = sum;
    }
    {
        double sum = X[n - 2];
        for (int k = of.fc1; k < n - 2; ++k) sum -= r1[k] * X[k];
        X[n - 2] = sum;
        sum = X[n - 1];
        for (int k = of.fc2; k < n - 1; ++k) sum -= r2[k] * X[k];
        X[n - 1] = sum;
    }
    for (int i = 0; i < n; ++i) X[i] /= D[i];
    {
        double xi = X[n - 1];
        for (int k = of.fc2; k < n - 1; ++k) X[k] -= r2[k] * xi;
        xi = X[n - 2];
        for (int k = of.fc1; k < n - 2; ++k) X[k] -= r1[k] * xi;
    }
    for (int i = n - 3; i >= 0; --i) {
        const double xi = X[i];
        if (i >= 2) X[i - 2] -= b2[i] * xi;
        if (i >= 1) X[i - 1] -= b1[i] * xi;
    }
    for (int k = 0; k < n; ++k) Y[P((k & 1) ? h + (k >> 1) : (k >> 1))] = X[k];
}

// ------------------------------------------------------------ apply / residual
// y = A u or r = f - A u with the Take/Give row of stencil.cpp:44-137 and the
// accumulation order of apply_take (stencil.cpp:166-171).
template <bool ONFLY, int MODE, bool NORM>
__global__ void __launch_bounds__(256) k_apply(LevelView L, const double* __restrict__ u,
                                               const double* __restrict__ f,
                                               double* __restrict__ out,
                                               double* __restrict__ partials, int norm_type,
                                               const int* __restrict__ active) {
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const long off = (long)b * L.n;
    const double* U = u + off;
    double val = 0.0;
    if (p < L.n) {
        int s, t;
        L.node(p, s, t);
        const CoefAt<ONFLY> cf{&L, off, b};
        const Nbr q = neighbours(L, s, t, p);
        const Row R = make_row_fast(L, cf, s, t, p, q);
        double acc;
        if (R.ident) {
            acc = 0.0;
            acc += 1.0 * U[p];
        } else {
            acc = 0.0;
            acc += R.d * U[p];
            if (R.has_sm) acc += R.sm * U[q.pSM];
            if (R.has_sp) acc += R.sp * U[q.pSP];
            acc += R.tm * U[q.pTM];
            acc += R.tp * U[q.pTP];
            if (R.has_sm) {
                acc += R.mm * U[q.pSMTM];
                acc += R.mp * U[q.pSMTP];
            }
            if (R.has_sp) {
                acc += R.pm * U[q.pSPTM];
                acc += R.pp * U[q.pSPTP];
            }
            if (R.origin) acc += R.ph * U[R.t2];
        }
        if (MODE == 0) {
            val = acc;
        } else {
            val = f[off + p] - acc;
        }
        out[off + p] = val;
    }
    if (NORM) {
        __shared__ double red[8];
        double v = norm_type == 2 ? fabs(val) : val * val;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const double o = __shfl_down_sync(FULL, v, d);
            v = norm_type == 2 ? fmax(v, o) : v + o;
        }
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double a = red[0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                a = norm_type == 2 ? fmax(a, red[w]) : a + red[w];
            partials[(long)b * gridDim.x + blockIdx.x] = a;
        }
    }
}

// ------------------------------------------------------------- circle sweep
// One block per circle line (ring s = parity + 2*blockIdx.x) of one section:
// rhs_t = f - sum_{off-line} A u (smoother.cpp:162-182), then the cyclic
// Sherman-Morrison solve (line_algebra.cpp:98-120), or the envelope solve of
// the across-origin ring 0 (smoother.cpp:144-152).
template <bool ONFLY, int K>
__global__ void __launch_bounds__(512) k_circle(LevelView L, double* __restrict__ u,
                                                const double* __restrict__ f,
                                                const double* __restrict__ cil,
                                                const double* __restrict__ cm,
                                                const double* __restrict__ corner,
                                                const double* __restrict__ cz,
                                                OriginFactor of, int parity, int serial,
                                                int exact_rings,
                                                const int* __restrict__ active) {
    extern __shared__ double smem[];
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int s = parity + 2 * blockIdx.x;
    const int nt = L.nt, T = blockDim.x;
    const long off = (long)b * L.n;
    double* U = u + off;
    const double* F = f + off;
    const int base = s * nt;
    if (L.dir(s)) {
        for (int t = threadIdx.x; t < nt; t += T) U[base + t] = F[base + t];
        return;
    }
    const int pn = padded(nt);
    double* Y = smem;
    double* IL = smem + pn;
    double* M = IL + pn;
    double* scr = M + pn;
    const CoefAt<ONFLY> cf{&L, off, b};
    for (int t = threadIdx.x; t < nt; t += T) {
        const int p = base + t;
        const Nbr q = neighbours(L, s, t, p);
        const Row R = make_row_fast(L, cf, s, t, p, q);
        double acc = F[p];
        if (R.has_sm) acc -= R.sm * U[q.pSM];
        if (R.has_sp) acc -= R.sp * U[q.pSP];
        if (R.has_sm) {
            acc -= R.mm * U[q.pSMTM];
            acc -= R.mp * U[q.pSMTP];
        }
        if (R.has_sp) {
            acc -= R.pm * U[q.pSPTM];
            acc -= R.pp * U[q.pSPTP];
        }
        Y[P(t)] = acc;
    }
    if (s == 0 && L.boundary == 0) {
        __syncthreads();
        if (serial || nt < PMG_ORIGIN_SCAN_MIN)
            origin_solve_exact(Y, IL, M, of, b, nt);
        else
            origin_solve<K>(Y, IL, of, b, nt, scr);
    } else {
        const long fo = (long)b * L.split * nt + (long)s * nt;
        const bool exact = serial || s <= exact_rings;  // block-uniform
        for (int t = threadIdx.x; t < nt; t += T) {
            IL[P(t)] = exact ? cil[fo + t] : __drcp_rn(cil[fo + t]);
            M[P(t)] = cm[fo + t];
        }
        __syncthreads();
        if (exact)
            cyc_solve_exact(Y, IL, M, nt, corner[(long)b * L.split + s], cz + fo, scr);
        else
            line_solve<K, true>(Y, IL, M, nt, corner[(long)b * L.split + s], scr);
    }
    for (int t = threadIdx.x; t < nt; t += T) U[base + t] = Y[P(t)];
}

// ------------------------------------------------------------- radial sweep
// One block per radial line (spoke t = parity + 2*blockIdx.x) of one section:
// rhs over rings split..n_r-1 (smoother.cpp:184-205) then the tridiagonal
// Cholesky solve (line_algebra.cpp:42-62); the Dirichlet row rides along as
// an identity row.
template <bool ONFLY, int K>
__global__ void __launch_bounds__(512) k_radial(LevelView L, double* __restrict__ u,
                                                const double* __restrict__ f,
                                                const double* __restrict__ ril,
                                                const double* __restrict__ rm, int parity,
                                                int serial, const int* __restrict__ active) {
    extern __shared__ double smem[];
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int t = parity + 2 * blockIdx.x;
    const int len = L.len, split = L.split, T = blockDim.x;
    const long off = (long)b * L.n;
    double* U = u + off;
    const double* F = f + off;
    const int base = split * L.nt + t * len;
    const int pn = padded(len);
    double* Y = smem;
    double* IL = smem + pn;
    double* M = IL + pn;
    double* scr = M + pn;
    const CoefAt<ONFLY> cf{&L, off, b};
    const long fo = ((long)b * L.nt + t) * len;
    for (int i = threadIdx.x; i < len; i += T) {
        const int s = split + i;
        const double lv = ril[fo + i];
        IL[P(i)] = serial ? lv : __drcp_rn(lv);
        M[P(i)] = rm[fo + i];
        const int p = base + i;
        if (L.dir(s)) {
            Y[P(i)] = F[p];
            continue;
        }
        const Nbr q = neighbours(L, s, t, p);
        const Row R = make_row_fast(L, cf, s, t, p, q);
        double acc = F[p];
        if (s == split && R.has_sm) acc -= R.sm * U[q.pSM];
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
        Y[P(i)] = acc;
    }
    __syncthreads();
    if (serial) {
        if (threadIdx.x == 0) tri_solve_exact(Y, IL, M, len);
        __syncthreads();
    } else {
        line_solve<K, false>(Y, IL, M, len, 0.0, scr);
    }
    for (int i = threadIdx.x; i < len; i += T) U[base + i] = Y[P(i)];
}

// ---------------------------------------------------------------- transfers
// restrict_transpose (interpolation.cpp:97-143) fused with
// mask_dirichlet_rows (multigrid.cpp:146-153) and the coarse u = 0 (:204).
__global__ void __launch_bounds__(256) k_restrict(LevelView F, LevelView C, Weights w,
                                                  const double* __restrict__ fr,
                                                  double* __restrict__ cf,
                                                  double* __restrict__ cu, int mask,
                                                  const int* __restrict__ active) {
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int pc = blockIdx.x * blockDim.x + threadIdx.x;
    if (pc >= C.n) return;
    int sc, tc;
    C.node(pc, sc, tc);
    const double* R = fr + (long)b * F.n;
    const int sf = 2 * sc, tf = 2 * tc;
    const int tdn = tf == 0 ? F.nt - 1 : tf - 1;
    const int tup = tf + 1;
    double acc = R[F.idx(sf, tf)];
    if (sf > 0) acc += w.rwa[sf - 1] * R[F.idx(sf - 1, tf)];
    if (sf < F.nr - 1) acc += w.rwb[sf + 1] * R[F.idx(sf + 1, tf)];
    acc += w.awa[tdn] * R[F.idx(sf, tdn)];
    acc += w.awb[tup] * R[F.idx(sf, tup)];
    if (sf > 0) {
        acc += w.rwa[sf - 1] * w.awa[tdn] * R[F.idx(sf - 1, tdn)];
        acc += w.rwa[sf - 1] * w.awb[tup] * R[F.idx(sf - 1, tup)];
    }
    if (sf < F.nr - 1) {
        acc += w.rwb[sf + 1] * w.awa[tdn] * R[F.idx(sf + 1, tdn)];
        acc += w.rwb[sf + 1] * w.awb[tup] * R[F.idx(sf + 1, tup)];
    }
    if (mask && C.dir(sc)) acc = 0.0;
    cf[(long)b * C.n + pc] = acc;
    if (cu) cu[(long)b * C.n + pc] = 0.0;
}

// prolongate(_add) (interpolation.cpp:38-95)
template <bool ADD>
__global__ void __launch_bounds__(256) k_prolong(LevelView F, LevelView C, Weights w,
                                                 const double* __restrict__ cu,
                                                 double* __restrict__ fu,
                                                 const int* __restrict__ active) {
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= F.n) return;
    int sf, tf;
    F.node(p, sf, tf);
    const double* X = cu + (long)b * C.n;
    const bool ro = sf & 1, so = tf & 1;
    const int sc = sf >> 1, tc = tf >> 1;
    const int tcu = tc + 1 == C.nt ? 0 : tc + 1;
    double v;
    if (!ro && !so) {
        v = X[C.idx(sc, tc)];
    } else if (ro && !so) {
        v = w.rwb[sf] * X[C.idx(sc, tc)] + w.rwa[sf] * X[C.idx(sc + 1, tc)];
    } else if (!ro && so) {
        v = w.awb[tf] * X[C.idx(sc, tc)] + w.awa[tf] * X[C.idx(sc, tcu)];
    } else {
        const double wb = w.rwb[sf], wa = w.rwa[sf], vb = w.awb[tf], va = w.awa[tf];
        v = wb * vb * X[C.idx(sc, tc)] + wb * va * X[C.idx(sc, tcu)] +
            wa * vb * X[C.idx(sc + 1, tc)] + wa * va * X[C.idx(sc + 1, tcu)];
    }
    double* Y = fu + (long)b * F.n;
    if (ADD)
        Y[p] += v;
    else
        Y[p] = v;
}

// coarsest-level direct solve: u = f; envelope LDL^T solve
// (multigrid.cpp:183-187, line_algebra.cpp:211-255), one thread per section.
__global__ void k_coarse(EnvFactor E, const double* __restrict__ f, double* __restrict__ u,
                         int B, const int* __restrict__ active) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B || (active && !active[b])) return;
    const int n = E.n;
    double* x = u + (long)b * n;
    const double* Lb = E.L + (long)b * E.nnz;
    const double* D = E.D + (long)b * n;
    for (int i = 0; i < n; ++i) x[i] = f[(long)b * n + i];
    for (int i = 0; i < n; ++i) {
        const int fi = E.fc[i];
        const double* ri = Lb + E.ro[i] - fi;
        double sum = x[i];
        for (int k = fi; k < i; ++k) sum -= ri[k] * x[k];
        x[i] = sum;
    }
    for (int i = 0; i < n; ++i) x[i] /= D[i];
    for (int i = n - 1; i >= 0; --i) {
        const int fi = E.fc[i];
        const double* ri = Lb + E.ro[i] - fi;
        const double xi = x[i];
        for (int k = fi; k < i; ++k) x[k] -= ri[k] * xi;
    }
}

// ------------------------------------------------------------------- norms
__global__ void __launch_bounds__(256) k_norm_partials(const double* __restrict__ v, long n,
                                                       int norm_type,
                                                       double* __restrict__ partials) {
    const int b = blockIdx.y;
    const double* V = v + (long)b * n;
    double a = 0.0;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long)gridDim.x * blockDim.x) {
        const double x = V[i];
        a = norm_type == 2 ? fmax(a, fabs(x)) : a + x * x;
    }
    __shared__ double red[8];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const double o = __shfl_down_sync(FULL, a, d);
        a = norm_type == 2 ? fmax(a, o) : a + o;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = red[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            s = norm_type == 2 ? fmax(s, red[w]) : s + red[w];
        partials[(long)b * gridDim.x + blockIdx.x] = s;
    }
}

// compute_norm (multigrid.cpp:48-59) from block partials; one block per section
__global__ void __launch_bounds__(256) k_norm_final(const double* __restrict__ partials,
                                                    int nblk, long n, int norm_type,
                                                    double* __restrict__ norms) {
    const int b = blockIdx.x;
    double a = 0.0;
    for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
        const double x = partials[(long)b * nblk + i];
        a = norm_type == 2 ? fmax(a, x) : a + x;
    }
    __shared__ double red[8];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const double o = __shfl_down_sync(FULL, a, d);
        a = norm_type == 2 ? fmax(a, o) : a + o;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = red[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            s = norm_type == 2 ? fmax(s, red[w]) : s + red[w];
        if (norm_type == 0)
            s = sqrt(s / (double)n);
        else if (norm_type == 1)
            s = sqrt(s);
        norms[b] = s;
    }
}

// convergence test of MultigridSolver::solve (multigrid.cpp:321-340)
__global__ void k_check(const double* __restrict__ norms, ConvState cs, int B, int max_it,
                        double rel_tol, double abs_tol) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B || !cs.active[b]) return;
    const int it = cs.count[b]++;  // residual norms taken so far = iteration index
    const double r = norms[b];
    if (it < cs.cap) cs.hist[(long)b * cs.cap + it] = r;
    bool conv;
    if (it == 0) {
        cs.r0[b] = r;
        conv = r == 0.0 || (abs_tol > 0.0 && r <= abs_tol);
    } else {
        conv = (abs_tol > 0.0 && r <= abs_tol) || (rel_tol > 0.0 && r <= rel_tol * cs.r0[b]);
    }
    cs.iters[b] = it;
    if (conv) cs.converged[b] = 1;
    if (conv || it >= max_it) {
        cs.active[b] = 0;
        atomicSub(cs.remaining, 1);
    }
}

__global__ void k_fill(double* p, long n, double v) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void k_set_active(int* active, int* count, int* conv, int* remaining, int B) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) {
        active[b] = 1;
        count[b] = 0;
        conv[b] = 0;
    }
    if (b == 0) *remaining = B;
}

__global__ void k_flush(double* p, long n) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long)gridDim.x * blockDim.x)
        p[i] = p[i] * 0.5 + 1.0;
}

// ------------------------------------------------------------ launch helpers
// Opt a kernel into the full 227 KB of dynamic shared memory once per
// (kernel, device); launches then pass their exact size.
template <class KernelT>
void set_smem(KernelT kern, size_t bytes) {
    (void)bytes;
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_pair(reinterpret_cast<const void*>(kern), dev);
    std::lock_guard<std::mutex> lock(mu);
    if (done.count(key)) return;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    done.insert(key);
}

// chunk size K and threads T for a line of n rows: T = 32*ceil(ceil(n/K)/32) <= 512
inline void line_shape(int n, int& K, int& T) {
    static const int ks[4] = {2, 4, 8, 16};
    K = 16;
    for (int q = 0; q < 4; ++q)
        if ((n + ks[q] - 1) / ks[q] <= 256 || ks[q] == 16) {
            K = ks[q];
            break;
        }
    const int chunks = (n + K - 1) / K;
    T = ((chunks + 31) / 32) * 32;
    if (T < 32) T = 32;
}

inline size_t line_smem(int n) { return (size_t)(3 * padded(n) + 32 * 6 + 16) * sizeof(double); }

}  // namespace

int apply_blocks(const LevelView& L) { return (L.n + 255) / 256; }

int launch_apply(const LevelView& L, bool onfly, int mode, const double* u, const double* f,
                 double* out, double* partials, int norm_type, const int* active,
                 cudaStream_t st) {
    const int nb = apply_blocks(L);
    dim3 grid(nb, L.B);
    const bool norm = partials != nullptr;
#define PMG_APPLY(ON, MO, NO) \
    k_apply<ON, MO, NO><<<grid, 256, 0, st>>>(L, u, f, out, partials, norm_type, active)
    if (onfly) {
        if (mode == 0) {
            if (norm) PMG_APPLY(true, 0, true); else PMG_APPLY(true, 0, false);
        } else {
            if (norm) PMG_APPLY(true, 1, true); else PMG_APPLY(true, 1, false);
        }
    } else {
        if (mode == 0) {
            if (norm) PMG_APPLY(false, 0, true); else PMG_APPLY(false, 0, false);
        } else {
            if (norm) PMG_APPLY(false, 1, true); else PMG_APPLY(false, 1, false);
        }
    }
#undef PMG_APPLY
    return nb;
}

template <bool ON, int K>
static void circle_k(const LevelView& L, double* u, const double* f, const double* cil,
                     const double* cm, const double* corner, const double* cz,
                     const OriginFactor& of, int parity, bool serial, int exact_rings,
                     const int* active, cudaStream_t st, int T, int lines) {
    const size_t sm = line_smem(L.nt);
    set_smem(k_circle<ON, K>, sm);
    k_circle<ON, K><<<dim3(lines, L.B), T, sm, st>>>(L, u, f, cil, cm, corner, cz, of, parity,
                                                      serial ? 1 : 0, exact_rings, active);
}

void launch_circle(const LevelView& L, bool onfly, double* u, const double* f, const double* cil,
                   const double* cm, const double* corner, const double* cz,
                   const OriginFactor& of, int parity, bool serial, int exact_rings,
                   const int* active, cudaStream_t st) {
    const int lines = L.split > parity ? (L.split - parity + 1) / 2 : 0;
    if (lines == 0) return;
    int K, T;
    line_shape(L.nt, K, T);
#define PMG_C(KK)                                                                            \
    (onfly ? circle_k<true, KK>(L, u, f, cil, cm, corner, cz, of, parity, serial, exact_rings, \
                                active, st, T, lines)                                      \
           : circle_k<false, KK>(L, u, f, cil, cm, corner, cz, of, parity, serial, exact_rings, \
                                 active, st, T, lines))
    switch (K) {
        case 2: PMG_C(2); break;
        case 4: PMG_C(4); break;
        case 8: PMG_C(8); break;
        default: PMG_C(16); break;
    }
#undef PMG_C
}

template <bool ON, int K>
static void radial_k(const LevelView& L, double* u, const double* f, const double* ril,
                     const double* rm, int parity, bool serial, const int* active,
                     cudaStream_t st, int T, int lines) {
    const size_t sm = line_smem(L.len);
    set_smem(k_radial<ON, K>, sm);
    k_radial<ON, K><<<dim3(lines, L.B), T, sm, st>>>(L, u, f, ril, rm, parity, serial ? 1 : 0,
                                                      active);
}

void launch_radial(const LevelView& L, bool onfly, double* u, const double* f, const double* ril,
                   const double* rm, int parity, bool serial, const int* active,
                   cudaStream_t st) {
    if (L.len <= 0) return;
    const int lines = (L.nt - parity + 1) / 2;
    int K, T;
    line_shape(L.len, K, T);
#define PMG_R(KK)                                                                       \
    (onfly ? radial_k<true, KK>(L, u, f, ril, rm, parity, serial, active, st, T, lines) \
           : radial_k<false, KK>(L, u, f, ril, rm, parity, serial, active, st, T, lines))
    switch (K) {
        case 2: PMG_R(2); break;
        case 4: PMG_R(4); break;
        case 8: PMG_R(8); break;
        default: PMG_R(16); break;
    }
#undef PMG_R
}

void launch_restrict(const LevelView& F, const LevelView& C, const Weights& w, const double* fr,
                     double* cf, double* cu_zero, bool mask, const int* active, cudaStream_t st) {
    k_restrict<<<dim3((C.n + 255) / 256, C.B), 256, 0, st>>>(F, C, w, fr, cf, cu_zero, mask ? 1 : 0,
                                                             active);
}

void launch_prolong(const LevelView& F, const LevelView& C, const Weights& w, const double* cu,
                    double* fu, bool add, const int* active, cudaStream_t st) {
    dim3 grid((F.n + 255) / 256, F.B);
    if (add)
        k_prolong<true><<<grid, 256, 0, st>>>(F, C, w, cu, fu, active);
    else
        k_prolong<false><<<grid, 256, 0, st>>>(F, C, w, cu, fu, active);
}

void launch_coarse(const LevelView& L, const EnvFactor& E, const double* f, double* u,
                   const int* active, cudaStream_t st) {
    k_coarse<<<(L.B + 63) / 64, 64, 0, st>>>(E, f, u, L.B, active);
}

int launch_norm_partials(const double* v, long n, int B, int norm_type, double* partials,
                         cudaStream_t st) {
    long nb = (n + 255) / 256;
    if (nb > 1024) nb = 1024;
    k_norm_partials<<<dim3((int)nb, B), 256, 0, st>>>(v, n, norm_type, partials);
    return (int)nb;
}

void launch_norm_final(const double* partials, int nblk, int B, long n, int norm_type,
                       double* norms, cudaStream_t st) {
    k_norm_final<<<B, 256, 0, st>>>(partials, nblk, n, norm_type, norms);
}

void launch_check(const double* norms, ConvState cs, int B, int max_it, double rel_tol,
                  double abs_tol, cudaStream_t st) {
    k_check<<<(B + 127) / 128, 128, 0, st>>>(norms, cs, B, max_it, rel_tol, abs_tol);
}

void launch_fill(double* p, long n, double v, cudaStream_t st) {
    long nb = (n + 255) / 256;
    if (nb > 4096) nb = 4096;
    if (nb < 1) nb = 1;
    k_fill<<<(int)nb, 256, 0, st>>>(p, n, v);
}

void launch_set_active(int* active, int* count, int* conv, int* remaining, int B,
                       cudaStream_t st) {
    k_set_active<<<(B + 127) / 128, 128, 0, st>>>(active, count, conv, remaining, B);
}

void launch_flush(double* buf, long n, cudaStream_t st) {
    k_flush<<<148 * 8, 256, 0, st>>>(buf, n);
}

}  // namespace pmg
