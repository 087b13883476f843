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
#include <atomic>
#include <cooperative_groups.h>
#include <cuda_pipeline.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

#include "pmg_kernels.h"
#include "pmg_lines.cuh"

namespace pmg {

namespace cg = cooperative_groups;

// unroll of the single-CTA radial rhs gather (rows whose loads are in flight together)
#ifndef PMG_RAD_UNROLL
#define PMG_RAD_UNROLL 2
#endif
constexpr int kRadUnroll = PMG_RAD_UNROLL;

#ifdef PMG_KTRACE
// diagnostics build only: clock64 marks of thread 0 of block (0,0)
__device__ unsigned long long g_ktrace[32];
#define KT(i)                                                       \
    do {                                                            \
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) \
            g_ktrace[i] = clock64();                                \
    } while (0)
#define KTS(slot, i)                                                \
    do {                                                            \
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && (slot) >= 0) \
            g_ktrace[16 + 5 * (slot) + (i)] = clock64();            \
    } while (0)
// a value (e.g. a wave count) of thread 0 of block (0,0)
#define KTV(i, v)                                                   \
    do {                                                            \
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) \
            g_ktrace[i] = (v);                                      \
    } while (0)
#else
#define KTV(i, v) \
    do {          \
    } while (0)
#define KT(i) \
    do {      \
    } while (0)
#define KTS(slot, i) \
    do {             \
    } while (0)
#endif

namespace {

// The across-origin ring is solved in the reference's exact substitution
// order (origin_solve_exact) in reference_order mode and for rings of at most
// this length; longer rings use the parallel 2x2-map scan (origin_solve).
// minimum resident CTAs of the cluster line kernels (register cap 64/thread at 4)
#ifndef PMG_CL_MINB
#define PMG_CL_MINB 4
#endif
// fused smoothing step: resident CTAs per SM (registers <= 65536 / (256 * MINB));
// measured: 2 (128 regs) c1 5.71 ms, 3 (80 regs) 5.42 ms, 4 (64 regs, spills) 5.52 ms;
// line_shape never picks more than 256 threads
// single-CTA line kernels with K <= 8 rows per thread run at most 256 threads
// (line_shape); K = 16 (reference-order solves of 8192-node lines) up to 512
#ifndef PMG_LINE_MINB
#define PMG_LINE_MINB 3
#endif
#ifndef PMG_FUSED_MINB
#define PMG_FUSED_MINB 3
#endif
// rows per solving thread of the exact-order parallel line solves
#ifndef PMG_EX_CHUNK
#define PMG_EX_CHUNK 16
#endif
constexpr int kExChunk = PMG_EX_CHUNK;
#ifndef PMG_ORIGIN_SCAN_MIN
#define PMG_ORIGIN_SCAN_MIN 0
#endif

// ------------------------------------------------ mbarrier + bulk copies (TMA engine)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n\t"
                 "fence.proxy.async.shared::cta;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// bulk global -> shared copy (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// loads of u inside a launch whose other CTAs write u (fused smoothing) go
// through L2 (ld.global.cg): L1 is not coherent across SMs
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
    KT(6);
    // the thread's factor entries are loaded up front (independent loads in
    // flight together), not inside the sequential compose chains
    double b1v[K + 1], b2v[K + 2];
#pragma unroll
    for (int q = 0; q < K + 2; ++q) {
        const int i = j0 + q;
        if (q < K + 1) b1v[q] = (i >= 1 && i < nb) ? b1[i] : 0.0;
        b2v[q] = (i >= 2 && i < nb) ? b2[i] : 0.0;
    }
    // forward band: z_i = x_i - L(i,i-2) z_{i-2} - L(i,i-1) z_{i-1}; state (z_{i-1}, z_i)
    Map2 m = {1.0, 0.0, 0.0, 1.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const int i = j0 + q;
        if (i < nb) {
            const Map2 mi = {0.0, 1.0, -b2v[q], -b1v[q], 0.0, X[P(i)]};
            m = compose2(mi, m);
        }
    }
    double zm2, zm1;
    KT(7);
    block_scan2<true>(m, zm2, zm1, scr);
    KT(8);
    double r1v[K], r2v[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const int i = j0 + q;
        r1v[q] = (i < nb && i >= of.fc1) ? r1[i] : 0.0;
        r2v[q] = (i < nb && i >= of.fc2) ? r2[i] : 0.0;
    }
    double s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const int i = j0 + q;
        if (i < nb) {
            double sum = X[P(i)];
            if (i >= 2) sum -= b2v[q] * zm2;
            if (i >= 1) sum -= b1v[q] * zm1;
            X[P(i)] = sum;
            zm2 = zm1;
            zm1 = sum;
            if (i >= of.fc1) s1 += r1v[q] * sum;
            if (i >= of.fc2) s2 += r2v[q] * sum;
        }
    }
    KT(9);
    s1 = block_sum(s1, scr);
    s2 = block_sum(s2, scr + 32);
    KT(10);
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
    KT(11);
    const double xn1 = X[P(n - 1)], xn2 = X[P(n - 2)];
    // backward band: x_k = g_k - L(k+2,k) x_{k+2} - L(k+1,k) x_{k+1},
    // g_k = w_k - L(n-1,k) x_{n-1} - L(n-2,k) x_{n-2}; state (x_{k+1}, x_{k+2})
    double dv[K];
#pragma unroll
    for (int q = 0; q < K; ++q) dv[q] = j0 + q < nb ? D[j0 + q] : 1.0;
    Map2 g = {1.0, 0.0, 0.0, 1.0, 0.0, 0.0};
#pragma unroll
    for (int q = K - 1; q >= 0; --q) {
        const int k = j0 + q;
        if (k < nb) {
            double gk = X[P(k)] / dv[q];
            if (k >= of.fc2) gk -= r2v[q] * xn1;
            if (k >= of.fc1) gk -= r1v[q] * xn2;
            X[P(k)] = gk;
            const double l1 = k + 1 < nb ? b1v[q + 1] : 0.0;
            const double l2 = k + 2 < nb ? b2v[q + 2] : 0.0;
            const Map2 mk = {-l1, -l2, 1.0, 0.0, gk, 0.0};
            g = compose2(mk, g);
        }
    }
    double xp1, xp2;
    KT(12);
    block_scan2<false>(g, xp1, xp2, scr);
    KT(13);
#pragma unroll
    for (int q = K - 1; q >= 0; --q) {
        const int k = j0 + q;
        if (k < nb) {
            double x = X[P(k)];
            if (k + 2 < nb) x -= b2v[q + 2] * xp2;
            if (k + 1 < nb) x -= b1v[q + 1] * xp1;
            X[P(k)] = x;
            xp2 = xp1;
            xp1 = x;
        }
    }
    __syncthreads();
    KT(14);
    for (int k = threadIdx.x; k < n; k += T) Y[P((k & 1) ? h + (k >> 1) : (k >> 1))] = X[P(k)];
    __syncthreads();
    KT(15);
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

// ------------------------------------------------ exact-order parallel solve
// Bitwise the reference's sequential substitution (tridiag_solve,
// line_algebra.cpp:42-62, and the Sherman-Morrison step of
// cyclic_tridiag_solve, :98-120), computed by all threads of the block:
//  1. the chunked affine scan of the fast path gives approximate values of
//     the iterate at every chunk boundary (a few ulps off);
//  2. every thread restarts the reference recurrence (its operation order,
//     division correctly rounded by Markstein's correction) one chunk early
//     from that approximation and runs it through its own chunk.  The
//     recurrences contract (|m/l| < 1), so after a few rows the rounding
//     makes the restarted trajectory coincide bit for bit with the
//     reference's;
//  3. a chunk whose trajectory at its predecessor's last row differs from the
//     predecessor's result is recomputed from that result, in waves, until
//     every chunk starts from its predecessor's end bit for bit.  The result
//     then IS the sequential substitution (induction from row 0), and every
//     wave settles at least the first inconsistent chunk, so it terminates.
// Y: rhs in / solution out, Ld: raw L diagonal, RC: RN(1/l), M: sub-diagonal
// (padded shared-memory rows); z: the Sherman-Morrison vector z = T^{-1}(e_1
// + e_n), computed at setup by the same exact sequence (k_circle_z).
// scr: >= 64 + 3*blockDim.x doubles (line_smem(n, true) reserves 64 + 6*512).
// forward row j of L y = b (tridiag_solve's first loop), v = y_{j-1}.
// Branch-free (selects, clamped indices): the rows of a chunk unroll into
// straight-line code whose shared-memory loads the scheduler hoists ahead of
// the dependent DMUL-DADD-DMUL-DFMA-DFMA chain.
// RCF: RN(1/l) evaluated on the fly (lines whose four arrays do not fit one
// CTA's shared memory keep three); it is off the dependency chain either way
template <bool RCF>
__device__ __forceinline__ double rc_at(const double* Ld, const double* RC, int j) {
    return RCF ? __drcp_rn(Ld[P(j)]) : RC[P(j)];
}
template <bool RCF = false>
__device__ __forceinline__ double ex_fwd(const double* Y, const double* Ld, const double* RC,
                                         const double* M, int j, double v) {
    const double b = Y[P(j)];
    const double m = M[P(j > 0 ? j - 1 : 0)];
    const double a = b - m * v;
    return xdiv(j == 0 ? b : a, Ld[P(j)], rc_at<RCF>(Ld, RC, j));
}
// backward row j of L^T x = y, v = x_{j+1}; yj = y_j
template <bool RCF = false>
__device__ __forceinline__ double ex_bwd(double yj, const double* Ld, const double* RC,
                                         const double* M, int n, int j, double v) {
    const double a = yj - M[P(j)] * v;
    return xdiv(j == n - 1 ? yj : a, Ld[P(j)], rc_at<RCF>(Ld, RC, j));
}

// KS rows per solving thread (independent of the kernel's chunk K: threads
// t >= ceil(n/KS) idle in the solve); warm-up = one chunk.  Each wave costs
// one barrier: the chunk results are double-buffered.
template <int KS, bool CYC, bool RCF = false>
__device__ __forceinline__ void line_solve_ex(double* Y, const double* Ld, const double* RC,
                                              const double* M, int n, double corner,
                                              const double* __restrict__ z, double* scr) {
    const int t = threadIdx.x, T = blockDim.x, j0 = t * KS;
    double* Sa = scr + 64;  // approximate chunk-entry values
    double* Se = Sa + T;    // chunk results at the chunk's far end, two buffers of T
    const bool live = j0 < n;
    double y[KS];
    int waves = 0;
    // ---- forward: y_j = (b_j - m_{j-1} y_{j-1}) / l_j  (b in Y)
    {
        double A = 1.0, Bv[1] = {0.0};
#pragma unroll
        for (int q = 0; q < KS; ++q) {
            const int j = j0 + q;
            if (j < n) {
                const double il = rc_at<RCF>(Ld, RC, j);
                const double a = j > 0 ? -(M[P(j - 1)] * il) : 0.0;
                Bv[0] = a * Bv[0] + Y[P(j)] * il;
                A = a * A;
            }
        }
        double yin[1];
        block_scan<1, true>(A, Bv, yin, scr);
        Sa[t] = yin[0];
        __syncthreads();
        double st = 0.0;  // this trajectory's value at row j0 - 1
        if (live && t >= 1) {
            double v = t >= 2 ? Sa[t - 1] : 0.0;  // thread 1 restarts at row 0: exact
#pragma unroll
            for (int q = 0; q < KS; ++q) v = ex_fwd<RCF>(Y, Ld, RC, M, j0 - KS + q, v);
            st = v;
        }
        // rows past n (last chunk) recompute row n-1 and are never stored;
        // the chunk's far-end value is then y_{n-1} (read by no one)
        auto chunk = [&](double v) {
#pragma unroll
            for (int q = 0; q < KS; ++q) {
                const int j = min(j0 + q, n - 1);
                const double w = ex_fwd<RCF>(Y, Ld, RC, M, j, v);
                v = j0 + q < n ? w : v;
                y[q] = v;
            }
            return v;
        };
        double e = live ? chunk(st) : 0.0;
        Se[t] = e;
        __syncthreads();
        for (int cur = 0;; cur ^= 1) {
            const double pe = t >= 1 ? Se[cur * T + t - 1] : 0.0;
            const bool bad = live && t >= 1 && !same_bits(st, pe);
            if (bad) {
                st = pe;
                e = chunk(st);
            }
            Se[(cur ^ 1) * T + t] = e;
            if (!__syncthreads_or(bad)) break;
            ++waves;
        }
    }
    // every read of b is behind the last barrier: Y now takes y
#pragma unroll
    for (int q = 0; q < KS; ++q)
        if (j0 + q < n) Y[P(j0 + q)] = y[q];
    // ---- backward: x_j = (y_j - m_j x_{j+1}) / l_j  (y in Y and in y[])
    {
        double G = 1.0, Dv[1] = {0.0};
#pragma unroll
        for (int q = KS - 1; q >= 0; --q) {
            const int j = j0 + q;
            if (j < n) {
                const double il = rc_at<RCF>(Ld, RC, j);
                const double g = j < n - 1 ? -(M[P(j)] * il) : 0.0;
                Dv[0] = g * Dv[0] + y[q] * il;
                G = g * G;
            }
        }
        double xin[1];
        block_scan<1, false>(G, Dv, xin, scr);  // its barriers publish Y
        Sa[t] = xin[0];
        __syncthreads();
        const bool succ = j0 + KS < n;  // a chunk follows (its rows are solved first)
        double st = 0.0;                // this trajectory's value at row j0 + KS
        if (live && succ) {
            // restart one chunk late from the approximate value at row j0+2KS;
            // if the next chunk is the last, its top row n-1 starts exactly
            double v = j0 + 2 * KS < n ? Sa[t + 1] : 0.0;
#pragma unroll
            for (int q = KS - 1; q >= 0; --q) {
                const int j = min(j0 + KS + q, n - 1);
                const double w = ex_bwd<RCF>(Y[P(j)], Ld, RC, M, n, j, v);
                v = j0 + KS + q < n ? w : v;
            }
            st = v;
        }
        // y_j is re-read from Y (one register array per thread)
        auto chunk = [&](double v) {
#pragma unroll
            for (int q = KS - 1; q >= 0; --q) {
                const int j = min(j0 + q, n - 1);
                const double w = ex_bwd<RCF>(Y[P(j)], Ld, RC, M, n, j, v);
                v = j0 + q < n ? w : v;
                y[q] = v;
            }
            return v;
        };
        double e = live ? chunk(st) : 0.0;
        Se[t] = e;
        __syncthreads();
        for (int cur = 0;; cur ^= 1) {
            const double pe = t + 1 < T ? Se[cur * T + t + 1] : 0.0;
            const bool bad = live && succ && !same_bits(st, pe);
            if (bad) {
                st = pe;
                e = chunk(st);
            }
            Se[(cur ^ 1) * T + t] = e;
            if (!__syncthreads_or(bad)) break;
            waves += 1000;
        }
    }
    KTV(30, waves);
    if (CYC) {
        // tau = c (x_0 + x_{n-1}) / (1 + c (z_0 + z_{n-1})); x -= tau z
#pragma unroll
        for (int q = 0; q < KS; ++q) {
            if (j0 + q == 0) scr[0] = y[q];
            if (j0 + q == n - 1) scr[2] = y[q];
        }
        __syncthreads();
        const double tau = corner * (scr[0] + scr[2]) / (1.0 + corner * (z[0] + z[n - 1]));
#pragma unroll
        for (int q = 0; q < KS; ++q)
            if (j0 + q < n) y[q] -= tau * z[j0 + q];
    }
    __syncthreads();  // every thread's reads of Y (and of scr) are done
#pragma unroll
    for (int q = 0; q < KS; ++q)
        if (j0 + q < n) Y[P(j0 + q)] = y[q];
    __syncthreads();
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
            double res = 0.0;
            // fully unrolled, branch-free (selects): the shuffles issue ahead of
            // the chain, which is one DMUL + DADD per row on zm1
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int i = g + j;
                const double yv = __shfl_sync(FULL, y_l, j);
                const double l1 = __shfl_sync(FULL, b1_l, j), l2 = __shfl_sync(FULL, b2_l, j);
                const double a1 = __shfl_sync(FULL, a1_l, j), a2 = __shfl_sync(FULL, a2_l, j);
                const double u2 = yv - l2 * zm2;
                const double sa = i >= 2 ? u2 : yv;
                const double u1 = sa - l1 * zm1;
                const double sum = i >= 1 ? u1 : sa;
                const bool valid = i < nb;
                zm2 = valid ? zm1 : zm2;
                zm1 = valid ? sum : zm1;
                const double t1 = s1 - a1 * sum, t2 = s2 - a2 * sum;
                s1 = (valid && i >= fc1) ? t1 : s1;
                s2 = (valid && i >= fc2) ? t2 : s2;
                res = lane == j ? sum : res;
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
            double res = 0.0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int k = g - j;
                const double xv = __shfl_sync(FULL, x_l, j);
                const double l2 = __shfl_sync(FULL, c2_l, j), l1 = __shfl_sync(FULL, c1_l, j);
                const double u2 = xv - l2 * xp2;
                const double sa = k + 2 < nb ? u2 : xv;
                const double u1 = sa - l1 * xp1;
                const double x = k + 1 < nb ? u1 : sa;
                const bool valid = k >= 0;
                xp2 = valid ? xp1 : xp2;
                xp1 = valid ? x : xp1;
                res = lane == j ? x : res;
            }
            if (ok) Y[P(operm(k_l, h))] = res;
        }
    }
    __syncthreads();
}

// Across-origin ring in the reference's exact order (line_algebra.cpp:211-255,
// permutation smoother.cpp:42-46), latency-optimised: the two band
// recurrences run on ONE thread with the operands of the next four rows
// loaded from shared memory while the current four are computed (the
// critical path is one DMUL + DADD per row); the dense closing rows'
// products are formed in parallel and their two sequential sums (the
// reference's k order) run on two warps; the diagonal scaling and the dense
// rows' column updates are per element.  Y: rhs in NATURAL order (padded) in,
// solution out; B1, B2, Q: padded workspaces (n).
__device__ void origin_solve_seq(double* Y, double* B1, double* B2, double* X,
                                 const OriginFactor& of, int b, int n) {
    const long o = (long)b * n;
    const double* __restrict__ r1 = of.row1 + o;
    const double* __restrict__ r2 = of.row2 + o;
    const double* __restrict__ D = of.D + o;
    const int h = n / 2, nb = n - 2, T = blockDim.x, t = threadIdx.x;
    // X: the rhs in the factor's (interleaved) order; B1, B2: the band
    for (int i = t; i < n; i += T) {
        X[P(i)] = Y[P(operm(i, h))];
        B1[P(i)] = of.band1[o + i];
        B2[P(i)] = of.band2[o + i];
    }
    __syncthreads();
    KT(6);
    if (t == 0) {  // forward band: z_i = (x_i - L(i,i-2) z_{i-2}) - L(i,i-1) z_{i-1}
        // rows 0, 1 (no L(i,i-2); row 0 no L(i,i-1)) peeled: the main loop is
        // straight-line, the next group's operands loaded before this group's
        // chain (critical path DMUL + DADD per row)
        double zm2 = X[P(0)];
        double zm1 = X[P(1)] - B1[P(1)] * zm2;
        X[P(1)] = zm1;
        int i = 2;
        if (i + 4 <= nb) {
            double xa[4], l1a[4], l2a[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                xa[q] = X[P(i + q)];
                l1a[q] = B1[P(i + q)];
                l2a[q] = B2[P(i + q)];
            }
            for (; i + 4 <= nb; i += 4) {
                double xb[4], l1b[4], l2b[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int k = min(i + 4 + q, nb - 1);
                    xb[q] = X[P(k)];
                    l1b[q] = B1[P(k)];
                    l2b[q] = B2[P(k)];
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double z = (xa[q] - l2a[q] * zm2) - l1a[q] * zm1;
                    X[P(i + q)] = z;
                    zm2 = zm1;
                    zm1 = z;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    xa[q] = xb[q];
                    l1a[q] = l1b[q];
                    l2a[q] = l2b[q];
                }
            }
        }
        for (; i < nb; ++i) {
            const double z = (X[P(i)] - B2[P(i)] * zm2) - B1[P(i)] * zm1;
            X[P(i)] = z;
            zm2 = zm1;
            zm1 = z;
        }
    }
    __syncthreads();
    KT(7);
    // dense closing rows: products in parallel (into Y and B2, free here),
    // then the two sequential sums of the reference's k order on two warps
    for (int k = t; k < nb; k += T) {
        const double zk = X[P(k)];
        Y[P(k)] = r1[k] * zk;
        B2[P(k)] = r2[k] * zk;  // B2 is reloaded before the backward band
    }
    __syncthreads();
    {
        const int w2 = T >= 64 ? 32 : 0;
        auto chain = [&](double s, const double* Q, int f) {
            // -= +0 past nb is an identity; loads one batch ahead
            double pa[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) pa[q] = f + q < nb ? Q[P(f + q)] : 0.0;
            for (int k0 = f; k0 < nb; k0 += 8) {
                double pb[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pb[q] = k0 + 8 + q < nb ? Q[P(k0 + 8 + q)] : 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q) s -= pa[q];
#pragma unroll
                for (int q = 0; q < 8; ++q) pa[q] = pb[q];
            }
            return s;
        };
        double s1 = 0.0, s2 = 0.0;
        if (t == 0) s1 = chain(X[P(n - 2)], Y, of.fc1);
        if (t == w2) s2 = chain(X[P(n - 1)], B2, of.fc2);
        __syncthreads();  // every read of X[n-2], X[n-1] done
        if (t == 0) X[P(n - 2)] = s1;
        if (t == w2) X[P(n - 1)] = s2;
    }
    __syncthreads();
    if (t == 0 && n - 2 >= of.fc2) X[P(n - 1)] -= r2[n - 2] * X[P(n - 2)];
    __syncthreads();
    KT(8);
    for (int i = t; i < n; i += T) {
        X[P(i)] /= D[i];
        B2[P(i)] = of.band2[o + i];
    }
    __syncthreads();
    if (t == 0 && n - 2 >= of.fc2) X[P(n - 2)] -= r2[n - 2] * X[P(n - 1)];
    __syncthreads();
    {
        const double xn1 = X[P(n - 1)], xn2 = X[P(n - 2)];
        for (int k = t; k < nb; k += T) {
            double x = X[P(k)];
            if (k >= of.fc2) x -= r2[k] * xn1;
            if (k >= of.fc1) x -= r1[k] * xn2;
            X[P(k)] = x;
        }
    }
    __syncthreads();
    KT(9);
    if (t == 0) {  // backward band: x_k = (g_k - L(k+2,k) x_{k+2}) - L(k+1,k) x_{k+1}
        // rows nb-1 (no terms) and nb-2 (no L(k+2,k)) peeled
        double xp2 = X[P(nb - 1)];
        double xp1 = X[P(nb - 2)] - B1[P(nb - 1)] * xp2;
        X[P(nb - 2)] = xp1;
        int k = nb - 3;
        if (k - 3 >= 0) {
            double ga[4], c1a[4], c2a[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                ga[q] = X[P(k - q)];
                c1a[q] = B1[P(k - q + 1)];
                c2a[q] = B2[P(k - q + 2)];
            }
            for (; k - 3 >= 0; k -= 4) {
                double gb[4], c1b[4], c2b[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int kk = max(k - 4 - q, 0);
                    gb[q] = X[P(kk)];
                    c1b[q] = B1[P(kk + 1)];
                    c2b[q] = B2[P(kk + 2)];
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double x = (ga[q] - c2a[q] * xp2) - c1a[q] * xp1;
                    X[P(k - q)] = x;
                    xp2 = xp1;
                    xp1 = x;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    ga[q] = gb[q];
                    c1a[q] = c1b[q];
                    c2a[q] = c2b[q];
                }
            }
        }
        for (; k >= 0; --k) {
            const double x = (X[P(k)] - B2[P(k + 2)] * xp2) - B1[P(k + 1)] * xp1;
            X[P(k)] = x;
            xp2 = xp1;
            xp1 = x;
        }
    }
    __syncthreads();
    KT(10);
    for (int i = t; i < n; i += T) Y[P(operm(i, h))] = X[P(i)];
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
// All operands of one row gathered into registers before any arithmetic, so
// the ~22 independent loads of a node are in flight together (the kernel is
// memory-latency bound otherwise).  Absent neighbours read the node itself.
struct Gather {
    double u, uSM, uSP, uTM, uTP, uSMTM, uSMTP, uSPTM, uSPTP, f;
    Coef P, TM, TP, SM, SP;
};

template <bool ONFLY, int MODE>
__device__ __forceinline__ double apply_node(const LevelView& L, const double* __restrict__ U,
                                             const double* __restrict__ F, long off, int b,
                                             int p) {
    int s, t;
    L.node(p, s, t);
    const Nbr q = neighbours(L, s, t, p);
    const CoefAt<ONFLY> cf{&L, off, b};
    if (L.dir(s)) {  // identity row
        double acc = 0.0;
        acc += 1.0 * U[p];
        return MODE == 0 ? acc : F[p] - acc;
    }
    const int N = L.nr - 1;
    const bool hs = s > 0, hp = s < N;
    Gather g;
    g.u = U[p];
    g.uTM = U[q.pTM];
    g.uTP = U[q.pTP];
    g.uSM = U[hs ? q.pSM : p];
    g.uSMTM = U[hs ? q.pSMTM : p];
    g.uSMTP = U[hs ? q.pSMTP : p];
    g.uSP = U[hp ? q.pSP : p];
    g.uSPTM = U[hp ? q.pSPTM : p];
    g.uSPTP = U[hp ? q.pSPTP : p];
    g.f = MODE == 0 ? 0.0 : F[p];
    g.P = cf(s, t, p);
    g.TM = cf(s, q.tm, q.pTM);
    g.TP = cf(s, q.tp, q.pTP);
    g.SM = hs ? cf(s - 1, t, q.pSM) : Coef{0.0, 0.0, 0.0, 0.0};
    g.SP = hp ? cf(s + 1, t, q.pSP) : Coef{0.0, 0.0, 0.0, 0.0};
    double anti = 0.0;
    if (s == 0 && L.boundary == 0) {
        const int t2 = t + L.nt / 2 >= L.nt ? t + L.nt / 2 - L.nt : t + L.nt / 2;
        anti = cf(0, t2, t2).arr;
    }
    const Row R = row_from(L, b, s, t, q.tm, g.P, g.TM, g.TP, g.SM, g.SP, anti);
    double acc = 0.0;
    acc += R.d * g.u;
    if (R.has_sm) acc += R.sm * g.uSM;
    if (R.has_sp) acc += R.sp * g.uSP;
    acc += R.tm * g.uTM;
    acc += R.tp * g.uTP;
    if (R.has_sm) {
        acc += R.mm * g.uSMTM;
        acc += R.mp * g.uSMTP;
    }
    if (R.has_sp) {
        acc += R.pm * g.uSPTM;
        acc += R.pp * g.uSPTP;
    }
    if (R.origin) acc += R.ph * U[R.t2];
    return MODE == 0 ? acc : g.f - acc;
}

// y = A u (MODE 0) or r = f - A u (MODE 1), NPT nodes per thread; optional
// per-block partial sums of r^2 (or max |r|) for the residual norm.
template <bool ONFLY, int MODE, bool NORM>
__global__ void __launch_bounds__(256) k_apply(LevelView L, const double* __restrict__ u,
                                               const double* __restrict__ f,
                                               double* __restrict__ out,
                                               double* __restrict__ partials, int norm_type,
                                               const int* __restrict__ active) {
    pdl_enter();
    constexpr int NPT = 2;
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const long off = (long)b * L.n;
    const double* U = u + off;
    const double* F = MODE == 0 ? nullptr : f + off;
    double v = 0.0;
    double val[NPT];
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int p = (blockIdx.x * NPT + k) * blockDim.x + threadIdx.x;
        val[k] = p < L.n ? apply_node<ONFLY, MODE>(L, U, F, off, b, p) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int p = (blockIdx.x * NPT + k) * blockDim.x + threadIdx.x;
        if (p < L.n) out[off + p] = val[k];
        if (NORM) v = norm_type == 2 ? fmax(v, fabs(val[k])) : v + val[k] * val[k];
    }
    if (NORM) {
        __shared__ double red[8];
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

// ------------------------------------------------------- tiled residual
// One launch covers a level with two tile families: circle tiles (kTR
// consecutive angles x kTS rings of the ring-major region, theta fast) and
// radial tiles (kTR consecutive rows x kTS spokes of the spoke-major region,
// r fast).  A tile stages u and the four coefficient arrays over the tile plus
// a one-node halo (cross-region halo nodes are gathered from their NodeIndexing
// position) with cp.async -- every load of the block is in flight at once --
// then computes its rows from shared memory with fixed +-1 / +-kTW neighbour
// offsets.  The across-origin phantom partner of ring 0 is read directly.
constexpr int kTS = 8, kTR = 64, kTW = kTR + 2, kTH = (kTS + 2) * kTW;

struct TileGeom {
    int nca, ncr;  // circle tiles: angle tiles x ring tiles
    int nrs, nrr;  // radial tiles: spoke tiles x row tiles
    int ntiles() const { return nca * ncr + nrs * nrr; }
};

inline TileGeom tile_geom(const LevelView& L) {
    TileGeom g;
    g.nca = (L.nt + kTR - 1) / kTR;
    g.ncr = (L.split + kTS - 1) / kTS;
    g.nrs = L.len > 0 ? (L.nt + kTS - 1) / kTS : 0;
    g.nrr = L.len > 0 ? (L.len + kTR - 1) / kTR : 0;
    return g;
}

template <bool ONFLY, int MODE, bool NORM>
__global__ void __launch_bounds__(256, 4) k_apply_tiled(LevelView L, TileGeom G,
                                                        const double* __restrict__ u,
                                                        const double* __restrict__ f,
                                                        double* __restrict__ out,
                                                        double* __restrict__ partials,
                                                        int norm_type,
                                                        const int* __restrict__ active) {
    pdl_enter();
    __shared__ double sU[kTH], sArr[kTH], sArt[kTH], sAtt[kTH], sDet[kTH], sF[kTS * kTR];
    __shared__ double red[8];
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const long off = (long)b * L.n;
    const double* U = u + off;
    const double* F = MODE == 0 ? nullptr : f + off;
    const int N = L.nr - 1, nt = L.nt, len = L.len, split = L.split;
    const int nct = G.nca * G.ncr;
    const bool circ = (int)blockIdx.x < nct;
    // tile origin: slow index (ring or spoke) and fast index (angle or row)
    int slow0, fast0;
    if (circ) {
        slow0 = ((int)blockIdx.x / G.nca) * kTS;  // first ring
        fast0 = ((int)blockIdx.x % G.nca) * kTR;  // first angle
    } else {
        const int tb = blockIdx.x - nct;
        slow0 = (tb / G.nrr) * kTS;  // first spoke
        fast0 = (tb % G.nrr) * kTR;  // first row (i = s - split)
    }
    // Per tile line j (slow index slow0 + j - 1): NodeIndexing base so that
    // node k of the line (fast index fast0 + k - 1) is at base + k whenever k
    // lies in [lo, hi]; nodes outside that range (cross-region halo, theta
    // wrap) take the general index; invalid nodes (outside the level) are 0.
    __shared__ long lBase[kTS + 2];
    __shared__ int lLo[kTS + 2], lHi[kTS + 2], lS[kTS + 2], lT[kTS + 2];
    if (threadIdx.x < kTS + 2) {
        const int j = threadIdx.x;
        if (circ) {
            const int sl = slow0 + j - 1;
            lS[j] = sl;
            lT[j] = 0;
            if (sl >= 0 && sl < split) {
                lBase[j] = (long)sl * nt + fast0 - 1;  // node k -> angle fast0 + k - 1
                lLo[j] = max(0, 1 - fast0);
                lHi[j] = min(kTR + 1, nt - fast0);
            } else {
                lBase[j] = 0;
                lLo[j] = 1;
                lHi[j] = 0;  // empty: general path
            }
        } else {
            int tl = slow0 + j - 1;
            tl = ((tl % nt) + nt) % nt;
            lS[j] = 0;
            lT[j] = tl;
            lBase[j] = (long)split * nt + (long)tl * len + fast0 - 1;  // node k -> row fast0+k-1
            lLo[j] = max(0, 1 - fast0);
            lHi[j] = min(kTR + 1, len - fast0);
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kTH; e += 256) {
        const int j = e / kTW, k = e - j * kTW;  // k in [0, kTW): fast index fast0 + k - 1
        int sv, tv;
        bool ok;
        long g;
        if (circ) {
            sv = lS[j];
            tv = fast0 + k - 1;
            if (tv < 0 || tv >= nt) tv = ((tv % nt) + nt) % nt;
            ok = sv >= 0 && sv <= N;
        } else {
            tv = lT[j];
            sv = split + fast0 + k - 1;
            ok = sv <= N;
        }
        if (k >= lLo[j] && k <= lHi[j])
            g = lBase[j] + k;
        else
            g = ok ? (long)L.idx(sv, tv) : 0;
        if (ok) {
            __pipeline_memcpy_async(&sU[e], U + g, 8);
            if (ONFLY) {
                const Coef c = transform(L.geo, L.alpha[(long)b * L.nr + sv], L.r[sv], L.sn[tv],
                                         L.cs[tv], nullptr);
                sArr[e] = c.arr;
                sArt[e] = c.art;
                sAtt[e] = c.att;
                sDet[e] = c.det;
            } else {
                __pipeline_memcpy_async(&sArr[e], L.arr + off + g, 8);
                __pipeline_memcpy_async(&sArt[e], L.art + off + g, 8);
                __pipeline_memcpy_async(&sAtt[e], L.att + off + g, 8);
                __pipeline_memcpy_async(&sDet[e], L.det + off + g, 8);
            }
            if (MODE == 1 && j >= 1 && j <= kTS && k >= 1 && k <= kTR)
                __pipeline_memcpy_async(&sF[(j - 1) * kTR + (k - 1)], F + g, 8);
        } else {
            sU[e] = 0.0;
            sArr[e] = sArt[e] = sAtt[e] = sDet[e] = 0.0;
        }
    }
    __pipeline_commit();
    __pipeline_wait_prior(0);
    __syncthreads();
    // neighbour strides in the tile: radial (s+-1) and angular (t+-1)
    const int dS = circ ? kTW : 1, dT = circ ? 1 : kTW;
    const int kk = threadIdx.x & (kTR - 1);
    // interior tile: every row of it and of its halo lines is a non-Dirichlet
    // ring away from the origin, so the row takes the lean form below (the
    // row_from expressions with has_sm = has_sp = true, no phantom)
    const bool lean = circ ? (slow0 >= 2 && slow0 + kTS + 1 <= min(split, N))
                           : (fast0 >= 1 && split + fast0 >= 2 && fast0 + kTR + 2 <= len);
    double v = 0.0;
    if (lean) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int jj = (threadIdx.x >> 6) + 4 * q;
            int s, t;
            bool mine;
            if (circ) {
                s = slow0 + jj;
                t = fast0 + kk;
                mine = t < nt;
            } else {
                t = slow0 + jj;
                s = split + fast0 + kk;
                mine = t < nt;
            }
            double val = 0.0;
            if (mine) {
                const int e = (jj + 1) * kTW + (kk + 1);
                const int tm = t == 0 ? nt - 1 : t - 1;
                const double km = L.k[tm], kp = L.k[t];
                const double hm = L.h[s - 1], hp = L.h[s];
                const double kbar = 0.5 * (km + kp);
                const double hbar = 0.5 * (hm + hp);
                const double qkm = xdiv(kbar, hm, L.rh[s - 1]);
                const double qkp = xdiv(kbar, hp, L.rh[s]);
                const double qhm = xdiv(hbar, km, L.rk[tm]);
                const double qhp = xdiv(hbar, kp, L.rk[t]);
                const double aP = sArr[e], aSM = sArr[e - dS], aSP = sArr[e + dS];
                const double tP = sAtt[e], tTM = sAtt[e - dT], tTP = sAtt[e + dT];
                const double rTM = sArt[e - dT], rTP = sArt[e + dT];
                const double rSM = sArt[e - dS], rSP = sArt[e + dS];
                double diag = 0.0;
                diag += qkm * (aP + aSM);
                diag += qkp * (aP + aSP);
                diag += qhm * (tP + tTM);
                diag += qhp * (tP + tTP);
                diag += L.beta[(long)b * L.nr + s] * sDet[e] * hbar * kbar;
                double acc = 0.0;
                acc += diag * sU[e];
                acc += (-qkm * (aP + aSM)) * sU[e - dS];
                acc += (-qkp * (aP + aSP)) * sU[e + dS];
                acc += (-qhm * (tP + tTM)) * sU[e - dT];
                acc += (-qhp * (tP + tTP)) * sU[e + dT];
                acc += (-(rTM + rSM) * 0.25) * sU[e - dS - dT];
                acc += ((rSM + rTP) * 0.25) * sU[e - dS + dT];
                acc += ((rTM + rSP) * 0.25) * sU[e + dS - dT];
                acc += (-(rSP + rTP) * 0.25) * sU[e + dS + dT];
                val = MODE == 0 ? acc : sF[jj * kTR + kk] - acc;
                out[off + (circ ? s * nt + t : split * nt + t * len + (s - split))] = val;
            }
            if (NORM) v = norm_type == 2 ? fmax(v, fabs(val)) : v + val * val;
        }
    } else
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int jj = (threadIdx.x >> 6) + 4 * q;
        int s, t;
        bool mine;
        if (circ) {
            s = slow0 + jj;
            t = fast0 + kk;
            mine = s < split && t < nt;
        } else {
            t = slow0 + jj;
            s = split + fast0 + kk;
            mine = t < nt && s <= N;
        }
        double val = 0.0;
        if (mine) {
            const int e = (jj + 1) * kTW + (kk + 1);
            const double up = sU[e];
            double acc = 0.0;
            if (L.dir(s)) {
                acc += 1.0 * up;
            } else {
                const int tm = t == 0 ? nt - 1 : t - 1;
                const Coef cP = {sArr[e], sArt[e], sAtt[e], sDet[e]};
                const Coef cTM = {sArr[e - dT], sArt[e - dT], sAtt[e - dT], sDet[e - dT]};
                const Coef cTP = {sArr[e + dT], sArt[e + dT], sAtt[e + dT], sDet[e + dT]};
                const Coef cSM = {sArr[e - dS], sArt[e - dS], sAtt[e - dS], sDet[e - dS]};
                const Coef cSP = {sArr[e + dS], sArt[e + dS], sAtt[e + dS], sDet[e + dS]};
                double anti = 0.0, uanti = 0.0;
                if (s == 0 && L.boundary == 0) {  // phantom partner (0, t + nt/2)
                    const int t2 = t + nt / 2 >= nt ? t + nt / 2 - nt : t + nt / 2;
                    anti = ONFLY ? transform(L.geo, L.alpha[(long)b * L.nr], L.r[0], L.sn[t2],
                                             L.cs[t2], nullptr).arr
                                 : L.arr[off + t2];
                    uanti = U[t2];
                }
                const Row R = row_from(L, b, s, t, tm, cP, cTM, cTP, cSM, cSP, anti);
                acc += R.d * up;
                if (R.has_sm) acc += R.sm * sU[e - dS];
                if (R.has_sp) acc += R.sp * sU[e + dS];
                acc += R.tm * sU[e - dT];
                acc += R.tp * sU[e + dT];
                if (R.has_sm) {
                    acc += R.mm * sU[e - dS - dT];
                    acc += R.mp * sU[e - dS + dT];
                }
                if (R.has_sp) {
                    acc += R.pm * sU[e + dS - dT];
                    acc += R.pp * sU[e + dS + dT];
                }
                if (R.origin) acc += R.ph * uanti;
            }
            val = MODE == 0 ? acc : sF[jj * kTR + kk] - acc;
            out[off + L.idx(s, t)] = val;
        }
        if (NORM) v = norm_type == 2 ? fmax(v, fabs(val)) : v + val * val;
    }
    if (NORM) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const double o = __shfl_down_sync(FULL, v, d);
            v = norm_type == 2 ? fmax(v, o) : v + o;
        }
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double a = red[0];
            for (int w = 1; w < 8; ++w) a = norm_type == 2 ? fmax(a, red[w]) : a + red[w];
            partials[(long)b * gridDim.x + blockIdx.x] = a;
        }
    }
}

// ------------------------------------------- TMA-streamed Take residual
// A CTA owns a strip of kTW2 = 240 consecutive nodes along the contiguous
// direction of a region (angles of a ring in the ring-major circle region;
// rows of a spoke in the spoke-major radial region) and walks R lines across
// it (rings, resp. spokes).  A producer warp streams each line -- u, arr, art,
// att, det, f over the 242-node halo segment -- into a kLines-deep ring of
// shared-memory slots with one bulk copy (TMA engine) per array and line,
// completion counted on the slot's `full` mbarrier; the 8 consumer warps (30
// output lanes + 2 halo lanes each) read each line once into a 3-line register
// window, take in-line neighbours by warp shuffles, and release the slot on
// its `empty` mbarrier.  HBM is read once per node; no per-element address
// arithmetic and no block barriers in the loop.  Segments are copied from
// their 16-byte-aligned start (node k of a line at slot position k + o, o the
// parity of the line's first index).  The theta wrap of the circle strips at
// both ends comes from two 16-byte edge copies per array.  Rings split-1 and
// split (the region interface: their ring/spoke neighbours lie in the other
// layout) are computed node-wise by extra CTAs of the same launch.
// the lean interior row (k_apply_tiled's lean branch, same order)
__device__ __forceinline__ double lean_row(double qkm, double qkp, double qhm, double qhp,
                                           double bdhk, double aP, double aSM, double aSP,
                                           double tP, double tTM, double tTP, double rTM,
                                           double rTP, double rSM, double rSP, double uP,
                                           double uSM, double uSP, double uTM, double uTP,
                                           double uMM, double uMP, double uPM, double uPP) {
    double diag = 0.0;
    diag += qkm * (aP + aSM);
    diag += qkp * (aP + aSP);
    diag += qhm * (tP + tTM);
    diag += qhp * (tP + tTP);
    diag += bdhk;
    double acc = 0.0;
    acc += diag * uP;
    acc += (-qkm * (aP + aSM)) * uSM;
    acc += (-qkp * (aP + aSP)) * uSP;
    acc += (-qhm * (tP + tTM)) * uTM;
    acc += (-qhp * (tP + tTP)) * uTP;
    acc += (-(rTM + rSM) * 0.25) * uMM;
    acc += ((rSM + rTP) * 0.25) * uMP;
    acc += ((rTM + rSP) * 0.25) * uPM;
    acc += (-(rSP + rTP) * 0.25) * uPP;
    return acc;
}

__device__ __forceinline__ bool lean_ring(const LevelView& L, int s) {
    return s >= 1 && s <= L.nr - 3 && !(L.boundary == 1 && s == 1);
}

// general row (origin, Dirichlet, next-to-Dirichlet rings) from the window
__device__ __forceinline__ double general_row(const LevelView& L, int b, long off,
                                              const double* __restrict__ u, int s, int t,
                                              const Coef& cP, const Coef& cTM, const Coef& cTP,
                                              const Coef& cSM, const Coef& cSP, double uP,
                                              double uSM, double uSP, double uTM, double uTP,
                                              double uMM, double uMP, double uPM, double uPP) {
    if (L.dir(s)) return 1.0 * uP;
    const int nt = L.nt;
    const int tm = t == 0 ? nt - 1 : t - 1;
    double anti = 0.0, uanti = 0.0;
    if (s == 0 && L.boundary == 0) {  // phantom partner (0, t + nt/2)
        const int t2 = t + nt / 2 >= nt ? t + nt / 2 - nt : t + nt / 2;
        anti = L.arr[off + t2];
        uanti = u[off + t2];
    }
    const Row R = row_from(L, b, s, t, tm, cP, cTM, cTP, cSM, cSP, anti);
    double acc = 0.0;
    acc += R.d * uP;
    if (R.has_sm) acc += R.sm * uSM;
    if (R.has_sp) acc += R.sp * uSP;
    acc += R.tm * uTM;
    acc += R.tp * uTP;
    if (R.has_sm) {
        acc += R.mm * uMM;
        acc += R.mp * uMP;
    }
    if (R.has_sp) {
        acc += R.pm * uPM;
        acc += R.pp * uPP;
    }
    if (R.origin) acc += R.ph * uanti;
    return acc;
}

constexpr int kTW2 = 240;             // output nodes per strip (8 warps x 30)
constexpr int kLn = 248;              // slot row: 242 halo nodes + alignment slack
#ifndef PMG_TMA_LINES
#define PMG_TMA_LINES 4
#endif
#ifndef PMG_TMA_MINB
#define PMG_TMA_MINB 2
#endif
constexpr int kLines = PMG_TMA_LINES;  // line slots per CTA
struct TmaSlot {
    double a[6][kLn];                 // u, arr, art, att, det, f
    double e[2][5][2];                // circle theta-wrap edges (left, right)
};
constexpr size_t kTmaSmem = kLines * sizeof(TmaSlot) + 2 * kLines * 8 + 16;

// Rows the strips compute are the lean interior rows: circle rings
// c0 .. split-2 and radial rows s = split+1 .. N-2.  The rest -- origin /
// interior-Dirichlet rings, the region interface rings split-1 and split, the
// Dirichlet ring N and ring N-1 -- are computed node-wise by the last CTAs of
// the launch.
struct TmaGeom {
    int c0;        // first strip ring (1, or 2 with an interior Dirichlet ring 0)
    int ncf, ncs;  // circle strips: angle strips x ring chunks
    int nrf, nrs;  // radial strips: row strips x spoke chunks
    int nif;       // node-wise CTAs (256 nodes each)
    int R;         // lines per strip
    int cps;       // CTAs per section
};

inline TmaGeom tma_geom(const LevelView& L, int R) {
    TmaGeom g;
    g.R = R;
    g.c0 = L.boundary == 1 ? 2 : 1;
    const int cr = L.split - 1 - g.c0;  // rings c0 .. split-2
    g.ncf = cr > 0 ? (L.nt + kTW2 - 1) / kTW2 : 0;
    g.ncs = cr > 0 ? (cr + R - 1) / R : 0;
    const int rr = L.len - 3;           // rows i = 1 .. len-3
    g.nrf = rr > 0 ? (rr + kTW2 - 1) / kTW2 : 0;
    g.nrs = rr > 0 ? (L.nt + R - 1) / R : 0;
    g.nif = (6 * L.nt + 255) / 256;     // up to 6 node-wise rings
    g.cps = g.ncf * g.ncs + g.nrf * g.nrs + g.nif;
    return g;
}

inline TmaGeom tma_geom_auto(const LevelView& L) {
    TmaGeom g = tma_geom(L, 64);
    for (int R = 64; R > 8; R >>= 1) {
        g = tma_geom(L, R);
        if ((long)g.cps * L.B >= 148L * 4) break;
    }
    return g;
}

inline long tma_min_nodes() {
    static const long v = [] {
        const char* e = std::getenv("PMG_TMA_MIN_NODES");
        return e ? std::atol(e) : (4L << 20);
    }();
    return v;
}
// whether the TMA kernel applies: long lines, even n_theta (16-byte aligned
// ring starts), and enough nodes that bandwidth, not latency, bounds the launch
// (latency-bound small levels keep the one-tile-per-CTA kernel)
inline bool tma_ok(const LevelView& L) {
    return L.nt >= 256 && (L.nt & 1) == 0 && L.len >= 64 && L.split >= 4 &&
           (long)L.n * L.B >= tma_min_nodes();
}

// ring of node-wise row e (0 .. 6 nt): 0, 1, split-1, split, N-1, N; -1 when
// that ring is a strip ring (or a duplicate)
__device__ __forceinline__ int tma_nodewise_ring(const LevelView& L, int c0, int j) {
    const int N = L.nr - 1;
    switch (j) {
        case 0: return 0;
        case 1: return c0 == 2 ? 1 : -1;
        case 2: return L.split - 1;
        case 3: return L.split;
        case 4: return N - 1 > L.split ? N - 1 : -1;
        default: return N > L.split ? N : -1;
    }
}

template <bool CIRC, int MODE, bool NORM>
__device__ __forceinline__ double tma_strip(const LevelView& L, const TmaGeom& G, int b, int w,
                                            const double* __restrict__ u,
                                            const double* __restrict__ f,
                                            double* __restrict__ out, int norm_type,
                                            TmaSlot* slot, unsigned long long* full,
                                            unsigned long long* empty) {
    const int nt = L.nt, split = L.split, len = L.len;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long off = (long)b * L.n;
    // strip: fast index of node k is f0 + k - 1; center lines l0 .. l1-1
    int f0, l0, l1;
    if (CIRC) {
        f0 = (w % G.ncf) * kTW2;
        l0 = G.c0 + (w / G.ncf) * G.R;
        l1 = min(l0 + G.R, split - 1);
    } else {
        f0 = 1 + (w % G.nrf) * kTW2;
        l0 = (w / G.nrf) * G.R;
        l1 = min(l0 + G.R, nt);
    }
    const int nlines = l1 - l0 + 2;  // halo line l0-1, lines l0..l1-1, halo line l1
    // global index of node k = 0 of line l (circle: ring l; radial: spoke l, wrapped)
    auto line_base = [&](int l) -> long {
        if (CIRC) return off + (long)l * nt + f0 - 1;
        const int tt = l < 0 ? l + nt : (l >= nt ? l - nt : l);
        return off + (long)split * nt + (long)tt * len + f0 - 1;
    };
    // last node of a line segment (circle: t <= nt-1; radial: row <= len-2)
    const int khi = CIRC ? min(kTW2 + 1, nt - f0) : min(kTW2 + 1, len - 1 - f0);
    const bool eL = CIRC && f0 == 0, eR = CIRC && f0 + kTW2 >= nt;
    if (warp == 8) {
        // ------------------------------------------------------ producer warp
        auto src = [&](int a) -> const double* {
            return a == 0 ? u : a == 1 ? L.arr : a == 2 ? L.art : a == 3 ? L.att : a == 4 ? L.det : f;
        };
        constexpr int narr = MODE == 1 ? 6 : 5;
        for (int q = 0; q < nlines; ++q) {
            const int sl = q % kLines;
            if (q >= kLines) mbar_wait(&empty[sl], (unsigned)((q / kLines) - 1) & 1u);
            const int l = l0 - 1 + q;
            TmaSlot& S = slot[sl];
            const long base = line_base(l);
            const int o = (int)(base & 1);
            const int p0 = ((eL ? 1 : 0) + o) & ~1;
            const int p1 = (khi + o) | 1;
            const long g0 = base + p0 - o;
            const unsigned bytes = (unsigned)(p1 - p0 + 1) * 8u;
            const unsigned ebytes = (eL ? 16u : 0u) + (eR ? 16u : 0u);
            // the slot was last read through the generic proxy
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (lane == 0) mbar_arrive_tx(&full[sl], bytes * narr + ebytes * 5);
            __syncwarp();
            if (lane < narr) bulk_g2s(&S.a[lane][p0], src(lane) + g0, bytes, &full[sl]);
            if (eL && lane >= 8 && lane < 13)  // t = nt-1 (odd index): the pair from nt-2
                bulk_g2s(&S.e[0][lane - 8][0], src(lane - 8) + off + (long)l * nt + nt - 2, 16,
                         &full[sl]);
            if (eR && lane >= 16 && lane < 21)  // t = 0 of the ring
                bulk_g2s(&S.e[1][lane - 16][0], src(lane - 16) + off + (long)l * nt, 16, &full[sl]);
        }
        return 0.0;
    }
    // ---------------------------------------------------------- consumer warps
    const int k = warp * 30 + lane;  // node k of the segment
    const int fi = f0 + k - 1;
    const bool outl = lane >= 1 && lane <= 30 && (CIRC ? fi < nt : fi <= len - 3);
    const bool useL = eL && k == 0;      // t = -1 -> nt-1
    const bool useR = CIRC && fi == nt;  // t = nt -> 0
    const int kc = min(k, kLn - 2);      // lanes past the segment read (unused) slot data
    struct V {
        double u, arr, art, att, det, f;
    };
    auto fetch = [&](int q) -> V {
        V x;
        const int sl = q % kLines;
        mbar_wait(&full[sl], (unsigned)(q / kLines) & 1u);
        const TmaSlot& S = slot[sl];
        if (useL || useR) {
            const int e = useL ? 0 : 1, i = useL ? 1 : 0;
            x.u = S.e[e][0][i];
            x.arr = S.e[e][1][i];
            x.art = S.e[e][2][i];
            x.att = S.e[e][3][i];
            x.det = S.e[e][4][i];
            x.f = 0.0;
        } else {
            const int pos = kc + (int)(line_base(l0 - 1 + q) & 1);
            x.u = S.a[0][pos];
            x.arr = S.a[1][pos];
            x.art = S.a[2][pos];
            x.att = S.a[3][pos];
            x.det = S.a[4][pos];
            x.f = MODE == 1 ? S.a[5][pos] : 0.0;
        }
        __syncwarp();
        if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[sl]))
                         : "memory");
        return x;
    };
    // per-lane constants along the strip
    double km = 0, kp = 0, rkm = 0, rkp = 0, kbar = 0;
    double hm = 0, hp = 0, rhm = 0, rhp = 0, hbar = 0, beta = 0;
    int t = 0;
    if (CIRC) {
        t = fi < 0 ? fi + nt : (fi >= nt ? fi - nt : fi);
        const int tm = t == 0 ? nt - 1 : t - 1;
        km = L.k[tm];
        kp = L.k[t];
        rkm = L.rk[tm];
        rkp = L.rk[t];
        kbar = 0.5 * (km + kp);
    } else {
        const int s = split + max(1, min(fi, len - 3));
        hm = L.h[s - 1];
        hp = L.h[s];
        rhm = L.rh[s - 1];
        rhp = L.rh[s];
        hbar = 0.5 * (hm + hp);
        beta = L.beta[(long)b * L.nr + s];
    }
    V M = fetch(0), C = fetch(1);
    double v = 0.0;
    for (int q = 2; q < nlines; ++q) {
        const V P = fetch(q);
        const int l = l0 + q - 2;  // center line
        double val = 0.0;
        if (CIRC) {
            const double uTM = __shfl_up_sync(FULL, C.u, 1), uTP = __shfl_down_sync(FULL, C.u, 1);
            const double uMM = __shfl_up_sync(FULL, M.u, 1), uMP = __shfl_down_sync(FULL, M.u, 1);
            const double uPM = __shfl_up_sync(FULL, P.u, 1), uPP = __shfl_down_sync(FULL, P.u, 1);
            const double tTM = __shfl_up_sync(FULL, C.att, 1), tTP = __shfl_down_sync(FULL, C.att, 1);
            const double rTM = __shfl_up_sync(FULL, C.art, 1), rTP = __shfl_down_sync(FULL, C.art, 1);
            if (outl) {
                const int s = l;
                const double hm2 = L.h[s - 1], hp2 = L.h[s];
                const double hb = 0.5 * (hm2 + hp2);
                const double qkm = xdiv(kbar, hm2, L.rh[s - 1]);
                const double qkp = xdiv(kbar, hp2, L.rh[s]);
                const double qhm = xdiv(hb, km, rkm);
                const double qhp = xdiv(hb, kp, rkp);
                const double acc =
                    lean_row(qkm, qkp, qhm, qhp, L.beta[(long)b * L.nr + s] * C.det * hb * kbar,
                             C.arr, M.arr, P.arr, C.att, tTM, tTP, rTM, rTP, M.art, P.art, C.u,
                             M.u, P.u, uTM, uTP, uMM, uMP, uPM, uPP);
                val = MODE == 0 ? acc : C.f - acc;
                out[off + (long)s * nt + t] = val;
            }
        } else {
            const double uSM = __shfl_up_sync(FULL, C.u, 1), uSP = __shfl_down_sync(FULL, C.u, 1);
            const double uMM = __shfl_up_sync(FULL, M.u, 1), uPM = __shfl_down_sync(FULL, M.u, 1);
            const double uMP = __shfl_up_sync(FULL, P.u, 1), uPP = __shfl_down_sync(FULL, P.u, 1);
            const double aSM = __shfl_up_sync(FULL, C.arr, 1), aSP = __shfl_down_sync(FULL, C.arr, 1);
            const double rSM = __shfl_up_sync(FULL, C.art, 1), rSP = __shfl_down_sync(FULL, C.art, 1);
            if (outl) {
                const int tc = l;
                const int tm = tc == 0 ? nt - 1 : tc - 1;
                const double km2 = L.k[tm], kp2 = L.k[tc];
                const double kb = 0.5 * (km2 + kp2);
                const double qkm = xdiv(kb, hm, rhm);
                const double qkp = xdiv(kb, hp, rhp);
                const double qhm = xdiv(hbar, km2, L.rk[tm]);
                const double qhp = xdiv(hbar, kp2, L.rk[tc]);
                const double acc =
                    lean_row(qkm, qkp, qhm, qhp, beta * C.det * hbar * kb, C.arr, aSM, aSP, C.att,
                             M.att, P.att, M.art, P.art, rSM, rSP, C.u, uSM, uSP, M.u, P.u, uMM,
                             uMP, uPM, uPP);
                val = MODE == 0 ? acc : C.f - acc;
                out[off + (long)split * nt + (long)tc * len + fi] = val;
            }
        }
        if (NORM) v = norm_type == 2 ? fmax(v, fabs(val)) : v + val * val;
        M = C;
        C = P;
    }
    return v;
}

// MINB: resident CTAs per SM the register allocation targets -- 2 (96
// registers) for single large grids (tuned at 8193x8192), 3 (72 registers) for
// batches of small sections, whose short strips leave more latency to cover
// (256 x 513x512: 0.914 -> 0.874 ms)
template <int MODE, bool NORM, int MINB = PMG_TMA_MINB>
__global__ void __launch_bounds__(288, MINB) k_apply_tma(LevelView L, TmaGeom G,
                                                      const double* __restrict__ u,
                                                      const double* __restrict__ f,
                                                      double* __restrict__ out,
                                                      double* __restrict__ partials, int norm_type,
                                                      const int* __restrict__ active) {
    pdl_enter();
    extern __shared__ __align__(128) unsigned char tsm[];
    __shared__ double red[9];
    const int b = blockIdx.x / G.cps;
    if (active && !active[b]) return;
    const int w = blockIdx.x - b * G.cps;
    const int nc = G.ncf * G.ncs, nrad = G.nrf * G.nrs;
    double v = 0.0;
    if (w < nc + nrad) {
        TmaSlot* slot = reinterpret_cast<TmaSlot*>(tsm);
        unsigned long long* full =
            reinterpret_cast<unsigned long long*>(tsm + kLines * sizeof(TmaSlot));
        unsigned long long* empty = full + kLines;
        if (threadIdx.x == 0)
            for (int i = 0; i < kLines; ++i) {
                mbar_init(&full[i], 1);
                mbar_init(&empty[i], 8);
            }
        __syncthreads();
        if (w < nc)
            v = tma_strip<true, MODE, NORM>(L, G, b, w, u, f, out, norm_type, slot, full, empty);
        else
            v = tma_strip<false, MODE, NORM>(L, G, b, w - nc, u, f, out, norm_type, slot, full,
                                             empty);
    } else if (threadIdx.x < 256) {
        // node-wise rings (origin, interior Dirichlet, region interface, N-1, N)
        const int e = (w - nc - nrad) * 256 + threadIdx.x;
        const int s = e < 6 * L.nt ? tma_nodewise_ring(L, G.c0, e / L.nt) : -1;
        if (s >= 0) {
            const int t = e % L.nt;
            const long off = (long)b * L.n;
            const double* U = u + off;
            const int p = L.idx(s, t);
            const Nbr q = neighbours(L, s, t, p);
            const CoefAt<false> cf{&L, off, b};
            const int N = L.nr - 1;
            const Coef z = {0.0, 0.0, 0.0, 0.0};
            const Coef cP = cf(s, t, p), cTM = cf(s, q.tm, q.pTM), cTP = cf(s, q.tp, q.pTP);
            const Coef cSM = s > 0 ? cf(s - 1, t, q.pSM) : z;
            const Coef cSP = s < N ? cf(s + 1, t, q.pSP) : z;
            const double uSM = s > 0 ? U[q.pSM] : 0.0, uSP = s < N ? U[q.pSP] : 0.0;
            const double uMM = s > 0 ? U[q.pSMTM] : 0.0, uMP = s > 0 ? U[q.pSMTP] : 0.0;
            const double uPM = s < N ? U[q.pSPTM] : 0.0, uPP = s < N ? U[q.pSPTP] : 0.0;
            const double acc = general_row(L, b, off, u, s, t, cP, cTM, cTP, cSM, cSP, U[p], uSM,
                                           uSP, U[q.pTM], U[q.pTP], uMM, uMP, uPM, uPP);
            const double val = MODE == 0 ? acc : f[off + p] - acc;
            out[off + p] = val;
            if (NORM) v = norm_type == 2 ? fabs(val) : val * val;
        }
    }
    if (NORM) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const double o = __shfl_down_sync(FULL, v, d);
            v = norm_type == 2 ? fmax(v, o) : v + o;
        }
        if (lane == 0) red[warp] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double a = red[0];
            for (int k2 = 1; k2 < 9; ++k2) a = norm_type == 2 ? fmax(a, red[k2]) : a + red[k2];
            partials[blockIdx.x] = a;
        }
    }
}

// ------------------------------------------------------------- circle sweep
// One block per circle line (ring s = parity + 2*blockIdx.x) of one section:
// rhs_t = f - sum_{off-line} A u (smoother.cpp:162-182), then the cyclic
// Sherman-Morrison solve (line_algebra.cpp:98-120), or the envelope solve of
// the across-origin ring 0 (smoother.cpp:144-152).
// One circle line (ring s of section b), reference smoother.cpp:95-116,
// 144-182: rhs gather, then the cyclic Sherman-Morrison solve
// (line_algebra.cpp:98-120) or the envelope solve of the across-origin ring.
// wait(): called once the line's own loads are in flight and before any u of
// another line is read (the fused smoothing step waits for those lines there).
template <bool ONFLY, int K, bool CG, class Wait>
__device__ __forceinline__ void circle_body(const LevelView& L, double* __restrict__ u,
                                            const double* __restrict__ f,
                                            const double* __restrict__ cil,
                                            const double* __restrict__ cm,
                                            const double* __restrict__ corner,
                                            const double* __restrict__ cz,
                                            const OriginFactor& of, int serial, int exact_rings,
                                            int b, int s, double* smem, const Wait& wait) {
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
    // serial: 0 fast (chunked scans), 1 exact order in parallel (line_solve_ex),
    // 2 exact order on one thread (lines whose 4 shared arrays do not fit)
    const bool par_ex = serial == 1 || (serial == 0 && exact_rings > 0);
    double* Y = smem;
    double* IL = smem + pn;
    double* M = IL + pn;
    double* RC = M + pn;  // RN(1/l) (par_ex only)
    double* scr = par_ex ? RC + pn : RC;
    const CoefAt<ONFLY> cf{&L, off, b};
    const bool origin = s == 0 && L.boundary == 0;
    const long fo = (long)b * L.split * nt + (long)s * nt;
    const bool exact = serial || s <= exact_rings;  // block-uniform
    if (!origin) {  // line factors: asynchronous copies, overlapped with the rhs
        for (int t = threadIdx.x; t < nt; t += T) {
            __pipeline_memcpy_async(&IL[P(t)], &cil[fo + t], 8);
            __pipeline_memcpy_async(&M[P(t)], &cm[fo + t], 8);
        }
        __pipeline_commit();
    }
    KT(1);
    wait();
    if (L.rows) {  // assembled rows (stencil.cpp:44-137 values, k_rows)
        const double* Rw = L.rows + (long)b * 10 * L.n;
        const int n = L.n;
        for (int t = threadIdx.x; t < nt; t += T) {
            const int p = base + t;
            const Nbr q = neighbours(L, s, t, p);
            double acc = F[p];
            acc -= Rw[1 * n + p] * ldu<CG>(&U[q.pSM]);
            acc -= Rw[2 * n + p] * ldu<CG>(&U[q.pSP]);
            acc -= Rw[5 * n + p] * ldu<CG>(&U[q.pSMTM]);
            acc -= Rw[6 * n + p] * ldu<CG>(&U[q.pSMTP]);
            acc -= Rw[7 * n + p] * ldu<CG>(&U[q.pSPTM]);
            acc -= Rw[8 * n + p] * ldu<CG>(&U[q.pSPTP]);
            Y[P(t)] = acc;
        }
    } else if (!ONFLY && circle_lean_ring(L, s)) {
        for (int t = threadIdx.x; t < nt; t += T) Y[P(t)] = circle_rhs_lean<CG>(L, off, s, t, U, F);
    } else
    for (int t = threadIdx.x; t < nt; t += T) {
        const int p = base + t;
        const Nbr q = neighbours(L, s, t, p);
        const Row R = make_row_fast(L, cf, s, t, p, q);
        double acc = F[p];
        if (R.has_sm) acc -= R.sm * ldu<CG>(&U[q.pSM]);
        if (R.has_sp) acc -= R.sp * ldu<CG>(&U[q.pSP]);
        if (R.has_sm) {
            acc -= R.mm * ldu<CG>(&U[q.pSMTM]);
            acc -= R.mp * ldu<CG>(&U[q.pSMTP]);
        }
        if (R.has_sp) {
            acc -= R.pm * ldu<CG>(&U[q.pSPTM]);
            acc -= R.pp * ldu<CG>(&U[q.pSPTP]);
        }
        Y[P(t)] = acc;
    }
    KT(2);
    if (origin) {
        __syncthreads();
        if (serial == 1)
            origin_solve_seq(Y, IL, M, RC, of, b, nt);
        else if (serial)
            origin_solve_exact(Y, IL, M, of, b, nt);
        else if (nt < PMG_ORIGIN_SCAN_MIN)
            origin_solve_exact(Y, IL, M, of, b, nt);
        else
            origin_solve<K>(Y, IL, of, b, nt, scr);
    } else {
        __pipeline_wait_prior(0);
        if (!exact)  // each thread converts the elements it copied
            for (int t = threadIdx.x; t < nt; t += T) IL[P(t)] = __drcp_rn(IL[P(t)]);
        else if (par_ex)
            for (int t = threadIdx.x; t < nt; t += T) RC[P(t)] = __drcp_rn(IL[P(t)]);
        __syncthreads();
        KT(3);
        if (exact && par_ex && nt <= 8 * T)
            line_solve_ex<8, true>(Y, IL, RC, M, nt, corner[(long)b * L.split + s], cz + fo, scr);
        else if (exact && par_ex)
            line_solve_ex<kExChunk, true>(Y, IL, RC, M, nt, corner[(long)b * L.split + s], cz + fo, scr);
        else if (serial == 3)
            line_solve_ex<kExChunk, true, true>(Y, IL, nullptr, M, nt, corner[(long)b * L.split + s],
                                                cz + fo, scr);
        else if (exact)
            cyc_solve_exact(Y, IL, M, nt, corner[(long)b * L.split + s], cz + fo, scr);
        else
            line_solve<K, true>(Y, IL, M, nt, corner[(long)b * L.split + s], scr);
    }
    KT(4);
    for (int t = threadIdx.x; t < nt; t += T) U[base + t] = Y[P(t)];
    KT(5);}
template <bool ONFLY, int K>
__global__ void __launch_bounds__(K >= 16 ? 512 : 256, K >= 16 ? 1 : PMG_LINE_MINB) k_circle(LevelView L, double* __restrict__ u,
                                                const double* __restrict__ f,
                                                const double* __restrict__ cil,
                                                const double* __restrict__ cm,
                                                const double* __restrict__ corner,
                                                const double* __restrict__ cz,
                                                OriginFactor of, int parity, int serial,
                                                int exact_rings,
                                                const int* __restrict__ active) {
    KT(0);
    pdl_enter();
    extern __shared__ double smem[];
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    circle_body<ONFLY, K, false>(L, u, f, cil, cm, corner, cz, of, serial, exact_rings, b,
                                 parity + 2 * blockIdx.x, smem, [] {});
}

// ------------------------------------------------------------- radial sweep
// One block per radial line (spoke t = parity + 2*blockIdx.x) of one section:
// rhs over rings split..n_r-1 (smoother.cpp:184-205) then the tridiagonal
// Cholesky solve (line_algebra.cpp:42-62); the Dirichlet row rides along as
// an identity row.
// One radial line (spoke t of section b), reference smoother.cpp:118-142,
// 184-205: rhs gather, then the tridiagonal LL^T solve (line_algebra.cpp:42-62).
template <bool ONFLY, int K, bool CG, class Wait>
__device__ __forceinline__ void radial_body(const LevelView& L, double* __restrict__ u,
                                            const double* __restrict__ f,
                                            const double* __restrict__ ril,
                                            const double* __restrict__ rm, int serial, int b,
                                            int t, double* smem, const Wait& wait) {
    const int len = L.len, split = L.split, T = blockDim.x;
    const long off = (long)b * L.n;
    double* U = u + off;
    const double* F = f + off;
    const int base = split * L.nt + t * len;
    const int pn = padded(len);
    double* Y = smem;
    double* IL = smem + pn;
    double* M = IL + pn;
    double* RC = M + pn;  // RN(1/l) (serial == 1 only)
    double* scr = serial == 1 ? RC + pn : RC;
    const CoefAt<ONFLY> cf{&L, off, b};
    const long fo = ((long)b * L.nt + t) * len;
    for (int i = threadIdx.x; i < len; i += T) {  // overlapped with the rhs
        __pipeline_memcpy_async(&IL[P(i)], &ril[fo + i], 8);
        __pipeline_memcpy_async(&M[P(i)], &rm[fo + i], 8);
    }
    __pipeline_commit();
    KT(1);
    wait();
    // interior rows split < s < n_r-1 (Take): only the off-line couplings --
    // angular (att) and corner (art) -- with direct spoke-major offsets; all
    // operands of two rows are loaded before any arithmetic (memory-level
    // parallelism).  Same expressions as row_from, so bitwise identical.
    int ifirst = 1, ilast = len - 2;  // rows 0 (s = split) and len-1 (s = n_r-1) below
    if (L.rows) {  // assembled rows (k_rows): every row the same ten products
        const double* Rw = L.rows + (long)b * 10 * L.n;
        const int n = L.n;
        for (int i = threadIdx.x; i < len; i += T) {
            const int s = split + i, p = base + i;
            const Nbr q = neighbours(L, s, t, p);
            double acc = F[p];
            if (s == split) acc -= Rw[1 * n + p] * ldu<CG>(&U[q.pSM]);
            acc -= Rw[3 * n + p] * ldu<CG>(&U[q.pTM]);
            acc -= Rw[4 * n + p] * ldu<CG>(&U[q.pTP]);
            acc -= Rw[5 * n + p] * ldu<CG>(&U[q.pSMTM]);
            acc -= Rw[6 * n + p] * ldu<CG>(&U[q.pSMTP]);
            acc -= Rw[7 * n + p] * ldu<CG>(&U[q.pSPTM]);
            acc -= Rw[8 * n + p] * ldu<CG>(&U[q.pSPTP]);
            Y[P(i)] = acc;
        }
        ifirst = len;
        ilast = -1;
    } else if (!ONFLY) {
        const int tm = L.tminus(t), tp = L.tplus(t);
        const double km = L.k[tm], kp = L.k[t], rkm = L.rk[tm], rkp = L.rk[t];
        const int dTM = (tm - t) * len, dTP = (tp - t) * len;
        const double* __restrict__ ATT = L.att + off;
        const double* __restrict__ ART = L.art + off;
        const int N = L.nr - 1;
#pragma unroll (kRadUnroll)
        for (int i = ifirst + threadIdx.x; i <= ilast; i += T) {
            const int s = split + i, p = base + i;
            const double fP = F[p];
            const double attP = ATT[p], attM = ATT[p + dTM], attQ = ATT[p + dTP];
            const double artM = ART[p + dTM], artQ = ART[p + dTP];
            const double artSM = ART[p - 1], artSP = ART[p + 1];
            const double uM = ldu<CG>(&U[p + dTM]), uQ = ldu<CG>(&U[p + dTP]);
            const double uMM = ldu<CG>(&U[p + dTM - 1]), uQM = ldu<CG>(&U[p + dTP - 1]);
            const double uMP = ldu<CG>(&U[p + dTM + 1]), uQP = ldu<CG>(&U[p + dTP + 1]);
            const double hbar = 0.5 * (L.h[s - 1] + L.h[s]);
            const double south = -xdiv(hbar, km, rkm) * (attP + attM);
            const double north = -xdiv(hbar, kp, rkp) * (attP + attQ);
            double acc = fP;
            acc -= south * uM;
            acc -= north * uQ;
            acc -= (-(artM + artSM) * 0.25) * uMM;
            acc -= ((artSM + artQ) * 0.25) * uQM;
            if (s + 1 < N || !L.dir(s + 1)) {  // coupling to ring s+1 kept
                acc -= ((artM + artSP) * 0.25) * uMP;
                acc -= (-(artSP + artQ) * 0.25) * uQP;
            }
            Y[P(i)] = acc;
        }
    } else {
        ifirst = len;  // Give: the general path below handles every row
        ilast = -1;
    }
    for (int i = threadIdx.x; i < len && !L.rows; i += T) {
        if (i >= ifirst && i <= ilast) continue;
        const int s = split + i;
        const int p = base + i;
        if (L.dir(s)) {
            Y[P(i)] = F[p];
            continue;
        }
        const Nbr q = neighbours(L, s, t, p);
        const Row R = make_row_fast(L, cf, s, t, p, q);
        double acc = F[p];
        if (s == split && R.has_sm) acc -= R.sm * ldu<CG>(&U[q.pSM]);
        acc -= R.tm * ldu<CG>(&U[q.pTM]);
        acc -= R.tp * ldu<CG>(&U[q.pTP]);
        if (R.has_sm) {
            acc -= R.mm * ldu<CG>(&U[q.pSMTM]);
            acc -= R.mp * ldu<CG>(&U[q.pSMTP]);
        }
        if (R.has_sp) {
            acc -= R.pm * ldu<CG>(&U[q.pSPTM]);
            acc -= R.pp * ldu<CG>(&U[q.pSPTP]);
        }
        Y[P(i)] = acc;
    }
    __pipeline_wait_prior(0);
    if (!serial)  // each thread converts the factor elements it copied
        for (int i = threadIdx.x; i < len; i += T) IL[P(i)] = __drcp_rn(IL[P(i)]);
    else if (serial == 1)
        for (int i = threadIdx.x; i < len; i += T) RC[P(i)] = __drcp_rn(IL[P(i)]);
    KT(2);
    __syncthreads();
    KT(3);
    if (serial == 1) {
        // 8 rows per solving thread where the CTA covers the line that way
        // (shorter dependent chains: c1 10.5 -> 9.5 ms), else 16
        if (len <= 8 * T)
            line_solve_ex<8, false>(Y, IL, RC, M, len, 0.0, nullptr, scr);
        else
            line_solve_ex<kExChunk, false>(Y, IL, RC, M, len, 0.0, nullptr, scr);
    } else if (serial == 3) {
        line_solve_ex<kExChunk, false, true>(Y, IL, nullptr, M, len, 0.0, nullptr, scr);
    } else if (serial) {
        if (threadIdx.x == 0) tri_solve_exact(Y, IL, M, len);
        __syncthreads();
    } else {
        line_solve<K, false>(Y, IL, M, len, 0.0, scr);
    }
    KT(4);
    for (int i = threadIdx.x; i < len; i += T) U[base + i] = Y[P(i)];
    KT(5);}
template <bool ONFLY, int K>
__global__ void __launch_bounds__(512) k_radial(LevelView L, double* __restrict__ u,
                                                const double* __restrict__ f,
                                                const double* __restrict__ ril,
                                                const double* __restrict__ rm, int parity,
                                                int serial, const int* __restrict__ active) {
    KT(0);
    pdl_enter();
    extern __shared__ double smem[];
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    radial_body<ONFLY, K, false>(L, u, f, ril, rm, serial, b, parity + 2 * blockIdx.x, smem,
                                 [] {});
}

// ------------------------------------------------- cluster-split line solves
// A long smoother line is split over a thread-block cluster of C CTAs (rows
// [r*R, r*R+R) on rank r).  Each CTA scans its chunk carries in-block
// (block_scan_ex), then the CTA composites are composed across the cluster
// through distributed shared memory, so shared memory per CTA shrinks by C and
// several lines run per SM (the single-CTA line kernels hold one 6889-row
// line per SM at 8193x8192).

// Block scan returning, per thread, the exclusive prefix map (Aex, Bex) of the
// earlier chunks of this CTA (scan order) and the CTA total (At, Bt).
template <int NV, bool FWD>
__device__ __forceinline__ void block_scan_ex(double A, double (&B)[NV], double& Aex,
                                              double (&Bex)[NV], double& At, double (&Bt)[NV],
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
        const int wi = FWD ? lane : nw - 1 - lane;
        double a = 1.0, bb[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) bb[v] = 0.0;
        if (lane < nw) {
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
            if (lane >= d) {
#pragma unroll
                for (int v = 0; v < NV; ++v) bb[v] = a * bo[v] + bb[v];
                a = a * ao;
            }
        }
        if (lane < nw) {
            scr[wi * (NV + 1)] = a;
#pragma unroll
            for (int v = 0; v < NV; ++v) scr[wi * (NV + 1) + 1 + v] = bb[v];
        }
    }
    __syncthreads();
    const int pw = FWD ? warp - 1 : warp + 1;
    double pA = 1.0, pB[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) pB[v] = 0.0;
    if (pw >= 0 && pw < nw) {
        pA = scr[pw * (NV + 1)];
#pragma unroll
        for (int v = 0; v < NV; ++v) pB[v] = scr[pw * (NV + 1) + 1 + v];
    }
    const double fA = A * pA;
    const double qa = FWD ? __shfl_up_sync(FULL, fA, 1) : __shfl_down_sync(FULL, fA, 1);
    const bool first = lane == (FWD ? 0 : 31);
    Aex = first ? pA : qa;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const double fB = A * pB[v] + B[v];
        const double qb = FWD ? __shfl_up_sync(FULL, fB, 1) : __shfl_down_sync(FULL, fB, 1);
        Bex[v] = first ? pB[v] : qb;
    }
    const int last = FWD ? nw - 1 : 0;  // last warp in scan order holds the CTA total
    At = scr[last * (NV + 1)];
#pragma unroll
    for (int v = 0; v < NV; ++v) Bt[v] = scr[last * (NV + 1) + 1 + v];
    __syncthreads();
}

// Cluster exchange of the line solves without cluster barriers: each CTA
// pushes its chunk total into a slot of every CTA that needs it with st.async
// (DSMEM store whose bytes complete a transaction count on the destination's
// mbarrier) and waits only on its own mbarrier for the totals it needs (the
// earlier ranks forward, the later ranks backward, the two end rows for the
// Sherman-Morrison correction).  Every CTA receives everything it waits for
// before it exits, so no CTA is written after exit.  (A cluster barrier
// compiles to a GPU-scope MEMBAR plus an L1 invalidate; three of them per line
// were the largest stall of the clustered line kernels.)
struct ClX {
    double slot[2][8][4];         // [forward/backward][rank] = A, B0, B1
    double ends[4];               // x0, z0, x_last, z_last
    unsigned long long bar[3];    // forward, backward, ends
};
__device__ __forceinline__ unsigned mapa(const void* p, int rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async2(unsigned raddr, double a, double b, unsigned rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
        "d"(a), "d"(b), "r"(rbar)
        : "memory");
}
__device__ __forceinline__ void st_async1(unsigned raddr, double a, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr),
                 "d"(a), "r"(rbar)
                 : "memory");
}
// At kernel start (all threads): barriers armed with the bytes this CTA will
// receive, then a cluster arrive; clx_ready() (the matching wait) must run
// before the first push -- call it after the rhs gather so its latency hides.
template <int NV, bool CYC>
__device__ __forceinline__ void clx_init(ClX& x) {
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank(), C = cl.num_blocks();
    constexpr unsigned push = NV == 1 ? 16u : 24u;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 3; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&x.bar[i])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // the single pending arrival gates each phase, so bytes may land
        // before their expect-tx (the tx-count may go transiently negative)
        mbar_arrive_tx(&x.bar[0], push * rank);
        mbar_arrive_tx(&x.bar[1], push * (C - 1 - rank));
        if (CYC) mbar_arrive_tx(&x.bar[2], 16u * ((rank != 0) + (rank != C - 1)));
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void clx_ready() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int NV, bool FWD>
__device__ __forceinline__ void cluster_carry(double At, const double (&Bt)[NV], ClX& x,
                                              double (&carry)[NV]) {
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank(), C = cl.num_blocks();
    const int bank = FWD ? 0 : 1;
    const int q = threadIdx.x;
    if (q < C && (FWD ? q > rank : q < rank)) {
        const unsigned ra = mapa(&x.slot[bank][rank][0], q), rb = mapa(&x.bar[bank], q);
        st_async2(ra, At, Bt[0], rb);
        if (NV == 2) st_async1(ra + 16, Bt[NV - 1], rb);
    }
    // one warp spins on the mbarrier, the others sleep in the block barrier
    if (threadIdx.x < 32 && (FWD ? rank > 0 : rank < C - 1)) mbar_wait(&x.bar[bank], 0);
    __syncthreads();
#pragma unroll
    for (int v = 0; v < NV; ++v) carry[v] = 0.0;
    if (FWD) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
            if (r < rank) {
                const double a = x.slot[0][r][0];
#pragma unroll
                for (int v = 0; v < NV; ++v) carry[v] = a * carry[v] + x.slot[0][r][1 + v];
            }
    } else {
#pragma unroll
        for (int r = 7; r >= 0; --r)
            if (r > rank && r < C) {
                const double a = x.slot[1][r][0];
#pragma unroll
                for (int v = 0; v < NV; ++v) carry[v] = a * carry[v] + x.slot[1][r][1 + v];
            }
    }
}


// Pull variant (radial lines, measured faster there): each CTA publishes its
// total locally, one cluster barrier, remote loads of the earlier (later)
// ranks' slots; the backward pass ends with a barrier so no CTA exits while
// its slot is read.
template <int NV, bool FWD>
__device__ __forceinline__ void cluster_carry_pull(double At, const double (&Bt)[NV], ClX& x,
                                                   double (&carry)[NV]) {
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank(), C = cl.num_blocks();
    double* slot = &x.slot[FWD ? 0 : 1][0][0];
    if (threadIdx.x == 0) {
        slot[0] = At;
#pragma unroll
        for (int v = 0; v < NV; ++v) slot[1 + v] = Bt[v];
    }
    cl.sync();
    double ra[8], rb[8][NV];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const bool use = FWD ? r < rank : (r > rank && r < C);
        ra[r] = 1.0;
#pragma unroll
        for (int v = 0; v < NV; ++v) rb[r][v] = 0.0;
        if (use) {
            const double* q = cl.map_shared_rank(slot, r);
            ra[r] = q[0];
#pragma unroll
            for (int v = 0; v < NV; ++v) rb[r][v] = q[1 + v];
        }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) carry[v] = 0.0;
    if (FWD) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int v = 0; v < NV; ++v) carry[v] = ra[r] * carry[v] + rb[r][v];
    } else {
#pragma unroll
        for (int r = 7; r >= 0; --r)
#pragma unroll
            for (int v = 0; v < NV; ++v) carry[v] = ra[r] * carry[v] + rb[r][v];
        cl.sync();
    }
}

// seg: rows per independent line when the cluster holds two lines back to
// back (ntot = 2 seg; the recurrences restart at row seg), else ntot.
// Circle (CYC) lines exchange chunk totals by st.async pushes, radial lines
// by the pull variant (each measured faster on its own lines).
template <int K, bool CYC>
__device__ __forceinline__ void line_solve_cl(double* Y, const double* IL, const double* Mx,
                                              int nloc, int row0, int ntot, double corner,
                                              double* scr, ClX& xch, int seg) {
    auto first = [&](int g) { return g == 0 || g == seg; };
    auto last = [&](int g) { return g == seg - 1 || g == ntot - 1; };
    constexpr int NV = CYC ? 2 : 1;
    const int j0 = threadIdx.x * K;
    double y[K], z[CYC ? K : 1];
    double A = 1.0, Bv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) Bv[v] = 0.0;
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const int j = j0 + q, g = row0 + j;
        if (j < nloc) {
            const double il = IL[P(j)];
            const double a = !first(g) ? -(Mx[P(j)] * il) : 0.0;
            const double b = Y[P(j)];
            y[q] = b;
            Bv[0] = a * Bv[0] + b * il;
            if (CYC) Bv[NV - 1] = a * Bv[NV - 1] + ((g == 0 || g == ntot - 1) ? il : 0.0);
            A = a * A;
        }
    }
    double Aex, Bex[NV], At, Bt[NV], carry[NV];
    block_scan_ex<NV, true>(A, Bv, Aex, Bex, At, Bt, scr);
    if (CYC) cluster_carry<NV, true>(At, Bt, xch, carry); else cluster_carry_pull<NV, true>(At, Bt, xch, carry);
    {
        double yp = Aex * carry[0] + Bex[0], zp = Aex * carry[NV - 1] + Bex[NV - 1];
#pragma unroll
        for (int q = 0; q < K; ++q) {
            const int j = j0 + q, g = row0 + j;
            if (j < nloc) {
                const double il = IL[P(j)];
                const double mp = !first(g) ? Mx[P(j)] : 0.0;
                yp = (y[q] - mp * yp) * il;
                y[q] = yp;
                if (CYC) {
                    zp = (((g == 0 || g == ntot - 1) ? 1.0 : 0.0) - mp * zp) * il;
                    z[CYC ? q : 0] = zp;
                }
            }
        }
    }
    double G = 1.0, Dv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) Dv[v] = 0.0;
#pragma unroll
    for (int q = K - 1; q >= 0; --q) {
        const int j = j0 + q, g = row0 + j;
        if (j < nloc) {
            const double il = IL[P(j)];
            const double gg = !last(g) ? -(Mx[P(j + 1)] * il) : 0.0;
            Dv[0] = gg * Dv[0] + y[q] * il;
            if (CYC) Dv[NV - 1] = gg * Dv[NV - 1] + z[CYC ? q : 0] * il;
            G = gg * G;
        }
    }
    block_scan_ex<NV, false>(G, Dv, Aex, Bex, At, Bt, scr);
    if (CYC) cluster_carry<NV, false>(At, Bt, xch, carry); else cluster_carry_pull<NV, false>(At, Bt, xch, carry);
    {
        double xp = Aex * carry[0] + Bex[0], zq = Aex * carry[NV - 1] + Bex[NV - 1];
#pragma unroll
        for (int q = K - 1; q >= 0; --q) {
            const int j = j0 + q, g = row0 + j;
            if (j < nloc) {
                const double il = IL[P(j)];
                const double mj = !last(g) ? Mx[P(j + 1)] : 0.0;
                xp = (y[q] - mj * xp) * il;
                y[q] = xp;
                if (CYC) {
                    zq = (z[CYC ? q : 0] - mj * zq) * il;
                    z[CYC ? q : 0] = zq;
                }
            }
        }
    }
    if (CYC) {
        // x, z at global rows 0 (rank 0) and ntot-1 (last rank), pushed into
        // every CTA of the cluster
        cg::cluster_group cl = cg::this_cluster();
        const int C = cl.num_blocks(), rank = cl.block_rank();
        double* ends = xch.ends;
#pragma unroll
        for (int q = 0; q < K; ++q) {
            const int j = j0 + q, g = row0 + j;
            if (j < nloc && (g == 0 || g == ntot - 1)) {
                const int e = g == 0 ? 0 : 2;
                ends[e] = y[q];
                ends[e + 1] = z[CYC ? q : 0];
                for (int r = 0; r < C; ++r)
                    if (r != rank)
                        st_async2(mapa(&ends[e], r), y[q], z[CYC ? q : 0], mapa(&xch.bar[2], r));
            }
        }
        if (threadIdx.x < 32) mbar_wait(&xch.bar[2], 0);  // C > 1: at least one end row arrives
        __syncthreads();  // (and this CTA's own end rows are written)
        const double tau = corner * (ends[0] + ends[2]) / (1.0 + corner * (ends[1] + ends[3]));
#pragma unroll
        for (int q = 0; q < K; ++q) y[q] -= tau * z[CYC ? q : 0];
    }
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const int j = j0 + q;
        if (j < nloc) Y[P(j)] = y[q];
    }
    __syncthreads();
}

inline __device__ int cl_rows(int n, int C) {  // rows per CTA
    return (n + C - 1) / C;
}

// Radial sweep with each spoke split over a cluster (fast mode, Take).
template <int K>
__global__ void __launch_bounds__(256, PMG_CL_MINB) k_radial_cl(LevelView L, double* __restrict__ u,
                                                   const double* __restrict__ f,
                                                   const double* __restrict__ ril,
                                                   const double* __restrict__ rm, int parity,
                                                   const int* __restrict__ active) {
    pdl_enter();
    extern __shared__ double smem[];
    __shared__ ClX xch;
    cg::cluster_group cl = cg::this_cluster();
    const int C = cl.num_blocks(), rank = cl.block_rank();
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int t = parity + 2 * (blockIdx.x / C);
    const int len = L.len, split = L.split, T = blockDim.x;
    const int R = cl_rows(len, C), row0 = rank * R;
    const int nloc = min(R, len - row0);
    const long off = (long)b * L.n;
    double* U = u + off;
    const double* F = f + off;
    const int base = split * L.nt + t * len;
    const int pn = padded(R + 1);
    double* Y = smem;
    double* IL = smem + pn;
    double* Mx = IL + pn;
    double* scr = Mx + pn;
    const long fo = ((long)b * L.nt + t) * len;
    // line factors: asynchronous copies overlapped with the rhs gather
    for (int j = threadIdx.x; j < nloc; j += T)
        __pipeline_memcpy_async(&IL[P(j)], &ril[fo + row0 + j], 8);
    for (int j = threadIdx.x; j <= nloc; j += T) {
        if (row0 + j > 0)
            __pipeline_memcpy_async(&Mx[P(j)], &rm[fo + row0 + j - 1], 8);
        else
            Mx[P(j)] = 0.0;
    }
    __pipeline_commit();
    const int tm = L.tminus(t), tp = L.tplus(t);
    const double km = L.k[tm], kp = L.k[t], rkm = L.rk[tm], rkp = L.rk[t];
    const int dTM = (tm - t) * len, dTP = (tp - t) * len;
    const double* __restrict__ ATT = L.att + off;
    const double* __restrict__ ART = L.art + off;
    const int N = L.nr - 1;
    const CoefAt<false> cf{&L, off, b};
#ifdef PMG_DIAG_NOGATHER
    for (int j = threadIdx.x; j < nloc; j += T) Y[P(j)] = F[base + row0 + j];
    if (false)
#endif
#pragma unroll 2
    for (int j = threadIdx.x; j < nloc; j += T) {
        const int i = row0 + j, s = split + i, p = base + i;
        double acc;
        if (i > 0 && s < N) {
            const double fP = F[p];
            const double attP = ATT[p], attM = ATT[p + dTM], attQ = ATT[p + dTP];
            const double artM = ART[p + dTM], artQ = ART[p + dTP];
            const double artSM = ART[p - 1], artSP = ART[p + 1];
            const double uM = U[p + dTM], uQ = U[p + dTP];
            const double uMM = U[p + dTM - 1], uQM = U[p + dTP - 1];
            const double uMP = U[p + dTM + 1], uQP = U[p + dTP + 1];
            const double hbar = 0.5 * (L.h[s - 1] + L.h[s]);
            const double south = -xdiv(hbar, km, rkm) * (attP + attM);
            const double north = -xdiv(hbar, kp, rkp) * (attP + attQ);
            acc = fP;
            acc -= south * uM;
            acc -= north * uQ;
            acc -= (-(artM + artSM) * 0.25) * uMM;
            acc -= ((artSM + artQ) * 0.25) * uQM;
            if (s + 1 < N || !L.dir(s + 1)) {
                acc -= ((artM + artSP) * 0.25) * uMP;
                acc -= (-(artSP + artQ) * 0.25) * uQP;
            }
        } else if (L.dir(s)) {
            acc = F[p];
        } else {
            const Nbr q = neighbours(L, s, t, p);
            const Row R2 = make_row_fast(L, cf, s, t, p, q);
            acc = F[p];
            if (s == split && R2.has_sm) acc -= R2.sm * U[q.pSM];
            acc -= R2.tm * U[q.pTM];
            acc -= R2.tp * U[q.pTP];
            if (R2.has_sm) {
                acc -= R2.mm * U[q.pSMTM];
                acc -= R2.mp * U[q.pSMTP];
            }
            if (R2.has_sp) {
                acc -= R2.pm * U[q.pSPTM];
                acc -= R2.pp * U[q.pSPTP];
            }
        }
        Y[P(j)] = acc;
    }
    __pipeline_wait_prior(0);
    for (int j = threadIdx.x; j < nloc; j += T) IL[P(j)] = __drcp_rn(IL[P(j)]);
    __syncthreads();
#ifndef PMG_DIAG_NOSOLVE
    line_solve_cl<K, false>(Y, IL, Mx, nloc, row0, len, 0.0, scr, xch, len);
#endif
    for (int j = threadIdx.x; j < nloc; j += T) U[base + row0 + j] = Y[P(j)];
}

// Circle sweep with each ring split over a cluster (fast mode); rings
// s = s_first + 2*line; the across-origin ring is launched separately.
template <bool ONFLY, int K>
__global__ void __launch_bounds__(256, PMG_CL_MINB) k_circle_cl(LevelView L, double* __restrict__ u,
                                                   const double* __restrict__ f,
                                                   const double* __restrict__ cil,
                                                   const double* __restrict__ cm,
                                                   const double* __restrict__ corner, int s_first,
                                                   const int* __restrict__ active) {
    pdl_enter();
    extern __shared__ double smem[];
    __shared__ ClX xch;
    cg::cluster_group cl = cg::this_cluster();
    const int C = cl.num_blocks(), rank = cl.block_rank();
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int s = s_first + 2 * (blockIdx.x / C);
    const int nt = L.nt, T = blockDim.x;
    const int R = cl_rows(nt, C), row0 = rank * R;
    const int nloc = min(R, nt - row0);
    const long off = (long)b * L.n;
    double* U = u + off;
    const double* F = f + off;
    const int base = s * nt;
    if (L.dir(s)) {
        for (int j = threadIdx.x; j < nloc; j += T) U[base + row0 + j] = F[base + row0 + j];
        return;
    }
    const int pn = padded(R + 1);
    double* Y = smem;
    double* IL = smem + pn;
    double* Mx = IL + pn;
    double* scr = Mx + pn;
    const long fo = (long)b * L.split * nt + (long)s * nt;
    clx_init<2, true>(xch);
    // line factors: asynchronous copies overlapped with the rhs gather
    for (int j = threadIdx.x; j < nloc; j += T)
        __pipeline_memcpy_async(&IL[P(j)], &cil[fo + row0 + j], 8);
    for (int j = threadIdx.x; j <= nloc; j += T) {
        if (row0 + j > 0)
            __pipeline_memcpy_async(&Mx[P(j)], &cm[fo + row0 + j - 1], 8);
        else
            Mx[P(j)] = 0.0;
    }
    __pipeline_commit();
    const CoefAt<ONFLY> cf{&L, off, b};
    const bool lean = !ONFLY && circle_lean_ring(L, s);
    if (lean)
        for (int j = threadIdx.x; j < nloc; j += T)
            Y[P(j)] = circle_rhs_lean(L, off, s, row0 + j, U, F);
    else
    for (int j = threadIdx.x; j < nloc; j += T) {
        const int t = row0 + j, p = base + t;
        const Nbr q = neighbours(L, s, t, p);
        const Row R2 = make_row_fast(L, cf, s, t, p, q);
        double acc = F[p];
        if (R2.has_sm) acc -= R2.sm * U[q.pSM];
        if (R2.has_sp) acc -= R2.sp * U[q.pSP];
        if (R2.has_sm) {
            acc -= R2.mm * U[q.pSMTM];
            acc -= R2.mp * U[q.pSMTP];
        }
        if (R2.has_sp) {
            acc -= R2.pm * U[q.pSPTM];
            acc -= R2.pp * U[q.pSPTP];
        }
        Y[P(j)] = acc;
    }
    __pipeline_wait_prior(0);
    for (int j = threadIdx.x; j < nloc; j += T) IL[P(j)] = __drcp_rn(IL[P(j)]);
    __syncthreads();
    clx_ready();
    line_solve_cl<K, true>(Y, IL, Mx, nloc, row0, nt, corner[(long)b * L.split + s], scr, xch, nt);
    for (int j = threadIdx.x; j < nloc; j += T) U[base + row0 + j] = Y[P(j)];
}


// ------------------------------------------------------ fused smoothing step
// Dependencies (reference smoother.cpp:72-81 order, Gauss-Seidel in place):
// a white ring needs the black rings s-1, s+1; a black spoke needs ring
// split-1 (its row split couples to it, and ring split-1 reads row split
// before the spokes overwrite it); a white spoke needs the black spokes
// t-1, t+1.  Black rings need nothing: the white lines they read are not
// written before they are done, since those wait for them.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// polling load: relaxed (an acquire load compiles to a load + L1 invalidate,
// which on every poll iteration would wipe the L1 of all CTAs on the SM);
// the waiter issues one acquire fence after its polls succeed
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acquire() {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool ONFLY, int K>
__global__ void __launch_bounds__(256, PMG_FUSED_MINB) k_smooth_fused(LevelView L, double* __restrict__ u,
                                                      const double* __restrict__ f,
                                                      const double* __restrict__ cil,
                                                      const double* __restrict__ cm,
                                                      const double* __restrict__ corner,
                                                      const double* __restrict__ cz,
                                                      OriginFactor of,
                                                      const double* __restrict__ ril,
                                                      const double* __restrict__ rm,
                                                      int exact_rings, int ex, FuseCtl fc,
                                                      const int* __restrict__ order, int nitems,
                                                      const int* __restrict__ active) {
    pdl_enter();
    extern __shared__ double smem[];
    __shared__ int s_item;
    __shared__ unsigned s_epoch;
    if (threadIdx.x == 0) {
        s_item = order[atomicAdd(&fc.ctl[0], 1u)];
        s_epoch = *reinterpret_cast<volatile unsigned*>(&fc.ctl[2]);
    }
    __syncthreads();
    const int per = L.split + L.nt;
    const int item = s_item, b = item / per, c = item - b * per;
    const unsigned ep = s_epoch;
    unsigned* flags = fc.flags + (long)b * per;
    if (!active || active[b]) {
        // the line's factors are prefetched before the wait (inside the body)
        auto wait = [&] {
        if (threadIdx.x == 0) {
            int dep[2] = {-1, -1};
            if (c < L.split) {
                if (c & 1) {  // white ring
                    dep[0] = c - 1;
                    dep[1] = c + 1 < L.split ? c + 1 : -1;
                }
            } else {
                const int t = c - L.split;
                if (t & 1) {  // white spoke
                    dep[0] = L.split + t - 1;
                    dep[1] = L.split + (t + 1 == L.nt ? 0 : t + 1);
                } else {
                    dep[0] = L.split - 1;
                }
            }
            bool waited = false;
            for (int d = 0; d < 2; ++d)
                if (dep[d] >= 0) {
                    while (ld_relaxed(&flags[dep[d]]) != ep) __nanosleep(32);
                    waited = true;
                }
            if (waited) fence_acquire();
        }
        __syncthreads();
        };
        if (c < L.split)
            circle_body<ONFLY, K, true>(L, u, f, cil, cm, corner, cz, of, ex, exact_rings, b, c,
                                        smem, wait);
        else
            radial_body<ONFLY, K, true>(L, u, f, ril, rm, ex, b, c - L.split, smem, wait);
        __syncthreads();  // every thread's stores of the line issued
        if (threadIdx.x == 0) st_release(&flags[c], ep);  // release: orders the CTA's stores
    }
    if (threadIdx.x == 0) {
        if (atomicAdd(&fc.ctl[1], 1u) == (unsigned)nitems - 1) {  // last CTA: reset for the next launch
            fc.ctl[0] = 0;
            fc.ctl[1] = 0;
            __threadfence();
            atomicAdd(&fc.ctl[2], 1u);
        }
    }
}


// ------------------------------------- two-colour radial wavefront (clusters)
// Both colours of the radial sweep of a level with clustered spokes in ONE
// launch.  Each cluster (one spoke, C CTAs of ~862 rows) takes the next spoke
// from a ticket counter in a host-built order in which every white spoke
// t = 2j+1 comes `lag` black spokes after black spoke 2j+2; CTA rank r of a
// white spoke waits for the epoch-stamped completion flags of chunks r-1..r+1
// of black spokes t-1 and t+1 (the rows its gather reads), then gathers
// (u through L2), solves and stamps its own chunk flag.  Black spokes wait for
// nothing (the white spokes they read are not written before they are done).
// A white spoke's own coefficients and its neighbours' were read by the black
// spokes shortly before, so its gather hits L2: 72 -> ~52 B/node of DRAM
// traffic for the B+W pair, and no kernel boundary between the colours.
template <int K>
__global__ void __launch_bounds__(256, PMG_CL_MINB) k_radial_wave(LevelView L, double* __restrict__ u,
                                                     const double* __restrict__ f,
                                                     const double* __restrict__ ril,
                                                     const double* __restrict__ rm,
                                                     FuseCtl fc, const int* __restrict__ order,
                                                     int nctas) {
    pdl_enter();
    extern __shared__ double smem[];
    __shared__ ClX xch;
    __shared__ int s_t;
    __shared__ unsigned s_ep;
    cg::cluster_group cl = cg::this_cluster();
    const int C = cl.num_blocks(), rank = cl.block_rank();
    if (rank == 0 && threadIdx.x == 0) {
        s_t = order[atomicAdd(&fc.ctl[0], 1u)];
        s_ep = *reinterpret_cast<volatile unsigned*>(&fc.ctl[2]);
    }
    cl.sync();
    const int t = *cl.map_shared_rank(&s_t, 0);
    const unsigned ep = *cl.map_shared_rank(&s_ep, 0);
    const int b = 0;
    const int len = L.len, split = L.split, T = blockDim.x;
    const int R = cl_rows(len, C), row0 = rank * R;
    const int nloc = min(R, len - row0);
    double* U = u;
    const double* F = f;
    const int base = split * L.nt + t * len;
    const int pn = padded(R + 1);
    double* Y = smem;
    double* IL = smem + pn;
    double* Mx = IL + pn;
    double* scr = Mx + pn;
    const long fo = ((long)b * L.nt + t) * len;
    for (int j = threadIdx.x; j < nloc; j += T)
        __pipeline_memcpy_async(&IL[P(j)], &ril[fo + row0 + j], 8);
    for (int j = threadIdx.x; j <= nloc; j += T) {
        if (row0 + j > 0)
            __pipeline_memcpy_async(&Mx[P(j)], &rm[fo + row0 + j - 1], 8);
        else
            Mx[P(j)] = 0.0;
    }
    __pipeline_commit();
    const int tm = L.tminus(t), tp = L.tplus(t);
    if (t & 1) {  // white: black neighbours' chunks r-1..r+1 done
        if (threadIdx.x < 6) {
            const int nb = threadIdx.x < 3 ? tm : tp;
            const int r = rank - 1 + (threadIdx.x % 3);
            if (r >= 0 && r < C)
                while (ld_acquire(&fc.flags[nb * C + r]) != ep) __nanosleep(64);
        }
        __syncthreads();
    }
    const double km = L.k[tm], kp = L.k[t], rkm = L.rk[tm], rkp = L.rk[t];
    const int dTM = (tm - t) * len, dTP = (tp - t) * len;
    const double* __restrict__ ATT = L.att;
    const double* __restrict__ ART = L.art;
    const int N = L.nr - 1;
    const CoefAt<false> cf{&L, 0, b};
#pragma unroll 2
    for (int j = threadIdx.x; j < nloc; j += T) {
        const int i = row0 + j, s = split + i, p = base + i;
        double acc;
        if (i > 0 && s < N) {
            const double fP = F[p];
            const double attP = ATT[p], attM = ATT[p + dTM], attQ = ATT[p + dTP];
            const double artM = ART[p + dTM], artQ = ART[p + dTP];
            const double artSM = ART[p - 1], artSP = ART[p + 1];
            const double uM = ldu<true>(&U[p + dTM]), uQ = ldu<true>(&U[p + dTP]);
            const double uMM = ldu<true>(&U[p + dTM - 1]), uQM = ldu<true>(&U[p + dTP - 1]);
            const double uMP = ldu<true>(&U[p + dTM + 1]), uQP = ldu<true>(&U[p + dTP + 1]);
            const double hbar = 0.5 * (L.h[s - 1] + L.h[s]);
            const double south = -xdiv(hbar, km, rkm) * (attP + attM);
            const double north = -xdiv(hbar, kp, rkp) * (attP + attQ);
            acc = fP;
            acc -= south * uM;
            acc -= north * uQ;
            acc -= (-(artM + artSM) * 0.25) * uMM;
            acc -= ((artSM + artQ) * 0.25) * uQM;
            if (s + 1 < N || !L.dir(s + 1)) {
                acc -= ((artM + artSP) * 0.25) * uMP;
                acc -= (-(artSP + artQ) * 0.25) * uQP;
            }
        } else if (L.dir(s)) {
            acc = F[p];
        } else {
            const Nbr q = neighbours(L, s, t, p);
            const Row R2 = make_row_fast(L, cf, s, t, p, q);
            acc = F[p];
            if (s == split && R2.has_sm) acc -= R2.sm * ldu<true>(&U[q.pSM]);
            acc -= R2.tm * ldu<true>(&U[q.pTM]);
            acc -= R2.tp * ldu<true>(&U[q.pTP]);
            if (R2.has_sm) {
                acc -= R2.mm * ldu<true>(&U[q.pSMTM]);
                acc -= R2.mp * ldu<true>(&U[q.pSMTP]);
            }
            if (R2.has_sp) {
                acc -= R2.pm * ldu<true>(&U[q.pSPTM]);
                acc -= R2.pp * ldu<true>(&U[q.pSPTP]);
            }
        }
        Y[P(j)] = acc;
    }
    __pipeline_wait_prior(0);
    for (int j = threadIdx.x; j < nloc; j += T) IL[P(j)] = __drcp_rn(IL[P(j)]);
    __syncthreads();
    line_solve_cl<K, false>(Y, IL, Mx, nloc, row0, len, 0.0, scr, xch, len);
    for (int j = threadIdx.x; j < nloc; j += T) U[base + row0 + j] = Y[P(j)];
    __syncthreads();  // every thread's stores of the chunk issued
    if (threadIdx.x == 0) {
        __threadfence();
        st_release(&fc.flags[t * C + rank], ep);
        if (atomicAdd(&fc.ctl[1], 1u) == (unsigned)nctas - 1) {  // last CTA: reset
            fc.ctl[0] = 0;
            fc.ctl[1] = 0;
            __threadfence();
            atomicAdd(&fc.ctl[2], 1u);
        }
    }
}

// ---------------------------------------------------------------- transfers
// restrict_transpose (interpolation.cpp:97-143) fused with
// mask_dirichlet_rows (multigrid.cpp:146-153) and the coarse u = 0 (:204).
// Loads of vectors another CTA of the same kernel may have written (the
// cluster-wide multigrid kernel) bypass L1: ld.global.cg.
template <bool CG>
__device__ __forceinline__ double ldv(const double* p) {
    if (CG) return __ldcg(p);
    return *p;
}

template <bool CG = false>
__device__ __forceinline__ void restrict_node(const LevelView& F, const LevelView& C,
                                              const Weights& w, const double* __restrict__ R,
                                              double* __restrict__ cf, double* __restrict__ cu,
                                              int mask, int pc) {
    int sc, tc;
    C.node(pc, sc, tc);
    const int sf = 2 * sc, tf = 2 * tc;
    const int tdn = tf == 0 ? F.nt - 1 : tf - 1;
    const int tup = tf + 1;
    double acc = ldv<CG>(R + F.idx(sf, tf));
    if (sf > 0) acc += w.rwa[sf - 1] * ldv<CG>(R + F.idx(sf - 1, tf));
    if (sf < F.nr - 1) acc += w.rwb[sf + 1] * ldv<CG>(R + F.idx(sf + 1, tf));
    acc += w.awa[tdn] * ldv<CG>(R + F.idx(sf, tdn));
    acc += w.awb[tup] * ldv<CG>(R + F.idx(sf, tup));
    if (sf > 0) {
        acc += w.rwa[sf - 1] * w.awa[tdn] * ldv<CG>(R + F.idx(sf - 1, tdn));
        acc += w.rwa[sf - 1] * w.awb[tup] * ldv<CG>(R + F.idx(sf - 1, tup));
    }
    if (sf < F.nr - 1) {
        acc += w.rwb[sf + 1] * w.awa[tdn] * ldv<CG>(R + F.idx(sf + 1, tdn));
        acc += w.rwb[sf + 1] * w.awb[tup] * ldv<CG>(R + F.idx(sf + 1, tup));
    }
    if (mask && C.dir(sc)) acc = 0.0;
    cf[pc] = acc;
    if (cu) cu[pc] = 0.0;
}

// restrict_transpose (interpolation.cpp:97-143) fused with
// mask_dirichlet_rows (multigrid.cpp:146-153) and the coarse u = 0 (:204).
__global__ void __launch_bounds__(256) k_restrict(LevelView F, LevelView C, Weights w,
                                                  const double* __restrict__ fr,
                                                  double* __restrict__ cf,
                                                  double* __restrict__ cu, int mask,
                                                  const int* __restrict__ active) {
    pdl_enter();
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int pc = blockIdx.x * blockDim.x + threadIdx.x;
    if (pc >= C.n) return;
    restrict_node(F, C, w, fr + (long)b * F.n, cf + (long)b * C.n,
                  cu ? cu + (long)b * C.n : nullptr, mask, pc);
}

template <bool ADD, bool CG = false>
__device__ __forceinline__ void prolong_node(const LevelView& F, const LevelView& C,
                                             const Weights& w, const double* __restrict__ X,
                                             double* __restrict__ Y, int p) {
    int sf, tf;
    F.node(p, sf, tf);
    const bool ro = sf & 1, so = tf & 1;
    const int sc = sf >> 1, tc = tf >> 1;
    const int tcu = tc + 1 == C.nt ? 0 : tc + 1;
    double v;
    if (!ro && !so) {
        v = ldv<CG>(X + C.idx(sc, tc));
    } else if (ro && !so) {
        v = w.rwb[sf] * ldv<CG>(X + C.idx(sc, tc)) + w.rwa[sf] * ldv<CG>(X + C.idx(sc + 1, tc));
    } else if (!ro && so) {
        v = w.awb[tf] * ldv<CG>(X + C.idx(sc, tc)) + w.awa[tf] * ldv<CG>(X + C.idx(sc, tcu));
    } else {
        const double wb = w.rwb[sf], wa = w.rwa[sf], vb = w.awb[tf], va = w.awa[tf];
        v = wb * vb * ldv<CG>(X + C.idx(sc, tc)) + wb * va * ldv<CG>(X + C.idx(sc, tcu)) +
            wa * vb * ldv<CG>(X + C.idx(sc + 1, tc)) + wa * va * ldv<CG>(X + C.idx(sc + 1, tcu));
    }
    if (ADD)
        Y[p] = ldv<CG>(Y + p) + v;
    else
        Y[p] = v;
}

// prolongate(_add) (interpolation.cpp:38-95)
template <bool ADD>
__global__ void __launch_bounds__(256) k_prolong(LevelView F, LevelView C, Weights w,
                                                 const double* __restrict__ cu,
                                                 double* __restrict__ fu,
                                                 const int* __restrict__ active) {
    pdl_enter();
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= F.n) return;
    prolong_node<ADD>(F, C, w, cu + (long)b * C.n, fu + (long)b * F.n, p);
}

__device__ __forceinline__ void env_solve(const EnvFactor& E, int b, double* __restrict__ x) {
    const int n = E.n;
    const double* Lb = E.L + (long)b * E.nnz;
    const double* D = E.D + (long)b * n;
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

// coarsest-level direct solve: u = f; envelope LDL^T solve
// (multigrid.cpp:183-187, line_algebra.cpp:211-255), one thread per section.
__global__ void k_coarse(EnvFactor E, const double* __restrict__ f, double* __restrict__ u,
                         int B, const int* __restrict__ active) {
    pdl_enter();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B || (active && !active[b])) return;
    double* x = u + (long)b * E.n;
    for (int i = 0; i < E.n; ++i) x[i] = f[(long)b * E.n + i];
    env_solve(E, b, x);
}

// ------------------------------------------------------- coarse-level cycle
// Below a size threshold every multigrid phase of a level is a few
// microseconds of latency, so the whole sub-cycle of the coarse levels runs in
// ONE launch: one block per section walks a host-generated op program
// (smooth / residual / restrict / prolongate / coarsest solve, the exact
// sequence of multigrid.cpp:189-220) with __syncthreads between phases.
// Smoother lines are solved one per warp: each lane owns kWK consecutive rows,
// the chunk carries are scanned with warp shuffles (no shared memory).
// KW = rows per lane (1, 2, 4 or 8: lines up to 32*KW nodes) is a template
// parameter so the kernel carries only the code of its own line length (the
// one-block tail is instruction-fetch bound when the code is large).

__device__ __forceinline__ void warp_scan2(Map2 a, bool fwd, double& in0, double& in1) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const Map2 o = shfl2(a, d, fwd);
        if (fwd ? (lane >= d) : (lane + d < 32)) a = compose2(a, o);
    }
    const double q0 = fwd ? __shfl_up_sync(FULL, a.c0, 1) : __shfl_down_sync(FULL, a.c0, 1);
    const double q1 = fwd ? __shfl_up_sync(FULL, a.c1, 1) : __shfl_down_sync(FULL, a.c1, 1);
    const bool first = lane == (fwd ? 0 : 31);
    in0 = first ? 0.0 : q0;
    in1 = first ? 0.0 : q1;
}

// Warp solve of L L^T x = y (+ Sherman-Morrison when CYC); y[] holds the
// lane's rows [lane*KW, +KW) on entry and the solution on exit.  Ld: raw L
// diagonal, Mo: sub-diagonal, both global (this line).
template <bool CYC, int KW>
__device__ __forceinline__ void warp_line_solve(double (&y)[KW], const double* __restrict__ Ld,
                                                const double* __restrict__ Mo, int n,
                                                double corner) {
    constexpr int NV = CYC ? 2 : 1;
    const int KE = (n + 31) >> 5;  // rows per lane (<= KW)
    const int j0 = (threadIdx.x & 31) * KE;
    double il[KW], mprev[KW], z[CYC ? KW : 1];
    double A = 1.0, Bv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) Bv[v] = 0.0;
#pragma unroll
    for (int q = 0; q < KW; ++q) {
        const int j = j0 + q;
        const bool in = q < KE && j < n;
        il[q] = in ? __drcp_rn(Ld[j]) : 0.0;
        mprev[q] = (in && j > 0) ? Mo[j - 1] : 0.0;
        if (in) {
            const double a = -(mprev[q] * il[q]);
            Bv[0] = a * Bv[0] + y[q] * il[q];
            if (CYC) Bv[NV - 1] = a * Bv[NV - 1] + ((j == 0 || j == n - 1) ? il[q] : 0.0);
            A = a * A;
        }
    }
    double yin[NV];
    warp_scan<NV, true>(A, Bv, yin);
    double yp = yin[0], zp = yin[NV - 1];
#pragma unroll
    for (int q = 0; q < KW; ++q) {
        if (q < KE && j0 + q < n) {
            yp = (y[q] - mprev[q] * yp) * il[q];
            y[q] = yp;
            if (CYC) {
                const int j = j0 + q;
                zp = (((j == 0 || j == n - 1) ? 1.0 : 0.0) - mprev[q] * zp) * il[q];
                z[CYC ? q : 0] = zp;
            }
        }
    }
    double G = 1.0, Dv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) Dv[v] = 0.0;
    double mj[KW];  // m_j couples row j to j+1
#pragma unroll
    for (int q = 0; q < KW; ++q) {
        const int j = j0 + q;
        mj[q] = (q < KE && j < n - 1) ? Mo[j] : 0.0;
    }
#pragma unroll
    for (int q = KW - 1; q >= 0; --q) {
        if (q < KE && j0 + q < n) {
            const double g = -(mj[q] * il[q]);
            Dv[0] = g * Dv[0] + y[q] * il[q];
            if (CYC) Dv[NV - 1] = g * Dv[NV - 1] + z[CYC ? q : 0] * il[q];
            G = g * G;
        }
    }
    double xin[NV];
    warp_scan<NV, false>(G, Dv, xin);
    double xp = xin[0], zq = xin[NV - 1];
#pragma unroll
    for (int q = KW - 1; q >= 0; --q) {
        if (q < KE && j0 + q < n) {
            xp = (y[q] - mj[q] * xp) * il[q];
            y[q] = xp;
            if (CYC) {
                zq = (z[CYC ? q : 0] - mj[q] * zq) * il[q];
                z[CYC ? q : 0] = zq;
            }
        }
    }
    if (CYC) {
        // x_0, z_0 live on lane 0; x_{n-1}, z_{n-1} on lane (n-1)/KW
        const int last = (n - 1) / KE, ql = (n - 1) - last * KE;
        double xl = 0.0, zl = 0.0;
#pragma unroll
        for (int q = 0; q < KW; ++q)
            if (q == ql) {
                xl = y[q];
                zl = z[CYC ? q : 0];
            }
        const double x0 = __shfl_sync(FULL, y[0], 0), z0 = __shfl_sync(FULL, z[0], 0);
        xl = __shfl_sync(FULL, xl, last);
        zl = __shfl_sync(FULL, zl, last);
        const double tau = corner * (x0 + xl) / (1.0 + corner * (z0 + zl));
#pragma unroll
        for (int q = 0; q < KW; ++q) y[q] -= tau * z[CYC ? q : 0];
    }
}

// Warp version of line_solve_ex: the reference's exact substitution order
// (line_algebra.cpp:42-62, 98-120) by speculation within one warp -- lane l
// restarts the recurrence over lane l-1's rows from the warp scan's
// approximate value, then waves (ballots, no block barriers) recompute the
// lanes whose start differs from their predecessor's result bit for bit.
// y[]: the lane's rows [lane*KE, +KE) of the rhs on entry, the solution on
// exit; Ld / Mo: raw L diagonal / sub-diagonal; z: exact Sherman-Morrison
// vector (CYC).
template <bool CYC, int KW>
__device__ __forceinline__ void warp_line_solve_ex(double (&y)[KW], const double* __restrict__ Ld,
                                                   const double* __restrict__ Mo, int n,
                                                   double corner, const double* __restrict__ z) {
    const int KE = (n + 31) >> 5;  // rows per lane (<= KW)
    const int lane = threadIdx.x & 31, j0 = lane * KE;
    if (n <= 32) {
        // one row per lane (the coarse tail's 4..32-node lines): the
        // substitution itself, row by row, each result broadcast by a shuffle
        // -- exact by construction, and for lines this short cheaper than the
        // scan, the restart and up to n verification waves
        const bool in = lane < n;
        const double l = in ? Ld[lane] : 1.0, rc = __drcp_rn(l);
        const double mp = (in && lane > 0) ? Mo[lane - 1] : 0.0;      // m_{j-1}
        const double mn = (in && lane < n - 1) ? Mo[lane] : 0.0;      // m_j
        double v = y[0];
        if (lane == 0) v = xdiv(v, l, rc);
        for (int k = 1; k < n; ++k) {
            const double p = __shfl_sync(FULL, v, k - 1);
            if (lane == k) v = xdiv(v - mp * p, l, rc);
        }
        if (lane == n - 1) v = xdiv(v, l, rc);
        for (int k = n - 2; k >= 0; --k) {
            const double p = __shfl_sync(FULL, v, k + 1);
            if (lane == k) v = xdiv(v - mn * p, l, rc);
        }
        if (CYC) {
            const double x0 = __shfl_sync(FULL, v, 0), xl = __shfl_sync(FULL, v, n - 1);
            const double tau = corner * (x0 + xl) / (1.0 + corner * (z[0] + z[n - 1]));
            if (in) v -= tau * z[lane];
        }
        y[0] = v;
        return;
    }
    const bool live = j0 < n;
    double b[KW];
#pragma unroll
    for (int q = 0; q < KW; ++q) b[q] = y[q];
    auto row_in = [&](int q, int j) { return q < KE && j < n; };
    // forward: y_j = (b_j - m_{j-1} y_{j-1}) / l_j
    double A = 1.0, Bv[1] = {0.0};
#pragma unroll
    for (int q = 0; q < KW; ++q) {
        const int j = j0 + q;
        if (row_in(q, j)) {
            const double il = __drcp_rn(Ld[j]);
            const double a = j > 0 ? -(Mo[j - 1] * il) : 0.0;
            Bv[0] = a * Bv[0] + b[q] * il;
            A = a * A;
        }
    }
    double yin[1];
    warp_scan<1, true>(A, Bv, yin);
    auto fstep = [&](double bj, int j, double v) {
        const double l = Ld[j];
        return xdiv(j == 0 ? bj : bj - Mo[j - 1] * v, l, __drcp_rn(l));
    };
    double st;
    {
        double v = __shfl_up_sync(FULL, yin[0], 1);  // approximate value at row j0 - KE - 1
#pragma unroll
        for (int q = 0; q < KW; ++q) {
            const double bp = __shfl_up_sync(FULL, b[q], 1);
            const int j = j0 - KE + q;
            if (lane >= 1 && live && q < KE) v = fstep(bp, j, v);
        }
        st = v;
    }
    auto fchunk = [&](double v) {
#pragma unroll
        for (int q = 0; q < KW; ++q) {
            const int j = j0 + q;
            if (row_in(q, j)) {
                v = fstep(b[q], j, v);
                y[q] = v;
            }
        }
        return v;
    };
    double e = live ? fchunk(st) : 0.0;
    for (;;) {
        const double pe = __shfl_up_sync(FULL, e, 1);
        const bool bad = lane >= 1 && live && !same_bits(st, pe);
        if (!__any_sync(FULL, bad)) break;
        if (bad) {
            st = pe;
            e = fchunk(st);
        }
    }
    // backward: x_j = (y_j - m_j x_{j+1}) / l_j
#pragma unroll
    for (int q = 0; q < KW; ++q) b[q] = y[q];
    double G = 1.0, Dv[1] = {0.0};
#pragma unroll
    for (int q = KW - 1; q >= 0; --q) {
        const int j = j0 + q;
        if (row_in(q, j)) {
            const double il = __drcp_rn(Ld[j]);
            const double g = j < n - 1 ? -(Mo[j] * il) : 0.0;
            Dv[0] = g * Dv[0] + b[q] * il;
            G = g * G;
        }
    }
    double xin[1];
    warp_scan<1, false>(G, Dv, xin);
    auto bstep = [&](double yj, int j, double v) {
        const double l = Ld[j];
        return xdiv(j == n - 1 ? yj : yj - Mo[j] * v, l, __drcp_rn(l));
    };
    const bool succ = j0 + KE < n;
    {
        // approximate value at row j0 + 2 KE (lane + 1's entry); exact start
        // when lane + 1 holds row n - 1
        double v = __shfl_down_sync(FULL, xin[0], 1);
#pragma unroll
        for (int q = KW - 1; q >= 0; --q) {
            const double yn = __shfl_down_sync(FULL, b[q], 1);
            const int j = j0 + KE + q;
            if (succ && q < KE && j < n) v = bstep(yn, j, v);
        }
        st = v;
    }
    auto bchunk = [&](double v) {
#pragma unroll
        for (int q = KW - 1; q >= 0; --q) {
            const int j = j0 + q;
            if (row_in(q, j)) {
                v = bstep(b[q], j, v);
                y[q] = v;
            }
        }
        return v;
    };
    e = live ? bchunk(st) : 0.0;
    for (;;) {
        const double pe = __shfl_down_sync(FULL, e, 1);
        const bool bad = live && succ && !same_bits(st, pe);
        if (!__any_sync(FULL, bad)) break;
        if (bad) {
            st = pe;
            e = bchunk(st);
        }
    }
    if (CYC) {
        const int last = (n - 1) / KE, ql = (n - 1) - last * KE;
        double xl = 0.0;
#pragma unroll
        for (int q = 0; q < KW; ++q)
            if (q == ql) xl = y[q];
        const double x0 = __shfl_sync(FULL, y[0], 0);
        xl = __shfl_sync(FULL, xl, last);
        const double tau = corner * (x0 + xl) / (1.0 + corner * (z[0] + z[n - 1]));
#pragma unroll
        for (int q = 0; q < KW; ++q)
            if (row_in(q, j0 + q)) y[q] -= tau * z[j0 + q];
    }
}

// Across-origin ring of a tail level in the reference's exact order
// (line_algebra.cpp:211-255 with the interleaved permutation of
// smoother.cpp:42-46), one warp, in place on ring 0 of U (natural order):
// the two recurrence chains run redundantly on every lane with the operands
// of 32 rows preloaded and broadcast by shuffles; diagonal scaling and the
// dense rows' column updates are per element.
__device__ void origin_exact_warp(double* X, const OriginFactor& of, int b, int n) {
    const long o = (long)b * n;
    const double* __restrict__ b1 = of.band1 + o;
    const double* __restrict__ b2 = of.band2 + o;
    const double* __restrict__ r1 = of.row1 + o;
    const double* __restrict__ r2 = of.row2 + o;
    const double* __restrict__ D = of.D + o;
    const int h = n / 2, nb = n - 2, lane = threadIdx.x & 31;
    {
        const int fc1 = of.fc1, fc2 = of.fc2;
        double zm2 = 0.0, zm1 = 0.0;
        double s1 = X[operm(n - 2, h)], s2 = X[operm(n - 1, h)];
        for (int g = 0; g < nb; g += 32) {
            const int i_l = g + lane;
            const bool ok = i_l < nb;
            const double y_l = ok ? X[operm(i_l, h)] : 0.0;
            const double b1_l = ok ? b1[i_l] : 0.0, b2_l = ok ? b2[i_l] : 0.0;
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
            __syncwarp();
            if (ok) X[operm(i_l, h)] = res;
        }
        __syncwarp();
        if (lane == 0) {
            if (n - 2 >= fc2) s2 -= r2[n - 2] * s1;
            X[operm(n - 2, h)] = s1;
            X[operm(n - 1, h)] = s2;
        }
    }
    __syncwarp();
    for (int i = lane; i < n; i += 32) X[operm(i, h)] /= D[i];
    __syncwarp();
    if (lane == 0 && n - 2 >= of.fc2) X[operm(n - 2, h)] -= r2[n - 2] * X[operm(n - 1, h)];
    __syncwarp();
    {
        const double xn1 = X[operm(n - 1, h)], xn2 = X[operm(n - 2, h)];
        for (int k = lane; k < nb; k += 32) {
            double x = X[operm(k, h)];
            if (k >= of.fc2) x -= r2[k] * xn1;
            if (k >= of.fc1) x -= r1[k] * xn2;
            X[operm(k, h)] = x;
        }
    }
    __syncwarp();
    {
        double xp1 = 0.0, xp2 = 0.0;  // x_{k+1}, x_{k+2}
        for (int g = nb - 1; g >= 0; g -= 32) {
            const int k_l = g - lane;
            const bool ok = k_l >= 0;
            const double x_l = ok ? X[operm(k_l, h)] : 0.0;
            const double c2_l = (ok && k_l + 2 < nb) ? b2[k_l + 2] : 0.0;
            const double c1_l = (ok && k_l + 1 < nb) ? b1[k_l + 1] : 0.0;
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
            __syncwarp();
            if (ok) X[operm(k_l, h)] = res;
        }
    }
    __syncwarp();
}

// The coarse tail evaluates the assembled rows of launch_rows (Rw = this
// section's [10][n] block): absent couplings are stored as 0 and their
// neighbour index is the node itself, so every row is the same 10 products.
// rhs of circle row (s,t): f - sum of the off-line couplings (smoother.cpp:162-182)
template <bool CG>
__device__ __forceinline__ double circle_rhs(const LevelView& L, const double* __restrict__ Rw,
                                             const double* __restrict__ U,
                                             const double* __restrict__ F, int s, int t) {
    const int p = s * L.nt + t, n = L.n;
    const Nbr q = neighbours(L, s, t, p);
    double acc = ldv<CG>(F + (p));
    acc -= Rw[1 * n + p] * ldv<CG>(U + (q.pSM));
    acc -= Rw[2 * n + p] * ldv<CG>(U + (q.pSP));
    acc -= Rw[5 * n + p] * ldv<CG>(U + (q.pSMTM));
    acc -= Rw[6 * n + p] * ldv<CG>(U + (q.pSMTP));
    acc -= Rw[7 * n + p] * ldv<CG>(U + (q.pSPTM));
    acc -= Rw[8 * n + p] * ldv<CG>(U + (q.pSPTP));
    return acc;
}

// r = f - A u of node p with the assembled row (apply_take order,
// stencil.cpp:166-171)
template <bool CG>
__device__ __forceinline__ double row_residual(const LevelView& L, const double* __restrict__ Rw,
                                               const double* __restrict__ U,
                                               const double* __restrict__ F, int p) {
    int s, t;
    L.node(p, s, t);
    const int n = L.n;
    const Nbr q = neighbours(L, s, t, p);
    int pph = p;
    if (s == 0 && L.boundary == 0) pph = t + L.nt / 2 >= L.nt ? t + L.nt / 2 - L.nt : t + L.nt / 2;
    double acc = 0.0;
    acc += Rw[p] * ldv<CG>(U + (p));
    acc += Rw[1 * n + p] * ldv<CG>(U + (q.pSM));
    acc += Rw[2 * n + p] * ldv<CG>(U + (q.pSP));
    acc += Rw[3 * n + p] * ldv<CG>(U + (q.pTM));
    acc += Rw[4 * n + p] * ldv<CG>(U + (q.pTP));
    acc += Rw[5 * n + p] * ldv<CG>(U + (q.pSMTM));
    acc += Rw[6 * n + p] * ldv<CG>(U + (q.pSMTP));
    acc += Rw[7 * n + p] * ldv<CG>(U + (q.pSPTM));
    acc += Rw[8 * n + p] * ldv<CG>(U + (q.pSPTP));
    acc += Rw[9 * n + p] * ldv<CG>(U + (pph));
    return ldv<CG>(F + (p)) - acc;
}

// r = f - A u from the assembled rows, one thread per node (latency-bound
// levels; same products and order as apply_node)
__global__ void __launch_bounds__(256) k_residual_rows(LevelView L, const double* __restrict__ u,
                                                       const double* __restrict__ f,
                                                       double* __restrict__ r,
                                                       const int* __restrict__ active) {
    pdl_enter();
    const int b = blockIdx.y;
    if (active && !active[b]) return;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= L.n) return;
    const long off = (long)b * L.n;
    r[off + p] = row_residual<false>(L, L.rows + (long)b * 10 * L.n, u + off, f + off, p);
}

// warp version of origin_solve (2nd-order recurrences as 2x2-map scans)
template <int KW, bool CG>
__device__ void origin_warp(const CoarseLevel& C, double* __restrict__ U,
                            const double* __restrict__ F, long off, int b) {
    const LevelView& L = C.v;
    if (C.of.inv && L.nt <= 32) {  // tiny ring: dense inverse, u_i = sum_j Ainv_ij rhs_j
        const int n = L.nt, lane = threadIdx.x & 31;
        const double* Rw = C.rows + (long)b * 10 * L.n;
        const double r = lane < n ? circle_rhs<CG>(L, Rw, U, F, 0, lane) : 0.0;
        const double* A = C.of.inv + (long)b * n * n;
        double a0 = 0.0, a1 = 0.0;
        for (int j = 0; j < n; j += 2) {
            const double r0 = __shfl_sync(FULL, r, j);
            const double r1 = __shfl_sync(FULL, r, j + 1 < n ? j + 1 : j);
            if (lane < n) {
                a0 += A[(long)j * n + lane] * r0;
                if (j + 1 < n) a1 += A[(long)(j + 1) * n + lane] * r1;
            }
        }
        __syncwarp();
        if (lane < n) U[lane] = a0 + a1;
        return;
    }
    const int n = L.nt, h = n / 2, nb = n - 2;
    const int KE = (n + 31) >> 5;  // rows per lane (<= KW)
    const int lane = threadIdx.x & 31, j0 = lane * KE;
    const long o = (long)b * n;
    const double* b1 = C.of.band1 + o;
    const double* b2 = C.of.band2 + o;
    const double* r1 = C.of.row1 + o;
    const double* r2 = C.of.row2 + o;
    const double* D = C.of.D + o;
    const double* Rw = C.rows + (long)b * 10 * L.n;
    double x[KW];
    Map2 m = {1.0, 0.0, 0.0, 1.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < KW; ++q) {
        const int i = j0 + q;
        const bool in = q < KE;
        x[q] = (in && i < n) ? circle_rhs<CG>(L, Rw, U, F, 0, operm(i, h)) : 0.0;
        if (in && i < nb) {
            const double l1 = i >= 1 ? b1[i] : 0.0, l2 = i >= 2 ? b2[i] : 0.0;
            const Map2 mi = {0.0, 1.0, -l2, -l1, 0.0, x[q]};
            m = compose2(mi, m);
        }
    }
    double zm2, zm1;
    warp_scan2(m, true, zm2, zm1);
    double s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int q = 0; q < KW; ++q) {
        const int i = j0 + q;
        if (q < KE && i < nb) {
            double sum = x[q];
            if (i >= 2) sum -= b2[i] * zm2;
            if (i >= 1) sum -= b1[i] * zm1;
            x[q] = sum;
            zm2 = zm1;
            zm1 = sum;
            if (i >= C.of.fc1) s1 += r1[i] * sum;
            if (i >= C.of.fc2) s2 += r2[i] * sum;
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        s1 += __shfl_xor_sync(FULL, s1, d);
        s2 += __shfl_xor_sync(FULL, s2, d);
    }
    double xr2 = 0.0, xr1 = 0.0;  // rhs of the closing rows n-2, n-1
#pragma unroll
    for (int q = 0; q < KW; ++q) {
        if (q < KE && j0 + q == n - 2) xr2 = x[q];
        if (q < KE && j0 + q == n - 1) xr1 = x[q];
    }
    xr2 = __shfl_sync(FULL, xr2, (n - 2) / KE);
    xr1 = __shfl_sync(FULL, xr1, (n - 1) / KE);
    const double zn2 = xr2 - s1;
    double zn1 = xr1 - s2;
    if (n - 2 >= C.of.fc2) zn1 -= r2[n - 2] * zn2;
    const double xn1 = zn1 / D[n - 1];
    double xn2 = zn2 / D[n - 2];
    if (n - 2 >= C.of.fc2) xn2 -= r2[n - 2] * xn1;
    Map2 g = {1.0, 0.0, 0.0, 1.0, 0.0, 0.0};
#pragma unroll
    for (int q = KW - 1; q >= 0; --q) {
        const int k = j0 + q;
        if (q < KE && k < nb) {
            double gk = x[q] / D[k];
            if (k >= C.of.fc2) gk -= r2[k] * xn1;
            if (k >= C.of.fc1) gk -= r1[k] * xn2;
            x[q] = gk;
            const double l1 = k + 1 < nb ? b1[k + 1] : 0.0;
            const double l2 = k + 2 < nb ? b2[k + 2] : 0.0;
            const Map2 mk = {-l1, -l2, 1.0, 0.0, gk, 0.0};
            g = compose2(mk, g);
        }
    }
    double xp1, xp2;
    warp_scan2(g, false, xp1, xp2);
#pragma unroll
    for (int q = KW - 1; q >= 0; --q) {
        const int k = j0 + q;
        if (q < KE && k < nb) {
            double xv = x[q];
            if (k + 2 < nb) xv -= b2[k + 2] * xp2;
            if (k + 1 < nb) xv -= b1[k + 1] * xp1;
            x[q] = xv;
            xp2 = xp1;
            xp1 = xv;
        }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < KW; ++q) {
        const int k = j0 + q;
        if (q >= KE) continue;
        if (k < nb) U[operm(k, h)] = x[q];
        if (k == n - 2) U[operm(k, h)] = xn2;
        if (k == n - 1) U[operm(k, h)] = xn1;
    }
}

template <int KW, bool CG, class Team>
__device__ void coarse_smooth(const CoarseLevel& C, int b, const Team& team) {
    const LevelView& L = C.v;
    const long off = (long)b * L.n;
    double* U = C.u + off;
    const double* F = C.f + off;
    const int warp = team.warp(), nw = team.nwarps(), lane = threadIdx.x & 31;
    const int nt = L.nt;
    const double* Rw = C.rows + (long)b * 10 * L.n;
    const int kslot = nt == 8 ? 0 : nt == 16 ? 1 : nt == 32 ? 2 : -1;
    (void)kslot;
    KTS(kslot, 0);
    for (int parity = 0; parity < 2; ++parity) {  // circle sweeps (smoother.cpp:95-116)
        const int lines = L.split > parity ? (L.split - parity + 1) / 2 : 0;
        for (int li = warp; li < lines; li += nw) {
            const int s = parity + 2 * li;
            if (L.dir(s)) {
                for (int t = lane; t < nt; t += 32) U[s * nt + t] = ldv<CG>(F + (s * nt + t));
                continue;
            }
            if (s == 0 && L.boundary == 0) {
                if (C.exact) {  // rhs into ring 0 of U, then the exact substitution in place
                    double rr[KW];
#pragma unroll
                    for (int q = 0; q < KW; ++q) {
                        const int t = lane + 32 * q;
                        rr[q] = t < nt ? circle_rhs<CG>(L, Rw, U, F, 0, t) : 0.0;
                    }
                    __syncwarp();
#pragma unroll
                    for (int q = 0; q < KW; ++q)
                        if (lane + 32 * q < nt) U[lane + 32 * q] = rr[q];
                    __syncwarp();
                    origin_exact_warp(U, C.of, b, nt);
                } else {
                    origin_warp<KW, CG>(C, U, F, off, b);
                }
                continue;
            }
            double y[KW];
            const int KE = (nt + 31) >> 5;
            const int j0 = lane * KE;
#pragma unroll
            for (int q = 0; q < KW; ++q)
                y[q] = (q < KE && j0 + q < nt) ? circle_rhs<CG>(L, Rw, U, F, s, j0 + q) : 0.0;
            const long fo = (long)b * L.split * nt + (long)s * nt;
#ifdef PMG_KTRACE
            if (kslot == 1 && parity == 1 && threadIdx.x == 0 && blockIdx.x == 0) g_ktrace[0] = clock64();
#endif
            if (C.exact)
                warp_line_solve_ex<true, KW>(y, C.cl + fo, C.cm + fo, nt,
                                             C.corner[(long)b * L.split + s], C.cz + fo);
            else
                warp_line_solve<true, KW>(y, C.cl + fo, C.cm + fo, nt,
                                          C.corner[(long)b * L.split + s]);
#ifdef PMG_KTRACE
            if (kslot == 1 && parity == 1 && threadIdx.x == 0 && blockIdx.x == 0) g_ktrace[1] = clock64();
#endif
            __syncwarp();
#pragma unroll
            for (int q = 0; q < KW; ++q)
                if (q < KE && j0 + q < nt) U[s * nt + j0 + q] = y[q];
        }
        team.sync();
        KTS(kslot, 1 + parity);
    }
    if (L.len <= 0) return;
    const int n = L.n;
    for (int parity = 0; parity < 2; ++parity) {  // radial sweeps (smoother.cpp:118-142)
        const int lines = (nt - parity + 1) / 2;
        for (int li = warp; li < lines; li += nw) {
            const int t = parity + 2 * li;
            const int base = L.split * nt + t * L.len;
            double y[KW];
            const int KE = (L.len + 31) >> 5;
            const int j0 = lane * KE;
#pragma unroll
            for (int q = 0; q < KW; ++q) {
                const int i = j0 + q, s = L.split + i;
                double acc = 0.0;
                if (q < KE && i < L.len) {
                    const int p = base + i;
                    const Nbr nb = neighbours(L, s, t, p);
                    acc = ldv<CG>(F + (p));
                    if (s == L.split) acc -= Rw[1 * n + p] * ldv<CG>(U + (nb.pSM));
                    acc -= Rw[3 * n + p] * ldv<CG>(U + (nb.pTM));
                    acc -= Rw[4 * n + p] * ldv<CG>(U + (nb.pTP));
                    acc -= Rw[5 * n + p] * ldv<CG>(U + (nb.pSMTM));
                    acc -= Rw[6 * n + p] * ldv<CG>(U + (nb.pSMTP));
                    acc -= Rw[7 * n + p] * ldv<CG>(U + (nb.pSPTM));
                    acc -= Rw[8 * n + p] * ldv<CG>(U + (nb.pSPTP));
                }
                y[q] = acc;
            }
            const long fo = ((long)b * nt + t) * L.len;
            if (C.exact)
                warp_line_solve_ex<false, KW>(y, C.rl + fo, C.rm + fo, L.len, 0.0, nullptr);
            else
                warp_line_solve<false, KW>(y, C.rl + fo, C.rm + fo, L.len, 0.0);
            __syncwarp();
#pragma unroll
            for (int q = 0; q < KW; ++q)
                if (q < KE && j0 + q < L.len) U[base + j0 + q] = y[q];
        }
        team.sync();
        KTS(kslot, 3 + parity);
    }
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Who executes a phase: one block (the resident tail) or every block of a
// thread-block cluster (the cluster-wide multigrid kernel).
struct BlockTeam {
    __device__ int warp() const { return threadIdx.x >> 5; }
    __device__ int nwarps() const { return blockDim.x >> 5; }
    __device__ int tid() const { return threadIdx.x; }
    __device__ int nthreads() const { return blockDim.x; }
    __device__ void sync() const { __syncthreads(); }
};
struct ClusterTeam {
    int rank, size;
    // consecutive lines go to different CTAs (SMs)
    __device__ int warp() const { return (threadIdx.x >> 5) * size + rank; }
    __device__ int nwarps() const { return size * (blockDim.x >> 5); }
    __device__ int tid() const { return rank * blockDim.x + threadIdx.x; }
    __device__ int nthreads() const { return size * blockDim.x; }
    __device__ void sync() const { cg::this_cluster().sync(); }
};

// One op of a program on level C (D = level below for transfers); `bb` is
// the section index of the per-section arrays (0 when shared-memory resident).
template <int KW, bool CG, class Team>
__device__ __forceinline__ void exec_op(int op, const CoarseLevel& C, const CoarseLevel& D,
                                        const EnvFactor& env, int bb, const Team& team) {
    const long off = (long)bb * C.v.n;
    switch (op) {
        case OP_SMOOTH:
            coarse_smooth<KW, CG>(C, bb, team);
            break;
        case OP_RESIDUAL:
            for (int p = team.tid(); p < C.v.n; p += team.nthreads())
                C.res[off + p] =
                    row_residual<CG>(C.v, C.rows + (long)bb * 10 * C.v.n, C.u + off, C.f + off, p);
            break;
        case OP_RESTRICT: {
            const long offc = (long)bb * D.v.n;
            for (int p = team.tid(); p < D.v.n; p += team.nthreads())
                restrict_node<CG>(C.v, D.v, C.w, C.res + off, D.f + offc, D.u + offc, 1, p);
            break;
        }
        case OP_PROLONG: {
            const long offc = (long)bb * D.v.n;
            for (int p = team.tid(); p < C.v.n; p += team.nthreads())
                prolong_node<true, CG>(C.v, D.v, C.w, D.u + offc, C.u + off, p);
            break;
        }
        default: {  // OP_COARSE: u = f, envelope LDL^T (multigrid.cpp:183-187)
            if (env.inv) {  // dense inverse: one row per thread
                const int n = env.n;
                const double* A = env.inv + (long)bb * n * n;
                for (int i = team.tid(); i < n; i += team.nthreads()) {
                    double a0 = 0.0, a1 = 0.0;
                    int j = 0;
                    for (; j + 1 < n; j += 2) {
                        a0 += A[(long)j * n + i] * C.f[off + j];
                        a1 += A[(long)(j + 1) * n + i] * C.f[off + j + 1];
                    }
                    if (j < n) a0 += A[(long)j * n + i] * C.f[off + j];
                    C.u[off + i] = a0 + a1;
                }
            } else if (env.n <= 32) {
                // the reference's envelope substitutions (line_algebra.cpp:229-251)
                // by one warp, lane i owning x_i: the forward sums run column by
                // column (x_k final -> every row i > k with first_col <= k subtracts
                // L(i,k) x_k), so each sum still receives its terms in increasing k,
                // and the backward column updates are per element as written --
                // the same operations on every x_i in the same order, bit for bit,
                // in 2 n broadcast steps instead of ~2 nnz dependent ones
                if (team.tid() < 32) {
                    const int lane = team.tid(), n = env.n;
                    const bool in = lane < n;
                    const double* Lb = env.L + (long)bb * env.nnz;
                    const int fi = in ? env.fc[lane] : 0;
                    const double* ri = Lb + (in ? env.ro[lane] - fi : 0);
                    double x = in ? C.f[off + lane] : 0.0;
                    for (int k = 0; k < n; ++k) {
                        const double xk = __shfl_sync(FULL, x, k);
                        if (in && lane > k && fi <= k) x -= ri[k] * xk;
                    }
                    if (in) x /= env.D[(long)bb * n + lane];
                    for (int i = n - 1; i >= 0; --i) {
                        const double xi = __shfl_sync(FULL, x, i);
                        const int fci = env.fc[i];
                        const double* rr = Lb + env.ro[i] - fci;
                        if (lane < i && lane >= fci) x -= rr[lane] * xi;
                    }
                    if (in) C.u[off + lane] = x;
                }
            } else if (team.tid() == 0) {
                double* x = C.u + off;
                for (int k = 0; k < env.n; ++k) x[k] = C.f[off + k];
                env_solve(env, bb, x);
            }
            break;
        }
    }
}

// The resident tail of section b, run by one block: stage this section's
// slice of every tail array into shared memory, run the op program, write the
// top level's correction back.
// (one instance per kernel, shared by the tail_body instantiations)
__shared__ __align__(16) TailImage simg;
__shared__ __align__(8) unsigned long long sbar;
__shared__ unsigned stx;

template <int KW>
__device__ void tail_body(const CoarseParams& cp, const int* __restrict__ prog, int nops, int b,
                          unsigned long long* trace) {
    extern __shared__ __align__(16) char sbuf[];
    // one thread per array issues a bulk (TMA) copy of its 16-byte aligned
    // part, completing on an mbarrier; leftovers go through cp.async
    if (threadIdx.x == 0) {
        mbar_init(&sbar, 1);
        stx = 0;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < cp.ncopy; c += blockDim.x) {
        const CopyDesc d = cp.copies[c];
        const char* src = static_cast<const char*>(d.src) + (long)b * d.stride;
        const int bulk = (reinterpret_cast<uintptr_t>(src) & 15) == 0 ? (d.bytes & ~15) : 0;
        if (bulk > 0) {
            bulk_g2s(sbuf + d.dst, src, bulk, &sbar);
            atomicAdd(&stx, (unsigned)bulk);
        }
        for (int o = bulk; o + 8 <= d.bytes; o += 8)
            __pipeline_memcpy_async(sbuf + d.dst + o, src + o, 8);
        if (d.bytes & 7)  // int arrays of odd length
            __pipeline_memcpy_async(sbuf + d.dst + (d.bytes - 4), src + (d.bytes - 4), 4);
    }
    __pipeline_commit();
    {  // level table image, rebased onto this block's shared window
        const unsigned long long base = reinterpret_cast<uintptr_t>(sbuf);
        unsigned long long* w = reinterpret_cast<unsigned long long*>(&simg);
        constexpr int words = sizeof(TailImage) / 8;
        for (int i = threadIdx.x; i < words; i += blockDim.x) {
            unsigned long long x = cp.image[i];
            if (((cp.image_mask[i >> 5] >> (i & 31)) & 1u) && x) x = x - 8 + base;
            w[i] = x;
        }
    }
    __syncthreads();
    if (trace && threadIdx.x == 0) trace[nops + 2] = globaltimer();
    if (threadIdx.x == 0) mbar_arrive_tx(&sbar, stx);
    __pipeline_wait_prior(0);
    mbar_wait(&sbar, 0);
    if (trace && threadIdx.x == 0) trace[nops + 3] = globaltimer();
    __syncthreads();
    if (trace && threadIdx.x == 0) trace[1] = globaltimer();
    const CoarseLevel* lv = simg.lv - cp.first;
    const BlockTeam team;
    for (int i = 0; i < nops; ++i) {
        const int op = prog[i] & 255, l = prog[i] >> 8;
        // level descriptors copied into registers: the shared-memory vectors
        // the phase stores to could alias the shared table, which would force
        // a reload of every field after every store
        const CoarseLevel Cl = lv[l], Dl = lv[l + (op == OP_COARSE ? 0 : 1)];
        const EnvFactor env = simg.env;
        exec_op<KW, false>(op, Cl, Dl, env, 0, team);
        __syncthreads();
        if (trace && threadIdx.x == 0) trace[2 + i] = globaltimer();
    }
    // the top level's correction goes back to global memory
    const CoarseLevel& top = simg.lv[0];
    for (int p = threadIdx.x; p < top.v.n; p += blockDim.x)
        cp.top_u_global[(long)b * top.v.n + p] = top.u[p];
}

template <int KW>
__global__ void __launch_bounds__(512) k_coarse_cycle(const __grid_constant__ CoarseParams cp,
                                                      const int* __restrict__ prog, int nops,
                                                      const int* __restrict__ active) {
    pdl_enter();
    const int b = blockIdx.x;
    if (active && !active[b]) return;
    unsigned long long* trace = b == 0 ? cp.trace : nullptr;
    if (trace && threadIdx.x == 0) trace[0] = globaltimer();
    tail_body<KW>(cp, prog, nops, b, trace);
}

__device__ __forceinline__ void tail_dispatch(const CoarseParams& cp, const int* prog, int nops,
                                              int b) {
    switch (cp.kw) {
        case 1: tail_body<1>(cp, prog, nops, b, nullptr); break;
        case 2: tail_body<2>(cp, prog, nops, b, nullptr); break;
        case 4: tail_body<4>(cp, prog, nops, b, nullptr); break;
        default: tail_body<8>(cp, prog, nops, b, nullptr); break;
    }
}

// Cluster-wide multigrid sub-cycle: the levels between the level kernels and
// the resident tail run in ONE launch, one thread-block cluster per section;
// every phase is spread over all warps / threads of the cluster and followed
// by a cluster barrier (instead of a kernel boundary).  Vectors written inside
// the launch are read with ld.global.cg.  OP_TAIL: block 0 runs the resident
// tail (tail_body) while the others wait at the barrier.
__global__ void __launch_bounds__(512) k_mid_cycle(const __grid_constant__ MidParams mp,
                                                   const int* __restrict__ prog, int nops,
                                                   const int* __restrict__ active) {
    pdl_enter();
    cg::cluster_group cluster = cg::this_cluster();
    const int b = blockIdx.x / mp.cl;
    if (active && !active[b]) return;  // uniform over the cluster
    const ClusterTeam team{static_cast<int>(cluster.block_rank()), mp.cl};
    unsigned long long* trace = (b == 0 && team.rank == 0 && threadIdx.x == 0) ? mp.trace : nullptr;
    if (trace) trace[0] = globaltimer();
    for (int i = 0; i < nops; ++i) {
        const int op = prog[i] & 255, l = prog[i] >> 8;
        if (op == OP_TAIL) {
            if (team.rank == 0) {
                asm volatile("fence.proxy.async.global;" ::: "memory");
                tail_dispatch(mp.tail, mp.tprog[l], mp.tlen[l], b);
            }
        } else {
            const int k = l - mp.first;
            const CoarseLevel& C = mp.lv[k];
            const CoarseLevel& D = mp.lv[k + 1];
            switch (mp.kw[k]) {
                case 1: exec_op<1, true>(op, C, D, mp.tail.env, b, team); break;
                case 2: exec_op<2, true>(op, C, D, mp.tail.env, b, team); break;
                case 4: exec_op<4, true>(op, C, D, mp.tail.env, b, team); break;
                default: exec_op<8, true>(op, C, D, mp.tail.env, b, team); break;
            }
        }
        cluster.sync();
        if (trace) trace[1 + i] = globaltimer();
    }
}

// ------------------------------------------------------------------- norms
__global__ void __launch_bounds__(256) k_norm_partials(const double* __restrict__ v, long n,
                                                       int norm_type,
                                                       double* __restrict__ partials) {
    pdl_enter();
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
// convergence bookkeeping of section b from its residual norm r
// (multigrid.cpp:321-340: history, r0, relative / absolute tolerance,
// max_iterations); per section, so the norm block of b can run it
__device__ __forceinline__ void check_section(int b, double r, const ConvState& cs, int max_it,
                                              double rel_tol, double abs_tol) {
    if (!cs.active[b]) return;
    const int it = cs.count[b]++;  // residual norms taken so far = iteration index
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

// CHECK: the block of section b also runs its convergence check (one launch
// instead of norm + check)
template <bool CHECK>
__global__ void __launch_bounds__(1024) k_norm_final(const double* __restrict__ partials,
                                                     int nblk, long n, int norm_type,
                                                     double* __restrict__ norms, ConvState cs,
                                                     int max_it, double rel_tol, double abs_tol) {
    pdl_enter();
    const int b = blockIdx.x;
    const double* Pb = partials + (long)b * nblk;
    // eight independent accumulators per thread so the loads overlap; fixed
    // combination order (deterministic for a given launch shape)
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.0;
    const int T = blockDim.x;
    for (int i0 = threadIdx.x; i0 < nblk; i0 += 8 * T) {
        double x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int i = i0 + k * T;
            x[k] = i < nblk ? Pb[i] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = norm_type == 2 ? fmax(acc[k], x[k]) : acc[k] + x[k];
    }
    double a = acc[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) a = norm_type == 2 ? fmax(a, acc[k]) : a + acc[k];
    __shared__ double red[32];
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
        if (CHECK) check_section(b, s, cs, max_it, rel_tol, abs_tol);
    }
}

// convergence test of MultigridSolver::solve (multigrid.cpp:321-340)
__global__ void k_check(const double* __restrict__ norms, ConvState cs, int B, int max_it,
                        double rel_tol, double abs_tol) {
    pdl_enter();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    check_section(b, norms[b], cs, max_it, rel_tol, abs_tol);
}

__global__ void k_fill(double* p, long n, double v) {
    pdl_enter();
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void k_set_active(int* active, int* count, int* conv, int* remaining, int B) {
    pdl_enter();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) {
        active[b] = 1;
        count[b] = 0;
        conv[b] = 0;
    }
    if (b == 0) *remaining = B;
}

// Loop condition of the solve's WHILE graph node (multigrid.cpp:328-340):
// another cycle runs while any section is still iterating.
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const int* __restrict__ remaining) {
    if (threadIdx.x == 0) cudaGraphSetConditional(h, *remaining != 0 ? 1u : 0u);
}

__global__ void k_flush(double* p, long n) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long)gridDim.x * blockDim.x)
        p[i] = p[i] * 0.5 + 1.0;
}

// ------------------------------------------------------------ launch helpers
// chunk size K and threads T for a line of n rows: T = 32*ceil(ceil(n/K)/32) <= 512
// Threads per line: wide CTAs (short per-thread chunks) when few lines run
// concurrently (latency), narrow CTAs when the batch of lines fills the GPU
// many times over (throughput, e.g. 256 sections of config 3).
inline void line_shape(int n, int& K, int& T, long lines_total = 0) {
    static const int ks[4] = {2, 4, 8, 16};
    static const int env_maxt = [] {
        const char* e = std::getenv("PMG_LINE_MAXT");
        // a multiple of 32 (full-mask shuffles in the block scans) within the
        // line kernels' launch bounds
        const int v = e ? std::atoi(e) : 0;
        return v > 0 ? std::min(256, std::max(32, (v + 31) / 32 * 32)) : 0;
    }();
    const int maxt = env_maxt > 0 ? env_maxt
                     : lines_total >= 4096 ? 64
                     : lines_total >= 2048 ? 128
                                           : 256;
    K = 16;
    for (int q = 0; q < 4; ++q)
        if ((n + ks[q] - 1) / ks[q] <= maxt || ks[q] == 16) {
            K = ks[q];
            break;
        }
    const int chunks = (n + K - 1) / K;
    T = ((chunks + 31) / 32) * 32;
    if (T < 32) T = 32;
}

// shared memory of a single-CTA line: Y, IL, M (+ RC and the chunk tables of
// the exact-order parallel solve when ex4)
inline size_t line_smem(int n, bool ex4 = false, int T = 512, bool ex3 = false) {
    if (ex3) return (size_t)(3 * padded(n) + 64 + 3 * T) * sizeof(double);
    return ex4 ? (size_t)(4 * padded(n) + 64 + 6 * T) * sizeof(double)
               : (size_t)(3 * padded(n) + 32 * 6 + 16) * sizeof(double);
}
// line-solve mode of an exact (reference_order) solve: 1 = parallel exact
// (line_solve_ex) when its four line arrays fit one CTA, else 2 = one thread
// (line_solve_ex), 3 = the same with RN(1/l) evaluated on the fly (three line
// arrays: 8192-node lines), 2 = one thread
// Radial lines (prefer3) also take mode 3 where it lets TWO lines be resident
// per SM and mode 1 only one (2048..4096-node lines: one CTA's rhs gather then
// overlaps the other's solve; c2-V radial 15.1 -> 12.5 ms).  Circle lines keep
// mode 1: the across-origin ring's fast exact solve needs the fourth array
// (measured 12.2 -> 19.7 ms in mode 3).  PMG_EXACT_MODE=1|3 forces a mode.
inline int exact_mode(int n, bool prefer3 = false) {
    static const int forced = [] {
        const char* e = std::getenv("PMG_EXACT_MODE");
        return e ? std::atoi(e) : 0;
    }();
    const int T = std::min(512, std::max(32, ((n + 15) / 16 + 31) / 32 * 32));  // 16 rows / thread
    const size_t m1 = line_smem(n, true, T), m3 = line_smem(n, false, T, true);
    const size_t cap = 227 * 1024, half = cap / 2 - 1024;
    if (forced == 1 && m1 <= cap) return 1;
    if (forced == 3 && m3 <= cap) return 3;
    if (m1 <= cap && !(prefer3 && m1 > half && m3 <= half)) return 1;
    return m3 <= cap ? 3 : 2;
}

}  // namespace

// First failed launch since the last check (a failed cudaLaunchKernelEx would
// otherwise only surface through cudaGetLastError, which other probes clear).
static std::atomic<int> g_launch_error{0};
void note_launch_error(cudaError_t e) {
    int z = 0;
    g_launch_error.compare_exchange_strong(z, (int)e);
}
cudaError_t last_error() {
    const cudaError_t e = (cudaError_t)g_launch_error.exchange(0);
    const cudaError_t g = cudaGetLastError();
    return e != cudaSuccess ? e : g;
}

int apply_launches(const LevelView& L) { return 1; }



int apply_blocks(const LevelView& L) {
    return std::max(tile_geom(L).ntiles(), tma_geom_auto(L).cps);
}

// Take residual/apply through the TMA-streamed kernel (PMG_TMA_APPLY=0: off)
static bool tma_apply_on() {
    static const bool on = [] {
        const char* e = std::getenv("PMG_TMA_APPLY");
        return e ? std::atoi(e) != 0 : true;
    }();
    return on;
}


int launch_apply(const LevelView& L, bool onfly, int mode, const double* u, const double* f,
                 double* out, double* partials, int norm_type, const int* active,
                 cudaStream_t st) {
    if (L.rows && mode == 1 && !partials) {
        launch_k(k_residual_rows, dim3((L.n + 255) / 256, L.B), 256, 0, st, L, u, f, out, active);
        return 0;
    }
    const bool norm = partials != nullptr;
    if (!onfly && tma_apply_on() && tma_ok(L)) {
        const TmaGeom S = tma_geom_auto(L);
#define PMG_TMA(MO, NO)                                                                     \
    do {                                                                                    \
        if (L.B > 1) {                                                                      \
            set_smem(k_apply_tma<MO, NO, 3>, kTmaSmem);                                     \
            launch_k(k_apply_tma<MO, NO, 3>, dim3(S.cps * L.B), 288, kTmaSmem, st, L, S, u, \
                     f, out, partials, norm_type, active);                                  \
        } else {                                                                            \
            set_smem(k_apply_tma<MO, NO>, kTmaSmem);                                        \
            launch_k(k_apply_tma<MO, NO>, dim3(S.cps * L.B), 288, kTmaSmem, st, L, S, u, f, \
                     out, partials, norm_type, active);                                     \
        }                                                                                   \
    } while (0)
        if (mode == 0) {
            if (norm) PMG_TMA(0, true); else PMG_TMA(0, false);
        } else {
            if (norm) PMG_TMA(1, true); else PMG_TMA(1, false);
        }
#undef PMG_TMA
        return S.cps;
    }
    const TileGeom G = tile_geom(L);
    const int nb = G.ntiles();
    dim3 grid(nb, L.B);
#define PMG_APPLY(ON, MO, NO) \
    launch_k(k_apply_tiled<ON, MO, NO>, grid, 256, 0, st, L, G, u, f, out, partials, norm_type, active)
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
    const int mode = serial ? exact_mode(L.nt) : 0;
    const size_t sm = line_smem(L.nt, mode == 1 || (mode == 0 && exact_rings > 0), T, mode == 3);
    set_smem(k_circle<ON, K>, sm);
    launch_k(k_circle<ON, K>, dim3(lines, L.B), T, sm, st, L, u, f, cil, cm, corner, cz, of, parity,
             mode, exact_rings, active);
}

// cluster size for a line of n rows in fast mode (1 = single-CTA kernels)
static int line_cluster(int n, int min_rows = 2048) {
    if (const char* e = std::getenv("PMG_CIRCLE_CLUSTER_ROWS")) {
        const int rows = std::atoi(e);
        if (rows <= 0) return 1;
        return std::min(8, std::max(1, (n + rows - 1) / rows));
    }
    if (n < min_rows) return 1;
    // ~1366 rows per CTA (measured: 8192-node rings 0.306 ms B+W at C = 4,
    // 0.276 ms at C = 6; 4096-node rings: c2-V 23.8 -> 23.2 ms at C = 3)
    return std::min(8, (n + 1365) / 1366);
}

template <class Kern, class... Args>
static void launch_cluster(Kern kern, int C, dim3 grid, int T, size_t smem, cudaStream_t st,
                           Args... args) {
    set_smem(kern, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(T, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_on() ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
    if (e != cudaSuccess) note_launch_error(e);
}

static void cl_shape(int n, int C, int& R, int& K, int& T, size_t& smem, int kpref = 8) {
    R = (n + C - 1) / C;
    K = R <= 1024 && kpref == 4 ? 4 : (R <= 2048 ? 8 : 16);
    T = (((R + K - 1) / K) + 31) / 32 * 32;
    smem = (size_t)(3 * padded(R + 1) + 32 * 3 + 16) * sizeof(double);
}

int line_launches(const LevelView& L, bool serial, bool onfly, int exact_rings, int kind,
                  int parity) {
    if (kind == 0) {
        const bool cl = !serial && exact_rings <= 0 && line_cluster(L.nt) > 1;
        return (cl && parity == 0 && L.boundary == 0) ? 2 : 1;
    }
    return 1;
}

void launch_circle(const LevelView& L, bool onfly, double* u, const double* f, const double* cil,
                   const double* cm, const double* corner, const double* cz,
                   const OriginFactor& of, int parity, bool serial, int exact_rings,
                   const int* active, cudaStream_t st) {
    int lines = L.split > parity ? (L.split - parity + 1) / 2 : 0;
    if (lines == 0) return;
    int K, T;
    // large batches of Take lines: one warp per ring (pmg_radial_warp.cu); the
    // across-origin ring, which is not a cyclic line, by the CTA kernel
    if (!onfly && !L.rows && exact_rings <= 0) {
        const bool org = parity == 0 && L.boundary == 0;
        const int s_first = org ? 2 : parity;
        const int nl = L.split > s_first ? (L.split - s_first + 1) / 2 : 0;
        // (fast mode keeps the CTA kernels: their two-rhs scans are quicker there)
        cudaStream_t side = st;
        cudaEvent_t fork = nullptr, join = nullptr;
        if (serial && org && nl > 0 && warp_batch_ok(L.nt, (long)nl * L.B)) {
            // ring 0 on a side stream, forked from / joined back into st: it
            // overlaps the other rings (a parallel branch of the cycle graph)
            static thread_local cudaStream_t s_side[64] = {};
            static thread_local cudaEvent_t s_fork[64] = {}, s_join[64] = {};
            int dev = 0;
            cudaGetDevice(&dev);
            if (!s_side[dev]) {
                cudaStreamCreateWithFlags(&s_side[dev], cudaStreamNonBlocking);
                cudaEventCreateWithFlags(&s_fork[dev], cudaEventDisableTiming);
                cudaEventCreateWithFlags(&s_join[dev], cudaEventDisableTiming);
            }
            side = s_side[dev];
            fork = s_fork[dev];
            join = s_join[dev];
            cudaEventRecord(fork, st);
            cudaStreamWaitEvent(side, fork, 0);
        }
        if (serial && nl > 0 &&
            launch_circle_warp(L, u, f, cil, cm, corner, cz, s_first, nl, serial, active, st)) {
            if (!org) return;
            struct Join {
                cudaStream_t st, side;
                cudaEvent_t join;
                ~Join() {
                    if (join) {
                        cudaEventRecord(join, side);
                        cudaStreamWaitEvent(st, join, 0);
                    }
                }
            } joiner{st, side, join};
            st = side;
            lines = 1;  // ring 0 below
            line_shape(L.nt, K, T, (long)L.B);
            switch (K) {
                case 2: circle_k<false, 2>(L, u, f, cil, cm, corner, cz, of, 0, serial, exact_rings, active, st, T, 1); break;
                case 4: circle_k<false, 4>(L, u, f, cil, cm, corner, cz, of, 0, serial, exact_rings, active, st, T, 1); break;
                case 8: circle_k<false, 8>(L, u, f, cil, cm, corner, cz, of, 0, serial, exact_rings, active, st, T, 1); break;
                default: circle_k<false, 16>(L, u, f, cil, cm, corner, cz, of, 0, serial, exact_rings, active, st, T, 1); break;
            }
            return;
        }
    }
    const int C = (!serial && exact_rings <= 0) ? line_cluster(L.nt) : 1;
    if (C > 1) {
        int s_first = parity, nl = lines;
        // the across-origin ring runs as a single-CTA kernel on a side stream,
        // forked from / joined back into st so it overlaps the clustered rings
        // (a parallel branch when captured into the cycle graph)
        cudaStream_t side = st;
        cudaEvent_t fork = nullptr, join = nullptr;
        if (parity == 0 && L.boundary == 0) {
            static thread_local cudaStream_t s_side[64] = {};
            static thread_local cudaEvent_t s_fork[64] = {}, s_join[64] = {};
            int dev = 0;
            cudaGetDevice(&dev);
            if (!s_side[dev]) {
                cudaStreamCreateWithFlags(&s_side[dev], cudaStreamNonBlocking);
                cudaEventCreateWithFlags(&s_fork[dev], cudaEventDisableTiming);
                cudaEventCreateWithFlags(&s_join[dev], cudaEventDisableTiming);
            }
            side = s_side[dev];
            fork = s_fork[dev];
            join = s_join[dev];
            cudaEventRecord(fork, st);
            cudaStreamWaitEvent(side, fork, 0);
        }
        if (parity == 0 && L.boundary == 0) {  // across-origin ring: single-CTA kernel
            line_shape(L.nt, K, T);
            const size_t sm = line_smem(L.nt);
#define PMG_C1(KK)                                                                               \
    do {                                                                                         \
        if (onfly) {                                                                             \
            set_smem(k_circle<true, KK>, sm);                                                    \
            k_circle<true, KK><<<dim3(1, L.B), T, sm, side>>>(L, u, f, cil, cm, corner, cz, of, 0, \
                                                              0, 0, active);                     \
        } else {                                                                                 \
            set_smem(k_circle<false, KK>, sm);                                                   \
            k_circle<false, KK><<<dim3(1, L.B), T, sm, side>>>(L, u, f, cil, cm, corner, cz, of, \
                                                               0, 0, 0, active);                 \
        }                                                                                        \
    } while (0)
            switch (K) {
                case 2: PMG_C1(2); break;
                case 4: PMG_C1(4); break;
                case 8: PMG_C1(8); break;
                default: PMG_C1(16); break;
            }
#undef PMG_C1
            s_first = 2;
            nl = L.split > 2 ? (L.split - 2 + 1) / 2 : 0;
        }
        if (nl > 0) {
            int R;
            size_t sm;
            cl_shape(L.nt, C, R, K, T, sm);
            const dim3 grid(nl * C, L.B);
            if (K == 8) {
                if (onfly)
                    launch_cluster(k_circle_cl<true, 8>, C, grid, T, sm, st, L, u, f, cil, cm,
                                   corner, s_first, active);
                else
                    launch_cluster(k_circle_cl<false, 8>, C, grid, T, sm, st, L, u, f, cil, cm,
                                   corner, s_first, active);
            } else {
                if (onfly)
                    launch_cluster(k_circle_cl<true, 16>, C, grid, T, sm, st, L, u, f, cil, cm,
                                   corner, s_first, active);
                else
                    launch_cluster(k_circle_cl<false, 16>, C, grid, T, sm, st, L, u, f, cil, cm,
                                   corner, s_first, active);
            }
        }
        if (join) {
            cudaEventRecord(join, side);
            cudaStreamWaitEvent(st, join, 0);
        }
        return;
    }
    line_shape(L.nt, K, T, (long)lines * L.B);
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
    const int mode = serial ? exact_mode(L.len, true) : 0;
    const size_t sm = line_smem(L.len, mode == 1, T, mode == 3);
    set_smem(k_radial<ON, K>, sm);
    launch_k(k_radial<ON, K>, dim3(lines, L.B), T, sm, st, L, u, f, ril, rm, parity, mode, active);
}

void launch_radial(const LevelView& L, bool onfly, double* u, const double* f, const double* ril,
                   const double* rm, int parity, bool serial, const int* active,
                   cudaStream_t st) {
    if (L.len <= 0) return;
    const int lines = (L.nt - parity + 1) / 2;
    if (launch_radial_tpl(L, onfly, u, f, ril, rm, parity, active, st)) return;
    if (launch_radial_warp(L, onfly, u, f, ril, rm, parity, serial, active, st)) return;
    int K, T;
    static const int cl_min = [] {
        const char* e = std::getenv("PMG_RADIAL_CL_MIN");
        return e ? std::atoi(e) : 1024;
    }();
    if (!serial && !onfly && L.len > cl_min) {
        int C = std::min(8, (L.len + 899) / 900);
        if (const char* e = std::getenv("PMG_LINE_CLUSTER_ROWS")) {
            const int rows = std::atoi(e);
            if (rows > 0) C = std::min(8, std::max(1, (L.len + rows - 1) / rows));
        }
        int R;
        size_t sm;
        int kp = 8;
        if (const char* e = std::getenv("PMG_RADIAL_K")) kp = std::atoi(e);
        cl_shape(L.len, C, R, K, T, sm, kp);
        const dim3 grid(lines * C, L.B);
        if (K == 4)
            launch_cluster(k_radial_cl<4>, C, grid, T, sm, st, L, u, f, ril, rm, parity, active);
        else if (K == 8)
            launch_cluster(k_radial_cl<8>, C, grid, T, sm, st, L, u, f, ril, rm, parity, active);
        else
            launch_cluster(k_radial_cl<16>, C, grid, T, sm, st, L, u, f, ril, rm, parity, active);
        return;
    }
    line_shape(L.len, K, T, (long)lines * L.B);
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

bool fused_ok(const LevelView& L, bool serial, int exact_rings) {
    static const bool on = [] {
        const char* e = std::getenv("PMG_FUSED_SMOOTH");
        return e ? std::atoi(e) != 0 : true;
    }();
    (void)serial;
    return on && exact_rings <= 0 && L.len > 1 && L.split >= 2 && L.nt <= 1024 &&
           L.len <= 1024 && (L.nt & 1) == 0;
}

void fused_order(int split, int nt, int B, int* out) {
    // black rings from the outside in (ring split-1, which the spokes wait
    // for, first), white rings, black spokes, white spokes; sections
    // interleaved within each phase
    const int per = split + nt;
    long k = 0;
    for (int s = (split - 1) & ~1; s >= 0; s -= 2)
        for (int b = 0; b < B; ++b) out[k++] = b * per + s;
    for (int s = (split - 1) | 1; s >= 1; s -= 2) {
        if (s >= split) continue;
        for (int b = 0; b < B; ++b) out[k++] = b * per + s;
    }
    for (int t = 0; t < nt; t += 2)
        for (int b = 0; b < B; ++b) out[k++] = b * per + split + t;
    for (int t = 1; t < nt; t += 2)
        for (int b = 0; b < B; ++b) out[k++] = b * per + split + t;
}

void launch_smooth_fused(const LevelView& L, bool onfly, double* u, const double* f,
                         const double* cil, const double* cm, const double* corner,
                         const double* cz, const OriginFactor& of, const double* ril,
                         const double* rm, int exact_rings, bool serial, const FuseCtl& fc,
                         const int* order, const int* active, cudaStream_t st) {
    const int n = std::max(L.nt, L.len);
    const int nitems = (L.split + L.nt) * L.B;
    int K, T;
    line_shape(n, K, T, nitems);
    // Short lines (<= 256 nodes, the latency-bound coarse levels): at least 128
    // threads per line even if some idle in the scans -- the rhs gather is the
    // latency, and more threads put more of its loads in flight (c1: 32/64-
    // thread lines 5.25 ms per solve, 128 threads 5.11 ms; PMG_FUSED_SMALL_T)
    static const int small_t = [] {
        const char* e = std::getenv("PMG_FUSED_SMALL_T");
        // 0 disables; else a multiple of 32 within k_smooth_fused's launch bounds
        const int v = e ? std::atoi(e) : 128;
        return v > 0 ? std::min(256, std::max(32, (v + 31) / 32 * 32)) : 0;
    }();
    if (small_t > 0 && n <= 256 && T < small_t) {
        T = small_t;
        K = 2;
        while (K < 16 && K * T < n) K *= 2;
    }
    const int ex = serial ? 1 : 0;  // lines <= 1024: the parallel exact solve always fits
    const size_t sm = line_smem(n, serial, T);
#define PMG_F(ON, KK)                                                                          \
    do {                                                                                       \
        set_smem(k_smooth_fused<ON, KK>, sm);                                                  \
        launch_k(k_smooth_fused<ON, KK>, dim3(nitems), T, sm, st, L, u, f, cil, cm, corner, cz, \
                 of, ril, rm, exact_rings, ex, fc, order, nitems, active);                     \
    } while (0)
#define PMG_FK(ON)                       \
    switch (K) {                         \
        case 2: PMG_F(ON, 2); break;     \
        case 4: PMG_F(ON, 4); break;     \
        case 8: PMG_F(ON, 8); break;     \
        default: PMG_F(ON, 16); break;   \
    }
    if (onfly) {
        PMG_FK(true)
    } else {
        PMG_FK(false)
    }
#undef PMG_FK
#undef PMG_F
}

// Two-colour radial wavefront (k_radial_wave): cluster size when it applies
// (one section, clustered Take spokes, fast mode, PMG_RADIAL_WAVE=1), else 0.
// Opt-in: measured slower than the two per-colour launches (8193x8192 B+W
// 1.35 vs 1.20 ms for lags 64-400; c2-V 23.9 vs 23.3 ms) -- the ticket
// broadcast barrier, L2 loads of u and flag waits cost more than the
// neighbour re-reads it saves.
int radial_wave_cluster(const LevelView& L, bool serial, bool onfly) {
    static const bool on = [] {
        const char* e = std::getenv("PMG_RADIAL_WAVE");
        return e ? std::atoi(e) != 0 : false;
    }();
    if (!on || serial || onfly || L.B != 1 || L.len <= 1024 || (L.nt & 1)) return 0;
    return std::min(8, (L.len + 899) / 900);
}

// claim order: black spokes in increasing t, white spoke 2j+1 `lag` items
// after black spoke 2j (so both its black neighbours were claimed before it)
void radial_wave_order(int nt, int C, int* out) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int lag = std::max(1, sms * 8 / C);
    if (const char* e = std::getenv("PMG_WAVE_LAG")) lag = std::max(1, std::atoi(e));
    const int nb = nt / 2;
    lag = std::min(lag, nb);
    int k = 0;
    for (int i = 0; i < nb; ++i) {
        out[k++] = 2 * i;
        if (i >= lag) out[k++] = 2 * (i - lag) + 1;
    }
    for (int j = nb - lag; j < nb; ++j) out[k++] = 2 * j + 1;
}

void launch_radial_wave(const LevelView& L, double* u, const double* f, const double* ril,
                        const double* rm, const FuseCtl& fc, const int* order, cudaStream_t st) {
    const int C = std::min(8, (L.len + 899) / 900);
    int R, K, T;
    size_t sm;
    cl_shape(L.len, C, R, K, T, sm, 8);
    const dim3 grid(L.nt * C);
    const int nctas = L.nt * C;
    if (K == 8)
        launch_cluster(k_radial_wave<8>, C, grid, T, sm, st, L, u, f, ril, rm, fc, order, nctas);
    else
        launch_cluster(k_radial_wave<16>, C, grid, T, sm, st, L, u, f, ril, rm, fc, order, nctas);
}

void launch_restrict(const LevelView& F, const LevelView& C, const Weights& w, const double* fr,
                     double* cf, double* cu_zero, bool mask, const int* active, cudaStream_t st) {
    launch_k(k_restrict, dim3((C.n + 255) / 256, C.B), 256, 0, st, F, C, w, fr, cf, cu_zero, mask ? 1 : 0,
                                                             active);
}

void launch_prolong(const LevelView& F, const LevelView& C, const Weights& w, const double* cu,
                    double* fu, bool add, const int* active, cudaStream_t st) {
    dim3 grid((F.n + 255) / 256, F.B);
    if (add)
        launch_k(k_prolong<true>, grid, 256, 0, st, F, C, w, cu, fu, active);
    else
        launch_k(k_prolong<false>, grid, 256, 0, st, F, C, w, cu, fu, active);
}

void launch_coarse(const LevelView& L, const EnvFactor& E, const double* f, double* u,
                   const int* active, cudaStream_t st) {
    launch_k(k_coarse, (L.B + 63) / 64, 64, 0, st, E, f, u, L.B, active);
}

int launch_norm_partials(const double* v, long n, int B, int norm_type, double* partials,
                         cudaStream_t st) {
    long nb = (n + 255) / 256;
    if (nb > 1024) nb = 1024;
    launch_k(k_norm_partials, dim3((int)nb, B), 256, 0, st, v, n, norm_type, partials);
    return (int)nb;
}

void launch_norm_final(const double* partials, int nblk, int B, long n, int norm_type,
                       double* norms, cudaStream_t st) {
    launch_k(k_norm_final<false>, B, nblk >= 4096 ? 1024 : 256, 0, st, partials, nblk, n,
             norm_type, norms, ConvState{}, 0, 0.0, 0.0);
}

void launch_norm_check(const double* partials, int nblk, int B, long n, int norm_type,
                       double* norms, ConvState cs, int max_it, double rel_tol, double abs_tol,
                       cudaStream_t st) {
    launch_k(k_norm_final<true>, B, nblk >= 4096 ? 1024 : 256, 0, st, partials, nblk, n,
             norm_type, norms, cs, max_it, rel_tol, abs_tol);
}

void launch_check(const double* norms, ConvState cs, int B, int max_it, double rel_tol,
                  double abs_tol, cudaStream_t st) {
    launch_k(k_check, (B + 127) / 128, 128, 0, st, norms, cs, B, max_it, rel_tol, abs_tol);
}

void launch_fill(double* p, long n, double v, cudaStream_t st) {
    long nb = (n + 255) / 256;
    if (nb > 4096) nb = 4096;
    if (nb < 1) nb = 1;
    launch_k(k_fill, (int)nb, 256, 0, st, p, n, v);
}

void launch_set_active(int* active, int* count, int* conv, int* remaining, int B,
                       cudaStream_t st) {
    launch_k(k_set_active, (B + 127) / 128, 128, 0, st, active, count, conv, remaining, B);
}

void launch_loop_cond(cudaGraphConditionalHandle h, const int* remaining, cudaStream_t st) {
    launch_k(k_loop_cond, 1, 32, 0, st, h, remaining);
}
void launch_flush(double* buf, long n, cudaStream_t st) {
    k_flush<<<148 * 8, 256, 0, st>>>(buf, n);
}

}  // namespace pmg

namespace pmg {
#ifdef PMG_KTRACE
void read_ktrace(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_ktrace, sizeof(g_ktrace)); }  // 32 entries
void reset_ktrace() {
    static const unsigned long long zero[32] = {};
    cudaMemcpyToSymbol(g_ktrace, zero, sizeof(zero));
}
#endif

void launch_mid_cycle(const MidParams& mp, const int* prog, int nops, int B, const int* active,
                      cudaStream_t st) {
    const size_t sm = (size_t)mp.tail.smem_bytes;
    set_smem(k_mid_cycle, sm);
    static std::set<int> nonportable;
    {
        static std::mutex mu;
        std::lock_guard<std::mutex> g(mu);
        int dev = 0;
        cudaGetDevice(&dev);
        if (!nonportable.count(dev)) {
            cudaFuncSetAttribute(k_mid_cycle, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            nonportable.insert(dev);
        }
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(mp.cl * B);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = mp.cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_on() ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_mid_cycle, mp, prog, nops, active);
    if (e != cudaSuccess) note_launch_error(e);
}

int mid_cluster_size(size_t smem, int want) {
    set_smem(k_mid_cycle, smem);
    cudaFuncSetAttribute(k_mid_cycle, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c = want; c >= 2; c /= 2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_mid_cycle, &cfg) == cudaSuccess && n > 0) return c;
        cudaGetLastError();
    }
    return 0;
}

void launch_coarse_cycle(const CoarseParams& cp, const int* prog, int nops, int B, bool onfly,
                         const int* active, cudaStream_t st) {
    (void)onfly;  // the tail evaluates assembled rows in both stencil modes
    const size_t sm = (size_t)cp.smem_bytes;
    switch (cp.kw) {
        case 1:
            set_smem(k_coarse_cycle<1>, sm);
            launch_k(k_coarse_cycle<1>, B, 512, sm, st, cp, prog, nops, active);
            break;
        case 2:
            set_smem(k_coarse_cycle<2>, sm);
            launch_k(k_coarse_cycle<2>, B, 512, sm, st, cp, prog, nops, active);
            break;
        case 4:
            set_smem(k_coarse_cycle<4>, sm);
            launch_k(k_coarse_cycle<4>, B, 512, sm, st, cp, prog, nops, active);
            break;
        default:
            set_smem(k_coarse_cycle<8>, sm);
            launch_k(k_coarse_cycle<8>, B, 512, sm, st, cp, prog, nops, active);
            break;
    }
}
}  // namespace pmg
