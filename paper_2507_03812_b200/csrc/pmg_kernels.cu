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
#include <cooperative_groups.h>

#include "pmg_kernels.h"

namespace pmg {

namespace {

constexpr unsigned FULL = 0xffffffffu;

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
        typename CF<ONFLY>::T cf{&L, b};
        const Row R = make_row(L, cf, s, t);
        double acc;
        if (R.ident) {
            acc = 0.0;
            acc += 1.0 * U[p];
        } else {
            const int tm = L.tminus(t), tp = L.tplus(t);
            acc = 0.0;
            acc += R.d * U[p];
            if (R.has_sm) acc += R.sm * U[L.idx(s - 1, t)];
            if (R.has_sp) acc += R.sp * U[L.idx(s + 1, t)];
            acc += R.tm * U[L.idx(s, tm)];
            acc += R.tp * U[L.idx(s, tp)];
            if (R.has_sm) {
                acc += R.mm * U[L.idx(s - 1, tm)];
                acc += R.mp * U[L.idx(s - 1, tp)];
            }
            if (R.has_sp) {
                acc += R.pm * U[L.idx(s + 1, tm)];
                acc += R.pp * U[L.idx(s + 1, tp)];
            }
            if (R.origin) acc += R.ph * U[L.idx(0, R.t2)];
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
                                                OriginFactor of, int parity,
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
    typename CF<ONFLY>::T cf{&L, b};
    for (int t = threadIdx.x; t < nt; t += T) {
        const Row R = make_row(L, cf, s, t);
        const int tm = L.tminus(t), tp = L.tplus(t);
        double acc = F[base + t];
        if (R.has_sm) acc -= R.sm * U[L.idx(s - 1, t)];
        if (R.has_sp) acc -= R.sp * U[L.idx(s + 1, t)];
        if (R.has_sm) {
            acc -= R.mm * U[L.idx(s - 1, tm)];
            acc -= R.mp * U[L.idx(s - 1, tp)];
        }
        if (R.has_sp) {
            acc -= R.pm * U[L.idx(s + 1, tm)];
            acc -= R.pp * U[L.idx(s + 1, tp)];
        }
        Y[P(t)] = acc;
    }
    if (s == 0 && L.boundary == 0) {
        __syncthreads();
        if (threadIdx.x == 0) origin_solve_serial(Y, IL, of, b, nt);
        __syncthreads();
    } else {
        const long fo = (long)b * L.split * nt + (long)s * nt;
        for (int t = threadIdx.x; t < nt; t += T) {
            IL[P(t)] = cil[fo + t];
            M[P(t)] = cm[fo + t];
        }
        __syncthreads();
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
                                                const int* __restrict__ active) {
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
    const int tm = L.tminus(t), tp = L.tplus(t);
    typename CF<ONFLY>::T cf{&L, b};
    const long fo = ((long)b * L.nt + t) * len;
    for (int i = threadIdx.x; i < len; i += T) {
        const int s = split + i;
        IL[P(i)] = ril[fo + i];
        M[P(i)] = rm[fo + i];
        if (L.dir(s)) {
            Y[P(i)] = F[base + i];
            continue;
        }
        const Row R = make_row(L, cf, s, t);
        double acc = F[base + i];
        if (s == split && R.has_sm) acc -= R.sm * U[L.idx(s - 1, t)];
        acc -= R.tm * U[L.idx(s, tm)];
        acc -= R.tp * U[L.idx(s, tp)];
        if (R.has_sm) {
            acc -= R.mm * U[L.idx(s - 1, tm)];
            acc -= R.mp * U[L.idx(s - 1, tp)];
        }
        if (R.has_sp) {
            acc -= R.pm * U[L.idx(s + 1, tm)];
            acc -= R.pp * U[L.idx(s + 1, tp)];
        }
        Y[P(i)] = acc;
    }
    __syncthreads();
    line_solve<K, false>(Y, IL, M, len, 0.0, scr);
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
__global__ void k_check(const double* __restrict__ norms, ConvState cs, int B, int it,
                        int max_it, double rel_tol, double abs_tol) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B || !cs.active[b]) return;
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

__global__ void k_set_active(int* active, int* remaining, int B) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) active[b] = 1;
    if (b == 0) *remaining = B;
}

__global__ void k_flush(double* p, long n) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long)gridDim.x * blockDim.x)
        p[i] = p[i] * 0.5 + 1.0;
}

// ------------------------------------------------------------ launch helpers
template <class KernelT>
void set_smem(KernelT kern, size_t bytes) {
    static thread_local bool done = false;  // per instantiation
    (void)done;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
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

inline size_t line_smem(int n) { return (size_t)(3 * padded(n) + 32 * 3 + 8) * sizeof(double); }

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
                     const double* cm, const double* corner, const OriginFactor& of, int parity,
                     const int* active, cudaStream_t st, int T, int lines) {
    const size_t sm = line_smem(L.nt);
    set_smem(k_circle<ON, K>, sm);
    k_circle<ON, K><<<dim3(lines, L.B), T, sm, st>>>(L, u, f, cil, cm, corner, of, parity,
                                                      active);
}

void launch_circle(const LevelView& L, bool onfly, double* u, const double* f, const double* cil,
                   const double* cm, const double* corner, const OriginFactor& of, int parity,
                   const int* active, cudaStream_t st) {
    const int lines = L.split > parity ? (L.split - parity + 1) / 2 : 0;
    if (lines == 0) return;
    int K, T;
    line_shape(L.nt, K, T);
#define PMG_C(KK)                                                                        \
    (onfly ? circle_k<true, KK>(L, u, f, cil, cm, corner, of, parity, active, st, T, lines) \
           : circle_k<false, KK>(L, u, f, cil, cm, corner, of, parity, active, st, T, lines))
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
                     const double* rm, int parity, const int* active, cudaStream_t st, int T,
                     int lines) {
    const size_t sm = line_smem(L.len);
    set_smem(k_radial<ON, K>, sm);
    k_radial<ON, K><<<dim3(lines, L.B), T, sm, st>>>(L, u, f, ril, rm, parity, active);
}

void launch_radial(const LevelView& L, bool onfly, double* u, const double* f, const double* ril,
                   const double* rm, int parity, const int* active, cudaStream_t st) {
    if (L.len <= 0) return;
    const int lines = (L.nt - parity + 1) / 2;
    int K, T;
    line_shape(L.len, K, T);
#define PMG_R(KK)                                                               \
    (onfly ? radial_k<true, KK>(L, u, f, ril, rm, parity, active, st, T, lines) \
           : radial_k<false, KK>(L, u, f, ril, rm, parity, active, st, T, lines))
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

void launch_check(const double* norms, ConvState cs, int B, int it, int max_it, double rel_tol,
                  double abs_tol, cudaStream_t st) {
    k_check<<<(B + 127) / 128, 128, 0, st>>>(norms, cs, B, it, max_it, rel_tol, abs_tol);
}

void launch_fill(double* p, long n, double v, cudaStream_t st) {
    long nb = (n + 255) / 256;
    if (nb > 4096) nb = 4096;
    if (nb < 1) nb = 1;
    k_fill<<<(int)nb, 256, 0, st>>>(p, n, v);
}

void launch_set_active(int* active, int* remaining, int B, cudaStream_t st) {
    k_set_active<<<(B + 127) / 128, 128, 0, st>>>(active, remaining, B);
}

void launch_flush(double* buf, long n, cudaStream_t st) {
    k_flush<<<148 * 8, 256, 0, st>>>(buf, n);
}

}  // namespace pmg
