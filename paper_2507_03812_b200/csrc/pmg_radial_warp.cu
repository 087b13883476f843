// Warp-per-line radial sweep for large batches of short lines (config 3):
// the kernel, its launch shape and dispatch.  Separate translation unit (it
// shares pmg_lines.cuh with the other line kernels) so that it rebuilds in
// seconds.
#include <cuda_pipeline.h>

#include <algorithm>
#include <cstdlib>

#include "pmg_kernels.h"
#include "pmg_lines.cuh"

#ifndef PMG_RAD_UNROLL
#define PMG_RAD_UNROLL 2
#endif

namespace pmg {
namespace {

constexpr int kRadUnroll = PMG_RAD_UNROLL;
// rows of a rhs gather in flight per lane.  Radial: 2 (120 registers, 16 warps
// per SM; measured 3 or 4 rows at 144-158 registers and 12 warps: 1.26-1.27 ms
// vs 1.11 ms; 3-4 rows with the +-1 operands taken by shuffles, 11 loads per
// row: 1.23-1.43 ms).  Circle: 4 (0.341 -> 0.305 ms).
#ifndef PMG_CIRC_UNROLL
#define PMG_CIRC_UNROLL 4
#endif
constexpr int kCircUnroll = PMG_CIRC_UNROLL;

// ---------------------------------------------- warp-per-line radial sweep
// Many radial lines of at most 32*KW nodes (config 3: 65536 spokes of 431
// nodes per colour): one WARP per spoke and no block barriers.  The warp
// gathers the rhs of rows lane, lane+32, ... (coalesced loads of the
// spoke-major arrays; all operands of a row issued before its arithmetic,
// the same expressions as radial_body, so the rhs is bitwise the same) and
// stages it with the line's factors in its own shared-memory slice.  Each
// lane then takes KE consecutive rows -- KE odd, so the 8-byte shared-memory
// reads of a half-warp hit 16 distinct banks pairs -- and the warp solves the
// line by warp scans: in the reference's exact order by speculation and
// verification waves (warp_tri_ex) or, fast mode, with the scans' values
// (warp_tri_fast).  The result goes back through the slice, coalesced.
// L L^T x = b of one line by one warp (tridiag_solve, line_algebra.cpp:42-62).
// The line is PADDED to 32 KE rows with identity rows (l = 1, m = 0, b = 0),
// and the sub-diagonal is stored shifted (Mp[j] = m_{j-1}, Mp[0] = 0), so no
// row of either substitution is special: the first row subtracts 0 * 0, the
// last real row subtracts m = 0 times the padding's x = 0 -- the same bits as
// the reference's unsubtracted rows -- and every loop below is straight-line.
// y[q]: row j0 + q (j0 = lane KE) of b on entry, of x on exit.
// EXACT: the reference's sequential substitution bit for bit -- the warp
// scan's approximate chunk-entry values seed a restart of the recurrence one
// chunk early (the recurrences contract, |m/l| < 1, so the restarted
// trajectory merges with the reference's bit for bit within a few rows);
// lanes whose trajectory at their predecessor's last row differs from the
// predecessor's result recompute from that result, in waves (ballots), until
// every lane starts from its predecessor's end bit for bit -- which is then
// the sequential substitution by induction from row 0.  Fast: the scan's
// values (reciprocal multiplies; differs in the last bits).
template <int KE, bool EXACT>
__device__ __forceinline__ void warp_tri(double (&y)[KE], const double* __restrict__ Ld,
                                         const double* __restrict__ Mp) {
    const int lane = threadIdx.x & 31, j0 = lane * KE;
    double b[KE], rc[KE];
#pragma unroll
    for (int q = 0; q < KE; ++q) {
        b[q] = y[q];
        rc[q] = __drcp_rn(Ld[j0 + q]);
    }
    // ---- forward: y_j = (b_j - m_{j-1} y_{j-1}) / l_j
    {
        double A = 1.0, Bv[1] = {0.0};
#pragma unroll
        for (int q = 0; q < KE; ++q) {
            const double a = -(Mp[j0 + q] * rc[q]);
            Bv[0] = a * Bv[0] + b[q] * rc[q];
            A = a * A;
        }
        double yin[1];
        warp_scan<1, true>(A, Bv, yin);
        if (!EXACT) {
            double v = yin[0];
#pragma unroll
            for (int q = 0; q < KE; ++q) {
                v = (b[q] - Mp[j0 + q] * v) * rc[q];
                y[q] = v;
            }
        } else {
            // lane-1's chunk from the approximate value entering it (lane 0:
            // clamped indices, result unused; lane 1 restarts at row 0: exact)
            const int jp = lane ? j0 - KE : 0;
            double v = __shfl_up_sync(FULL, yin[0], 1);
#pragma unroll
            for (int q = 0; q < KE; ++q) {
                const double bp = __shfl_up_sync(FULL, b[q], 1);
                const double rp = __shfl_up_sync(FULL, rc[q], 1);
                v = xdiv(bp - Mp[jp + q] * v, Ld[jp + q], rp);
            }
            double st = lane ? v : 0.0;
            auto chunk = [&](double w) {
#pragma unroll
                for (int q = 0; q < KE; ++q) {
                    w = xdiv(b[q] - Mp[j0 + q] * w, Ld[j0 + q], rc[q]);
                    y[q] = w;
                }
                return w;
            };
            double e = chunk(st);
            for (;;) {
                const double pe = __shfl_up_sync(FULL, e, 1);
                const bool bad = lane >= 1 && !same_bits(st, pe);
                if (!__any_sync(FULL, bad)) break;
                if (bad) {
                    st = pe;
                    e = chunk(st);
                }
            }
        }
    }
    // ---- backward: x_j = (y_j - m_j x_{j+1}) / l_j, m_j = Mp[j + 1]
#pragma unroll
    for (int q = 0; q < KE; ++q) b[q] = y[q];
    double G = 1.0, Dv[1] = {0.0};
#pragma unroll
    for (int q = KE - 1; q >= 0; --q) {
        const double g = -(Mp[j0 + q + 1] * rc[q]);
        Dv[0] = g * Dv[0] + b[q] * rc[q];
        G = g * G;
    }
    double xin[1];
    warp_scan<1, false>(G, Dv, xin);
    if (!EXACT) {
        double v = xin[0];
#pragma unroll
        for (int q = KE - 1; q >= 0; --q) {
            v = (b[q] - Mp[j0 + q + 1] * v) * rc[q];
            y[q] = v;
        }
        return;
    }
    // lane+1's chunk from the approximate value entering it from above (lane
    // 31: clamped, unused; lane 30 restarts at the padded end: exact)
    const int jn = lane < 31 ? j0 + KE : j0;
    double v = __shfl_down_sync(FULL, xin[0], 1);
#pragma unroll
    for (int q = KE - 1; q >= 0; --q) {
        const double yn = __shfl_down_sync(FULL, b[q], 1);
        const double rn = __shfl_down_sync(FULL, rc[q], 1);
        v = xdiv(yn - Mp[jn + q + 1] * v, Ld[jn + q], rn);
    }
    double st = lane < 31 ? v : 0.0;
    auto chunk = [&](double w) {
#pragma unroll
        for (int q = KE - 1; q >= 0; --q) {
            w = xdiv(b[q] - Mp[j0 + q + 1] * w, Ld[j0 + q], rc[q]);
            y[q] = w;
        }
        return w;
    };
    double e = chunk(st);
    for (;;) {
        const double pe = __shfl_down_sync(FULL, e, 1);
        const bool bad = lane < 31 && !same_bits(st, pe);
        if (!__any_sync(FULL, bad)) break;
        if (bad) {
            st = pe;
            e = chunk(st);
        }
    }
}

// rows per lane >= ceil(n / 32), odd (conflict-free chunked shared-memory reads)
__host__ __device__ __forceinline__ int warp_ke(int n) { return ((n + 31) >> 5) | 1; }
// shared-memory doubles per line: rhs / solution, L diagonal, shifted sub-diagonal (+1, even)
__host__ __device__ __forceinline__ int warp_slice(int ke) { return 3 * 32 * ke + 2; }

template <bool ONFLY, int KE, bool EXACT>
__global__ void __launch_bounds__(128) k_radial_warp(LevelView L, double* __restrict__ u,
                                                     const double* __restrict__ f,
                                                     const double* __restrict__ ril,
                                                     const double* __restrict__ rm, int parity,
                                                     const int* __restrict__ active) {
    pdl_enter();
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int lines = (L.nt - parity + 1) >> 1;
    const long g = (long)blockIdx.x * (blockDim.x >> 5) + w;
    if (g >= (long)lines * L.B) return;  // whole warps only
    const int b = (int)(g / lines);
    const int t = parity + 2 * (int)(g - (long)b * lines);
    if (active && !active[b]) return;
    constexpr int stride = 32 * KE;
    const int len = L.len;
    const long off = (long)b * L.n;
    double* U = u + off;
    const double* F = f + off;
    const int base = L.split * L.nt + t * len;
    const long fo = ((long)b * L.nt + t) * len;
    double* Y = smem + (long)w * warp_slice(KE);
    double* Ld = Y + stride;
    double* Mp = Ld + stride;  // stride + 1 entries
    RadLine R;
    {
        const int tm = L.tminus(t), tp = L.tplus(t);
        R.dTM = (tm - t) * len;
        R.dTP = (tp - t) * len;
        R.km = L.k[tm];
        R.kp = L.k[t];
        R.rkm = L.rk[tm];
        R.rkp = L.rk[t];
    }
    const CoefAt<ONFLY> cf{&L, off, b};
    // factors of the line (asynchronous copies, in flight under the rhs
    // gather) and the identity padding
#pragma unroll 4
    for (int i = lane; i < stride; i += 32) {
        if (i < len)
            __pipeline_memcpy_async(&Ld[i], &ril[fo + i], 8);
        else
            Ld[i] = 1.0;
        if (i < len - 1)
            __pipeline_memcpy_async(&Mp[i + 1], &rm[fo + i], 8);
        else
            Mp[i + 1] = 0.0;
        if (i >= len) Y[i] = 0.0;
    }
    __pipeline_commit();
    if (lane == 0) Mp[0] = 0.0;
#ifdef PMG_DIAG_NOGATHER
    if (true) {
        for (int i = lane; i < len; i += 32) Y[i] = F[base + i];
    } else
#endif
    if (!ONFLY && !L.rows && len >= 4) {
        // Take: rows 1 .. len-3 are lean and branch-free -- the operands of
        // kRadUnroll rows are in flight per lane before any arithmetic; the
        // first row (coupled to the circle region) and the two rows at the
        // outer boundary go through the general row on three lanes
        for (int i0 = 1 + lane; i0 <= len - 3; i0 += 32 * kRadUnroll) {
            RadOps o[kRadUnroll];
#pragma unroll
            for (int q = 0; q < kRadUnroll; ++q)
                if (i0 + 32 * q <= len - 3) rad_load(L, U, F, off, base, R, i0 + 32 * q, o[q]);
#pragma unroll
            for (int q = 0; q < kRadUnroll; ++q)
                if (i0 + 32 * q <= len - 3) Y[i0 + 32 * q] = rad_eval(o[q], R);
        }
        if (lane < 3) {
            const int i = lane == 0 ? 0 : len - 3 + lane;
            Y[i] = radial_rhs<ONFLY>(L, cf, U, F, off, t, base, R, i);
        }
    } else {
#pragma unroll 2
        for (int i = lane; i < len; i += 32)
            Y[i] = radial_rhs<ONFLY>(L, cf, U, F, off, t, base, R, i);
    }
    __pipeline_wait_prior(0);
    __syncwarp();
    const int j0 = lane * KE;
    double y[KE];
#pragma unroll
    for (int q = 0; q < KE; ++q) y[q] = Y[j0 + q];
#ifndef PMG_DIAG_NOSOLVE
    warp_tri<KE, EXACT>(y, Ld, Mp);
#endif
    __syncwarp();
#pragma unroll
    for (int q = 0; q < KE; ++q) Y[j0 + q] = y[q];
    __syncwarp();
    for (int i = lane; i < len; i += 32) U[base + i] = Y[i];
}

// ---------------------------------------------- warp-per-line circle sweep
// The same scheme for large batches of circle lines (config 3: 10496 rings of
// 512 nodes per colour): one warp per ring, rhs gather (smoother.cpp:162-182;
// lean interior rings branch-free with the operands of kRadUnroll nodes in
// flight per lane, the ring next to the radial region through the general
// row), the core solve T y = b by warp_tri on the identity-padded line, then
// the Sherman-Morrison correction of cyclic_tridiag_solve
// (line_algebra.cpp:112-118) with the precomputed z = T^{-1}(e_1 + e_n)
// (k_circle_z, the reference's own sequence).  The across-origin ring is not
// a cyclic line and stays with k_circle.
template <int KE, bool EXACT>
__global__ void __launch_bounds__(128) k_circle_warp(LevelView L, double* __restrict__ u,
                                                     const double* __restrict__ f,
                                                     const double* __restrict__ cil,
                                                     const double* __restrict__ cm,
                                                     const double* __restrict__ corner,
                                                     const double* __restrict__ cz, int s_first,
                                                     int nl, const int* __restrict__ active) {
    pdl_enter();
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long g = (long)blockIdx.x * (blockDim.x >> 5) + w;
    if (g >= (long)nl * L.B) return;  // whole warps only
    const int b = (int)(g / nl);
    const int s = s_first + 2 * (int)(g - (long)b * nl);
    if (active && !active[b]) return;
    constexpr int stride = 32 * KE;
    const int nt = L.nt;
    const long off = (long)b * L.n;
    double* U = u + off;
    const double* F = f + off;
    const int base = s * nt;
    if (L.dir(s)) {
        for (int t = lane; t < nt; t += 32) U[base + t] = F[base + t];
        return;
    }
    const long fo = (long)b * L.split * nt + (long)s * nt;
    double* Y = smem + (long)w * warp_slice(KE);
    double* Ld = Y + stride;
    double* Mp = Ld + stride;  // stride + 1 entries
#pragma unroll 4
    for (int i = lane; i < stride; i += 32) {
        if (i < nt)
            __pipeline_memcpy_async(&Ld[i], &cil[fo + i], 8);
        else
            Ld[i] = 1.0;
        if (i < nt - 1)
            __pipeline_memcpy_async(&Mp[i + 1], &cm[fo + i], 8);
        else
            Mp[i + 1] = 0.0;
        if (i >= nt) Y[i] = 0.0;
    }
    __pipeline_commit();
    if (lane == 0) Mp[0] = 0.0;
    if (circle_lean_ring(L, s)) {
        const double hm = L.h[s - 1], rhm = L.rh[s - 1], hp = L.h[s], rhp = L.rh[s];
        for (int t0 = lane; t0 < nt; t0 += 32 * kCircUnroll) {
            CircOps o[kCircUnroll];
#pragma unroll
            for (int q = 0; q < kCircUnroll; ++q)
                if (t0 + 32 * q < nt) circ_load<false>(L, off, s, t0 + 32 * q, U, F, o[q]);
#pragma unroll
            for (int q = 0; q < kCircUnroll; ++q)
                if (t0 + 32 * q < nt) Y[t0 + 32 * q] = circ_eval(o[q], hm, rhm, hp, rhp);
        }
    } else {
        const CoefAt<false> cf{&L, off, b};
        for (int t = lane; t < nt; t += 32) {
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
            Y[t] = acc;
        }
    }
    __pipeline_wait_prior(0);
    __syncwarp();
    const int j0 = lane * KE;
    double y[KE];
#pragma unroll
    for (int q = 0; q < KE; ++q) y[q] = Y[j0 + q];
    warp_tri<KE, EXACT>(y, Ld, Mp);
    __syncwarp();
#pragma unroll
    for (int q = 0; q < KE; ++q) Y[j0 + q] = y[q];
    __syncwarp();
    // tau = c (x_0 + x_{n-1}) / (1 + c (z_0 + z_{n-1})); x -= tau z
    const double c = corner[(long)b * L.split + s];
    const double* __restrict__ z = cz + fo;
    const double tau = c * (Y[0] + Y[nt - 1]) / (1.0 + c * (z[0] + z[nt - 1]));
    for (int t = lane; t < nt; t += 32) U[base + t] = Y[t] - tau * z[t];
}

}  // namespace

// rows per lane of the warp-per-line kernels for a line of n nodes when the
// batch of lines_total concurrent lines is large enough (0: CTA-per-line
// kernels).  PMG_WARP_LINES=0 disables; PMG_WARP_MIN_LINES sets the batch.
static int warp_kw(int n, long lines_total) {
    static const long min_lines = [] {
        const char* e = std::getenv("PMG_WARP_MIN_LINES");
        return e ? std::atol(e) : 1024L;
    }();
    static const bool on = [] {
        const char* e = std::getenv("PMG_WARP_LINES");
        return e ? std::atoi(e) != 0 : true;
    }();
    if (!on || lines_total < min_lines || n < 2) return 0;
    const int ke = warp_ke(n);
    return ke <= 17 ? ke : 0;  // odd, 1 .. 17
}

template <bool ON, int KW>
static void radial_warp_k(const LevelView& L, double* u, const double* f, const double* ril,
                          const double* rm, int parity, bool exact, const int* active,
                          cudaStream_t st, long lines_total) {
    constexpr int WPB = 4;  // warps (lines) per CTA
    const size_t sm = (size_t)WPB * warp_slice(KW) * sizeof(double);
    const dim3 grid((unsigned)((lines_total + WPB - 1) / WPB));
    if (exact) {
        set_smem(k_radial_warp<ON, KW, true>, sm);
        launch_k(k_radial_warp<ON, KW, true>, grid, 32 * WPB, sm, st, L, u, f, ril, rm, parity,
                 active);
    } else {
        set_smem(k_radial_warp<ON, KW, false>, sm);
        launch_k(k_radial_warp<ON, KW, false>, grid, 32 * WPB, sm, st, L, u, f, ril, rm, parity,
                 active);
    }
}


bool launch_radial_warp(const LevelView& L, bool onfly, double* u, const double* f,
                        const double* ril, const double* rm, int parity, bool serial,
                        const int* active, cudaStream_t st) {
    const int lines = (L.nt - parity + 1) / 2;
    if (const int kw = warp_kw(L.len, (long)lines * L.B)) {
        const long lt = (long)lines * L.B;
#define PMG_RW(ON, KK) radial_warp_k<ON, KK>(L, u, f, ril, rm, parity, serial, active, st, lt)
        // Take: the exact odd rows-per-lane count; Give (on-the-fly
        // coefficients) rounds up to fewer instantiations (identity padding)
        if (onfly) {
            if (kw <= 5) PMG_RW(true, 5);
            else if (kw <= 9) PMG_RW(true, 9);
            else PMG_RW(true, 17);
        } else {
            switch (kw) {
                case 1: case 3: PMG_RW(false, 3); break;
                case 5: PMG_RW(false, 5); break;
                case 7: PMG_RW(false, 7); break;
                case 9: PMG_RW(false, 9); break;
                case 11: PMG_RW(false, 11); break;
                case 13: PMG_RW(false, 13); break;
                case 15: PMG_RW(false, 15); break;
                default: PMG_RW(false, 17); break;
            }
        }
#undef PMG_RW
        return true;
    }
    return false;
}


bool warp_batch_ok(int n, long lines_total) { return warp_kw(n, lines_total) != 0; }

template <int KW>
static void circle_warp_k(const LevelView& L, double* u, const double* f, const double* cil,
                          const double* cm, const double* corner, const double* cz, int s_first,
                          int nl, bool exact, const int* active, cudaStream_t st) {
    constexpr int WPB = 4;  // warps (lines) per CTA
    const size_t sm = (size_t)WPB * warp_slice(KW) * sizeof(double);
    const dim3 grid((unsigned)(((long)nl * L.B + WPB - 1) / WPB));
    if (exact) {
        set_smem(k_circle_warp<KW, true>, sm);
        launch_k(k_circle_warp<KW, true>, grid, 32 * WPB, sm, st, L, u, f, cil, cm, corner, cz,
                 s_first, nl, active);
    } else {
        set_smem(k_circle_warp<KW, false>, sm);
        launch_k(k_circle_warp<KW, false>, grid, 32 * WPB, sm, st, L, u, f, cil, cm, corner, cz,
                 s_first, nl, active);
    }
}

// Rings s_first, s_first + 2, ... (nl of them, none the across-origin ring) of
// a Take level with cached coefficients; false: batch too small / lines too long.
bool launch_circle_warp(const LevelView& L, double* u, const double* f, const double* cil,
                        const double* cm, const double* corner, const double* cz, int s_first,
                        int nl, bool serial, const int* active, cudaStream_t st) {
    if (L.rows || !cz) return false;
    const int kw = warp_kw(L.nt, (long)nl * L.B);
    if (!kw) return false;
#define PMG_CW(KK) circle_warp_k<KK>(L, u, f, cil, cm, corner, cz, s_first, nl, serial, active, st)
    switch (kw) {
        case 1: case 3: PMG_CW(3); break;
        case 5: PMG_CW(5); break;
        case 7: PMG_CW(7); break;
        case 9: PMG_CW(9); break;
        case 11: PMG_CW(11); break;
        case 13: PMG_CW(13); break;
        case 15: PMG_CW(15); break;
        default: PMG_CW(17); break;
    }
#undef PMG_CW
    return true;
}

}  // namespace pmg
