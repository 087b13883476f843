// Thread-per-line radial sweep for large batches of short lines (config 3).
// See the comment above k_radial_tpl.  Separate translation unit: it shares
// only pmg_lines.cuh with the other line kernels.
#include <cuda_pipeline.h>

#include <algorithm>
#include <cstdlib>

#include "pmg_kernels.h"
#include "pmg_lines.cuh"

namespace pmg {
namespace {

// ------------------------------------------- thread-per-line radial sweep
// Large batches of short radial lines (config 3: 65536 spokes of 431 nodes per
// colour).  The reference's substitution (tridiag_solve, line_algebra.cpp:
// 42-62) is sequential along a line; with this many independent lines the
// cheapest schedule that reproduces it is ONE THREAD PER LINE running it as
// written -- 10 dependent FP64 operations per row, no speculation, no scans --
// so the result is the reference's bit for bit in every mode.  What has to be
// organised is the data movement (a line is contiguous in HBM, a thread walks
// one line):
//   A. all threads of the CTA gather the rhs of its G lines into Y[G][len] in
//      shared memory, the only line-resident array (consecutive threads take
//      consecutive rows of a line: coalesced; the operands of four rows are in
//      flight per thread before any arithmetic);
//   B. forward substitution: the factor rows (L diagonal, sub-diagonal) stream
//      through a ring of [G][R]-row tiles, copied asynchronously by all
//      threads (cp.async, R-row segments of a line are contiguous); thread
//      j < G of warp 0 walks line j through each tile (odd strides: no bank
//      conflicts), one barrier per tile;
//   C. backward substitution with the tiles streamed in reverse order;
//   D. all threads store Y to u, coalesced.
// Several CTAs per SM: one's gather (HBM-bound) overlaps another's
// substitution (one warp, latency-bound).
constexpr int kTplR = 16;   // rows per factor tile
constexpr int kTplS = 5;    // factor tiles in the ring (3 in flight ahead of the reciprocals)
constexpr int kTplT = 128;  // threads per CTA
constexpr int kTplB = 2;    // rhs rows in flight per thread (registers: four CTAs per SM)
constexpr int kTplArrays = 3;  // L diagonal, sub-diagonal, RN(1/l)

// L2 prefetch of the sectors rad_load will touch for row i (no register
// destination: the loads of a later line then come back at L2 latency)
__device__ __forceinline__ void pf_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ void rad_prefetch(const LevelView& L, const double* __restrict__ U,
                                             const double* __restrict__ F, long off, int base,
                                             const RadLine& R, int i) {
    const double* __restrict__ ATT = L.att + off;
    const double* __restrict__ ART = L.art + off;
    const int p = base + i;
    pf_l2(F + p);
    pf_l2(ATT + p);
    pf_l2(ATT + p + R.dTM);
    pf_l2(ATT + p + R.dTP);
    pf_l2(ART + p);
    pf_l2(ART + p + R.dTM);
    pf_l2(ART + p + R.dTP);
    pf_l2(U + p + R.dTM);
    pf_l2(U + p + R.dTP);
}
__device__ __forceinline__ RadLine rad_line(const LevelView& L, int t) {
    RadLine R;
    const int tm = L.tminus(t), tp = L.tplus(t);
    R.dTM = (tm - t) * L.len;
    R.dTP = (tp - t) * L.len;
    R.km = L.k[tm];
    R.kp = L.k[t];
    R.rkm = L.rk[tm];
    R.rkp = L.rk[t];
    return R;
}

// PMG_TPL_TRACE=1: per-phase time (globaltimer ns, thread 0 of every CTA)
// summed over CTAs: [0] gather, [1] forward, [2] backward, [3] store, [4] CTAs
__device__ unsigned long long g_tpl_trace[8];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TPL_MARK(slot)                                              \
    do {                                                            \
        if (trace && threadIdx.x == 0) {                            \
            const unsigned long long now = gtimer();                \
            atomicAdd(&g_tpl_trace[slot], now - tmark);             \
            tmark = now;                                            \
        }                                                           \
    } while (0)

template <bool ONFLY>
__global__ void __launch_bounds__(kTplT, 4) k_radial_tpl(LevelView L, double* __restrict__ u,
                                                         const double* __restrict__ f,
                                                         const double* __restrict__ ril,
                                                         const double* __restrict__ rm,
                                                         int parity,
                                                         const int* __restrict__ active, int G,
                                                         int groups, int flags) {
    pdl_enter();
    const int trace = flags & 1;
    unsigned long long tmark = trace ? gtimer() : 0ull;
    extern __shared__ double smem[];
    const int tid = threadIdx.x;
    const int lines = (L.nt - parity + 1) >> 1;
    const int b = blockIdx.x / groups, grp = blockIdx.x - b * groups;
    if (active && !active[b]) return;
    const int j0 = grp * G;
    const int g = min(G, lines - j0);  // lines of this CTA
    const int len = L.len, ys = len | 1;
    constexpr int RS = kTplR + 1;
    double* Y = smem;                               // [G][ys]
    double* TL = Y + (size_t)G * ys;                // [S][G][R+1] L diagonal
    double* TM = TL + (size_t)kTplS * G * RS;       // [S][G][R+1] sub-diagonal
    double* TR = TM + (size_t)kTplS * G * RS;       // [S][G][R+1] RN(1/l)
    const long off = (long)b * L.n;
    double* U = u + off;
    const double* F = f + off;
    const int NT = (len + kTplR - 1) / kTplR;
    const long fo0 = ((long)b * L.nt + parity + 2 * j0) * len;  // line j: fo0 + 2 j len
    // factor tile k (rows k R ..) into a ring slot, by the warps that do not solve
    auto issue = [&](int k, int slot) {
        if (k >= 0 && k < NT) {
            const int r0 = k * kTplR;
            for (int e = tid - 32; e >= 0 && e < g * kTplR; e += kTplT - 32) {
                const int j = e / kTplR, r = e - j * kTplR, i = r0 + r;
                if (i < len) {
                    const long fo = fo0 + (long)2 * j * len + i;
                    const int d = (slot * G + j) * RS + r;
                    __pipeline_memcpy_async(&TL[d], &ril[fo], 8);
                    __pipeline_memcpy_async(&TM[d], &rm[fo], 8);
                }
            }
        }
        __pipeline_commit();
    };
    auto recips = [&](int k, int slot) {  // TR of tile k, by the warps that do not solve
        if (k < 0 || k >= NT || tid < 32) return;
        const int r0 = k * kTplR;
        for (int e = tid - 32; e < g * kTplR; e += kTplT - 32) {
            const int j = e / kTplR, r = e - j * kTplR;
            if (r0 + r < len) {
                const int d = (slot * G + j) * RS + r;
                TR[d] = __drcp_rn(TL[d]);
            }
        }
    };
    // the first factor tiles travel under the gather
#pragma unroll
    for (int k = 0; k < kTplS - 1; ++k) issue(k, k);
    // ---- A: rhs of every line (reference smoother.cpp:184-205)
    {
        const CoefAt<ONFLY> cf{&L, off, b};
        const bool lean_ok = !ONFLY && !L.rows;
        const int lo = lean_ok ? 1 : len, hi = lean_ok ? len - 3 : -1;  // lean rows lo..hi
        // a lane in four prefetches its sector of the line two ahead
        auto prefetch_line = [&](int j) {
            if (!lean_ok || j >= g || (tid & 3) || !(flags & 2)) return;
            const int t = parity + 2 * (j0 + j);
            const RadLine R = rad_line(L, t);
            for (int i = tid; i < len; i += kTplT)
                rad_prefetch(L, U, F, off, L.split * L.nt + t * len, R, min(i + 2, len - 1));
        };
        prefetch_line(0);
        prefetch_line(1);
        for (int j = 0; j < g; ++j) {
            const int t = parity + 2 * (j0 + j);
            const int base = L.split * L.nt + t * len;
            const RadLine R = rad_line(L, t);
            double* Yj = Y + (size_t)j * ys;
            prefetch_line(j + 2);
            for (int i0 = tid; i0 < len; i0 += kTplB * kTplT) {
                RadOps o[kTplB];
#pragma unroll
                for (int q = 0; q < kTplB; ++q) {
                    const int i = i0 + q * kTplT;
                    if (i >= lo && i <= hi) rad_load(L, U, F, off, base, R, i, o[q]);
                }
#pragma unroll
                for (int q = 0; q < kTplB; ++q) {
                    const int i = i0 + q * kTplT;
                    if (i >= lo && i <= hi) Yj[i] = rad_eval(o[q], R);
                }
            }
        }
        // the other rows (first row, the rows next to the outer boundary;
        // every row of Give / assembled-row levels) of all lines together
        const int nlean = hi >= lo ? hi - lo + 1 : 0, nrest = len - nlean;
        for (int e = tid; e < g * nrest; e += kTplT) {
            const int j = e / nrest, q = e - j * nrest;
            const int i = nlean == 0 ? q : (q == 0 ? 0 : hi + q);
            const int t = parity + 2 * (j0 + j);
            const RadLine R = rad_line(L, t);
            Y[(size_t)j * ys + i] =
                radial_rhs<ONFLY>(L, cf, U, F, off, t, L.split * L.nt + t * len, R, i);
        }
    }
    // ---- B, C: substitution (tridiag_solve, line_algebra.cpp:42-62)
    const int sj = tid < g ? tid : 0;
    double* Yj = Y + (size_t)sj * ys;
    double y = 0.0;
    __pipeline_wait_prior(kTplS - 2);
    __syncthreads();  // tile 0 landed, Y complete
    recips(0, 0);
    TPL_MARK(0);
    {  // forward: y_i = (b_i - m_{i-1} y_{i-1}) / l_i
        double mprev = 0.0;
        for (int k = 0; k < NT; ++k) {
            __pipeline_wait_prior(kTplS - 3);
            __syncthreads();  // tile k+1 landed, TR of tile k written, tile k-1 consumed
            issue(k + kTplS - 1, (k + kTplS - 1) % kTplS);
            recips(k + 1, (k + 1) % kTplS);
            if (tid < g) {
                const int d = ((k % kTplS) * G + sj) * RS;
                const double* tl = TL + d;
                const double* tm = TM + d;
                const double* tr = TR + d;
                const int r0 = k * kTplR;
                if (r0 > 0 && r0 + kTplR <= len) {  // full interior tile: straight-line code
                    const double* yr = Yj + r0;
                    double bq[kTplR];
#pragma unroll
                    for (int r = 0; r < kTplR; ++r) bq[r] = yr[r];
#pragma unroll
                    for (int r = 0; r < kTplR; ++r) {
                        y = xdiv(bq[r] - mprev * y, tl[r], tr[r]);
                        bq[r] = y;
                        mprev = tm[r];
                    }
#pragma unroll
                    for (int r = 0; r < kTplR; ++r) Yj[r0 + r] = bq[r];
                } else {
                    for (int r = 0; r < kTplR; ++r) {
                        const int i = r0 + r;
                        if (i < len) {
                            const double bq = Yj[i];
                            const double a = bq - mprev * y;
                            y = xdiv(i > 0 ? a : bq, tl[r], tr[r]);
                            Yj[i] = y;
                            mprev = tm[r];
                        }
                    }
                }
            }
        }
    }
    __pipeline_wait_prior(0);
    __syncthreads();
    TPL_MARK(1);
#pragma unroll
    for (int k = 0; k < kTplS - 1; ++k) issue(NT - 1 - k, k);
    __pipeline_wait_prior(kTplS - 2);
    __syncthreads();
    recips(NT - 1, 0);
    {  // backward: x_i = (y_i - m_i x_{i+1}) / l_i
        for (int kk = 0; kk < NT; ++kk) {
            const int k = NT - 1 - kk;
            __pipeline_wait_prior(kTplS - 3);
            __syncthreads();
            issue(k - (kTplS - 1), (kk + kTplS - 1) % kTplS);
            recips(k - 1, (kk + 1) % kTplS);
            if (tid < g) {
                const int d = ((kk % kTplS) * G + sj) * RS;
                const double* tl = TL + d;
                const double* tm = TM + d;
                const double* tr = TR + d;
                const int r0 = k * kTplR;
                if (r0 + kTplR < len) {  // full tile below the last row
                    double yq[kTplR];
#pragma unroll
                    for (int r = 0; r < kTplR; ++r) yq[r] = Yj[r0 + r];
#pragma unroll
                    for (int r = kTplR - 1; r >= 0; --r) {
                        y = xdiv(yq[r] - tm[r] * y, tl[r], tr[r]);
                        yq[r] = y;
                    }
#pragma unroll
                    for (int r = 0; r < kTplR; ++r) Yj[r0 + r] = yq[r];
                } else {
                    for (int r = kTplR - 1; r >= 0; --r) {
                        const int i = r0 + r;
                        if (i < len) {
                            const double yq = Yj[i];
                            const double a = yq - tm[r] * y;
                            y = xdiv(i < len - 1 ? a : yq, tl[r], tr[r]);
                            Yj[i] = y;
                        }
                    }
                }
            }
        }
    }
    __syncthreads();
    TPL_MARK(2);
    // ---- D: store
    for (int j = 0; j < g; ++j) {
        const int base = L.split * L.nt + (parity + 2 * (j0 + j)) * len;
        const double* Yr = Y + (size_t)j * ys;
        for (int i = tid; i < len; i += kTplT) U[base + i] = Yr[i];
    }
    TPL_MARK(3);
    if (trace && tid == 0) atomicAdd(&g_tpl_trace[4], 1ull);
}

}  // namespace

// Thread-per-line sweep (k_radial_tpl) for batches of at least
// PMG_TPL_MIN_LINES lines (default 4096) whose rhs fits shared memory with at
// least 8 lines per CTA and two CTAs per SM; PMG_TPL=0 disables.  Returns the
// lines per CTA (0: not applicable).
static int tpl_lines(int len, int lines, long lines_total) {
    static const long min_lines = [] {
        const char* e = std::getenv("PMG_TPL_MIN_LINES");
        return e ? std::atol(e) : 4096L;
    }();
    // opt-in (PMG_TPL=1): measured on config 3 at 1.74 ms per finest B+W sweep
    // against 1.54 ms for the warp-per-line kernel -- a thread's substitution
    // advances one row per ~77 cycles (5 dependent FP64 operations) and shared
    // memory holds only ~32 lines per SM, which bounds the sweep at ~0.45 ms per
    // colour however the data movement is arranged
    static const bool on = [] {
        const char* e = std::getenv("PMG_TPL");
        return e ? std::atoi(e) != 0 : false;
    }();
    if (!on || lines_total < min_lines || len < 24) return 0;
    const size_t per_line =
        ((size_t)(len | 1) + kTplArrays * kTplS * (kTplR + 1)) * sizeof(double);
    int gmax = (int)std::min<size_t>(32, (size_t)44 * 1024 / per_line);  // four CTAs per SM
    if (gmax < 8) gmax = (int)std::min<size_t>(32, (size_t)112 * 1024 / per_line);
    if (const char* e = std::getenv("PMG_TPL_G"))
        gmax = (int)std::min<size_t>(std::min<size_t>(32, (size_t)224 * 1024 / per_line),
                                     std::max(1, std::atoi(e)));
    if (gmax < 8) return 0;
    const int groups = (lines + gmax - 1) / gmax;
    return (lines + groups - 1) / groups;  // balanced groups
}


bool launch_radial_tpl(const LevelView& L, bool onfly, double* u, const double* f,
                       const double* ril, const double* rm, int parity, const int* active,
                       cudaStream_t st) {
    const int lines = (L.nt - parity + 1) / 2;
    if (const int G = tpl_lines(L.len, lines, (long)lines * L.B)) {
        const int groups = (lines + G - 1) / G;
        const size_t sm = ((size_t)G * (L.len | 1) + (size_t)kTplArrays * kTplS * G * (kTplR + 1)) *
                          sizeof(double);
        const dim3 grid((unsigned)(groups * L.B));
        // bit 0: phase trace (PMG_TPL_TRACE), bit 1: L2 prefetch two lines ahead
        // (PMG_TPL_PF; measured slower: the gather is bandwidth-bound, not latency-bound)
        static const int trace = [] {
            const char* e = std::getenv("PMG_TPL_TRACE");
            const char* n = std::getenv("PMG_TPL_PF");
            return (e && std::atoi(e) ? 1 : 0) | (n && std::atoi(n) ? 2 : 0);
        }();
        if (onfly) {
            set_smem(k_radial_tpl<true>, sm);
            launch_k(k_radial_tpl<true>, grid, kTplT, sm, st, L, u, f, ril, rm, parity, active, G,
                     groups, trace);
        } else {
            set_smem(k_radial_tpl<false>, sm);
            launch_k(k_radial_tpl<false>, grid, kTplT, sm, st, L, u, f, ril, rm, parity, active, G,
                     groups, trace);
        }
        return true;
    }
    return false;
}

}  // namespace pmg

// diagnostics (PMG_TPL_TRACE=1): read and clear the phase sums of k_radial_tpl
extern "C" int pmg_debug_tpl_trace(unsigned long long* out8) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out8, pmg::g_tpl_trace, sizeof(unsigned long long) * 8);
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(pmg::g_tpl_trace, z, sizeof z);
    return 0;
}
