// Pieces shared by the line-sweep translation units (pmg_kernels.cu,
// pmg_tpl.cu): exact division, the rhs of a radial line row, launch helpers.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

#include "pmg_common.cuh"

namespace pmg {

void note_launch_error(cudaError_t e);

// Programmatic dependent launch: every kernel of the solve lets the next one
// in the stream start launching at once and waits for its predecessor's
// results before touching them (griddepcontrol; no-ops without the launch
// attribute).
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

struct RadLine {  // per-spoke constants of the lean interior rows
    int dTM, dTP;
    double km, kp, rkm, rkp;
};

// rhs row i of radial line t (reference smoother.cpp:184-205): the branches
// of radial_body for one row.
template <bool ONFLY>
__device__ __forceinline__ double radial_rhs(const LevelView& L, const CoefAt<ONFLY>& cf,
                                             const double* __restrict__ U,
                                             const double* __restrict__ F, long off, int t,
                                             int base, const RadLine& R, int i) {
    const int s = L.split + i, p = base + i;
    if (L.rows) {
        const double* Rw = L.rows + (off / L.n) * 10 * L.n;
        const int n = L.n;
        const Nbr q = neighbours(L, s, t, p);
        double acc = F[p];
        if (s == L.split) acc -= Rw[1 * n + p] * U[q.pSM];
        acc -= Rw[3 * n + p] * U[q.pTM];
        acc -= Rw[4 * n + p] * U[q.pTP];
        acc -= Rw[5 * n + p] * U[q.pSMTM];
        acc -= Rw[6 * n + p] * U[q.pSMTP];
        acc -= Rw[7 * n + p] * U[q.pSPTM];
        acc -= Rw[8 * n + p] * U[q.pSPTP];
        return acc;
    }
    if (!ONFLY && i >= 1 && i <= L.len - 2) {
        const double* __restrict__ ATT = L.att + off;
        const double* __restrict__ ART = L.art + off;
        const int dTM = R.dTM, dTP = R.dTP;
        const double fP = F[p];
        const double attP = ATT[p], attM = ATT[p + dTM], attQ = ATT[p + dTP];
        const double artM = ART[p + dTM], artQ = ART[p + dTP];
        const double artSM = ART[p - 1], artSP = ART[p + 1];
        const double uM = U[p + dTM], uQ = U[p + dTP];
        const double uMM = U[p + dTM - 1], uQM = U[p + dTP - 1];
        const double uMP = U[p + dTM + 1], uQP = U[p + dTP + 1];
        const double hbar = 0.5 * (L.h[s - 1] + L.h[s]);
        const double south = -xdiv(hbar, R.km, R.rkm) * (attP + attM);
        const double north = -xdiv(hbar, R.kp, R.rkp) * (attP + attQ);
        double acc = fP;
        acc -= south * uM;
        acc -= north * uQ;
        acc -= (-(artM + artSM) * 0.25) * uMM;
        acc -= ((artSM + artQ) * 0.25) * uQM;
        if (s + 1 < L.nr - 1 || !L.dir(s + 1)) {
            acc -= ((artM + artSP) * 0.25) * uMP;
            acc -= (-(artSP + artQ) * 0.25) * uQP;
        }
        return acc;
    }
    if (L.dir(s)) return F[p];
    const Nbr q = neighbours(L, s, t, p);
    const Row Rr = make_row_fast(L, cf, s, t, p, q);
    double acc = F[p];
    if (s == L.split && Rr.has_sm) acc -= Rr.sm * U[q.pSM];
    acc -= Rr.tm * U[q.pTM];
    acc -= Rr.tp * U[q.pTP];
    if (Rr.has_sm) {
        acc -= Rr.mm * U[q.pSMTM];
        acc -= Rr.mp * U[q.pSMTP];
    }
    if (Rr.has_sp) {
        acc -= Rr.pm * U[q.pSPTM];
        acc -= Rr.pp * U[q.pSPTP];
    }
    return acc;
}

struct RadOps {  // operands of one lean interior rhs row (see radial_rhs)
    double fP, attP, attM, attQ, artM, artQ, artSM, artSP, uM, uQ, uMM, uQM, uMP, uQP, hm, hp;
};
__device__ __forceinline__ void rad_load(const LevelView& L, const double* __restrict__ U,
                                         const double* __restrict__ F, long off, int base,
                                         const RadLine& R, int i, RadOps& o) {
    const double* __restrict__ ATT = L.att + off;
    const double* __restrict__ ART = L.art + off;
    const int s = L.split + i, p = base + i;
    const int dTM = R.dTM, dTP = R.dTP;
    o.fP = F[p];
    o.attP = ATT[p];
    o.attM = ATT[p + dTM];
    o.attQ = ATT[p + dTP];
    o.artM = ART[p + dTM];
    o.artQ = ART[p + dTP];
    o.artSM = ART[p - 1];
    o.artSP = ART[p + 1];
    o.uM = U[p + dTM];
    o.uQ = U[p + dTP];
    o.uMM = U[p + dTM - 1];
    o.uQM = U[p + dTP - 1];
    o.uMP = U[p + dTM + 1];
    o.uQP = U[p + dTP + 1];
    o.hm = L.h[s - 1];
    o.hp = L.h[s];
}
// rows 1 .. len-3 of a Take line: the lean branch of radial_rhs with both
// outer corners present, the same expressions in the same order
__device__ __forceinline__ double rad_eval(const RadOps& o, const RadLine& R) {
    const double hbar = 0.5 * (o.hm + o.hp);
    const double south = -xdiv(hbar, R.km, R.rkm) * (o.attP + o.attM);
    const double north = -xdiv(hbar, R.kp, R.rkp) * (o.attP + o.attQ);
    double acc = o.fP;
    acc -= south * o.uM;
    acc -= north * o.uQ;
    acc -= (-(o.artM + o.artSM) * 0.25) * o.uMM;
    acc -= ((o.artSM + o.artQ) * 0.25) * o.uQM;
    acc -= ((o.artM + o.artSP) * 0.25) * o.uMP;
    acc -= (-(o.artSP + o.artQ) * 0.25) * o.uQP;
    return acc;
}
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ bool same_bits(double a, double b) {
    return __double_as_longlong(a) == __double_as_longlong(b);
}

// Inclusive affine scan across the lanes of a warp (see block_scan); yin = the
// value entering the lane's rows.
template <int NV, bool FWD>
__device__ __forceinline__ void warp_scan(double A, double (&B)[NV], double (&yin)[NV]) {
    const int lane = threadIdx.x & 31;
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
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const double prev = FWD ? __shfl_up_sync(FULL, B[v], 1) : __shfl_down_sync(FULL, B[v], 1);
        yin[v] = lane == (FWD ? 0 : 31) ? 0.0 : prev;
    }
}


template <bool CG>
__device__ __forceinline__ double ldu(const double* p) {
    if (CG) return __ldcg(p);
    return *p;
}

// Circle-line rhs (smoother.cpp:162-182) of an interior Take ring: rings
// s-1, s+1 are circle rings and not Dirichlet, so the off-line couplings are
// the row_from expressions with has_sm = has_sp = true (same values).
__device__ __forceinline__ bool circle_lean_ring(const LevelView& L, int s) {
#ifdef PMG_NO_CIRCLE_LEAN
    return false;
#endif
    return s >= 1 && s + 1 < L.split && s + 1 < L.nr - 1 && !(s == 1 && L.boundary == 1);
}
struct CircOps {  // operands of one node of a lean ring
    double aP, aSM, aSP, rTM, rTP, rSM, rSP, uSM, uSP, uSMTM, uSMTP, uSPTM, uSPTP, fP, km, kp;
};
template <bool CG = false>
__device__ __forceinline__ void circ_load(const LevelView& L, long off, int s, int t,
                                          const double* __restrict__ U,
                                          const double* __restrict__ F, CircOps& o) {
    const int nt = L.nt, p = s * nt + t;
    const int tm = t == 0 ? nt - 1 : t - 1, tp = t + 1 == nt ? 0 : t + 1;
    const int pTM = s * nt + tm, pTP = s * nt + tp;
    const double* A = L.arr + off;
    const double* R = L.art + off;
    o.aP = A[p];
    o.aSM = A[p - nt];
    o.aSP = A[p + nt];
    o.rTM = R[pTM];
    o.rTP = R[pTP];
    o.rSM = R[p - nt];
    o.rSP = R[p + nt];
    o.uSM = ldu<CG>(&U[p - nt]);
    o.uSP = ldu<CG>(&U[p + nt]);
    o.uSMTM = ldu<CG>(&U[pTM - nt]);
    o.uSMTP = ldu<CG>(&U[pTP - nt]);
    o.uSPTM = ldu<CG>(&U[pTM + nt]);
    o.uSPTP = ldu<CG>(&U[pTP + nt]);
    o.fP = F[p];
    o.km = L.k[tm];
    o.kp = L.k[t];
}
// hm, rhm, hp, rhp: h_{s-1}, RN(1/h_{s-1}), h_s, RN(1/h_s)
__device__ __forceinline__ double circ_eval(const CircOps& o, double hm, double rhm, double hp,
                                            double rhp) {
    const double kbar = 0.5 * (o.km + o.kp);
    const double qkm = xdiv(kbar, hm, rhm);
    const double qkp = xdiv(kbar, hp, rhp);
    double acc = o.fP;
    acc -= (-qkm * (o.aP + o.aSM)) * o.uSM;
    acc -= (-qkp * (o.aP + o.aSP)) * o.uSP;
    acc -= (-(o.rTM + o.rSM) * 0.25) * o.uSMTM;
    acc -= ((o.rSM + o.rTP) * 0.25) * o.uSMTP;
    acc -= ((o.rTM + o.rSP) * 0.25) * o.uSPTM;
    acc -= (-(o.rSP + o.rTP) * 0.25) * o.uSPTP;
    return acc;
}
template <bool CG = false>
__device__ __forceinline__ double circle_rhs_lean(const LevelView& L, long off, int s, int t,
                                                  const double* __restrict__ U,
                                                  const double* __restrict__ F) {
    CircOps o;
    circ_load<CG>(L, off, s, t, U, F, o);
    return circ_eval(o, L.h[s - 1], L.rh[s - 1], L.h[s], L.rh[s]);
}

// Opt a kernel into the full 227 KB of dynamic shared memory once per
// (kernel, device); launches then pass their exact size.
template <class KernelT>
inline void set_smem(KernelT kern, size_t bytes) {
    (void)bytes;
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_pair(reinterpret_cast<const void*>(kern), dev);
    std::lock_guard<std::mutex> lock(mu);
    if (done.count(key)) return;
    cudaFuncAttributes fa;
    int optin = 227 * 1024;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess) optin -= (int)fa.sharedSizeBytes;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    done.insert(key);
}

// Launch with programmatic stream serialization (PDL) when PMG_PDL=1 (off by
// default: no measurable gain inside the replayed cycle graph, r01).
inline bool pdl_on() {
    static const bool on = [] {
        const char* e = std::getenv("PMG_PDL");
        return e ? std::atoi(e) != 0 : false;
    }();
    return on;
}
template <class... KArgs, class... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_on() ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    if (e != cudaSuccess) note_launch_error(e);
}


}  // namespace pmg
