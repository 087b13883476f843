// Host side of the B200 multigrid solve path: level hierarchy in device
// memory, the V/W/F cycle driver, and the extern "C" ABI of
// include/polarmg_b200.h.  Mirrors reference polarmg::MultigridSolver
// (multigrid.hpp:86-151, multigrid.cpp:61-357).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/polarmg_b200.h"
#include "pmg_common.cuh"
#include "pmg_grid.hpp"
#include "pmg_kernels.h"

namespace pmg {

// ------------------------------------------------------------------ errors
struct PmgError : std::runtime_error {
    int code;
    PmgError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

thread_local std::string g_err;

#define PMG_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw PmgError(PMG_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                          " at " #call);                                \
    } while (0)

// --------------------------------------------- envelope LDL^T (host setup)
// Restates reference SparseDirectFactor (line_algebra.cpp:122-209).
struct Trip {
    int row, col;
    double v;
};

struct HostEnv {
    int n = 0;
    std::vector<int> perm, iperm, fc;
    std::vector<long> ro;
    std::vector<double> L, D;

    void factor(int n_, const std::vector<Trip>& tr, const std::vector<int>& permutation) {
        n = n_;
        perm = permutation;
        if (perm.empty()) {
            perm.resize(n);
            for (int i = 0; i < n; ++i) perm[i] = i;
        }
        iperm.assign(n, -1);
        for (int k = 0; k < n; ++k) iperm[perm[k]] = k;
        fc.resize(n);
        for (int i = 0; i < n; ++i) fc[i] = i;
        for (const Trip& t : tr) {
            if (t.row < 0 || t.row >= n || t.col < 0 || t.col > t.row)
                throw PmgError(PMG_EINVAL, "sparse factor: triplets must address the lower triangle");
            const int pi = iperm[t.row], pj = iperm[t.col];
            const int hi = std::max(pi, pj), lo = std::min(pi, pj);
            fc[hi] = std::min(fc[hi], lo);
        }
        ro.assign(n + 1, 0);
        for (int i = 0; i < n; ++i) ro[i + 1] = ro[i] + (i - fc[i]);
        L.assign(ro[n], 0.0);
        D.assign(n, 0.0);
        std::vector<char> seen(n, 0);
        for (const Trip& t : tr) {
            const int pi = iperm[t.row], pj = iperm[t.col];
            if (pi == pj) {
                D[pi] += t.v;
                seen[pi] = 1;
            } else {
                const int hi = std::max(pi, pj), lo = std::min(pi, pj);
                L[ro[hi] + (lo - fc[hi])] += t.v;
            }
        }
        for (int i = 0; i < n; ++i)
            if (!seen[i])
                throw PmgError(PMG_ERUNTIME,
                               "sparse factor: structurally singular (missing diagonal at row " +
                                   std::to_string(perm[i]) + ")");
        double scale = 0.0;
        for (int i = 0; i < n; ++i) scale = std::max(scale, std::abs(D[i]));
        for (int i = 0; i < n; ++i) {
            const int fi = fc[i];
            double* ri = L.data() + ro[i] - fi;
            for (int j = fi; j < i; ++j) {
                const int fj = fc[j];
                const double* rj = L.data() + ro[j] - fj;
                const int k0 = std::max(fi, fj);
                double sum = ri[j];
                for (int k = k0; k < j; ++k) sum -= ri[k] * D[k] * rj[k];
                ri[j] = sum / D[j];
            }
            double d = D[i];
            for (int k = fi; k < i; ++k) d -= ri[k] * ri[k] * D[k];
            if (std::abs(d) < 1e-14 * std::max(scale, 1.0))
                throw PmgError(PMG_ERUNTIME,
                               "sparse factor: zero pivot at row " + std::to_string(perm[i]));
            D[i] = d;
        }
    }
    double at(int i, int k) const {  // L(i,k) within the envelope, else 0
        if (k < fc[i] || k >= i) return 0.0;
        return L[ro[i] + (k - fc[i])];
    }
};

// host coefficient provider (same transform() as the device)
struct HostCoef {
    const LevelView* L;
    int b;
    Coef operator()(int s, int t) const {
        return transform(L->geo, L->alpha[(long)b * L->nr + s], L->r[s], L->sn[t], L->cs[t],
                         nullptr);
    }
};

// assemble_coo (stencil.cpp:355-373) of a node subset given in NODE indices
static std::vector<Trip> assemble_coo(const LevelView& HL, const HostGrid& g, int b,
                                      const std::vector<int>& nodes) {
    std::vector<int> local(g.n(), -1);
    for (std::size_t i = 0; i < nodes.size(); ++i) local[nodes[i]] = static_cast<int>(i);
    std::vector<Trip> out;
    out.reserve(nodes.size() * 6);
    HostCoef cf{&HL, b};
    for (std::size_t i = 0; i < nodes.size(); ++i) {
        int s, t;
        HL.node(nodes[i], s, t);
        const Row R = make_row(HL, cf, s, t);
        const int lr = static_cast<int>(i);
        auto push = [&](int col, double v) {
            const int lc = local[col];
            if (lc >= 0 && lc <= lr) out.push_back({lr, lc, v});
        };
        const int p = g.idx(s, t);
        if (R.ident) {
            push(p, 1.0);
            continue;
        }
        const int tm = HL.tminus(t), tp = HL.tplus(t);
        push(p, R.d);
        if (R.has_sm) push(g.idx(s - 1, t), R.sm);
        if (R.has_sp) push(g.idx(s + 1, t), R.sp);
        push(g.idx(s, tm), R.tm);
        push(g.idx(s, tp), R.tp);
        if (R.has_sm) {
            push(g.idx(s - 1, tm), R.mm);
            push(g.idx(s - 1, tp), R.mp);
        }
        if (R.has_sp) {
            push(g.idx(s + 1, tm), R.pm);
            push(g.idx(s + 1, tp), R.pp);
        }
        if (R.origin) push(g.idx(0, R.t2), R.ph);
    }
    return out;
}

// ------------------------------------------------------------------ solver
struct Level {
    HostGrid g;
    LevelView v{};
    std::vector<double> h_alpha, h_beta, h_sn, h_cs;
    double *u = nullptr, *f = nullptr, *res = nullptr;
    double *arr = nullptr, *art = nullptr, *att = nullptr, *det = nullptr;
    double *cil = nullptr, *cm = nullptr, *corner = nullptr, *ril = nullptr, *rm = nullptr;
    double* cz = nullptr;  // Sherman-Morrison vectors of the circle lines (exact path)
    double* rows = nullptr;  // assembled rows [B][10][n] (coarse-tail levels)
    double *ob1 = nullptr, *ob2 = nullptr, *or1 = nullptr, *or2 = nullptr, *oD = nullptr;
    double* oinv = nullptr;  // dense inverse of the origin ring (n_theta <= 32)
    int ofc1 = 0, ofc2 = 0;
    Weights w{};
    EnvFactor env{};
    OriginFactor of() const { return OriginFactor{ob1, ob2, or1, or2, oD, ofc1, ofc2}; }
    // fused smoothing step (fused_ok levels): claim order and completion flags
    int* forder = nullptr;
    unsigned* fflags = nullptr;
    // two-colour radial wavefront (clustered spokes): claim order and chunk flags
    int* worder = nullptr;
    unsigned* wflags = nullptr;
};

struct Solver {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    Geo geo{};
    pmg_problem prob{};
    pmg_settings set{};
    int B = 1;
    std::vector<double> scales;
    double tol = 1e-12;
    bool onfly = false;
    bool serial = false;  // reference_order: exact-order (bitwise) line solves
    int exact_rings = 0;  // innermost circle rings solved in exact order (fast mode)
    std::vector<Level> lv;
    std::vector<void*> allocs;
    size_t bytes = 0;
    // convergence state
    double *norms = nullptr, *partials = nullptr, *r0 = nullptr, *hist = nullptr;
    int *active = nullptr, *iters = nullptr, *conv = nullptr, *remaining = nullptr;
    // the per-section activity mask the cycle kernels test; a single section
    // is only cycled while it is active, so its kernels skip the dependent load
    const int* act_mask() const { return B > 1 ? active : nullptr; }
    int* count = nullptr;
    // single-launch coarse tail: levels >= coarse_start run in k_coarse_cycle
    int coarse_start = -1;
    CoarseParams coarse_params{};
    int* d_prog[3] = {nullptr, nullptr, nullptr};
    int prog_len[3] = {0, 0, 0};
    std::vector<int> h_prog[3];
    MidParams mid_params{};
    int mid_start = -1;
    int* d_mprog[3] = {nullptr, nullptr, nullptr};
    int mprog_len[3] = {0, 0, 0};
    // CUDA graph of one cycle + residual norm + convergence check
    cudaGraphExec_t cycle_exec = nullptr;
    // the whole iteration as ONE graph launch: a WHILE node whose body is the
    // cycle graph and whose condition a device kernel sets from `remaining`
    cudaGraphExec_t loop_exec = nullptr;
    bool use_loop = true;
    long long cycle_nodes = 0;
    bool use_graph = true;
    int* h_remaining = nullptr;
    int hist_cap = 0;
    int partial_cap = 0;
    double* flush_buf = nullptr;
    long flush_n = 0;
    long long launches = 0;
    bool prof = false;
    struct Ev {
        int kind;
        cudaEvent_t a, b;
    };
    std::vector<Ev> evs;
    std::vector<cudaEvent_t> ev_pool;
    double prof_ms[KK_COUNT] = {};
    long long prof_n[KK_COUNT] = {};
    double setup_seconds = 0.0;
    double last_solve_ms = 0.0;

    ~Solver() {
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        for (auto& e : evs) {
            cudaEventDestroy(e.a);
            cudaEventDestroy(e.b);
        }
        for (auto e : ev_pool) cudaEventDestroy(e);
        if (cycle_exec) cudaGraphExecDestroy(cycle_exec);
        if (loop_exec) cudaGraphExecDestroy(loop_exec);
        for (void* p : allocs) cudaFree(p);
        if (h_remaining) cudaFreeHost(h_remaining);
        if (own_stream && stream) cudaStreamDestroy(stream);
    }

    template <class T>
    T* alloc(size_t count, bool zero = true) {
        void* p = nullptr;
        // 64 bytes of tail padding: aligned bulk copies may round a segment's
        // end up to the next 16-byte boundary
        const size_t nb = std::max<size_t>(count, 1) * sizeof(T) + 64;
        PMG_CUDA(cudaMalloc(&p, nb));
        allocs.push_back(p);
        bytes += nb;
        if (zero) PMG_CUDA(cudaMemsetAsync(p, 0, nb, stream));
        return static_cast<T*>(p);
    }
    template <class T>
    T* upload(const std::vector<T>& v) {
        T* p = alloc<T>(v.size(), false);
        if (!v.empty())
            PMG_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice,
                                     stream));
        return p;
    }

    // ---- kernel launch wrapper: counts launches, optional per-class timing
    cudaEvent_t pool_event() {
        if (!ev_pool.empty()) {
            cudaEvent_t e = ev_pool.back();
            ev_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        PMG_CUDA(cudaEventCreate(&e));
        return e;
    }
    template <class F>
    void run(int kind, int nlaunch, F&& fn) {
        if (prof) {
            Ev e{kind, pool_event(), pool_event()};
            PMG_CUDA(cudaEventRecord(e.a, stream));
            fn();
            PMG_CUDA(cudaEventRecord(e.b, stream));
            evs.push_back(e);
            prof_n[kind] += nlaunch;
        } else {
            fn();
        }
        launches += nlaunch;
    }
    void collect_profile() {
        if (evs.empty()) return;
        PMG_CUDA(cudaStreamSynchronize(stream));
        for (auto& e : evs) {
            float ms = 0.f;
            PMG_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
            prof_ms[e.kind] += ms;
            ev_pool.push_back(e.a);
            ev_pool.push_back(e.b);
        }
        evs.clear();
    }

    // ------------------------------------------------------------ setup
    void build(const pmg_grid& gp) {
        const auto t0 = std::chrono::steady_clock::now();
        tol = gp.pair_tolerance > 0.0 ? gp.pair_tolerance : 1e-12;
        HostGrid g0;
        if (gp.mode == 0)
            g0 = uniform_grid(gp.R0, gp.Rmax, gp.n_r, gp.n_theta, tol);
        else if (gp.mode == 1)
            g0 = build_grid(gp.R0, gp.Rmax, gp.nr_exp, gp.ntheta_exp, gp.anisotropic_factor,
                            gp.divide_by_2, tol);
        else {
            if (!gp.radii || !gp.angles || gp.n_r <= 0 || gp.n_theta <= 0)
                throw PmgError(PMG_EINVAL, "explicit grid requires radii and angles");
            g0 = make_grid(std::vector<double>(gp.radii, gp.radii + gp.n_r),
                           std::vector<double>(gp.angles, gp.angles + gp.n_theta), tol);
        }
        std::vector<HostGrid> grids;
        grids.push_back(std::move(g0));
        while ((set.max_levels == 0 || static_cast<int>(grids.size()) < set.max_levels) &&
               can_coarsen(grids.back(), tol))
            grids.push_back(coarsen(grids.back(), tol));
        const int L = static_cast<int>(grids.size());
        if (set.extrapolation && L < 2)
            throw PmgError(PMG_EINVAL, "extrapolation requires at least two levels");
        lv.resize(L);
        onfly = set.stencil_mode == 1 && !set.cache_geometry;
        serial = set.reference_order != 0;
        if (const char* e = std::getenv("PMG_EXACT_RINGS")) exact_rings = std::atoi(e);
        int* bad = alloc<int>(1);
        for (int l = 0; l < L; ++l) {
            Level& V = lv[l];
            V.g = std::move(grids[l]);
            setup_level(V, l == L - 1, bad);
        }
        setup_rows();
        setup_coarse_tail();
        setup_mid();
        setup_fused();
        if (set.extrapolation) ex_g = alloc<double>((size_t)B * lv[0].v.n);
        // convergence state
        hist_cap = std::max(set.max_iterations, 0) + 1;
        norms = alloc<double>(B);
        r0 = alloc<double>(B);
        hist = alloc<double>((size_t)B * hist_cap);
        active = alloc<int>(B);
        iters = alloc<int>(B);
        conv = alloc<int>(B);
        count = alloc<int>(B);
        remaining = alloc<int>(1);
        partial_cap = std::max(apply_blocks(lv[0].v), 1024);
        partials = alloc<double>((size_t)B * partial_cap);
        PMG_CUDA(cudaMallocHost(&h_remaining, sizeof(int)));
        PMG_CUDA(cudaStreamSynchronize(stream));
        setup_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }

    void setup_level(Level& V, bool coarsest, int* bad) {
        const HostGrid& g = V.g;
        const int nr = g.nr(), nt = g.nt();
        V.h_sn.resize(nt);
        V.h_cs.resize(nt);
        for (int t = 0; t < nt; ++t) {  // level_cache.cpp:27-32
            V.h_sn[t] = std::sin(g.th[t]);
            V.h_cs[t] = std::cos(g.th[t]);
        }
        V.h_alpha.resize((size_t)B * nr);
        V.h_beta.resize((size_t)B * nr);
        for (int b = 0; b < B; ++b)
            for (int s = 0; s < nr; ++s) {  // problem.cpp:86-94
                const double r = g.r[s];
                const double a = prob.alpha_coeff == 0
                                     ? 1.0
                                     : scales[b] * std::exp(-std::tanh(
                                                       (r / prob.rmax - prob.alpha_jump) /
                                                       prob.delta_r));
                V.h_alpha[(size_t)b * nr + s] = a;
                V.h_beta[(size_t)b * nr + s] = prob.beta_coeff == 0 ? 0.0 : 1.0 / a;
            }
        LevelView& v = V.v;
        v.nr = nr;
        v.nt = nt;
        v.split = g.split;
        v.len = nr - g.split;
        v.n = nr * nt;
        v.B = B;
        v.boundary = set.boundary_mode;
        v.r0 = g.r[0];
        v.geo = geo;
        v.r = upload(g.r);
        v.h = upload(g.h);
        v.k = upload(g.k);
        {  // exact reciprocals RN(1/h), RN(1/k) for the Markstein quotients
            std::vector<double> rh(g.h.size()), rk(g.k.size());
            for (std::size_t i = 0; i < rh.size(); ++i) rh[i] = 1.0 / g.h[i];
            for (std::size_t i = 0; i < rk.size(); ++i) rk[i] = 1.0 / g.k[i];
            v.rh = upload(rh);
            v.rk = upload(rk);
        }
        v.sn = upload(V.h_sn);
        v.cs = upload(V.h_cs);
        v.alpha = upload(V.h_alpha);
        v.beta = upload(V.h_beta);
        const size_t N = (size_t)B * v.n;
        V.u = alloc<double>(N);
        V.f = alloc<double>(N);
        V.res = alloc<double>(N);
        // coefficients: stored for Take (and Give+cacheDomainGeometry); for
        // on-the-fly Give a temporary set validates |det DF| once.
        {
            double* a = alloc<double>(N, false);
            double* c = alloc<double>(N, false);
            double* t_ = alloc<double>(N, false);
            double* d = alloc<double>(N, false);
            v.arr = a;
            v.art = c;
            v.att = t_;
            v.det = d;
            PMG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), stream));
            launch_coeffs(v, a, c, t_, d, bad, stream);
            check_bad(bad, "singular Jacobian: mapping degenerate at queried point");
            if (onfly) {  // release: Give recomputes coefficients
                release(a);
                release(c);
                release(t_);
                release(d);
                v.arr = v.art = v.att = v.det = nullptr;
            }
        }
        if (!coarsest) {
            if (!g.uniform_angles)
                throw PmgError(PMG_ERUNTIME,
                               "smoother split undefined: non-uniform angular spacing; a more "
                               "general switching condition or overlapping smoothers would be "
                               "needed");
            if (nt > 8192 || v.len > 8192)
                throw PmgError(PMG_EINVAL,
                               "line length above 8192 is not supported by the on-chip line "
                               "solver (n_theta and n_r - split must be <= 8192)");
            if (nt < 3)
                throw PmgError(PMG_EINVAL,
                               "cyclic_tridiag_factor: need n >= 3 (corner would duplicate a band)");
            V.cil = alloc<double>((size_t)B * v.split * nt, false);
            V.cm = alloc<double>((size_t)B * v.split * nt, false);
            V.corner = alloc<double>((size_t)B * v.split);
            PMG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), stream));
            launch_factor_circle(v, onfly, V.cil, V.cm, V.corner, bad, stream);
            check_bad(bad, "cyclic core not positive definite after rank-one shift");
            V.cz = alloc<double>((size_t)B * v.split * nt, false);
            launch_circle_z(v, V.cil, V.cm, V.cz, stream);
            if (v.len > 0) {
                V.ril = alloc<double>((size_t)B * nt * v.len, false);
                V.rm = alloc<double>((size_t)B * nt * v.len, false);
                PMG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), stream));
                launch_factor_radial(v, onfly, V.ril, V.rm, bad, stream);
                check_bad(bad, "not positive definite (radial line factor)");
            }
            if (set.boundary_mode == 0) setup_origin(V);
            setup_weights(V);
        } else {
            setup_coarsest(V);
        }
    }

    // op program of cycle(l, type) (multigrid.cpp:189-220) for k_coarse_cycle
    void gen_prog(int l, int type, std::vector<int>& prog) const {
        const int L = static_cast<int>(lv.size());
        if (l == L - 1) {
            prog.push_back(OP_COARSE | (l << 8));
            return;
        }
        for (int i = 0; i < set.pre_smoothing; ++i) prog.push_back(OP_SMOOTH | (l << 8));
        prog.push_back(OP_RESIDUAL | (l << 8));
        prog.push_back(OP_RESTRICT | (l << 8));
        if (type == 0) {
            gen_prog(l + 1, 0, prog);
        } else if (type == 1) {
            gen_prog(l + 1, 1, prog);
            gen_prog(l + 1, 1, prog);
        } else {
            gen_prog(l + 1, 2, prog);
            gen_prog(l + 1, 0, prog);
        }
        prog.push_back(OP_PROLONG | (l << 8));
        for (int i = 0; i < set.post_smoothing; ++i) prog.push_back(OP_SMOOTH | (l << 8));
    }

    // Levels qualify for the single-block coarse tail when every line fits a
    // warp (<= 32*kWK nodes).  Resident mode (default): the tail is the largest
    // set of coarsest levels whose per-section data fits the shared-memory
    // budget; the block stages it into shared memory and runs the whole
    // sub-cycle there.
    void setup_coarse_tail() {
        const int L = static_cast<int>(lv.size());
        long budget = 200 * 1024;
        if (const char* e = std::getenv("PMG_COARSE_SMEM")) budget = std::atol(e);
        if (budget <= 0) return;
        auto fits_warp = [&](int l) {
            const HostGrid& g = lv[l].g;
            return g.nt() <= 32 * 8 && (g.nr() - g.split) <= 32 * 8 && g.uniform_angles;
        };
        // bytes of one section's slice of level l in the resident tail
        auto level_bytes = [&](int l, bool top) {
            const HostGrid& g = lv[l].g;
            const long n = g.n(), nr = g.nr(), nt = g.nt(), sp = g.split, len = nr - sp;
            const bool coarsest = l == L - 1;
            long d = 2 * n;                         // u, f
            if (!coarsest) {
                d += 11 * n;                        // res, assembled rows
                d += 2 * sp * nt + sp + 2 * nt * len + 5 * nt + 2 * nr + 2 * nt;
                if (serial) d += sp * nt;        // Sherman-Morrison vectors
                else if (nt <= 32) d += nt * nt;  // origin ring inverse
            } else {
                d += n <= 64 ? n * n : lv[l].env.nnz + n + n / 2 + n + 2;  // inv | L, D, fc, ro
            }
            (void)top;
            return d * 8 + 40 * 16;                 // + alignment slack
        };
        int start = L;
        long total = 0;
        for (int l = L - 1; l >= 0; --l) {
            if (!fits_warp(l) && l != L - 1) break;
            const long bl = level_bytes(l, true);
            if (total + bl > budget) break;
            total += bl;
            start = l;
        }
        if (L - start > kMaxCoarse) start = L - kMaxCoarse;
        if (set.extrapolation && start < 1) start = 1;  // level 0 runs the extrapolated kernels
        if (start >= L - 1) return;  // only the coarsest: nothing to gain
        coarse_start = start;
        std::memset(&coarse_params, 0, sizeof coarse_params);
        coarse_params.first = start;
        std::vector<CopyDesc> plan;
        long off = 0;
        // allocate `count` elements of `esz` bytes at a 16-byte aligned offset;
        // copy from src (stride = per-section bytes, 0 = shared) if src != null
        auto place = [&](const void* src, long stride, long count, int esz) -> void* {
            off = (off + 15) & ~15L;
            const long at = off;
            off += count * esz;
            if (src) plan.push_back(CopyDesc{src, stride, static_cast<int>(count * esz),
                                             static_cast<int>(at)});
            return reinterpret_cast<void*>(at + 8);
        };
        for (int l = start; l < L; ++l) {
            Level& V = lv[l];
            const HostGrid& g = V.g;
            const long n = g.n(), nr = g.nr(), nt = g.nt(), sp = g.split, len = nr - sp;
            const bool coarsest = l == L - 1, top = l == start;
            CoarseLevel& c = coarse_params.lv[l - start];
            c.v = V.v;
            LevelView& v = c.v;
            // the tail works from assembled rows: geometry/coefficients stay behind
            v.r = v.h = v.rh = v.k = v.rk = v.sn = v.cs = v.alpha = v.beta = nullptr;
            v.arr = v.art = v.att = v.det = nullptr;
            v.rows = nullptr;
            if (!coarsest) {
                if (!V.rows) {
                    V.rows = alloc<double>((size_t)B * 10 * n, false);
                    launch_rows(V.v, onfly, V.rows, stream);
                }
                c.rows = static_cast<double*>(place(V.rows, 10 * n * 8, 10 * n, 8));
            }
            c.u = static_cast<double*>(place(top ? V.u : nullptr, n * 8, n, 8));
            c.f = static_cast<double*>(place(top ? V.f : nullptr, n * 8, n, 8));
            if (!coarsest) {
                c.res = static_cast<double*>(place(nullptr, 0, n, 8));
                c.cl = static_cast<double*>(place(V.cil, sp * nt * 8, sp * nt, 8));
                c.cm = static_cast<double*>(place(V.cm, sp * nt * 8, sp * nt, 8));
                c.corner = static_cast<double*>(place(V.corner, sp * 8, sp, 8));
                if (serial) c.cz = static_cast<double*>(place(V.cz, sp * nt * 8, sp * nt, 8));
                c.exact = serial ? 1 : 0;
                if (len > 0) {
                    c.rl = static_cast<double*>(place(V.ril, nt * len * 8, nt * len, 8));
                    c.rm = static_cast<double*>(place(V.rm, nt * len * 8, nt * len, 8));
                }
                if (set.boundary_mode == 0) {
                    c.of.band1 = static_cast<double*>(place(V.ob1, nt * 8, nt, 8));
                    c.of.band2 = static_cast<double*>(place(V.ob2, nt * 8, nt, 8));
                    c.of.row1 = static_cast<double*>(place(V.or1, nt * 8, nt, 8));
                    c.of.row2 = static_cast<double*>(place(V.or2, nt * 8, nt, 8));
                    c.of.D = static_cast<double*>(place(V.oD, nt * 8, nt, 8));
                    c.of.fc1 = V.ofc1;
                    c.of.fc2 = V.ofc2;
                    // dense inverse on coarse levels only: on the finest level the
                    // substitution's backward stability matters at the roundoff floor
                    if (V.oinv && l > 0)
                        c.of.inv = static_cast<double*>(place(V.oinv, nt * nt * 8, nt * nt, 8));
                }
                c.w.rwb = static_cast<double*>(place(V.w.rwb, 0, nr, 8));
                c.w.rwa = static_cast<double*>(place(V.w.rwa, 0, nr, 8));
                c.w.awb = static_cast<double*>(place(V.w.awb, 0, nt, 8));
                c.w.awa = static_cast<double*>(place(V.w.awa, 0, nt, 8));
            } else {
                const EnvFactor& E = V.env;
                coarse_params.env = E;
                coarse_params.env.fc = nullptr;
                coarse_params.env.ro = nullptr;
                coarse_params.env.L = coarse_params.env.D = coarse_params.env.inv = nullptr;
                if (E.inv) {
                    coarse_params.env.inv =
                        static_cast<double*>(place(E.inv, (long)E.n * E.n * 8, (long)E.n * E.n, 8));
                } else {
                    coarse_params.env.fc = static_cast<int*>(place(E.fc, 0, E.n, 4));
                    coarse_params.env.ro = static_cast<long*>(place(E.ro, 0, E.n + 1, 8));
                    coarse_params.env.L = static_cast<double*>(place(E.L, E.nnz * 8, E.nnz, 8));
                    coarse_params.env.D = static_cast<double*>(place(E.D, E.n * 8, E.n, 8));
                }
            }
        }
        if (off > 220 * 1024) {  // budget estimate too small: stay non-resident
            coarse_start = -1;
            return;
        }
        coarse_params.resident = 1;
        {  // level table image + pointer-word mask (see TailImage)
            TailImage img;
            std::memset(&img, 0, sizeof img);
            for (int i = 0; i < kMaxCoarse; ++i) {
                img.lv[i] = coarse_params.lv[i];
                if (img.lv[i].v.nr > 0) img.lv[i].v.B = 1;
            }
            img.env = coarse_params.env;
            constexpr size_t words = sizeof(TailImage) / 8;
            std::vector<unsigned> mask((words + 31) / 32, 0u);
            auto mark = [&](size_t byte) {
                const size_t w = byte / 8;
                mask[w >> 5] |= 1u << (w & 31);
            };
            for (int i = 0; i < kMaxCoarse; ++i) {
                const size_t c = offsetof(TailImage, lv) + i * sizeof(CoarseLevel);
                const size_t v = c + offsetof(CoarseLevel, v);
                for (size_t f : {offsetof(LevelView, r), offsetof(LevelView, h),
                                 offsetof(LevelView, k), offsetof(LevelView, sn),
                                 offsetof(LevelView, cs), offsetof(LevelView, alpha),
                                 offsetof(LevelView, beta), offsetof(LevelView, arr),
                                 offsetof(LevelView, art), offsetof(LevelView, att),
                                 offsetof(LevelView, det), offsetof(LevelView, rh),
                                 offsetof(LevelView, rk)})
                    mark(v + f);
                for (size_t f : {offsetof(CoarseLevel, u), offsetof(CoarseLevel, f),
                                 offsetof(CoarseLevel, res), offsetof(CoarseLevel, cl),
                                 offsetof(CoarseLevel, cm), offsetof(CoarseLevel, corner),
                                 offsetof(CoarseLevel, rl), offsetof(CoarseLevel, rm),
                                 offsetof(CoarseLevel, rows), offsetof(CoarseLevel, cz)})
                    mark(c + f);
                const size_t o = c + offsetof(CoarseLevel, of);
                for (size_t f : {offsetof(OriginFactor, band1), offsetof(OriginFactor, band2),
                                 offsetof(OriginFactor, row1), offsetof(OriginFactor, row2),
                                 offsetof(OriginFactor, D), offsetof(OriginFactor, inv)})
                    mark(o + f);
                const size_t w = c + offsetof(CoarseLevel, w);
                for (size_t f : {offsetof(Weights, rwb), offsetof(Weights, rwa),
                                 offsetof(Weights, awb), offsetof(Weights, awa)})
                    mark(w + f);
            }
            const size_t e = offsetof(TailImage, env);
            for (size_t f : {offsetof(EnvFactor, fc), offsetof(EnvFactor, ro), offsetof(EnvFactor, L),
                             offsetof(EnvFactor, D), offsetof(EnvFactor, inv)})
                mark(e + f);
            std::vector<unsigned long long> iw(words);
            std::memcpy(iw.data(), &img, sizeof img);
            coarse_params.image = upload(iw);
            coarse_params.image_mask = upload(mask);
        }
        int kw = 1;
        for (int l = start; l < L - 1; ++l) {
            const HostGrid& g = lv[l].g;
            const int m = std::max(g.nt(), g.nr() - g.split);
            while (32 * kw < m) kw *= 2;
        }
        coarse_params.kw = kw;
        coarse_params.ncopy = static_cast<int>(plan.size());
        coarse_params.smem_bytes = static_cast<int>((off + 15) & ~15L);
        coarse_params.copies = upload(plan);
        coarse_params.top_u_global = lv[start].u;
        int maxlen = 0;
        for (int type = 0; type < 3; ++type) {
            std::vector<int> prog;
            gen_prog(start, type, prog);
            d_prog[type] = upload(prog);
            prog_len[type] = static_cast<int>(prog.size());
            h_prog[type] = prog;
            maxlen = std::max(maxlen, prog_len[type]);
        }
        if (std::getenv("PMG_TAIL_TRACE"))
            coarse_params.trace = alloc<unsigned long long>(maxlen + 4);
    }

    // Latency-bound levels (all sections together at most PMG_ROWS_NODES nodes,
    // level 0 excluded) keep their assembled rows: the line kernels and the
    // residual then evaluate ten products per node instead of re-deriving the
    // stencil (same values, k_rows).
    void setup_rows() {
        long max_nodes = 300000;
        if (const char* e = std::getenv("PMG_ROWS_NODES")) max_nodes = std::atol(e);
        for (size_t l = 1; l < lv.size(); ++l) {
            Level& V = lv[l];
            if ((long)B * V.v.n > max_nodes) continue;
            V.rows = alloc<double>((size_t)B * 10 * V.v.n, false);
            launch_rows(V.v, onfly, V.rows, stream);
            V.v.rows = V.rows;
        }
    }

    // Fused smoothing steps: levels with one-CTA lines run all four zebra
    // sweeps in one launch (launch_smooth_fused); one control block (ticket,
    // done count, epoch) serves every launch since they are stream-ordered.
    unsigned* fuse_ctl = nullptr;
    void setup_fused() {
        for (size_t l = 0; l < lv.size(); ++l) {
            Level& V = lv[l];
            if (coarse_start >= 0 && (int)l >= coarse_start) break;  // resident tail
            if (l == 0 && set.extrapolation) continue;
            if (!fused_ok(V.v, serial, exact_rings)) continue;
            // large batches keep the per-colour launches (c3, 256 sections:
            // 14% slower fused -- ticket contention over 152K lines)
            // batches whose lines run on the warp-per-line kernels keep the
            // per-colour launches too: measured on the 32-section slice an
            // 8-GPU rank owns, 20.7 -> 17.5 ms per solve (the fused step's
            // CTA-per-line exact solves are slower than a warp per line)
            if (B > 1 && !onfly && warp_batch_ok(V.v.len, (long)(V.v.nt / 2) * B)) continue;
            static const long max_lines = [] {
                const char* e = std::getenv("PMG_FUSED_MAX_LINES");
                return e ? std::atol(e) : 16384L;
            }();
            if ((long)B * (V.v.split + V.v.nt) > max_lines) continue;
            if (!fuse_ctl) {
                fuse_ctl = alloc<unsigned>(4);
                const unsigned init[4] = {0u, 0u, 1u, 0u};
                PMG_CUDA(cudaMemcpyAsync(fuse_ctl, init, sizeof init, cudaMemcpyHostToDevice,
                                         stream));
            }
            const int per = V.v.split + V.v.nt;
            std::vector<int> order((size_t)B * per);
            fused_order(V.v.split, V.v.nt, B, order.data());
            V.forder = upload(order);
            V.fflags = alloc<unsigned>((size_t)B * per);
        }
        for (size_t l = 0; l < lv.size(); ++l) {
            Level& V = lv[l];
            if (V.forder || (coarse_start >= 0 && (int)l >= coarse_start)) continue;
            if (l == 0 && set.extrapolation) continue;
            const int C = radial_wave_cluster(V.v, serial, onfly);
            if (C <= 0) continue;
            if (!fuse_ctl) {
                fuse_ctl = alloc<unsigned>(4);
                const unsigned init[4] = {0u, 0u, 1u, 0u};
                PMG_CUDA(cudaMemcpyAsync(fuse_ctl, init, sizeof init, cudaMemcpyHostToDevice,
                                         stream));
            }
            std::vector<int> order(V.v.nt);
            radial_wave_order(V.v.nt, C, order.data());
            V.worder = upload(order);
            V.wflags = alloc<unsigned>((size_t)V.v.nt * C);
        }
        PMG_CUDA(cudaStreamSynchronize(stream));
    }

    // Cluster-wide sub-cycle (k_mid_cycle): the levels just above the resident
    // tail whose lines fit a warp and whose vectors stay in L2 run in one
    // launch per cycle, one thread-block cluster per section.  Opt-in
    // (PMG_MID_NODES=5000): measured 1-2% slower than the per-level kernels on
    // c0, c1, c2-V and c2-W once those got faster.
    void setup_mid() {
        if (coarse_start <= 0) return;
        long max_nodes = 0;
        if (const char* e = std::getenv("PMG_MID_NODES")) max_nodes = std::atol(e);
        int max_b = 16;
        if (const char* e = std::getenv("PMG_MID_SECTIONS")) max_b = std::atoi(e);
        if (max_nodes <= 0 || B > max_b) return;
        int first = coarse_start;
        const int lowest = set.extrapolation ? 1 : 0;
        while (first - 1 >= lowest && coarse_start - (first - 1) <= kMaxMid) {
            const HostGrid& g = lv[first - 1].g;
            if (!(g.nt() <= 256 && g.nr() - g.split <= 256 && g.uniform_angles &&
                  g.n() <= max_nodes))
                break;
            --first;
        }
        if (first == coarse_start) return;
        int want = 16;
        if (const char* e = std::getenv("PMG_MID_CLUSTER")) want = std::atoi(e);
        const int cl = mid_cluster_size((size_t)coarse_params.smem_bytes, want);
        if (cl < 2) return;
        std::memset(&mid_params, 0, sizeof mid_params);
        mid_params.first = first;
        mid_params.nmid = coarse_start - first;
        mid_params.cl = cl;
        mid_params.tail = coarse_params;
        for (int t = 0; t < 3; ++t) {
            mid_params.tprog[t] = d_prog[t];
            mid_params.tlen[t] = prog_len[t];
        }
        for (int l = first; l <= coarse_start; ++l) {
            Level& V = lv[l];
            const HostGrid& g = V.g;
            const long n = g.n();
            CoarseLevel& c = mid_params.lv[l - first];
            c.v = V.v;
            c.u = V.u;
            c.f = V.f;
            if (l == coarse_start) break;  // tail top: restrict target / prolong source
            c.res = V.res;
            c.cl = V.cil;
            c.cm = V.cm;
            c.corner = V.corner;
            c.rl = V.ril;
            c.rm = V.rm;
            if (!V.rows) {
                V.rows = alloc<double>((size_t)B * 10 * n, false);
                launch_rows(V.v, onfly, V.rows, stream);
            }
            c.rows = V.rows;
            c.cz = V.cz;
            c.exact = serial ? 1 : 0;
            if (set.boundary_mode == 0) {
                c.of.band1 = V.ob1;
                c.of.band2 = V.ob2;
                c.of.row1 = V.or1;
                c.of.row2 = V.or2;
                c.of.D = V.oD;
                c.of.fc1 = V.ofc1;
                c.of.fc2 = V.ofc2;
            }
            c.w = V.w;
            int kw = 1;
            while (32 * kw < std::max(g.nt(), g.nr() - g.split)) kw *= 2;
            mid_params.kw[l - first] = kw;
        }
        for (int type = 0; type < 3; ++type) {
            std::vector<int> prog;
            gen_mid_prog(first, type, prog);
            d_mprog[type] = upload(prog);
            mprog_len[type] = static_cast<int>(prog.size());
        }
        mid_start = first;
        if (std::getenv("PMG_TAIL_TRACE")) {
            int mx = 0;
            for (int t = 0; t < 3; ++t) mx = std::max(mx, mprog_len[t]);
            mid_params.trace = alloc<unsigned long long>(mx + 1);
            h_mprog_type = set.cycle;
            gen_mid_prog(first, set.cycle, h_mprog);
        }
    }
    std::vector<int> h_mprog;
    int h_mprog_type = 0;
    void print_mid_trace() {
        std::vector<unsigned long long> t(h_mprog.size() + 1);
        PMG_CUDA(cudaMemcpy(t.data(), mid_params.trace, t.size() * 8, cudaMemcpyDeviceToHost));
        static const char* names[] = {"smooth", "residual", "restrict", "prolong", "coarse", "tail"};
        double sum[6][kMaxCoarse + 1] = {};
        for (size_t i = 0; i < h_mprog.size(); ++i) {
            const int op = h_mprog[i] & 255;
            const int l = op == OP_TAIL ? kMaxCoarse : (h_mprog[i] >> 8);
            sum[op][l] += (t[1 + i] - t[i]) * 1e-3;
        }
        for (int o = 0; o < 6; ++o)
            for (int l = 0; l <= kMaxCoarse; ++l)
                if (sum[o][l] > 0)
                    std::fprintf(stderr, "mid trace: level %d %-8s %.2f us\n", l, names[o],
                                 sum[o][l]);
        std::fprintf(stderr, "mid trace: total %.2f us\n", (t.back() - t[0]) * 1e-3);
    }
    void gen_mid_prog(int l, int type, std::vector<int>& prog) const {
        if (l == coarse_start) {
            prog.push_back(OP_TAIL | (type << 8));
            return;
        }
        for (int i = 0; i < set.pre_smoothing; ++i) prog.push_back(OP_SMOOTH | (l << 8));
        prog.push_back(OP_RESIDUAL | (l << 8));
        prog.push_back(OP_RESTRICT | (l << 8));
        if (type == 0) {
            gen_mid_prog(l + 1, 0, prog);
        } else if (type == 1) {
            gen_mid_prog(l + 1, 1, prog);
            gen_mid_prog(l + 1, 1, prog);
        } else {
            gen_mid_prog(l + 1, 2, prog);
            gen_mid_prog(l + 1, 0, prog);
        }
        prog.push_back(OP_PROLONG | (l << 8));
        for (int i = 0; i < set.post_smoothing; ++i) prog.push_back(OP_SMOOTH | (l << 8));
    }

    void release(double* p) {
        auto it = std::find(allocs.begin(), allocs.end(), static_cast<void*>(p));
        if (it != allocs.end()) {
            PMG_CUDA(cudaStreamSynchronize(stream));
            cudaFree(p);
            allocs.erase(it);
        }
    }

    void check_bad(int* bad, const char* msg) {
        int hb = 0;
        PMG_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, stream));
        PMG_CUDA(cudaStreamSynchronize(stream));
        PMG_CUDA(last_error());
        if (hb) throw PmgError(PMG_ERUNTIME, msg);
    }

    LevelView host_view(const Level& V) const {
        LevelView h = V.v;
        h.r = V.g.r.data();
        h.h = V.g.h.data();
        h.k = V.g.k.data();
        h.sn = V.h_sn.data();
        h.cs = V.h_cs.data();
        h.alpha = V.h_alpha.data();
        h.beta = V.h_beta.data();
        h.arr = h.art = h.att = h.det = nullptr;
        h.rh = h.rk = nullptr;
        h.rows = nullptr;
        return h;
    }

    // across-origin ring: envelope LDL^T in antipodal order (smoother.cpp:33-49)
    void setup_origin(Level& V) {
        const int nt = V.g.nt();
        const LevelView HL = host_view(V);
        std::vector<int> nodes(nt), perm(nt);
        for (int t = 0; t < nt; ++t) nodes[t] = t;
        for (int i = 0; i < nt / 2; ++i) {
            perm[2 * i] = i;
            perm[2 * i + 1] = nt / 2 + i;
        }
        std::vector<double> b1((size_t)B * nt, 0.0), b2((size_t)B * nt, 0.0),
            r1((size_t)B * nt, 0.0), r2((size_t)B * nt, 0.0), D((size_t)B * nt, 0.0), oinv;
        for (int b = 0; b < B; ++b) {
            HostEnv E;
            E.factor(nt, assemble_coo(HL, V.g, b, nodes), perm);
            for (int i = 0; i < nt - 2; ++i)
                if (E.fc[i] < i - 2)
                    throw PmgError(PMG_ERUNTIME,
                                   "origin ring factor: unexpected envelope structure");
            if (b == 0) {
                V.ofc1 = E.fc[nt - 2];
                V.ofc2 = E.fc[nt - 1];
            } else if (V.ofc1 != E.fc[nt - 2] || V.ofc2 != E.fc[nt - 1]) {
                throw PmgError(PMG_ERUNTIME, "origin ring factor: section structures differ");
            }
            const size_t o = (size_t)b * nt;
            for (int i = 0; i < nt; ++i) {
                D[o + i] = E.D[i];
                if (i < nt - 2) {
                    b1[o + i] = E.at(i, i - 1);
                    b2[o + i] = E.at(i, i - 2);
                }
            }
            for (int k = 0; k < nt - 2; ++k) r1[o + k] = E.at(nt - 2, k);
            for (int k = 0; k < nt - 1; ++k) r2[o + k] = E.at(nt - 1, k);
            if (nt <= 32 && !serial) {  // dense inverse for the warp solves of the one-block tail
                if (b == 0) oinv.assign((size_t)B * nt * nt, 0.0);
                std::vector<double> y(nt);
                for (int j = 0; j < nt; ++j) {
                    for (int k = 0; k < nt; ++k) y[k] = perm[k] == j ? 1.0 : 0.0;
                    for (int i = 0; i < nt; ++i)
                        for (int k = E.fc[i]; k < i; ++k) y[i] -= E.at(i, k) * y[k];
                    for (int i = 0; i < nt; ++i) y[i] /= E.D[i];
                    for (int i = nt - 1; i >= 0; --i)
                        for (int k = E.fc[i]; k < i; ++k) y[k] -= E.at(i, k) * y[i];
                    for (int k = 0; k < nt; ++k) oinv[((size_t)b * nt + j) * nt + perm[k]] = y[k];
                }
            }
        }
        V.oinv = oinv.empty() ? nullptr : upload(oinv);
        V.ob1 = upload(b1);
        V.ob2 = upload(b2);
        V.or1 = upload(r1);
        V.or2 = upload(r2);
        V.oD = upload(D);
    }

    // coarsest direct factor (multigrid.cpp:112-121)
    void setup_coarsest(Level& V) {
        const int n = static_cast<int>(V.g.n());
        const LevelView HL = host_view(V);
        std::vector<int> nodes(n);
        for (int i = 0; i < n; ++i) nodes[i] = i;
        std::vector<double> Lall, Dall, inv;
        std::vector<int> fc;
        std::vector<long> ro;
        for (int b = 0; b < B; ++b) {
            HostEnv E;
            E.factor(n, assemble_coo(HL, V.g, b, nodes), {});
            if (b == 0) {
                fc = E.fc;
                ro = E.ro;
                Lall.resize((size_t)B * E.L.size());
                Dall.resize((size_t)B * n);
            } else if (E.fc != fc) {
                throw PmgError(PMG_ERUNTIME, "coarsest factor: section structures differ");
            }
            std::copy(E.L.begin(), E.L.end(), Lall.begin() + (size_t)b * E.L.size());
            std::copy(E.D.begin(), E.D.end(), Dall.begin() + (size_t)b * n);
            if (n <= 64 && !serial) {  // dense inverse for the one-block coarse tail
                if (b == 0) inv.resize((size_t)B * n * n);
                std::vector<double> x(n);
                for (int j = 0; j < n; ++j) {
                    std::fill(x.begin(), x.end(), 0.0);
                    x[j] = 1.0;
                    for (int i = 0; i < n; ++i)
                        for (int k = E.fc[i]; k < i; ++k) x[i] -= E.at(i, k) * x[k];
                    for (int i = 0; i < n; ++i) x[i] /= E.D[i];
                    for (int i = n - 1; i >= 0; --i)
                        for (int k = E.fc[i]; k < i; ++k) x[k] -= E.at(i, k) * x[i];
                    std::copy(x.begin(), x.end(), inv.begin() + ((size_t)b * n + j) * n);
                }
            }
        }
        V.env.n = n;
        V.env.nnz = ro.back();
        V.env.fc = upload(fc);
        V.env.ro = upload(ro);
        V.env.L = upload(Lall);
        V.env.D = upload(Dall);
        V.env.inv = inv.empty() ? nullptr : upload(inv);
    }

    // interpolation weights of this level as the fine grid (interpolation.cpp:19-36)
    void setup_weights(Level& V) {
        const HostGrid& g = V.g;
        std::vector<double> rwb(g.nr(), 0.0), rwa(g.nr(), 0.0), awb(g.nt(), 0.0),
            awa(g.nt(), 0.0);
        for (int sf = 1; sf + 1 < g.nr(); ++sf) {
            rwb[sf] = g.h[sf] / (g.h[sf - 1] + g.h[sf]);
            rwa[sf] = g.h[sf - 1] / (g.h[sf - 1] + g.h[sf]);
        }
        for (int tf = 1; tf < g.nt(); ++tf) {
            awb[tf] = g.k[tf] / (g.k[tf - 1] + g.k[tf]);
            awa[tf] = g.k[tf - 1] / (g.k[tf - 1] + g.k[tf]);
        }
        V.w.rwb = upload(rwb);
        V.w.rwa = upload(rwa);
        V.w.awb = upload(awb);
        V.w.awa = upload(awa);
    }

    // ------------------------------------------------------------ cycle
    // smooth_level (multigrid.cpp:170-181): level 0 with extrapolation runs
    // smooth_extrapolated (smoother.cpp:83-91)
    void smooth(int l, const int* act) {
        Level& V = lv[l];
        if (l == 0 && set.extrapolation) {
            run(KK_OTHER, 1, [&] { launch_ex_fhat(V.v, V.f, ex_g, act, stream); });
            run(KK_CIRCLE, line_launches(V.v, serial, onfly, exact_rings, 0, 1), [&] {
                launch_circle(V.v, onfly, V.u, ex_g, V.cil, V.cm, V.corner, V.cz, V.of(), 1,
                              serial, exact_rings, act, stream);
            });
            if (V.v.len > 0)
                run(KK_RADIAL, 1, [&] {
                    launch_radial(V.v, onfly, V.u, ex_g, V.ril, V.rm, 1, serial, act, stream);
                });
            run(KK_SMOOTH, 3, [&] { launch_ex_pointwise(V.v, onfly, V.u, V.f, act, stream); });
            return;
        }
        if (V.forder) {
            run(KK_SMOOTH, 1, [&] {
                launch_smooth_fused(V.v, onfly, V.u, V.f, V.cil, V.cm, V.corner, V.cz, V.of(),
                                    V.ril, V.rm, exact_rings, serial, FuseCtl{fuse_ctl, V.fflags},
                                    V.forder, act, stream);
            });
            return;
        }
        for (int parity = 0; parity < 2; ++parity)
            run(KK_CIRCLE, line_launches(V.v, serial, onfly, exact_rings, 0, parity), [&] {
                launch_circle(V.v, onfly, V.u, V.f, V.cil, V.cm, V.corner, V.cz, V.of(), parity,
                              serial, exact_rings, act, stream);
            });
        if (V.worder) {
            run(KK_RADIAL, 1, [&] {
                launch_radial_wave(V.v, V.u, V.f, V.ril, V.rm, FuseCtl{fuse_ctl, V.wflags},
                                   V.worder, stream);
            });
        } else if (V.v.len > 0)
            for (int parity = 0; parity < 2; ++parity)
                run(KK_RADIAL, 1, [&] {
                    launch_radial(V.v, onfly, V.u, V.f, V.ril, V.rm, parity, serial, act, stream);
                });
    }
    // extrapolated_residual (multigrid.cpp:224-248) into lv[0].res
    void ex_residual(const int* act) {
        Level& F = lv[0];
        Level& C = lv[1];
        run(KK_RESIDUAL, 2 * apply_launches(F.v) + 2, [&] {
            launch_apply(F.v, onfly, 0, F.u, nullptr, F.res, nullptr, 0, act, stream);
            launch_inject(F.v, C.v, F.u, C.u, act, stream);
            launch_apply(C.v, onfly, 0, C.u, nullptr, C.res, nullptr, 0, act, stream);
            launch_ex_residual(F.v, C.v, F.u, F.f, C.res, F.res, act, stream);
        });
    }
    // build_extrapolated_rhs (multigrid.cpp:159-168)
    void build_extrapolated_rhs() {
        run(KK_OTHER, 1, [&] { launch_ex_rhs(lv[0].v, lv[1].v, lv[0].f, lv[1].f, stream); });
        set_dirichlet_rows(0, lv[0].f);
    }
    void residual(int l, const int* act) {
        Level& V = lv[l];
        if (l == 0 && set.extrapolation) {
            ex_residual(act);
            return;
        }
        run(KK_RESIDUAL, apply_launches(V.v), [&] {
            launch_apply(V.v, onfly, 1, V.u, V.f, V.res, nullptr, 0, act, stream);
        });
    }
    void restrict_to(int l, const int* act) {
        Level& F = lv[l];
        Level& C = lv[l + 1];
        run(KK_RESTRICT, 1,
            [&] { launch_restrict(F.v, C.v, F.w, F.res, C.f, C.u, true, act, stream); });
    }
    void prolong_add(int l, const int* act) {
        Level& F = lv[l];
        Level& C = lv[l + 1];
        run(KK_PROLONG, 1, [&] { launch_prolong(F.v, C.v, F.w, C.u, F.u, true, act, stream); });
    }
    void coarse(int l, const int* act) {
        Level& V = lv[l];
        run(KK_COARSE, 1, [&] { launch_coarse(V.v, V.env, V.f, V.u, act, stream); });
    }
    // multigrid.cpp:189-220
    void cycle(int l, int type, const int* act) {
        const int L = static_cast<int>(lv.size());
        if (l == mid_start) {
            run(KK_COARSE, 1, [&] {
                launch_mid_cycle(mid_params, d_mprog[type], mprog_len[type], B, act, stream);
            });
            return;
        }
        if (l == coarse_start) {
            run(KK_COARSE, 1, [&] {
                launch_coarse_cycle(coarse_params, d_prog[type], prog_len[type], B, onfly, act,
                                    stream);
            });
            return;
        }
        if (l == L - 1) {
            coarse(l, act);
            return;
        }
        for (int i = 0; i < set.pre_smoothing; ++i) smooth(l, act);
        residual(l, act);
        restrict_to(l, act);
        if (type == 0) {
            cycle(l + 1, 0, act);
        } else if (type == 1) {
            cycle(l + 1, 1, act);
            cycle(l + 1, 1, act);
        } else {
            cycle(l + 1, 2, act);
            cycle(l + 1, 0, act);
        }
        prolong_add(l, act);
        for (int i = 0; i < set.post_smoothing; ++i) smooth(l, act);
    }

    // residual norm + convergence bookkeeping of the next iteration index
    void norm_check() {
        Level& V = lv[0];
        int nb = 0;
        if (set.extrapolation) {  // residual_norm (multigrid.cpp:267-275)
            ex_residual(act_mask());
            run(KK_NORM, 1, [&] {
                nb = launch_norm_partials(V.res, V.v.n, B, set.norm_type, partials, stream);
            });
        } else {
            run(KK_RESIDUAL, apply_launches(V.v), [&] {
                nb = launch_apply(V.v, onfly, 1, V.u, V.f, V.res, partials, set.norm_type, act_mask(),
                                  stream);
            });
        }
        run(KK_NORM, 1, [&] {
            ConvState cs{r0, hist, active, iters, conv, remaining, count, hist_cap};
            launch_norm_check(partials, nb, B, V.v.n, set.norm_type, norms, cs,
                              set.max_iterations, set.relative_tolerance, set.absolute_tolerance,
                              stream);
        });
    }

    // one multigrid cycle + residual norm + convergence check, captured once
    // and replayed every iteration (the active mask and the per-section
    // iteration counters live on the device)
    void build_cycle_graph() {
        const long long l0 = launches;
        cudaGraph_t g = nullptr;
        PMG_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
        cycle(0, set.cycle, act_mask());
        norm_check();
        PMG_CUDA(cudaStreamEndCapture(stream, &g));
        PMG_CUDA(cudaGraphInstantiate(&cycle_exec, g, 0));
        cudaGraphDestroy(g);
        cycle_nodes = launches - l0;
        launches = l0;
    }

    // The solve loop of multigrid.cpp:328-340 on the device: a conditional
    // WHILE node replays {cycle, residual norm, convergence check, condition}
    // until no section is iterating -- no host round trip between cycles.
    // Falls back to the per-cycle graph launches (host loop) if the driver
    // rejects the conditional graph.
    bool build_loop_graph() {
        const long long l0 = launches;
        cudaGraph_t g = nullptr;
        bool ok = cudaGraphCreate(&g, 0) == cudaSuccess;
        cudaGraphConditionalHandle h{};
        ok = ok && cudaGraphConditionalHandleCreate(&h, g, 0, 0) == cudaSuccess;
        cudaGraphNode_t first = nullptr;
        if (ok) {  // condition of the first pass, from the initial norm check
            cudaGraph_t tmp = nullptr;
            ok = cudaStreamBeginCaptureToGraph(stream, g, nullptr, nullptr, 0,
                                               cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                launch_loop_cond(h, remaining, stream);
                ok = cudaStreamEndCapture(stream, &tmp) == cudaSuccess;
            }
            size_t nn = 1;
            ok = ok && cudaGraphGetNodes(g, &first, &nn) == cudaSuccess && nn == 1;
        }
        if (ok) {
            cudaGraphNodeParams cp{};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            cudaGraphNode_t wn = nullptr;
            ok = cudaGraphAddNode(&wn, g, &first, 1, &cp) == cudaSuccess;
            if (ok) {
                cudaGraph_t body = cp.conditional.phGraph_out[0], tmp = nullptr;
                ok = cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0,
                                                   cudaStreamCaptureModeThreadLocal) == cudaSuccess;
                if (ok) {
                    cycle(0, set.cycle, act_mask());
                    norm_check();
                    launch_loop_cond(h, remaining, stream);
                    ok = cudaStreamEndCapture(stream, &tmp) == cudaSuccess;
                }
            }
        }
        ok = ok && cudaGraphInstantiate(&loop_exec, g, 0) == cudaSuccess;
        if (g) cudaGraphDestroy(g);
        cycle_nodes = launches - l0;
        launches = l0;
        if (!ok) {
            cudaGetLastError();
            last_error();
            loop_exec = nullptr;
            use_loop = false;
        }
        return ok;
    }

    // PMG_TAIL_TRACE: per-op durations of the last coarse-tail launch (stderr)
    void print_tail_trace() {
        const std::vector<int>& prog = h_prog[set.cycle];
        std::vector<unsigned long long> t(prog.size() + 4);
        PMG_CUDA(cudaMemcpy(t.data(), coarse_params.trace, t.size() * 8, cudaMemcpyDeviceToHost));
        static const char* names[] = {"smooth", "residual", "restrict", "prolong", "coarse"};
        const size_t np = prog.size();
        std::fprintf(stderr, "tail trace: staging %.2f us (issue %.2f, wait %.2f, rebase %.2f)\n",
                     (t[1] - t[0]) * 1e-3, (t[np + 2] - t[0]) * 1e-3,
                     (t[np + 3] - t[np + 2]) * 1e-3, (t[1] - t[np + 3]) * 1e-3);
        double sum[5][kMaxCoarse] = {};
        for (size_t i = 0; i < prog.size(); ++i)
            sum[prog[i] & 255][(prog[i] >> 8) - coarse_start] += (t[2 + i] - t[1 + i]) * 1e-3;
        for (int o = 0; o < 5; ++o)
            for (int l = 0; l < kMaxCoarse; ++l)
                if (sum[o][l] > 0)
                    std::fprintf(stderr, "tail trace: level %d %-8s %.2f us\n", coarse_start + l,
                                 names[o], sum[o][l]);
        std::fprintf(stderr, "tail trace: total %.2f us\n", (t[prog.size() + 1] - t[0]) * 1e-3);
    }

    // ---------------------------------------------- manufactured problem
    // (problem.cpp:48-148, stencil.cpp:297-353, multigrid.cpp:133-143,250-296)
    std::vector<RhsTables> rhs_tabs;
    int* d_bad = nullptr;
    int fmg_run = 0;
    double* ex_g = nullptr;  // 3/4 f of the extrapolated line sweeps (level 0)

    void build_rhs_tables() {
        if (!rhs_tabs.empty()) return;
        const double two_pi = 2.0 * 3.141592653589793;  // kTwoPi (problem.cpp:10)
        for (Level& V : lv) {
            const HostGrid& g = V.g;
            const int nr = g.nr(), nt = g.nt();
            std::vector<double> aR((size_t)B * nr * 8), sT((size_t)nt * 8), cT((size_t)nt * 8),
                s11((size_t)nt * 8), c11((size_t)nt * 8), s0(nt), c0(nt);
            const auto alpha = [&](int b, double r) {  // problem.cpp:86-89
                return prob.alpha_coeff == 0
                           ? 1.0
                           : scales[b] * std::exp(-std::tanh((r / prob.rmax - prob.alpha_jump) /
                                                             prob.delta_r));
            };
            for (int b = 0; b < B; ++b)
                for (int s = 0; s < nr; ++s) {  // rhs_f radial stencil (problem.cpp:135-142)
                    const double r = g.r[s];
                    const double a1 = 1e-4 * prob.rmax, a2 = r / 3.0;
                    const double er = a2 < a1 ? a2 : a1;
                    for (int k = 0; k < 2; ++k) {
                        const double e = er * (k == 0 ? 1.0 : 0.5);
                        const double xs[4] = {r - 2.0 * e, r - e, r + e, r + 2.0 * e};
                        for (int j = 0; j < 4; ++j)
                            aR[((size_t)b * nr + s) * 8 + 4 * k + j] = alpha(b, xs[j]);
                    }
                }
            const double et = 1e-4 * two_pi;
            for (int t = 0; t < nt; ++t) {
                const double th = g.th[t];
                s0[t] = std::sin(11.0 * th);
                c0[t] = std::cos(11.0 * th);
                for (int k = 0; k < 2; ++k) {
                    const double e = et * (k == 0 ? 1.0 : 0.5);
                    const double ts[4] = {th - 2.0 * e, th - e, th + e, th + 2.0 * e};
                    for (int j = 0; j < 4; ++j) {
                        const size_t i = (size_t)t * 8 + 4 * k + j;
                        sT[i] = std::sin(ts[j]);
                        cT[i] = std::cos(ts[j]);
                        s11[i] = std::sin(11.0 * ts[j]);
                        c11[i] = std::cos(11.0 * ts[j]);
                    }
                }
            }
            RhsTables T{};
            T.th = upload(g.th);
            T.aR = upload(aR);
            T.sT = upload(sT);
            T.cT = upload(cT);
            T.s11 = upload(s11);
            T.c11 = upload(c11);
            T.s11_0 = upload(s0);
            T.c11_0 = upload(c0);
            T.rmax = prob.rmax;
            T.sol = prob.solution;
            rhs_tabs.push_back(T);
        }
        d_bad = alloc<int>(1);
    }
    // MultigridSolver::assemble_level_rhs (multigrid.cpp:155-157)
    void assemble_level_rhs(int l) {
        build_rhs_tables();
        PMG_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), stream));
        run(KK_OTHER, 1, [&] { launch_assemble_rhs(lv[l].v, rhs_tabs[l], lv[l].f, d_bad, stream); });
        int hb = 0;
        PMG_CUDA(cudaMemcpyAsync(&hb, d_bad, sizeof(int), cudaMemcpyDeviceToHost, stream));
        PMG_CUDA(cudaStreamSynchronize(stream));
        PMG_CUDA(last_error());
        if (hb == 1) throw PmgError(PMG_ERUNTIME, "singular Jacobian: mapping degenerate at queried point");
        if (hb == 2)
            throw PmgError(PMG_ERUNTIME,
                           "rhs_f lost accuracy: Richardson step-halving check disagrees by more "
                           "than 1e-7");
        if (hb == 3) throw PmgError(PMG_EINVAL, "rhs_f requires r > 0");
    }
    void set_dirichlet_rows(int l, double* u) {
        build_rhs_tables();
        run(KK_OTHER, 1, [&] { launch_set_dirichlet(lv[l].v, rhs_tabs[l], u, stream); });
    }
    // multigrid.cpp:250-265
    void fmg_initialize() {
        const int L = static_cast<int>(lv.size());
        assemble_level_rhs(L - 1);
        coarse(L - 1, act_mask());
        for (int lf = L - 2; lf >= 0; --lf) {
            Level& F = lv[lf];
            Level& C = lv[lf + 1];
            run(KK_PROLONG, 1,
                [&] { launch_prolong(F.v, C.v, F.w, C.u, F.u, false, act_mask(), stream); });
            set_dirichlet_rows(lf, F.u);
            assemble_level_rhs(lf);
            if (lf == 0 && set.extrapolation) build_extrapolated_rhs();
            for (int c = 0; c < set.fmg_iterations; ++c) {
                cycle(lf, set.fmg_cycle, act_mask());
                if (lf == 0) ++fmg_run;
            }
        }
    }
    // multigrid.cpp:277-296 (device reduction order; -1 without a solution)
    void exact_errors(const double* u, double* w, double* inf) {
        build_rhs_tables();
        const LevelView& v = lv[0].v;
        const int nb = launch_exact_errors(v, rhs_tabs[0], u, partials, partial_cap / 2, stream);
        std::vector<double> hp((size_t)B * nb * 2);
        PMG_CUDA(cudaMemcpyAsync(hp.data(), partials, hp.size() * sizeof(double),
                                 cudaMemcpyDeviceToHost, stream));
        PMG_CUDA(cudaStreamSynchronize(stream));
        for (int b = 0; b < B; ++b) {
            double a = 0.0, m = 0.0;
            for (int i = 0; i < nb; ++i) {
                a += hp[((size_t)b * nb + i) * 2];
                m = std::max(m, hp[((size_t)b * nb + i) * 2 + 1]);
            }
            w[b] = prob.solution ? std::sqrt(a / v.n) : -1.0;
            inf[b] = prob.solution ? m : -1.0;
        }
    }

    int solve(pmg_report* reports, double* history, int history_cap) {
        PMG_CUDA(cudaSetDevice(device));
        cudaEvent_t e0, e1;
        PMG_CUDA(cudaEventCreate(&e0));
        PMG_CUDA(cudaEventCreate(&e1));
        PMG_CUDA(cudaEventRecord(e0, stream));
        Level& V = lv[0];
        fmg_run = 0;
        if (set.fmg) {  // multigrid.cpp:306-307
            run(KK_OTHER, 1, [&] { launch_set_active(active, count, conv, remaining, B, stream); });
            fmg_initialize();
        } else {  // multigrid.cpp:309-316 (the RHS is the current f)
            if (set.extrapolation) {  // the extrapolated RHS needs f on levels 0 and 1
                assemble_level_rhs(0);
                assemble_level_rhs(1);
                build_extrapolated_rhs();
            }
            run(KK_OTHER, 2, [&] {
                launch_set_active(active, count, conv, remaining, B, stream);
                launch_fill(V.u, (long)B * V.v.n, 0.0, stream);
            });
            if (prob.solution) set_dirichlet_rows(0, V.u);
        }
        norm_check();
        const bool graph = use_graph && !prof;
        bool looped = false;
        if (const char* e = std::getenv("PMG_LOOP_GRAPH")) use_loop = use_loop && std::atoi(e) != 0;
        if (graph && use_loop && !set.verbose) {
            if (!loop_exec) build_loop_graph();
            if (loop_exec) {
                PMG_CUDA(cudaGraphLaunch(loop_exec, stream));
                looped = true;
            }
        }
        if (graph && !looped && !cycle_exec) build_cycle_graph();
        int it = 0;
        for (; !looped;) {
            PMG_CUDA(cudaMemcpyAsync(h_remaining, remaining, sizeof(int), cudaMemcpyDeviceToHost,
                                     stream));
            PMG_CUDA(cudaStreamSynchronize(stream));
            if (set.verbose) {
                double r;
                PMG_CUDA(cudaMemcpy(&r, norms, sizeof(double), cudaMemcpyDeviceToHost));
                std::printf("cycle %3d  residual %.6e\n", it, r);
            }
            if (*h_remaining == 0) break;
            if (graph) {
                PMG_CUDA(cudaGraphLaunch(cycle_exec, stream));
                launches += cycle_nodes;
            } else {
                cycle(0, set.cycle, act_mask());
                norm_check();
            }
            ++it;
        }
        PMG_CUDA(cudaEventRecord(e1, stream));
        PMG_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        PMG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        PMG_CUDA(last_error());
        last_solve_ms = ms;
        collect_profile();
        if (coarse_params.trace && mid_start < 0) print_tail_trace();
        if (mid_params.trace) print_mid_trace();
        // reports
        std::vector<int> h_it(B), h_conv(B);
        std::vector<double> h_hist((size_t)B * hist_cap);
        PMG_CUDA(cudaMemcpy(h_it.data(), iters, sizeof(int) * B, cudaMemcpyDeviceToHost));
        if (looped) launches += cycle_nodes * *std::max_element(h_it.begin(), h_it.end());
        PMG_CUDA(cudaMemcpy(h_conv.data(), conv, sizeof(int) * B, cudaMemcpyDeviceToHost));
        PMG_CUDA(cudaMemcpy(h_hist.data(), hist, sizeof(double) * h_hist.size(),
                            cudaMemcpyDeviceToHost));
        std::vector<double> ew(B, -1.0), ei(B, -1.0);
        if (reports && prob.solution) exact_errors(lv[0].u, ew.data(), ei.data());
        bool all = true;
        for (int b = 0; b < B; ++b) {
            const int itb = h_it[b];
            const double* hb = h_hist.data() + (size_t)b * hist_cap;
            if (reports) {
                pmg_report& r = reports[b];
                std::memset(&r, 0, sizeof r);
                r.converged = h_conv[b];
                r.iterations = itb;
                r.fine_cycles_total = itb + fmg_run;
                r.exact_error_weighted = ew[b];
                r.exact_error_infinity = ei[b];
                r.num_residuals = itb + 1;
                r.initial_residual = hb[0];
                r.final_residual = hb[itb];
                r.reduction_factor_mean = (itb > 0 && hb[0] > 0.0 && hb[itb] > 0.0)
                                              ? std::pow(hb[itb] / hb[0], 1.0 / itb)
                                              : 0.0;
                r.setup_seconds = setup_seconds;
                r.solve_seconds = ms * 1e-3;
                r.device_bytes = bytes;
            }
            if (history && history_cap > 0)
                for (int k = 0; k < history_cap; ++k)
                    history[(size_t)b * history_cap + k] = k <= itb ? hb[k] : 0.0;
            all = all && h_conv[b];
        }
        return all ? PMG_OK : PMG_ENOTCONV;
    }

    // ------------------------------------------------------------ helpers
    void to_node(int l, const double* in, double* out, int layout) const {
        const HostGrid& g = lv[l].g;
        const long n = g.n();
        if (layout == PMG_LAYOUT_NODE) {
            std::memcpy(out, in, sizeof(double) * n * B);
            return;
        }
        for (int b = 0; b < B; ++b)
            for (int s = 0; s < g.nr(); ++s)
                for (int t = 0; t < g.nt(); ++t)
                    out[(long)b * n + g.idx(s, t)] = in[(long)b * n + (long)s * g.nt() + t];
    }
    void from_node(int l, const double* in, double* out, int layout) const {
        const HostGrid& g = lv[l].g;
        const long n = g.n();
        if (layout == PMG_LAYOUT_NODE) {
            std::memcpy(out, in, sizeof(double) * n * B);
            return;
        }
        for (int b = 0; b < B; ++b)
            for (int s = 0; s < g.nr(); ++s)
                for (int t = 0; t < g.nt(); ++t)
                    out[(long)b * n + (long)s * g.nt() + t] = in[(long)b * n + g.idx(s, t)];
    }
    void h2d(double* d, const double* h, long count) {
        PMG_CUDA(cudaMemcpyAsync(d, h, sizeof(double) * count, cudaMemcpyHostToDevice, stream));
    }
    void d2h(double* h, const double* d, long count) {
        PMG_CUDA(cudaMemcpyAsync(h, d, sizeof(double) * count, cudaMemcpyDeviceToHost, stream));
        PMG_CUDA(cudaStreamSynchronize(stream));
    }
    void check_level(int l, bool need_smoother = false) const {
        if (l < 0 || l >= static_cast<int>(lv.size()))
            throw PmgError(PMG_EINVAL, "level out of range");
        if (need_smoother && l == static_cast<int>(lv.size()) - 1)
            throw PmgError(PMG_EINVAL, "the coarsest level has no smoother");
    }
    void sync_check() {
        PMG_CUDA(cudaStreamSynchronize(stream));
        PMG_CUDA(last_error());
    }
    void ensure_flush() {
        if (!flush_buf) {
            flush_n = (256l << 20) / 8;  // 256 MiB > 126 MB L2
            flush_buf = alloc<double>(flush_n);
        }
    }
};

// ------------------------------------------------------------- validation
// SolverConfig::validate (config.cpp:150-183) on the ABI structs
static void validate(const pmg_geometry* g, const pmg_problem* p, const pmg_grid* gr,
                     const pmg_settings* s) {
    if (!g || !p || !gr || !s) throw PmgError(PMG_EINVAL, "null argument");
    if (s->extrapolation != 0 && s->extrapolation != 1)
        throw PmgError(PMG_EINVAL, "extrapolation=" + std::to_string(s->extrapolation) +
                                       " is not supported by this solver (use 0 or 1)");
    if (s->extrapolation == 1 && s->max_levels == 1)
        throw PmgError(PMG_EINVAL,
                       "extrapolation requires at least two levels (maxLevels=1 given)");
    if (s->fmg && (s->fmg_cycle < 0 || s->fmg_cycle > 2))
        throw PmgError(PMG_EINVAL, "unknown FMG_cycle type (expected V, W, or F)");
    if (p->solution < 0 || p->solution > 1)
        throw PmgError(PMG_EINVAL, "unknown problem (expected None or Polar)");
    if (p->rmax <= 0.0) throw PmgError(PMG_EINVAL, "Rmax must be positive");
    if (p->delta_r <= 0.0) throw PmgError(PMG_EINVAL, "delta_r must be positive");
    if (gr->mode != 2 && (gr->R0 <= 0.0 || gr->R0 >= gr->Rmax))
        throw PmgError(PMG_EINVAL, "R0 must lie in (0, Rmax)");
    if (gr->mode == 1) {
        if (gr->nr_exp < 2) throw PmgError(PMG_EINVAL, "nr_exp must be at least 2");
        if (gr->ntheta_exp < 2) throw PmgError(PMG_EINVAL, "ntheta_exp must be at least 2");
        if (gr->anisotropic_factor < 0)
            throw PmgError(PMG_EINVAL, "anisotropic_factor must be >= 0");
        if (gr->divide_by_2 < 0) throw PmgError(PMG_EINVAL, "divideBy2 must be >= 0");
    }
    if (s->max_levels < 0) throw PmgError(PMG_EINVAL, "maxLevels must be >= 0");
    if (s->pre_smoothing < 0 || s->post_smoothing < 0)
        throw PmgError(PMG_EINVAL, "preSmoothingSteps/postSmoothingSteps must be >= 0");
    if (s->max_iterations < 0) throw PmgError(PMG_EINVAL, "maxIterations must be >= 0");
    if (s->fmg_iterations < 1) throw PmgError(PMG_EINVAL, "FMG_iterations must be >= 1");
    if (s->max_threads < 0) throw PmgError(PMG_EINVAL, "maxOpenMPThreads must be >= 0");
    if (s->stencil_mode != 0 && s->stencil_mode != 1)
        throw PmgError(PMG_EINVAL, "unknown stencilDistributionMethod (expected Take or Give)");
    if (s->cycle < 0 || s->cycle > 2)
        throw PmgError(PMG_EINVAL, "unknown cycle type (expected V, W, or F)");
    if (s->norm_type < 0 || s->norm_type > 2)
        throw PmgError(PMG_EINVAL,
                       "unknown residualNormType (expected weighted-l2, euclidean, or infinity)");
    if (s->boundary_mode != 0 && s->boundary_mode != 1)
        throw PmgError(PMG_EINVAL, "unknown boundary mode");
    if (g->kind < 0 || g->kind > 2) throw PmgError(PMG_EINVAL, "unknown geometry");
    if (g->kind == 2 && (g->kappa_eps <= 0.0 || g->kappa_eps >= 2.0))
        throw PmgError(PMG_EINVAL, "Czarny requires 0 < epsilon < 2");
}

}  // namespace pmg

// =================================================================== C ABI
using pmg::PmgError;
using pmg::Solver;

struct pmg_solver {
    std::unique_ptr<Solver> s;
};

template <class F>
static int guarded(F&& fn) {
    try {
        fn();
        return PMG_OK;
    } catch (const PmgError& e) {
        pmg::g_err = e.what();
        return e.code;
    } catch (const std::invalid_argument& e) {
        pmg::g_err = e.what();
        return PMG_EINVAL;
    } catch (const std::bad_alloc&) {
        pmg::g_err = "out of host memory";
        return PMG_ERUNTIME;
    } catch (const std::exception& e) {
        pmg::g_err = e.what();
        return PMG_ERUNTIME;
    }
}

static Solver& S(pmg_handle h) {
    if (!h || !h->s) throw PmgError(PMG_EINVAL, "null solver handle");
    cudaSetDevice(h->s->device);
    return *h->s;
}

extern "C" {

const char* pmg_last_error(void) { return pmg::g_err.c_str(); }
const char* pmg_version(void) { return "polarmg_b200 0.1 (sm_100a, fp64)"; }

void pmg_default_settings(pmg_settings* s) {
    std::memset(s, 0, sizeof *s);
    s->stencil_mode = 0;
    s->boundary_mode = 0;
    s->cache_profile = 1;
    s->cache_geometry = 0;
    s->max_levels = 0;
    s->pre_smoothing = 1;
    s->post_smoothing = 1;
    s->cycle = 0;
    s->extrapolation = 0;
    s->fmg = 0;
    s->fmg_iterations = 2;
    s->fmg_cycle = 2;
    s->norm_type = 0;
    s->max_iterations = 150;
    s->reference_order = 1;  // bitwise reference parity (the drop-in default)
    s->absolute_tolerance = -1.0;
    s->relative_tolerance = 1e-8;
    s->max_threads = 0;
    s->verbose = 0;
}

int pmg_create_batch(const pmg_geometry* geom, const pmg_problem* prob, const pmg_grid* grid,
                     const pmg_settings* settings, int n_sections, const double* alpha_scales,
                     int device, void* stream, pmg_handle* out) {
    return guarded([&] {
        if (!out) throw PmgError(PMG_EINVAL, "null output handle");
        *out = nullptr;
        pmg::validate(geom, prob, grid, settings);
        if (n_sections < 1) throw PmgError(PMG_EINVAL, "n_sections must be >= 1");
        int ndev = 0;
        PMG_CUDA(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev)
            throw PmgError(PMG_EINVAL, "CUDA device " + std::to_string(device) + " not present");
        PMG_CUDA(cudaSetDevice(device));
        auto s = std::make_unique<Solver>();
        s->device = device;
        if (stream) {
            s->stream = static_cast<cudaStream_t>(stream);
        } else {
            PMG_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
            s->own_stream = true;
        }
        s->geo.kind = geom->kind;
        s->geo.ke = geom->kappa_eps;
        s->geo.de = geom->delta_e;
        s->geo.xi = geom->kind == 2
                        ? 1.0 / std::sqrt(1.0 - geom->kappa_eps * geom->kappa_eps / 4.0)
                        : 1.0;
        s->prob = *prob;
        s->set = *settings;
        s->B = n_sections;
        s->scales.assign(n_sections, 1.0);
        // alpha_scale multiplies the per-section scale (both 1 => reference alpha)
        for (int b = 0; b < n_sections; ++b)
            s->scales[b] = (alpha_scales ? alpha_scales[b] : 1.0) * prob->alpha_scale;
        s->build(*grid);
        auto* h = new pmg_solver;
        h->s = std::move(s);
        *out = h;
    });
}

int pmg_create(const pmg_geometry* geom, const pmg_problem* prob, const pmg_grid* grid,
               const pmg_settings* settings, int device, void* stream, pmg_handle* out) {
    return pmg_create_batch(geom, prob, grid, settings, 1, nullptr, device, stream, out);
}

int pmg_grid_hierarchy(const pmg_grid* gp, int max_levels, int capacity, int* levels, int* n_r,
                       int* n_theta, int* split) {
    return guarded([&] {
        if (!gp || !levels) throw PmgError(PMG_EINVAL, "null argument");
        const double tol = gp->pair_tolerance > 0.0 ? gp->pair_tolerance : 1e-12;
        pmg::HostGrid g;
        if (gp->mode == 0)
            g = pmg::uniform_grid(gp->R0, gp->Rmax, gp->n_r, gp->n_theta, tol);
        else if (gp->mode == 1)
            g = pmg::build_grid(gp->R0, gp->Rmax, gp->nr_exp, gp->ntheta_exp,
                                gp->anisotropic_factor, gp->divide_by_2, tol);
        else
            g = pmg::make_grid(std::vector<double>(gp->radii, gp->radii + gp->n_r),
                               std::vector<double>(gp->angles, gp->angles + gp->n_theta), tol);
        int L = 0;
        for (;;) {
            if (L < capacity) {
                n_r[L] = g.nr();
                n_theta[L] = g.nt();
                split[L] = g.split;
            }
            ++L;
            if ((max_levels != 0 && L >= max_levels) || !pmg::can_coarsen(g, tol)) break;
            g = pmg::coarsen(g, tol);
        }
        *levels = L;
    });
}

int pmg_destroy(pmg_handle h) {
    return guarded([&] { delete h; });
}

int pmg_num_levels(pmg_handle h, int* levels) {
    return guarded([&] { *levels = static_cast<int>(S(h).lv.size()); });
}
int pmg_num_sections(pmg_handle h, int* sections) {
    return guarded([&] { *sections = S(h).B; });
}
int pmg_level_info(pmg_handle h, int level, int* n_r, int* n_theta, int* split) {
    return guarded([&] {
        Solver& s = S(h);
        s.check_level(level);
        const auto& g = s.lv[level].g;
        *n_r = g.nr();
        *n_theta = g.nt();
        *split = g.split;
    });
}
int pmg_level_grid(pmg_handle h, int level, double* radii, double* angles) {
    return guarded([&] {
        Solver& s = S(h);
        s.check_level(level);
        const auto& g = s.lv[level].g;
        std::copy(g.r.begin(), g.r.end(), radii);
        std::copy(g.th.begin(), g.th.end(), angles);
    });
}

int pmg_set_rhs(pmg_handle h, const double* f_host, int layout) {
    return guarded([&] {
        Solver& s = S(h);
        const long N = (long)s.B * s.lv[0].v.n;
        if (layout == PMG_LAYOUT_NODE) {  // device layout: one direct copy
            s.h2d(s.lv[0].f, f_host, N);
        } else {
            std::vector<double> tmp(N);
            s.to_node(0, f_host, tmp.data(), layout);
            s.h2d(s.lv[0].f, tmp.data(), N);
        }
        s.sync_check();
    });
}

int pmg_get_rhs(pmg_handle h, double* f_host, int layout) {
    return guarded([&] {
        Solver& s = S(h);
        const long N = (long)s.B * s.lv[0].v.n;
        std::vector<double> tmp(N);
        s.d2h(tmp.data(), s.lv[0].f, N);
        s.from_node(0, tmp.data(), f_host, layout);
    });
}

int pmg_set_rhs_device(pmg_handle h, const void* f_device) {
    return guarded([&] {
        Solver& s = S(h);
        const long N = (long)s.B * s.lv[0].v.n;
        PMG_CUDA(cudaMemcpyAsync(s.lv[0].f, f_device, sizeof(double) * N,
                                 cudaMemcpyDeviceToDevice, s.stream));
    });
}

int pmg_seeded_rhs(pmg_handle h, unsigned seed, double* ustar_host, int layout) {
    return guarded([&] {
        Solver& s = S(h);
        pmg::Level& V = s.lv[0];
        const auto& g = V.g;
        const long n = g.n();
        std::vector<double> us((size_t)s.B * n);
        for (int b = 0; b < s.B; ++b) {
            std::mt19937 rng(seed + static_cast<unsigned>(b));
            std::uniform_real_distribution<double> dist(-1.0, 1.0);
            double* ub = us.data() + (size_t)b * n;
            for (int si = 0; si < g.nr(); ++si)
                for (int t = 0; t < g.nt(); ++t) ub[g.idx(si, t)] = dist(rng);
            for (int t = 0; t < g.nt(); ++t) ub[g.idx(g.nr() - 1, t)] = 0.0;
        }
        s.h2d(V.res, us.data(), (long)us.size());
        s.run(pmg::KK_RESIDUAL, pmg::apply_launches(V.v), [&] {
            pmg::launch_apply(V.v, s.onfly, 0, V.res, nullptr, V.f, nullptr, 0, nullptr,
                              s.stream);
        });
        s.sync_check();
        if (ustar_host) s.from_node(0, us.data(), ustar_host, layout);
    });
}

int pmg_solve(pmg_handle h, pmg_report* reports, double* history, int history_cap) {
    int rc = PMG_OK;
    const int g = guarded([&] { rc = S(h).solve(reports, history, history_cap); });
    if (g != PMG_OK) return g;
    if (rc == PMG_ENOTCONV) pmg::g_err = "solve ended without meeting a tolerance";
    return rc;
}

#ifdef PMG_KTRACE
int pmg_debug_ktrace(unsigned long long* out) {
    pmg::read_ktrace(out);
    return 0;
}
int pmg_debug_ktrace_reset() {
    pmg::reset_ktrace();
    return 0;
}
#endif

int pmg_assemble_rhs(pmg_handle h) {
    return guarded([&] {
        Solver& s = S(h);
        PMG_CUDA(cudaSetDevice(s.device));
        s.assemble_level_rhs(0);
    });
}

int pmg_exact_errors(pmg_handle h, double* weighted, double* infinity) {
    return guarded([&] {
        Solver& s = S(h);
        if (!weighted || !infinity) throw PmgError(PMG_EINVAL, "null argument");
        PMG_CUDA(cudaSetDevice(s.device));
        s.exact_errors(s.lv[0].u, weighted, infinity);
    });
}

int pmg_get_solution(pmg_handle h, double* u_host, int layout) {
    return guarded([&] {
        Solver& s = S(h);
        const long N = (long)s.B * s.lv[0].v.n;
        if (layout == PMG_LAYOUT_NODE) {
            s.d2h(u_host, s.lv[0].u, N);
            return;
        }
        std::vector<double> tmp(N);
        s.d2h(tmp.data(), s.lv[0].u, N);
        s.from_node(0, tmp.data(), u_host, layout);
    });
}

int pmg_solution_device(pmg_handle h, const void** u_device) {
    return guarded([&] { *u_device = S(h).lv[0].u; });
}

// ---- operator seams on host buffers
int pmg_apply(pmg_handle h, int level, const double* u, double* y) {
    return guarded([&] {
        Solver& s = S(h);
        s.check_level(level);
        pmg::Level& V = s.lv[level];
        const long N = (long)s.B * V.v.n;
        s.h2d(V.u, u, N);
        s.run(pmg::KK_RESIDUAL, pmg::apply_launches(V.v), [&] {
            pmg::launch_apply(V.v, s.onfly, 0, V.u, nullptr, V.res, nullptr, 0, nullptr,
                              s.stream);
        });
        s.d2h(y, V.res, N);
        s.sync_check();
    });
}

int pmg_residual(pmg_handle h, int level, const double* u, const double* f, double* r) {
    return guarded([&] {
        Solver& s = S(h);
        s.check_level(level);
        pmg::Level& V = s.lv[level];
        const long N = (long)s.B * V.v.n;
        s.h2d(V.u, u, N);
        s.h2d(V.f, f, N);
        s.residual(level, nullptr);
        s.d2h(r, V.res, N);
        s.sync_check();
    });
}

int pmg_smooth(pmg_handle h, int level, double* u, const double* f) {
    return guarded([&] {
        Solver& s = S(h);
        s.check_level(level, true);
        pmg::Level& V = s.lv[level];
        const long N = (long)s.B * V.v.n;
        s.h2d(V.u, u, N);
        s.h2d(V.f, f, N);
        s.smooth(level, nullptr);
        s.d2h(u, V.u, N);
        s.sync_check();
    });
}

int pmg_sweep(pmg_handle h, int level, int kind, int parity, double* u, const double* f) {
    return guarded([&] {
        Solver& s = S(h);
        s.check_level(level, true);
        if (parity != 0 && parity != 1) throw PmgError(PMG_EINVAL, "parity must be 0 or 1");
        pmg::Level& V = s.lv[level];
        const long N = (long)s.B * V.v.n;
        s.h2d(V.u, u, N);
        s.h2d(V.f, f, N);
        if (kind == 0)
            s.run(pmg::KK_CIRCLE, 1, [&] {
                pmg::launch_circle(V.v, s.onfly, V.u, V.f, V.cil, V.cm, V.corner, V.cz, V.of(),
                                   parity, s.serial, s.exact_rings, nullptr, s.stream);
            });
        else if (V.v.len > 0)
            s.run(pmg::KK_RADIAL, 1, [&] {
                pmg::launch_radial(V.v, s.onfly, V.u, V.f, V.ril, V.rm, parity, s.serial, nullptr,
                                   s.stream);
            });
        s.d2h(u, V.u, N);
        s.sync_check();
    });
}

int pmg_restrict(pmg_handle h, int level, const double* fine, double* coarse) {
    return guarded([&] {
        Solver& s = S(h);
        s.check_level(level, true);
        pmg::Level& F = s.lv[level];
        pmg::Level& C = s.lv[level + 1];
        s.h2d(F.res, fine, (long)s.B * F.v.n);
        // plain restrict_transpose: no Dirichlet masking at this seam
        s.run(pmg::KK_RESTRICT, 1, [&] {
            pmg::launch_restrict(F.v, C.v, F.w, F.res, C.f, nullptr, false, nullptr, s.stream);
        });
        s.d2h(coarse, C.f, (long)s.B * C.v.n);
        s.sync_check();
    });
}

int pmg_prolongate(pmg_handle h, int level, const double* coarse, double* fine, int add) {
    return guarded([&] {
        Solver& s = S(h);
        s.check_level(level, true);
        pmg::Level& F = s.lv[level];
        pmg::Level& C = s.lv[level + 1];
        s.h2d(C.u, coarse, (long)s.B * C.v.n);
        if (add) s.h2d(F.u, fine, (long)s.B * F.v.n);
        s.run(pmg::KK_PROLONG, 1, [&] {
            pmg::launch_prolong(F.v, C.v, F.w, C.u, F.u, add != 0, nullptr, s.stream);
        });
        s.d2h(fine, F.u, (long)s.B * F.v.n);
        s.sync_check();
    });
}

int pmg_coarse_solve(pmg_handle h, const double* f, double* u) {
    return guarded([&] {
        Solver& s = S(h);
        const int l = static_cast<int>(s.lv.size()) - 1;
        pmg::Level& V = s.lv[l];
        s.h2d(V.f, f, (long)s.B * V.v.n);
        s.coarse(l, nullptr);
        s.d2h(u, V.u, (long)s.B * V.v.n);
        s.sync_check();
    });
}

int pmg_norm(pmg_handle h, int type, const double* v_host, long n, double* out) {
    return guarded([&] {
        Solver& s = S(h);
        if (type < 0 || type > 2) throw PmgError(PMG_EINVAL, "unknown norm type");
        double* buf = s.alloc<double>(n, false);
        double* part = s.alloc<double>(1024, false);
        double* res = s.alloc<double>(1, false);
        s.h2d(buf, v_host, n);
        const int nb = pmg::launch_norm_partials(buf, n, 1, type, part, s.stream);
        pmg::launch_norm_final(part, nb, 1, n, type, res, s.stream);
        s.d2h(out, res, 1);
        s.release(buf);
        s.release(part);
        s.release(res);
        s.sync_check();
    });
}

int pmg_launch_count(pmg_handle h, long long* count) {
    return guarded([&] { *count = S(h).launches; });
}

int pmg_time_kernel(pmg_handle h, int kind, int level, int reps, int flush_l2,
                    double* ms_per_call) {
    return guarded([&] {
        Solver& s = S(h);
        s.check_level(level, kind != 0);
        if (reps < 1) throw PmgError(PMG_EINVAL, "reps must be >= 1");
        if (flush_l2) s.ensure_flush();
        cudaEvent_t a, b;
        PMG_CUDA(cudaEventCreate(&a));
        PMG_CUDA(cudaEventCreate(&b));
        double total = 0.0;
        // two untimed warm-up repetitions (lazy module loading, attribute setup)
        for (int r = -2; r < reps; ++r) {
            if (flush_l2) pmg::launch_flush(s.flush_buf, s.flush_n, s.stream);
            PMG_CUDA(cudaEventRecord(a, s.stream));
            pmg::Level& V = s.lv[level];
            switch (kind) {
                case 0: s.residual(level, nullptr); break;
                case 1:
                    for (int p = 0; p < 2; ++p)
                        s.run(pmg::KK_CIRCLE, 1, [&] {
                            pmg::launch_circle(V.v, s.onfly, V.u, V.f, V.cil, V.cm, V.corner,
                                               V.cz, V.of(), p, s.serial, s.exact_rings,
                                               nullptr, s.stream);
                        });
                    break;
                case 2:
                    if (V.worder) {  // both colours in one wavefront launch, as in smooth()
                        s.run(pmg::KK_RADIAL, 1, [&] {
                            pmg::launch_radial_wave(V.v, V.u, V.f, V.ril, V.rm,
                                                    pmg::FuseCtl{s.fuse_ctl, V.wflags}, V.worder,
                                                    s.stream);
                        });
                        break;
                    }
                    for (int p = 0; p < 2; ++p)
                        s.run(pmg::KK_RADIAL, 1, [&] {
                            pmg::launch_radial(V.v, s.onfly, V.u, V.f, V.ril, V.rm, p, s.serial,
                                               nullptr, s.stream);
                        });
                    break;
                case 3: s.smooth(level, nullptr); break;
                case 4: s.restrict_to(level, nullptr); break;
                case 5: s.prolong_add(level, nullptr); break;
                default: throw PmgError(PMG_EINVAL, "unknown kernel kind");
            }
            PMG_CUDA(cudaEventRecord(b, s.stream));
            PMG_CUDA(cudaEventSynchronize(b));
            float ms = 0.f;
            PMG_CUDA(cudaEventElapsedTime(&ms, a, b));
            if (r >= 0) total += ms;
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        PMG_CUDA(pmg::last_error());
        *ms_per_call = total / reps;
    });
}

int pmg_profile_enable(pmg_handle h, int on) {
    return guarded([&] {
        Solver& s = S(h);
        s.collect_profile();
        s.prof = on != 0;
        if (on)
            for (int k = 0; k < pmg::KK_COUNT; ++k) {
                s.prof_ms[k] = 0.0;
                s.prof_n[k] = 0;
            }
    });
}

int pmg_profile_read(pmg_handle h, int kind, double* total_ms, long long* launches) {
    return guarded([&] {
        Solver& s = S(h);
        if (kind < 0 || kind >= pmg::KK_COUNT) throw PmgError(PMG_EINVAL, "unknown kernel kind");
        s.collect_profile();
        *total_ms = s.prof_ms[kind];
        *launches = s.prof_n[kind];
    });
}

}  // extern "C"
