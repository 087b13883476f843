/* TEST INFRASTRUCTURE ONLY -- the CPU oracle of the GPU solve path.
 *
 * A plain-C, single-threaded restatement of the reference polarmg multigrid
 * solve path (reference = /root/reference/proj/core, "ref" below).  Every
 * function names the reference file:line whose algorithm it restates, with
 * the same operation order, so that on identical inputs it reproduces the
 * reference bit-for-bit (pinned by tests/test_oracle.py against the compiled
 * reference oracle/_ref/libpolarmg_ref.so and the committed golden fixtures).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this code; the product (paper_2507_03812_b200) never does.
 *
 * Vectors use the reference NodeIndexing order (polar_grid.hpp:17-37).
 */
#include "polarmg_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define TWO_PI (2.0 * 3.141592653589793)

static _Thread_local char g_err[512];
static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}
const char* orc_last_error(void) { return g_err; }

static void* xcalloc(size_t n, size_t sz) {
    void* p = calloc(n ? n : 1, sz);
    if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
    return p;
}
#define NEWD(n) ((double*)xcalloc((size_t)(n), sizeof(double)))
#define NEWI(n) ((int*)xcalloc((size_t)(n), sizeof(int)))

/* ------------------------------------------------------------------ grid */
/* ref polar_grid.cpp:42-113, 131-225 */
typedef struct {
    int nr, nt, split, uniform_angles;
    double *r, *th, *h, *k;
} Grid;

static void grid_free(Grid* g) {
    free(g->r); free(g->th); free(g->h); free(g->k);
    memset(g, 0, sizeof *g);
}

static int gidx(const Grid* g, int s, int t) { /* polar_grid.hpp:24-27 */
    if (s < g->split) return s * g->nt + t;
    return g->split * g->nt + t * (g->nr - g->split) + (s - g->split);
}
static void gnode(const Grid* g, int idx, int* s, int* t) { /* polar_grid.hpp:30-36 */
    const int cn = g->split * g->nt;
    if (idx < cn) { *s = idx / g->nt; *t = idx % g->nt; return; }
    const int z = idx - cn, len = g->nr - g->split;
    *s = g->split + z % len;
    *t = z / len;
}
static int wrap(const Grid* g, int t) { t %= g->nt; return t < 0 ? t + g->nt : t; }
static double k_below(const Grid* g, int t) { return g->k[t == 0 ? g->nt - 1 : t - 1]; }

static int paired(const double* sp, int n, double tol) { /* polar_grid.cpp:18-26 */
    if (n <= 0) return 1;
    double scale = sp[0];
    for (int i = 1; i < n; ++i) if (sp[i] > scale) scale = sp[i];
    for (int i = 0; i + 1 < n; i += 2)
        if (fabs(sp[i] - sp[i + 1]) > tol * scale) return 0;
    return 1;
}

/* Takes ownership of r, th.  polar_grid.cpp:42-97 */
static int grid_init(Grid* g, double* r, int nr, double* th, int nt, double tol) {
    memset(g, 0, sizeof *g);
    g->r = r; g->th = th; g->nr = nr; g->nt = nt;
    g->h = NEWD(nr > 1 ? nr - 1 : 1);
    g->k = NEWD(nt);
    for (int i = 0; i + 1 < nr; ++i) g->h[i] = r[i + 1] - r[i];
    for (int j = 0; j + 1 < nt; ++j) g->k[j] = th[j + 1] - th[j];
    if (nt > 0) g->k[nt - 1] = TWO_PI - th[nt - 1];
    if (nr < 3 || nt < 2) return fail(1, "grid too small: need at least 3 radii and 2 angles");
    if (r[0] <= 0.0) return fail(1, "invertible mapping requires r_1 > 0 (inner radius must be positive)");
    for (int i = 0; i + 1 < nr; ++i) if (r[i + 1] <= r[i]) return fail(1, "radii must be strictly increasing");
    if (th[0] != 0.0) return fail(1, "angles must start at 0");
    for (int j = 0; j + 1 < nt; ++j) if (th[j + 1] <= th[j]) return fail(1, "angles must be strictly increasing");
    if (th[nt - 1] >= TWO_PI) return fail(1, "angles must lie in [0, 2pi)");
    if (nr % 2 != 1) return fail(1, "n_r must be odd (pairing constraint)");
    if (nt % 2 != 0) return fail(1, "n_theta must be even (pairing constraint)");
    if (!paired(g->h, nr - 1, tol)) return fail(1, "radial spacings violate the pairing constraint");
    if (!paired(g->k, nt, tol)) return fail(1, "angular spacings violate the pairing constraint");
    double sum = 0.0;
    for (int j = 0; j < nt; ++j) sum += g->k[j];
    if (fabs(sum - TWO_PI) > 1e-14 * TWO_PI) return fail(1, "angular spacings must sum to 2pi");
    g->uniform_angles = 1;
    const double k0 = g->k[0];
    for (int j = 0; j < nt; ++j)
        if (fabs(g->k[j] - k0) > tol * k0) { g->uniform_angles = 0; break; }
    int split = -1;
    if (g->uniform_angles) { /* polar_grid.cpp:30-40, clamp :63-65 */
        split = nr;
        for (int i = 0; i < nr; ++i) {
            const double hh = g->h[i < nr - 2 ? i : nr - 2];
            if (r[i] * k0 > hh) { split = i; break; }
        }
        if (split < 1) split = 1;
        if (split > nr) split = nr;
    }
    g->split = split >= 0 ? split : nr;
    if (split < 0) g->uniform_angles = 0;
    return 0;
}

static int grid_uniform(Grid* g, double R0, double Rmax, int nr, int nt, double tol) { /* :99-113 */
    if (R0 <= 0.0) return fail(1, "invertible mapping requires r_1 > 0 (inner radius must be positive)");
    if (Rmax <= R0) return fail(1, "Rmax must exceed R0");
    if (nr < 3 || nt < 2) return fail(1, "grid too small");
    double* r = NEWD(nr);
    const double hh = (Rmax - R0) / (nr - 1);
    for (int i = 0; i < nr; ++i) r[i] = R0 + i * hh;
    r[nr - 1] = Rmax;
    double* th = NEWD(nt);
    const double kk = TWO_PI / nt;
    for (int j = 0; j < nt; ++j) th[j] = j * kk;
    return grid_init(g, r, nr, th, nt, tol);
}

static int grid_refine(Grid* out, const Grid* g, double tol) { /* :209-225 */
    double* r = NEWD(2 * g->nr - 1);
    int n = 0;
    for (int i = 0; i + 1 < g->nr; ++i) {
        r[n++] = g->r[i];
        r[n++] = 0.5 * (g->r[i] + g->r[i + 1]);
    }
    r[n++] = g->r[g->nr - 1];
    double* th = NEWD(2 * g->nt);
    for (int j = 0; j < g->nt; ++j) {
        th[2 * j] = g->th[j];
        const double next = j + 1 < g->nt ? g->th[j + 1] : TWO_PI;
        th[2 * j + 1] = 0.5 * (g->th[j] + next);
    }
    return grid_init(out, r, n, th, 2 * g->nt, tol);
}

static int grid_build(Grid* g, double R0, double Rmax, int nr_exp, int nt_exp, int aniso,
                      int d2, double tol) { /* :131-178 */
    if (R0 <= 0.0) return fail(1, "invertible mapping requires r_1 > 0 (set R0 > 0)");
    if (Rmax <= R0) return fail(1, "Rmax must exceed R0");
    if (nr_exp < 2 || nr_exp > 24) return fail(1, "nr_exp out of range [2, 24]");
    if (nt_exp < 2 || nt_exp > 24) return fail(1, "ntheta_exp out of range [2, 24]");
    if (aniso < 0) return fail(1, "anisotropic_factor must be >= 0");
    if (d2 < 0) return fail(1, "divideBy2 must be >= 0");
    int rc = grid_uniform(g, R0, Rmax, (1 << nr_exp) + 1, 1 << nt_exp, tol);
    if (rc) return rc;
    const double lo = 0.6 * Rmax, hi = 0.8 * Rmax;
    for (int round = 0; round < aniso; ++round) {
        double* nrad = NEWD(2 * g->nr);
        int n = 0;
        for (int p = 0; 2 * p + 2 < g->nr; ++p) {
            const double left = g->r[2 * p], mid = g->r[2 * p + 1], right = g->r[2 * p + 2];
            nrad[n++] = left;
            if (left >= lo && right <= hi) {
                nrad[n++] = 0.5 * (left + mid);
                nrad[n++] = mid;
                nrad[n++] = 0.5 * (mid + right);
            } else {
                nrad[n++] = mid;
            }
        }
        nrad[n++] = g->r[g->nr - 1];
        double* th = NEWD(g->nt);
        memcpy(th, g->th, sizeof(double) * g->nt);
        const int nt = g->nt;
        grid_free(g);
        if ((rc = grid_init(g, nrad, n, th, nt, tol))) return rc;
    }
    for (int d = 0; d < d2; ++d) {
        Grid fine;
        rc = grid_refine(&fine, g, tol);
        grid_free(g);
        *g = fine;
        if (rc) return rc;
    }
    return 0;
}

static int can_coarsen(const Grid* g, double tol) { /* :180-196 */
    const int cnr = (g->nr + 1) / 2, cnt = g->nt / 2;
    if (cnr % 2 != 1 || cnt % 2 != 0) return 0;
    if (cnr < 5 || cnt < 4) return 0;
    double* ch = NEWD(cnr - 1);
    for (int m = 0; m + 1 < cnr; ++m) ch[m] = g->r[2 * m + 2] - g->r[2 * m];
    const int ok = paired(ch, cnr - 1, tol);
    free(ch);
    return ok;
}

static int grid_coarsen(Grid* out, const Grid* g, double tol) { /* :198-207 */
    const int cnr = (g->nr + 1) / 2, cnt = g->nt / 2;
    double* r = NEWD(cnr);
    double* th = NEWD(cnt);
    for (int i = 0; i < cnr; ++i) r[i] = g->r[2 * i];
    for (int j = 0; j < cnt; ++j) th[j] = g->th[2 * j];
    return grid_init(out, r, cnr, th, cnt, tol);
}

/* -------------------------------------------------------------- geometry */
/* ref geometry.cpp:8-108, problem.cpp:86-94 */
typedef struct { int kind; double ke, de, xi; } Geom;
typedef struct { double arr, art, att, det; } Coef;

static int transform(const Geom* G, double alpha, double r, double s, double c, Coef* out) {
    double xr, xt, yr, yt;
    if (G->kind == 0) {
        xr = c; xt = -r * s; yr = s; yt = r * c;
    } else if (G->kind == 1) {
        const double kap = G->ke, del = G->de;
        xr = (1.0 - kap) * c - 2.0 * del * r;
        xt = -(1.0 - kap) * r * s;
        yr = (1.0 + kap) * s;
        yt = (1.0 + kap) * r * c;
    } else {
        const double eps = G->ke, e = G->de;
        const double root = sqrt(1.0 + eps * (eps + 2.0 * r * c));
        const double denom = 2.0 - root;
        xr = -c / root;
        xt = r * s / root;
        yr = e * G->xi * s * (denom + r * eps * c / root) / (denom * denom);
        yt = e * G->xi * r * (c * denom - eps * r * s * s / root) / (denom * denom);
    }
    const double det = xr * yt - xt * yr;
    if (fabs(det) < 1e-14) return fail(2, "singular Jacobian: mapping degenerate at queried point");
    const double da = fabs(det);
    out->arr = 0.5 * alpha * (xt * xt + yt * yt) / da;
    out->att = 0.5 * alpha * (xr * xr + yr * yr) / da;
    out->art = -alpha * (xr * xt + yr * yt) / da;
    out->det = da;
    return 0;
}

typedef struct { int zoni, inv_beta; double rmax, jump, dr, scale; } Prob;
static double p_alpha(const Prob* P, double r) {
    if (!P->zoni) return 1.0;
    return P->scale * exp(-tanh((r / P->rmax - P->jump) / P->dr));
}
static double p_beta(const Prob* P, double r) { return P->inv_beta ? 1.0 / p_alpha(P, r) : 0.0; }

/* ---------------------------------------------------------- line algebra */
/* ref line_algebra.cpp:10-120 */
static int tri_factor(int n, const double* diag, const double* off, double* l, double* m) {
    if (diag[0] <= 0.0) return fail(2, "not positive definite at index 0");
    l[0] = sqrt(diag[0]);
    for (int i = 1; i < n; ++i) {
        const double mm = off[i - 1] / l[i - 1];
        const double piv = diag[i] - mm * mm;
        if (piv <= 0.0) return fail(2, "not positive definite at index %d", i);
        m[i - 1] = mm;
        l[i] = sqrt(piv);
    }
    return 0;
}
static void tri_solve(int n, const double* l, const double* m, double* b) {
    b[0] /= l[0];
    for (int i = 1; i < n; ++i) b[i] = (b[i] - m[i - 1] * b[i - 1]) / l[i];
    b[n - 1] /= l[n - 1];
    for (int i = n - 2; i >= 0; --i) b[i] = (b[i] - m[i] * b[i + 1]) / l[i];
}
static void cyc_solve(int n, const double* l, const double* m, double c, double* b, double* w) {
    tri_solve(n, l, m, b);
    for (int i = 0; i < n; ++i) w[i] = 0.0;
    w[0] = 1.0;
    w[n - 1] = 1.0;
    tri_solve(n, l, m, w);
    const double tau = c * (b[0] + b[n - 1]) / (1.0 + c * (w[0] + w[n - 1]));
    for (int i = 0; i < n; ++i) b[i] -= tau * w[i];
}

/* Envelope LDL^T, ref line_algebra.cpp:122-255 */
typedef struct { int row, col; double v; } Trip;
typedef struct {
    int n, identity;
    int *perm, *iperm, *fc;
    long* ro;
    double *L, *D;
} Env;

static void env_free(Env* e) {
    free(e->perm); free(e->iperm); free(e->fc); free(e->ro); free(e->L); free(e->D);
    memset(e, 0, sizeof *e);
}

static int env_factor(Env* e, int n, const Trip* tr, int nt, const int* perm) {
    memset(e, 0, sizeof *e);
    e->n = n;
    e->perm = NEWI(n); e->iperm = NEWI(n); e->fc = NEWI(n);
    e->ro = (long*)xcalloc(n + 1, sizeof(long));
    e->identity = 1;
    for (int i = 0; i < n; ++i) {
        e->perm[i] = perm ? perm[i] : i;
        if (e->perm[i] != i) e->identity = 0;
    }
    for (int k = 0; k < n; ++k) e->iperm[e->perm[k]] = k;
    for (int i = 0; i < n; ++i) e->fc[i] = i;
    for (int q = 0; q < nt; ++q) {
        if (tr[q].row < 0 || tr[q].row >= n || tr[q].col < 0 || tr[q].col > tr[q].row)
            return fail(1, "sparse factor: triplets must address the lower triangle");
        const int pi = e->iperm[tr[q].row], pj = e->iperm[tr[q].col];
        const int hi = pi > pj ? pi : pj, lo = pi < pj ? pi : pj;
        if (lo < e->fc[hi]) e->fc[hi] = lo;
    }
    for (int i = 0; i < n; ++i) e->ro[i + 1] = e->ro[i] + (i - e->fc[i]);
    e->L = NEWD(e->ro[n]);
    e->D = NEWD(n);
    char* seen = (char*)xcalloc(n, 1);
    for (int q = 0; q < nt; ++q) {
        const int pi = e->iperm[tr[q].row], pj = e->iperm[tr[q].col];
        if (pi == pj) { e->D[pi] += tr[q].v; seen[pi] = 1; }
        else {
            const int hi = pi > pj ? pi : pj, lo = pi < pj ? pi : pj;
            e->L[e->ro[hi] + (lo - e->fc[hi])] += tr[q].v;
        }
    }
    for (int i = 0; i < n; ++i)
        if (!seen[i]) { free(seen); return fail(2, "sparse factor: structurally singular (missing diagonal at row %d)", e->perm[i]); }
    free(seen);
    double scale = 0.0;
    for (int i = 0; i < n; ++i) if (fabs(e->D[i]) > scale) scale = fabs(e->D[i]);
    for (int i = 0; i < n; ++i) {
        const int fi = e->fc[i];
        double* ri = e->L + e->ro[i] - fi;
        for (int j = fi; j < i; ++j) {
            const int fj = e->fc[j];
            const double* rj = e->L + e->ro[j] - fj;
            const int k0 = fi > fj ? fi : fj;
            double sum = ri[j];
            for (int k = k0; k < j; ++k) sum -= ri[k] * e->D[k] * rj[k];
            ri[j] = sum / e->D[j];
        }
        double d = e->D[i];
        for (int k = fi; k < i; ++k) d -= ri[k] * ri[k] * e->D[k];
        if (fabs(d) < 1e-14 * (scale > 1.0 ? scale : 1.0))
            return fail(2, "sparse factor: zero pivot at row %d", e->perm[i]);
        e->D[i] = d;
    }
    return 0;
}

static void env_solve(const Env* e, double* rhs, double* work) {
    const int n = e->n;
    double* x = rhs;
    if (!e->identity) {
        for (int k = 0; k < n; ++k) work[k] = rhs[e->perm[k]];
        x = work;
    }
    for (int i = 0; i < n; ++i) {
        const int fi = e->fc[i];
        const double* ri = e->L + e->ro[i] - fi;
        double sum = x[i];
        for (int k = fi; k < i; ++k) sum -= ri[k] * x[k];
        x[i] = sum;
    }
    for (int i = 0; i < n; ++i) x[i] /= e->D[i];
    for (int i = n - 1; i >= 0; --i) {
        const int fi = e->fc[i];
        const double* ri = e->L + e->ro[i] - fi;
        const double xi = x[i];
        for (int k = fi; k < i; ++k) x[k] -= ri[k] * xi;
    }
    if (!e->identity)
        for (int k = 0; k < n; ++k) rhs[e->perm[k]] = work[k];
}

/* ----------------------------------------------------------------- level */
typedef struct { int count; int cols[10]; double vals[10]; } Row;

typedef struct {
    Grid g;
    double *sn, *cs, *alpha, *beta;
    double *arr, *art, *att, *det; /* ring-major s*nt+t, level_cache.cpp:44-58 */
    int smoother;                  /* 0 on the coarsest level */
    double **cl, **cm, *cc;        /* circle factors (core LL^T + corner) */
    Env origin;
    double **rl, **rm;             /* radial factors */
    Env direct;
    double *u, *f, *res;
} Level;

typedef struct {
    Geom G;
    Prob P;
    int mode, boundary, pre, post, cycle, norm, max_it;
    double abs_tol, rel_tol, tol;
    int L;
    Level* lv;
    double* work; /* max(nr, nt) scratch */
    int sol;                     /* 1: PolarOscillation manufactured solution */
    int fmg, fmg_it, fmg_cycle;  /* multigrid.hpp:42-45 */
    int ex;                      /* implicit extrapolation (multigrid.hpp:41) */
    int fmg_run;
} Solver;

static int is_dir(const Solver* S, const Level* l, int s) {
    return s == l->g.nr - 1 || (s == 0 && S->boundary == 1);
}

static Coef coef(const Level* l, int s, int t) {
    const size_t i = (size_t)s * l->g.nt + t;
    Coef c = {l->arr[i], l->art[i], l->att[i], l->det[i]};
    return c;
}

static void row_add(Row* r, int col, double v) { r->cols[r->count] = col; r->vals[r->count] = v; r->count++; }

/* ref stencil.cpp:44-137 (build_row) */
static void build_row(const Solver* S, const Level* l, int s, int t, int elim, Row* out) {
    const Grid* g = &l->g;
    const int N = g->nr - 1;
    const int p = gidx(g, s, t);
    out->count = 0;
    if (elim && is_dir(S, l, s)) { row_add(out, p, 1.0); return; }
    const int tm = wrap(g, t - 1), tp = wrap(g, t + 1);
    const double km = k_below(g, t), kp = g->k[t];
    const double hm = s > 0 ? g->h[s - 1] : 0.0, hp = s < N ? g->h[s] : 0.0;
    const double kbar = 0.5 * (km + kp), hbar = 0.5 * (hm + hp);
    const Coef cP = coef(l, s, t), cTM = coef(l, s, tm), cTP = coef(l, s, tp);
    Coef cSM = {0, 0, 0, 0}, cSP = {0, 0, 0, 0};
    if (s > 0) cSM = coef(l, s - 1, t);
    if (s < N) cSP = coef(l, s + 1, t);
    const int origin = s == 0 && S->boundary == 0;
    double diag = 0.0;
    if (s > 0) diag += (kbar / hm) * (cP.arr + cSM.arr);
    if (s < N) diag += (kbar / hp) * (cP.arr + cSP.arr);
    diag += (hbar / km) * (cP.att + cTM.att);
    diag += (hbar / kp) * (cP.att + cTP.att);
    diag += l->beta[s] * cP.det * hbar * kbar;
    double wph = 0.0;
    int t2 = -1;
    if (origin) {
        t2 = wrap(g, t + g->nt / 2);
        const int tlo = t < t2 ? t : t2, thi = t < t2 ? t2 : t;
        const double klo = 0.5 * (k_below(g, tlo) + g->k[tlo]);
        const double khi = 0.5 * (k_below(g, thi) + g->k[thi]);
        const double omega = (klo + khi) / (4.0 * g->r[0]);
        wph = omega * (coef(l, 0, tlo).arr + coef(l, 0, thi).arr);
        diag += wph;
    }
    row_add(out, p, diag);
#define KEEP(ring) (!elim || !is_dir(S, l, (ring)))
    if (s > 0 && KEEP(s - 1)) row_add(out, gidx(g, s - 1, t), -(kbar / hm) * (cP.arr + cSM.arr));
    if (s < N && KEEP(s + 1)) row_add(out, gidx(g, s + 1, t), -(kbar / hp) * (cP.arr + cSP.arr));
    {
        double south = -(hbar / km) * (cP.att + cTM.att);
        double north = -(hbar / kp) * (cP.att + cTP.att);
        if (s == 0) {
            south += (cP.art - cTM.art) * 0.25;
            north += (cTP.art - cP.art) * 0.25;
        } else if (s == N) {
            south += (cTM.art - cP.art) * 0.25;
            north += (cP.art - cTP.art) * 0.25;
        }
        row_add(out, gidx(g, s, tm), south);
        row_add(out, gidx(g, s, tp), north);
    }
    if (s > 0 && KEEP(s - 1)) {
        row_add(out, gidx(g, s - 1, tm), -(cTM.art + cSM.art) * 0.25);
        row_add(out, gidx(g, s - 1, tp), (cSM.art + cTP.art) * 0.25);
    }
    if (s < N && KEEP(s + 1)) {
        row_add(out, gidx(g, s + 1, tm), (cTM.art + cSP.art) * 0.25);
        row_add(out, gidx(g, s + 1, tp), -(cSP.art + cTP.art) * 0.25);
    }
#undef KEEP
    if (origin) row_add(out, gidx(g, 0, t2), -wph);
}

static double row_at(const Row* r, int col) {
    for (int i = 0; i < r->count; ++i) if (r->cols[i] == col) return r->vals[i];
    return 0.0;
}

/* ref stencil.cpp:161-174 */
static void apply_take(const Solver* S, const Level* l, const double* u, double* y) {
    Row r;
    for (int s = 0; s < l->g.nr; ++s)
        for (int t = 0; t < l->g.nt; ++t) {
            build_row(S, l, s, t, 1, &r);
            double acc = 0.0;
            for (int i = 0; i < r.count; ++i) acc += r.vals[i] * u[r.cols[i]];
            y[gidx(&l->g, s, t)] = acc;
        }
}

/* ref stencil.cpp:176-272 (scatter_ring) */
static void scatter_ring(const Solver* S, const Level* l, int s, const double* u, double* y) {
    const Grid* g = &l->g;
    const int N = g->nr - 1, nt = g->nt;
    const double hm = s > 0 ? g->h[s - 1] : 0.0, hp = s < N ? g->h[s] : 0.0;
    const double hbar = 0.5 * (hm + hp);
    const int pD = is_dir(S, l, s);
    const int smD = s > 0 && is_dir(S, l, s - 1);
    const int spD = s < N && is_dir(S, l, s + 1);
    const double beta_s = l->beta[s];
    for (int t = 0; t < nt; ++t) {
        const int p = gidx(g, s, t);
        const int tm = wrap(g, t - 1), tp = wrap(g, t + 1);
        const double km = k_below(g, t), kp = g->k[t];
        const double kbar = 0.5 * (km + kp);
        const Coef cP = coef(l, s, t);
        if (pD) {
            y[p] = u[p];
            for (int side = 0; side < 2; ++side) {
                const int inward = side == 0;
                if (inward ? s == 0 : s == N) continue;
                const int q = inward ? gidx(g, s - 1, t) : gidx(g, s + 1, t);
                if (inward ? smD : spD) continue;
                y[q] += (kbar / (inward ? hm : hp)) * cP.arr * u[q];
            }
            continue;
        }
        y[p] += beta_s * cP.det * hbar * kbar * u[p];
        for (int side = 0; side < 2; ++side) {
            const int inward = side == 0;
            if (inward ? s == 0 : s == N) continue;
            const int q = inward ? gidx(g, s - 1, t) : gidx(g, s + 1, t);
            const int qD = inward ? smD : spD;
            const double w = (kbar / (inward ? hm : hp)) * cP.arr;
            y[p] += w * u[p];
            if (!qD) {
                y[p] -= w * u[q];
                y[q] += w * u[q];
                y[q] -= w * u[p];
            }
        }
        for (int side = 0; side < 2; ++side) {
            const int q = gidx(g, s, side == 0 ? tm : tp);
            const double w = (hbar / (side == 0 ? km : kp)) * cP.att;
            y[p] += w * (u[p] - u[q]);
            y[q] += w * (u[q] - u[p]);
        }
        for (int rho = 0; rho < 2; ++rho) {
            const int below = rho == 0;
            if (below ? s == 0 : s == N) continue;
            for (int tau = 0; tau < 2; ++tau) {
                const int left = tau == 1;
                const double sigma = (below != left) ? 1.0 : -1.0;
                const int R = below ? gidx(g, s - 1, t) : gidx(g, s + 1, t);
                const int RD = below ? smD : spD;
                const int T = gidx(g, s, left ? tp : tm);
                const double v = sigma * cP.art * 0.25;
                y[p] += 2.0 * v * u[p];
                if (!RD) {
                    y[p] -= v * u[R];
                    y[R] -= v * u[p];
                    y[R] += v * u[T];
                }
                y[p] -= v * u[T];
                y[T] -= v * u[p];
                if (!RD) y[T] += v * u[R];
            }
        }
    }
    if (s == 0 && S->boundary == 0) { /* phantom edges, stencil.cpp:440-456 */
        const int half = nt / 2;
        for (int t = 0; t < half; ++t) {
            const int t2 = t + half;
            const double klo = 0.5 * (k_below(g, t) + g->k[t]);
            const double khi = 0.5 * (k_below(g, t2) + g->k[t2]);
            const double omega = (klo + khi) / (4.0 * g->r[0]);
            const double w = omega * (coef(l, 0, t).arr + coef(l, 0, t2).arr);
            const int p = gidx(g, 0, t), q = gidx(g, 0, t2);
            y[p] += w * (u[p] - u[q]);
            y[q] += w * (u[q] - u[p]);
        }
    }
}

/* ref stencil.cpp:274-287 */
static void apply_give(const Solver* S, const Level* l, const double* u, double* y) {
    const int n = l->g.nr * l->g.nt;
    for (int i = 0; i < n; ++i) y[i] = 0.0;
    for (int phase = 0; phase < 3; ++phase) {
        const int count = (l->g.nr - phase + 2) / 3;
        for (int i = 0; i < count; ++i) scatter_ring(S, l, phase + 3 * i, u, y);
    }
}

static void apply_op(const Solver* S, const Level* l, int mode, const double* u, double* y) {
    if (mode == 0) apply_take(S, l, u, y); else apply_give(S, l, u, y);
}

/* ref stencil.cpp:289-295 */
static void residual(const Solver* S, const Level* l, int mode, const double* u, const double* f, double* r) {
    apply_op(S, l, mode, u, r);
    const int n = l->g.nr * l->g.nt;
    for (int i = 0; i < n; ++i) r[i] = f[i] - r[i];
}

/* ref stencil.cpp:355-373 */
static Trip* assemble_coo(const Solver* S, const Level* l, const int* nodes, int nn, int* count) {
    const int n = l->g.nr * l->g.nt;
    int* local = NEWI(n);
    for (int i = 0; i < n; ++i) local[i] = -1;
    for (int i = 0; i < nn; ++i) local[nodes[i]] = i;
    Trip* tr = (Trip*)xcalloc((size_t)nn * 10, sizeof(Trip));
    int c = 0;
    Row r;
    for (int i = 0; i < nn; ++i) {
        int s, t;
        gnode(&l->g, nodes[i], &s, &t);
        build_row(S, l, s, t, 1, &r);
        for (int e = 0; e < r.count; ++e) {
            const int lc = local[r.cols[e]];
            if (lc >= 0 && lc <= i) { tr[c].row = i; tr[c].col = lc; tr[c].v = r.vals[e]; ++c; }
        }
    }
    free(local);
    *count = c;
    return tr;
}

/* -------------------------------------------------------------- smoother */
/* ctor: ref smoother.cpp:18-68; lines: stencil.cpp:375-409 */
static int smoother_init(const Solver* S, Level* l) {
    const Grid* g = &l->g;
    if (!g->uniform_angles)
        return fail(2, "smoother split undefined: non-uniform angular spacing; a more general "
                       "switching condition or overlapping smoothers would be needed");
    const int nt = g->nt, split = g->split;
    l->cl = (double**)xcalloc(split, sizeof(double*));
    l->cm = (double**)xcalloc(split, sizeof(double*));
    l->cc = NEWD(split);
    double* diag = NEWD(nt > g->nr ? nt : g->nr);
    double* off = NEWD(nt > g->nr ? nt : g->nr);
    Row r;
    int rc = 0;
    for (int s = 0; s < split && !rc; ++s) {
        if (s == 0 && S->boundary == 0) {
            int* nodes = NEWI(nt);
            for (int t = 0; t < nt; ++t) nodes[t] = t;
            int ntr;
            Trip* tr = assemble_coo(S, l, nodes, nt, &ntr);
            int* perm = NEWI(nt);
            for (int i = 0; i < nt / 2; ++i) { perm[2 * i] = i; perm[2 * i + 1] = nt / 2 + i; }
            rc = env_factor(&l->origin, nt, tr, ntr, perm);
            free(nodes); free(tr); free(perm);
            continue;
        }
        double corner = 0.0;
        for (int t = 0; t < nt; ++t) {
            build_row(S, l, s, t, 1, &r);
            diag[t] = row_at(&r, gidx(g, s, t));
            if (t < nt - 1) off[t] = row_at(&r, gidx(g, s, t + 1));
            else corner = row_at(&r, gidx(g, s, 0));
        }
        if (nt < 3) { rc = fail(1, "cyclic_tridiag_factor: need n >= 3 (corner would duplicate a band)"); break; }
        diag[0] -= corner;
        diag[nt - 1] -= corner;
        l->cl[s] = NEWD(nt);
        l->cm[s] = NEWD(nt);
        l->cc[s] = corner;
        if ((rc = tri_factor(nt, diag, off, l->cl[s], l->cm[s]))) {
            char why[600];
            snprintf(why, sizeof why, "%s", g_err);
            rc = fail(2, "cyclic core not positive definite after rank-one shift: %s", why);
        }
    }
    if (!rc && split < g->nr) {
        const int len = g->nr - split;
        l->rl = (double**)xcalloc(nt, sizeof(double*));
        l->rm = (double**)xcalloc(nt, sizeof(double*));
        for (int t = 0; t < nt && !rc; ++t) {
            for (int i = 0; i < len; ++i) {
                const int s = split + i;
                build_row(S, l, s, t, 1, &r);
                diag[i] = row_at(&r, gidx(g, s, t));
                if (i < len - 1) off[i] = row_at(&r, gidx(g, s + 1, t));
            }
            l->rl[t] = NEWD(len);
            l->rm[t] = NEWD(len);
            rc = tri_factor(len, diag, off, l->rl[t], l->rm[t]);
        }
    }
    free(diag);
    free(off);
    l->smoother = 1;
    return rc;
}

/* ref smoother.cpp:162-182 */
static void take_rhs_circle(const Solver* S, const Level* l, int s, double* u, const double* f, int ex) {
    const int nt = l->g.nt, base = s * nt;
    if (is_dir(S, l, s)) { for (int t = 0; t < nt; ++t) u[base + t] = f[base + t]; return; }
    Row r;
    for (int t = 0; t < nt; ++t) {
        const int p = base + t;
        build_row(S, l, s, t, 1, &r);
        double acc = ex ? 0.75 * f[p] : f[p];
        for (int i = 0; i < r.count; ++i) {
            const int c = r.cols[i];
            if (c >= base && c < base + nt) continue;
            acc -= r.vals[i] * u[c];
        }
        u[p] = acc;
    }
}

/* ref smoother.cpp:184-205 */
static void take_rhs_radial(const Solver* S, const Level* l, int t, double* u, const double* f, int ex) {
    const int split = l->g.split, len = l->g.nr - split, base = split * l->g.nt + t * len;
    Row r;
    for (int i = 0; i < len; ++i) {
        const int s = split + i, p = base + i;
        if (is_dir(S, l, s)) { u[p] = f[p]; continue; }
        build_row(S, l, s, t, 1, &r);
        double acc = ex ? 0.75 * f[p] : f[p];
        for (int e = 0; e < r.count; ++e) {
            const int c = r.cols[e];
            if (c >= base && c < base + len) continue;
            acc -= r.vals[e] * u[c];
        }
        u[p] = acc;
    }
}

/* ref smoother.cpp:220-302 */
static void give_rhs_circle(const Solver* S, const Level* l, int parity, double* u, const double* f) {
    const Grid* g = &l->g;
    const int nt = g->nt, N = g->nr - 1, split = g->split;
    const int targets = split > parity ? (split - parity + 1) / 2 : 0;
    for (int i = 0; i < targets; ++i) {
        const int s = parity + 2 * i, base = s * nt;
        if (is_dir(S, l, s)) { for (int t = 0; t < nt; ++t) u[base + t] = f[base + t]; continue; }
        const double hm = s > 0 ? g->h[s - 1] : 0.0, hp = s < N ? g->h[s] : 0.0;
        const int in_ok = s > 0 && !is_dir(S, l, s - 1);
        const int out_ok = s < N && !is_dir(S, l, s + 1);
        for (int t = 0; t < nt; ++t) u[base + t] = f[base + t];
        for (int t = 0; t < nt; ++t) {
            const int tm = t == 0 ? nt - 1 : t - 1, tp = t + 1 == nt ? 0 : t + 1;
            const double kbar = 0.5 * (k_below(g, t) + g->k[t]);
            const Coef cP = coef(l, s, t);
            const double v = 0.25 * cP.art;
            if (in_ok) {
                const double ur = u[gidx(g, s - 1, t)];
                u[base + t] += (kbar / hm) * cP.arr * ur;
                u[base + tp] += v * ur;
                u[base + tm] -= v * ur;
            }
            if (out_ok) {
                const double ur = u[gidx(g, s + 1, t)];
                u[base + t] += (kbar / hp) * cP.arr * ur;
                u[base + tp] -= v * ur;
                u[base + tm] += v * ur;
            }
        }
    }
    const int max_source = split < N ? split : N;
    for (int group = 0; group < 2; ++group) {
        const int first = (parity + 1 + 2 * group) % 4;
        const int count = max_source >= first ? (max_source - first) / 4 + 1 : 0;
        for (int i = 0; i < count; ++i) {
            const int sq = first + 4 * i;
            if (is_dir(S, l, sq)) continue;
            const int in_t = sq > 0 && sq - 1 < split && !is_dir(S, l, sq - 1);
            const int out_t = sq + 1 < split && !is_dir(S, l, sq + 1);
            if (!in_t && !out_t) continue;
            const double hm = sq > 0 ? g->h[sq - 1] : 0.0, hp = sq < N ? g->h[sq] : 0.0;
            for (int tc = 0; tc < nt; ++tc) {
                const int tm = tc == 0 ? nt - 1 : tc - 1, tp = tc + 1 == nt ? 0 : tc + 1;
                const double kbar = 0.5 * (k_below(g, tc) + g->k[tc]);
                const Coef cS = coef(l, sq, tc);
                const double uc = u[gidx(g, sq, tc)];
                const double v = 0.25 * cS.art;
                if (in_t) {
                    const int q = gidx(g, sq - 1, tc);
                    u[q] += (kbar / hm) * cS.arr * uc;
                    u[q] += v * u[gidx(g, sq, tp)];
                    u[q] -= v * u[gidx(g, sq, tm)];
                }
                if (out_t) {
                    const int q = gidx(g, sq + 1, tc);
                    u[q] += (kbar / hp) * cS.arr * uc;
                    u[q] -= v * u[gidx(g, sq, tp)];
                    u[q] += v * u[gidx(g, sq, tm)];
                }
            }
        }
    }
}

/* ref smoother.cpp:304-396 */
static void give_rhs_radial(const Solver* S, const Level* l, int parity, double* u, const double* f) {
    const Grid* g = &l->g;
    const int nt = g->nt, N = g->nr - 1, split = g->split, len = g->nr - split;
    const int region = split * nt;
    const int targets = (nt - parity + 1) / 2;
    for (int i = 0; i < targets; ++i) {
        const int t = parity + 2 * i, base = region + t * len;
        const int tm = t == 0 ? nt - 1 : t - 1, tp = t + 1 == nt ? 0 : t + 1;
        const double km = k_below(g, t), kp = g->k[t], kbar = 0.5 * (km + kp);
        for (int j = 0; j < len; ++j) u[base + j] = f[base + j];
        for (int j = 0; j < len; ++j) {
            const int s = split + j;
            if (is_dir(S, l, s)) continue;
            const double hm = g->h[s - 1], hp = s < N ? g->h[s] : 0.0, hbar = 0.5 * (hm + hp);
            const Coef cP = coef(l, s, t);
            const double v = 0.25 * cP.art;
            u[base + j] += (hbar / km) * cP.att * u[gidx(g, s, tm)];
            u[base + j] += (hbar / kp) * cP.att * u[gidx(g, s, tp)];
            if (s == split && !is_dir(S, l, split - 1))
                u[base + j] += (kbar / hm) * cP.arr * u[gidx(g, split - 1, t)];
            if (s > split && !is_dir(S, l, s - 1)) {
                u[base + j - 1] += v * u[gidx(g, s, tp)];
                u[base + j - 1] -= v * u[gidx(g, s, tm)];
            }
            if (s < N && !is_dir(S, l, s + 1)) {
                u[base + j + 1] -= v * u[gidx(g, s, tp)];
                u[base + j + 1] += v * u[gidx(g, s, tm)];
            }
        }
        if (!is_dir(S, l, split) && !is_dir(S, l, split - 1)) {
            const Coef c2 = coef(l, split - 1, t);
            const double v2 = 0.25 * c2.art;
            u[base] += (kbar / g->h[split - 1]) * c2.arr * u[gidx(g, split - 1, t)];
            u[base] += v2 * u[gidx(g, split - 1, tm)];
            u[base] -= v2 * u[gidx(g, split - 1, tp)];
        }
    }
    for (int group = 0; group < 2; ++group) {
        const int first = (parity + 1 + 2 * group) % 4;
        const int count = nt > first ? (nt - 1 - first) / 4 + 1 : 0;
        for (int i = 0; i < count; ++i) {
            const int tq = first + 4 * i;
            const int tm = tq == 0 ? nt - 1 : tq - 1, tp = tq + 1 == nt ? 0 : tq + 1;
            const double km = k_below(g, tq), kp = g->k[tq];
            const int bq = region + tq * len, bm = region + tm * len, bp = region + tp * len;
            for (int j = 0; j < len; ++j) {
                const int s = split + j;
                if (is_dir(S, l, s)) continue;
                const double hm = g->h[s - 1], hp = s < N ? g->h[s] : 0.0, hbar = 0.5 * (hm + hp);
                const Coef cS = coef(l, s, tq);
                const double uc = u[bq + j];
                const double v = 0.25 * cS.art;
                u[bp + j] += (hbar / kp) * cS.att * uc;
                u[bm + j] += (hbar / km) * cS.att * uc;
                if (!is_dir(S, l, s - 1)) {
                    const double ub = u[gidx(g, s - 1, tq)];
                    u[bp + j] += v * ub;
                    u[bm + j] -= v * ub;
                }
                if (s < N && !is_dir(S, l, s + 1)) {
                    const double ua = u[gidx(g, s + 1, tq)];
                    u[bp + j] -= v * ua;
                    u[bm + j] += v * ua;
                }
            }
        }
    }
}

/* ref smoother.cpp:95-152 */
static void sweep_circle_x(const Solver* S, const Level* l, int parity, double* u, const double* f, double* w, int ex) {
    const int take = ex || S->mode == 0;
    if (!take) give_rhs_circle(S, l, parity, u, f);
    const int split = l->g.split, nt = l->g.nt;
    const int lines = split > parity ? (split - parity + 1) / 2 : 0;
    for (int i = 0; i < lines; ++i) {
        const int s = parity + 2 * i;
        if (take) take_rhs_circle(S, l, s, u, f, ex);
        if (s == 0 && S->boundary == 0) env_solve(&l->origin, u, w);
        else cyc_solve(nt, l->cl[s], l->cm[s], l->cc[s], u + s * nt, w);
    }
}

static void sweep_radial_x(const Solver* S, const Level* l, int parity, double* u, const double* f, int ex) {
    const int take = ex || S->mode == 0;
    if (!take) give_rhs_radial(S, l, parity, u, f);
    const int nt = l->g.nt, split = l->g.split, len = l->g.nr - split;
    const int lines = (nt - parity + 1) / 2;
    for (int i = 0; i < lines; ++i) {
        const int t = parity + 2 * i;
        if (take) take_rhs_radial(S, l, t, u, f, ex);
        tri_solve(len, l->rl[t], l->rm[t], u + split * nt + t * len);
    }
}

static void sweep_circle(const Solver* S, const Level* l, int parity, double* u, const double* f, double* w) {
    sweep_circle_x(S, l, parity, u, f, w, 0);
}
static void sweep_radial(const Solver* S, const Level* l, int parity, double* u, const double* f) {
    sweep_radial_x(S, l, parity, u, f, 0);
}

/* ref smoother.cpp:400-465: fine-only nodes of even circle rings (odd t),
 * then of even spokes (odd rings), pointwise with 3/4 f */
static void extrapolated_pointwise(const Solver* S, const Level* l, double* u, const double* fhat) {
    const Grid* g = &l->g;
    const int nt = g->nt, N = g->nr - 1, split = g->split;
    const int origin_pairs = S->boundary == 0;
    const int even_rings = (split + 1) / 2;
    Row r;
    for (int i = 0; i < even_rings; ++i) {
        const int s = 2 * i;
        if (s == 0 && origin_pairs) continue;
        const int base = s * nt;
        if (is_dir(S, l, s)) {
            for (int t = 1; t < nt; t += 2) u[base + t] = fhat[base + t];
            continue;
        }
        for (int t = 1; t < nt; t += 2) {
            const int p = base + t;
            build_row(S, l, s, t, 1, &r);
            double diag = 1.0;
            double acc = 0.75 * fhat[p];
            for (int e = 0; e < r.count; ++e) {
                if (r.cols[e] == p) diag = r.vals[e];
                else acc -= r.vals[e] * u[r.cols[e]];
            }
            u[p] = acc / diag;
        }
    }
    if (split < g->nr) {
        const int len = g->nr - split;
        const int spokes = (nt + 1) / 2;
        for (int i = 0; i < spokes; ++i) {
            const int t = 2 * i;
            for (int s = split % 2 == 0 ? split + 1 : split; s <= N; s += 2) {
                const int p = split * nt + t * len + (s - split);
                if (is_dir(S, l, s)) { u[p] = fhat[p]; continue; }
                build_row(S, l, s, t, 1, &r);
                double diag = 1.0;
                double acc = 0.75 * fhat[p];
                for (int e = 0; e < r.count; ++e) {
                    if (r.cols[e] == p) diag = r.vals[e];
                    else acc -= r.vals[e] * u[r.cols[e]];
                }
                u[p] = acc / diag;
            }
        }
    }
}

/* ref smoother.cpp:467-503: antipodal fine-only pairs of the origin ring */
static void extrapolated_origin_pairs(const Solver* S, const Level* l, double* u, const double* fhat) {
    const Grid* g = &l->g;
    const int nt = g->nt, half = nt / 2;
    Row r;
    for (int i = 0; i < half / 2; ++i) {
        const int t = 2 * i + 1, t2 = t + half;
        const int p = gidx(g, 0, t), q = gidx(g, 0, t2);
        double a11 = 1.0, a12 = 0.0, a21 = 0.0, a22 = 1.0, b1, b2;
        build_row(S, l, 0, t, 1, &r);
        b1 = 0.75 * fhat[p];
        for (int e = 0; e < r.count; ++e) {
            const int c = r.cols[e];
            if (c == p) a11 = r.vals[e];
            else if (c == q) a12 = r.vals[e];
            else b1 -= r.vals[e] * u[c];
        }
        build_row(S, l, 0, t2, 1, &r);
        b2 = 0.75 * fhat[q];
        for (int e = 0; e < r.count; ++e) {
            const int c = r.cols[e];
            if (c == q) a22 = r.vals[e];
            else if (c == p) a21 = r.vals[e];
            else b2 -= r.vals[e] * u[c];
        }
        const double det = a11 * a22 - a12 * a21;
        u[p] = (b1 * a22 - a12 * b2) / det;
        u[q] = (a11 * b2 - a21 * b1) / det;
    }
}

/* ref smoother.cpp:83-91 */
static void smooth_extrapolated(const Solver* S, const Level* l, double* u, const double* fhat) {
    sweep_circle_x(S, l, 1, u, fhat, S->work, 1);
    if (l->g.split < l->g.nr) sweep_radial_x(S, l, 1, u, fhat, 1);
    extrapolated_pointwise(S, l, u, fhat);
    if (S->boundary == 0) extrapolated_origin_pairs(S, l, u, fhat);
}

/* ref smoother.cpp:72-81 */
static void smooth(const Solver* S, const Level* l, double* u, const double* f) {
    sweep_circle(S, l, 0, u, f, S->work);
    sweep_circle(S, l, 1, u, f, S->work);
    if (l->g.split < l->g.nr) {
        sweep_radial(S, l, 0, u, f);
        sweep_radial(S, l, 1, u, f);
    }
}

/* ------------------------------------------------------------- transfers */
/* ref interpolation.cpp:19-143 */
static double rw_below(const Grid* f, int sf) { return f->h[sf] / (f->h[sf - 1] + f->h[sf]); }
static double rw_above(const Grid* f, int sf) { return f->h[sf - 1] / (f->h[sf - 1] + f->h[sf]); }
static double aw_below(const Grid* f, int tf) { return f->k[tf] / (f->k[tf - 1] + f->k[tf]); }
static double aw_above(const Grid* f, int tf) { return f->k[tf - 1] / (f->k[tf - 1] + f->k[tf]); }

static void prolongate(const Grid* fine, const Grid* coarse, const double* cu, double* fu, int add) {
    const int ntc = coarse->nt;
    for (int sf = 0; sf < fine->nr; ++sf) {
        const int ro = sf & 1, sc = sf / 2;
        for (int tf = 0; tf < fine->nt; ++tf) {
            const int so = tf & 1, tc = tf / 2, tcu = (tc + 1) % ntc;
            double v;
            if (!ro && !so) v = cu[gidx(coarse, sc, tc)];
            else if (ro && !so)
                v = rw_below(fine, sf) * cu[gidx(coarse, sc, tc)] + rw_above(fine, sf) * cu[gidx(coarse, sc + 1, tc)];
            else if (!ro && so)
                v = aw_below(fine, tf) * cu[gidx(coarse, sc, tc)] + aw_above(fine, tf) * cu[gidx(coarse, sc, tcu)];
            else {
                const double wb = rw_below(fine, sf), wa = rw_above(fine, sf);
                const double vb = aw_below(fine, tf), va = aw_above(fine, tf);
                v = wb * vb * cu[gidx(coarse, sc, tc)] + wb * va * cu[gidx(coarse, sc, tcu)] +
                    wa * vb * cu[gidx(coarse, sc + 1, tc)] + wa * va * cu[gidx(coarse, sc + 1, tcu)];
            }
            const int p = gidx(fine, sf, tf);
            if (add) fu[p] += v; else fu[p] = v;
        }
    }
}

static void restrict_t(const Grid* fine, const Grid* coarse, const double* fr, double* cr) {
    const int nr = fine->nr, nt = fine->nt;
    for (int sc = 0; sc < coarse->nr; ++sc) {
        const int sf = 2 * sc;
        for (int tc = 0; tc < coarse->nt; ++tc) {
            const int tf = 2 * tc, tdn = tf == 0 ? nt - 1 : tf - 1, tup = tf + 1;
            double acc = fr[gidx(fine, sf, tf)];
            if (sf > 0) acc += rw_above(fine, sf - 1) * fr[gidx(fine, sf - 1, tf)];
            if (sf < nr - 1) acc += rw_below(fine, sf + 1) * fr[gidx(fine, sf + 1, tf)];
            acc += aw_above(fine, tdn) * fr[gidx(fine, sf, tdn)];
            acc += aw_below(fine, tup) * fr[gidx(fine, sf, tup)];
            if (sf > 0) {
                acc += rw_above(fine, sf - 1) * aw_above(fine, tdn) * fr[gidx(fine, sf - 1, tdn)];
                acc += rw_above(fine, sf - 1) * aw_below(fine, tup) * fr[gidx(fine, sf - 1, tup)];
            }
            if (sf < nr - 1) {
                acc += rw_below(fine, sf + 1) * aw_above(fine, tdn) * fr[gidx(fine, sf + 1, tdn)];
                acc += rw_below(fine, sf + 1) * aw_below(fine, tup) * fr[gidx(fine, sf + 1, tup)];
            }
            cr[gidx(coarse, sc, tc)] = acc;
        }
    }
}

/* ------------------------------------------------------------- multigrid */
/* ref multigrid.cpp:48-59 */
/* ref interpolation.cpp:145-165 */
static void inject(const Grid* fine, const Grid* coarse, const double* fu, double* cu) {
    for (int sc = 0; sc < coarse->nr; ++sc)
        for (int tc = 0; tc < coarse->nt; ++tc)
            cu[gidx(coarse, sc, tc)] = fu[gidx(fine, 2 * sc, 2 * tc)];
}
static void inject_transpose_add(const Grid* fine, const Grid* coarse, const double* cu, double* fu) {
    for (int sc = 0; sc < coarse->nr; ++sc)
        for (int tc = 0; tc < coarse->nt; ++tc)
            fu[gidx(fine, 2 * sc, 2 * tc)] += cu[gidx(coarse, sc, tc)];
}

double orc_norm(int type, const double* v, long n) {
    if (type == 2) {
        double m = 0.0;
        for (long i = 0; i < n; ++i) if (fabs(v[i]) > m) m = fabs(v[i]);
        return m;
    }
    double acc = 0.0;
    for (long i = 0; i < n; ++i) acc += v[i] * v[i];
    return type == 0 ? sqrt(acc / (double)n) : sqrt(acc);
}

/* ------------------------------------------- manufactured solution / RHS */
/* PolarOscillation, ref problem.cpp:48-72 (rmax = ProblemCase rmax) */
static double sol_u(double rmax, double r, double th) {
    const double rho = r / rmax;
    const double a = rho * rho * rho;
    const double omr = 1.0 - rho;
    const double b = omr * omr * omr;
    return 0.4096 * (a * a) * (b * b) * cos(11.0 * th);
}
static double sol_ur(double rmax, double r, double th) {
    const double rho = r / rmax;
    const double rho5 = rho * rho * rho * rho * rho;
    const double omr = 1.0 - rho;
    const double omr5 = omr * omr * omr * omr * omr;
    return 0.4096 * 6.0 * rho5 * omr5 * (1.0 - 2.0 * rho) * cos(11.0 * th) / rmax;
}
static double sol_ut(double rmax, double r, double th) {
    const double rho = r / rmax;
    const double a = rho * rho * rho;
    const double omr = 1.0 - rho;
    const double b = omr * omr * omr;
    return -11.0 * 0.4096 * (a * a) * (b * b) * sin(11.0 * th);
}
/* ref problem.cpp:104-106 */
static double dirichlet_u(const Solver* S, double r, double th) {
    return S->sol ? sol_u(S->P.rmax, r, th) : 0.0;
}
/* logical fluxes of rhs_f, ref problem.cpp:126-133 */
static int flux_r(const Solver* S, double rr, double tt, double* out) {
    Coef tc;
    const int rc = transform(&S->G, p_alpha(&S->P, rr), rr, sin(tt), cos(tt), &tc);
    if (rc) return rc;
    *out = 2.0 * tc.arr * sol_ur(S->P.rmax, rr, tt) + tc.art * sol_ut(S->P.rmax, rr, tt);
    return 0;
}
static int flux_t(const Solver* S, double rr, double tt, double* out) {
    Coef tc;
    const int rc = transform(&S->G, p_alpha(&S->P, rr), rr, sin(tt), cos(tt), &tc);
    if (rc) return rc;
    *out = tc.art * sol_ur(S->P.rmax, rr, tt) + 2.0 * tc.att * sol_ut(S->P.rmax, rr, tt);
    return 0;
}
/* ProblemCase::rhs_f, ref problem.cpp:108-148: fourth-order central
 * differences (diff4, :99-103) of the fluxes, Richardson step halving */
static int rhs_f(const Solver* S, double r, double th, double* out) {
    if (!S->sol) { *out = 0.0; return 0; }
    if (r <= 0.0) return fail(1, "rhs_f requires r > 0");
    const double rmax = S->P.rmax;
    const double a = 1e-4 * rmax, b = r / 3.0;
    const double er = b < a ? b : a;
    const double et = 1e-4 * TWO_PI;
    Coef c0;
    int rc = transform(&S->G, 1.0, r, sin(th), cos(th), &c0);
    if (rc) return rc;
    const double det_abs = c0.det;
    const double bu = p_beta(&S->P, r) * sol_u(rmax, r, th);
    double fs[2];
    for (int k = 0; k < 2; ++k) {
        const double scale = k == 0 ? 1.0 : 0.5;
        double g[4], q[4];
        const double e = er * scale, f = et * scale;
        const double xs[4] = {r - 2.0 * e, r - e, r + e, r + 2.0 * e};
        const double ts[4] = {th - 2.0 * f, th - f, th + f, th + 2.0 * f};
        for (int j = 0; j < 4; ++j) {
            if ((rc = flux_r(S, xs[j], th, &g[j]))) return rc;
            if ((rc = flux_t(S, r, ts[j], &q[j]))) return rc;
        }
        const double d_r = (g[0] - 8.0 * g[1] + 8.0 * g[2] - g[3]) / (12.0 * e);
        const double d_t = (q[0] - 8.0 * q[1] + 8.0 * q[2] - q[3]) / (12.0 * f);
        fs[k] = (-d_r - d_t) / det_abs + bu;
    }
    if (fabs(fs[0] - fs[1]) > 1e-7)
        return fail(2, "rhs_f lost accuracy: Richardson step-halving check disagrees by more than 1e-7");
    *out = (16.0 * fs[1] - fs[0]) / 15.0;
    return 0;
}
/* ref stencil.cpp:297-305 */
static double node_weight(const Grid* g, int s, int t) {
    const int N = g->nr - 1;
    const double hm = s > 0 ? g->h[s - 1] : 0.0;
    const double hp = s < N ? g->h[s] : 0.0;
    const double km = k_below(g, t);
    const double kp = g->k[t];
    return 0.5 * (hm + hp) * 0.5 * (km + kp);
}
/* DiscreteOperator::assemble_rhs_raw + assemble_rhs (Dirichlet lifting),
 * ref stencil.cpp:307-353 */
static int assemble_rhs(const Solver* S, const Level* l, double* b) {
    const Grid* g = &l->g;
    const int N = g->nr - 1;
    for (int s = 0; s < g->nr; ++s)
        for (int t = 0; t < g->nt; ++t) {
            double f;
            const int rc = rhs_f(S, g->r[s], g->th[t], &f);
            if (rc) return rc;
            b[gidx(g, s, t)] = f * coef(l, s, t).det * node_weight(g, s, t);
        }
    for (int s = 0; s < g->nr; ++s) {
        const int lift = (s > 0 && is_dir(S, l, s - 1)) || (s < N && is_dir(S, l, s + 1));
        if (!is_dir(S, l, s) && !lift) continue;
        for (int t = 0; t < g->nt; ++t) {
            const int p = gidx(g, s, t);
            if (is_dir(S, l, s)) {
                b[p] = dirichlet_u(S, g->r[s], g->th[t]);
                continue;
            }
            Row r;
            build_row(S, l, s, t, 0, &r);
            for (int i = 0; i < r.count; ++i) {
                int cs, ct;
                gnode(g, r.cols[i], &cs, &ct);
                if (!is_dir(S, l, cs)) continue;
                b[p] -= r.vals[i] * dirichlet_u(S, g->r[cs], g->th[ct]);
            }
        }
    }
    return 0;
}
/* ref multigrid.cpp:133-143 */
static void set_dirichlet_rows(const Solver* S, const Level* l, double* u) {
    const Grid* g = &l->g;
    const int N = g->nr - 1;
    for (int t = 0; t < g->nt; ++t) u[gidx(g, N, t)] = dirichlet_u(S, g->r[N], g->th[t]);
    if (S->boundary == 1)
        for (int t = 0; t < g->nt; ++t) u[gidx(g, 0, t)] = dirichlet_u(S, g->r[0], g->th[t]);
}

/* ref multigrid.cpp:145-153 */
static void mask_dirichlet(const Solver* S, const Level* l, double* v) {
    const int N = l->g.nr - 1;
    for (int t = 0; t < l->g.nt; ++t) v[gidx(&l->g, N, t)] = 0.0;
    if (S->boundary == 1)
        for (int t = 0; t < l->g.nt; ++t) v[gidx(&l->g, 0, t)] = 0.0;
}

/* ref multigrid.cpp:224-248: r = fhat - (4/3 A0 u - I^T (1/3) A1 I u), Dirichlet rows f - u */
static void extrapolated_residual(Solver* S, double* out) {
    Level* l0 = &S->lv[0];
    Level* l1 = &S->lv[1];
    const Grid* g0 = &l0->g;
    const long n0 = (long)g0->nr * g0->nt, n1 = (long)l1->g.nr * l1->g.nt;
    apply_op(S, l0, S->mode, l0->u, out);
    inject(g0, &l1->g, l0->u, l1->u);
    apply_op(S, l1, S->mode, l1->u, l1->res);
    for (long p = 0; p < n0; ++p) out[p] = l0->f[p] - (4.0 / 3.0) * out[p];
    for (long p = 0; p < n1; ++p) l1->res[p] *= 1.0 / 3.0;
    inject_transpose_add(g0, &l1->g, l1->res, out);
    const int N = g0->nr - 1;
    for (int t = 0; t < g0->nt; ++t) {
        const int p = gidx(g0, N, t);
        out[p] = l0->f[p] - l0->u[p];
    }
    if (S->boundary == 1)
        for (int t = 0; t < g0->nt; ++t) {
            const int p = gidx(g0, 0, t);
            out[p] = l0->f[p] - l0->u[p];
        }
}

/* ref multigrid.cpp:159-168: fhat = 4/3 f0 - I^T (1/3) f1 */
static void build_extrapolated_rhs(Solver* S) {
    Level* l0 = &S->lv[0];
    Level* l1 = &S->lv[1];
    const long n0 = (long)l0->g.nr * l0->g.nt, n1 = (long)l1->g.nr * l1->g.nt;
    for (long p = 0; p < n0; ++p) l0->f[p] *= 4.0 / 3.0;
    for (long p = 0; p < n1; ++p) l1->res[p] = -l1->f[p] / 3.0;
    inject_transpose_add(&l0->g, &l1->g, l1->res, l0->f);
    set_dirichlet_rows(S, l0, l0->f);
}

/* ref multigrid.cpp:183-220 */
static void cycle(Solver* S, int lev, int type) {
    Level* l = &S->lv[lev];
    const int n = l->g.nr * l->g.nt;
    if (lev == S->L - 1) {
        memcpy(l->u, l->f, sizeof(double) * n);
        env_solve(&l->direct, l->u, NULL);
        return;
    }
    Level* c = &S->lv[lev + 1];
    const int ex = lev == 0 && S->ex;  /* smooth_level (multigrid.cpp:170-181) */
    for (int i = 0; i < S->pre; ++i) {
        if (ex) smooth_extrapolated(S, l, l->u, l->f);
        else smooth(S, l, l->u, l->f);
    }
    if (ex) extrapolated_residual(S, l->res);
    else residual(S, l, S->mode, l->u, l->f, l->res);
    restrict_t(&l->g, &c->g, l->res, c->f);
    mask_dirichlet(S, c, c->f);
    memset(c->u, 0, sizeof(double) * c->g.nr * c->g.nt);
    if (type == 0) cycle(S, lev + 1, 0);
    else if (type == 1) { cycle(S, lev + 1, 1); cycle(S, lev + 1, 1); }
    else { cycle(S, lev + 1, 2); cycle(S, lev + 1, 0); }
    prolongate(&l->g, &c->g, c->u, l->u, 1);
    for (int i = 0; i < S->post; ++i) {
        if (ex) smooth_extrapolated(S, l, l->u, l->f);
        else smooth(S, l, l->u, l->f);
    }
}

/* ref multigrid.cpp:267-275 */
static double residual_norm(Solver* S) {
    Level* l = &S->lv[0];
    if (S->ex) extrapolated_residual(S, l->res);
    else residual(S, l, S->mode, l->u, l->f, l->res);
    return orc_norm(S->norm, l->res, (long)l->g.nr * l->g.nt);
}

static void coarse_direct(Solver* S, int lev) { /* ref multigrid.cpp:183-187 */
    Level* l = &S->lv[lev];
    memcpy(l->u, l->f, sizeof(double) * l->g.nr * l->g.nt);
    env_solve(&l->direct, l->u, NULL);
}

/* ref multigrid.cpp:250-265 */
static int fmg_initialize(Solver* S) {
    const int L = S->L;
    Level* lc = &S->lv[L - 1];
    int rc = assemble_rhs(S, lc, lc->f);
    if (rc) return rc;
    coarse_direct(S, L - 1);
    for (int lf = L - 2; lf >= 0; --lf) {
        Level* l = &S->lv[lf];
        Level* c = &S->lv[lf + 1];
        prolongate(&l->g, &c->g, c->u, l->u, 0);
        set_dirichlet_rows(S, l, l->u);
        if ((rc = assemble_rhs(S, l, l->f))) return rc;
        if (lf == 0 && S->ex) build_extrapolated_rhs(S);
        for (int k = 0; k < S->fmg_it; ++k) {
            cycle(S, lf, S->fmg_cycle);
            if (lf == 0) ++S->fmg_run;
        }
    }
    return 0;
}

/* ref multigrid.cpp:277-296 */
static void exact_errors(const Solver* S, const double* u, double* w, double* inf) {
    if (!S->sol) { *w = -1.0; *inf = -1.0; return; }
    const Grid* g = &S->lv[0].g;
    double acc = 0.0, mx = 0.0;
    for (int s = 0; s < g->nr; ++s)
        for (int t = 0; t < g->nt; ++t) {
            const double e = u[gidx(g, s, t)] - sol_u(S->P.rmax, g->r[s], g->th[t]);
            acc += e * e;
            const double ae = fabs(e);
            mx = mx < ae ? ae : mx;
        }
    *w = sqrt(acc / (double)(g->nr * g->nt));
    *inf = mx;
}

static void solver_free(Solver* S) {
    if (!S) return;
    for (int i = 0; i < S->L; ++i) {
        Level* l = &S->lv[i];
        if (l->cl) { for (int s = 0; s < l->g.split; ++s) { free(l->cl[s]); free(l->cm[s]); } }
        free(l->cl); free(l->cm); free(l->cc);
        if (l->rl) { for (int t = 0; t < l->g.nt; ++t) { free(l->rl[t]); free(l->rm[t]); } }
        free(l->rl); free(l->rm);
        env_free(&l->origin); env_free(&l->direct);
        free(l->sn); free(l->cs); free(l->alpha); free(l->beta);
        free(l->arr); free(l->art); free(l->att); free(l->det);
        free(l->u); free(l->f); free(l->res);
        grid_free(&l->g);
    }
    free(S->lv);
    free(S->work);
    free(S);
}

/* level cache, ref level_cache.cpp:7-67 */
static int level_init(Solver* S, Level* l) {
    const Grid* g = &l->g;
    const int nr = g->nr, nt = g->nt;
    const size_t n = (size_t)nr * nt;
    l->sn = NEWD(nt); l->cs = NEWD(nt);
    for (int t = 0; t < nt; ++t) { l->sn[t] = sin(g->th[t]); l->cs[t] = cos(g->th[t]); }
    l->alpha = NEWD(nr); l->beta = NEWD(nr);
    for (int s = 0; s < nr; ++s) { l->alpha[s] = p_alpha(&S->P, g->r[s]); l->beta[s] = p_beta(&S->P, g->r[s]); }
    l->arr = NEWD(n); l->art = NEWD(n); l->att = NEWD(n); l->det = NEWD(n);
    for (int s = 0; s < nr; ++s)
        for (int t = 0; t < nt; ++t) {
            Coef c;
            int rc = transform(&S->G, l->alpha[s], g->r[s], l->sn[t], l->cs[t], &c);
            if (rc) return rc;
            const size_t i = (size_t)s * nt + t;
            l->arr[i] = c.arr; l->art[i] = c.art; l->att[i] = c.att; l->det[i] = c.det;
        }
    l->u = NEWD(n); l->f = NEWD(n); l->res = NEWD(n);
    return 0;
}

static _Thread_local int g_extra[5]; /* solution, fmg, fmg_iterations, fmg_cycle, extrapolation */
static _Thread_local int g_extra_set;
int orc_set_extra(int solution, int fmg, int fmg_iterations, int fmg_cycle, int extrapolation) {
    g_extra[0] = solution; g_extra[1] = fmg; g_extra[2] = fmg_iterations; g_extra[3] = fmg_cycle;
    g_extra[4] = extrapolation;
    g_extra_set = 1;
    return 0;
}

int orc_create(int geom_kind, double kappa_eps, double delta_e, int alpha_coeff,
               int beta_coeff, double rmax, double alpha_jump, double delta_r,
               double alpha_scale, int grid_mode, double R0, int a, int b,
               int aniso, int divide_by_2, double pair_tol, int stencil_mode,
               int boundary_mode, int max_levels, int pre, int post, int cyc,
               int norm_type, int max_iterations, double abs_tol,
               double rel_tol, int threads, void** out) {
    (void)threads;
    Solver* S = (Solver*)xcalloc(1, sizeof(Solver));
    S->G.kind = geom_kind; S->G.ke = kappa_eps; S->G.de = delta_e; S->G.xi = 1.0;
    if (geom_kind == 2) {
        if (kappa_eps <= 0.0 || kappa_eps >= 2.0) { free(S); return fail(1, "Czarny requires 0 < epsilon < 2"); }
        S->G.xi = 1.0 / sqrt(1.0 - kappa_eps * kappa_eps / 4.0);
    }
    if (rmax <= 0.0) { free(S); return fail(1, "Rmax must be positive"); }
    if (delta_r <= 0.0) { free(S); return fail(1, "delta_r must be positive"); }
    S->P.zoni = alpha_coeff; S->P.inv_beta = beta_coeff; S->P.rmax = rmax;
    S->P.jump = alpha_jump; S->P.dr = delta_r; S->P.scale = alpha_scale;
    S->mode = stencil_mode; S->boundary = boundary_mode; S->pre = pre; S->post = post;
    S->cycle = cyc; S->norm = norm_type; S->max_it = max_iterations;
    S->abs_tol = abs_tol; S->rel_tol = rel_tol; S->tol = pair_tol;
    S->fmg_it = 2; S->fmg_cycle = 2;
    if (g_extra_set) {
        S->sol = g_extra[0]; S->fmg = g_extra[1]; S->fmg_it = g_extra[2]; S->fmg_cycle = g_extra[3];
        S->ex = g_extra[4];
        g_extra_set = 0;
    }
    Grid g0;
    int rc = grid_mode == 0 ? grid_uniform(&g0, R0, rmax, a, b, pair_tol)
                            : grid_build(&g0, R0, rmax, a, b, aniso, divide_by_2, pair_tol);
    if (rc) { grid_free(&g0); free(S); return rc; }
    /* hierarchy, ref multigrid.cpp:81-124 */
    int cap = 32;
    Grid* grids = (Grid*)xcalloc(cap, sizeof(Grid));
    int L = 0;
    grids[L++] = g0;
    while ((max_levels == 0 || L < max_levels) && can_coarsen(&grids[L - 1], pair_tol)) {
        rc = grid_coarsen(&grids[L], &grids[L - 1], pair_tol);
        ++L;
        if (rc) break;
    }
    S->L = L;
    S->lv = (Level*)xcalloc(L, sizeof(Level));
    for (int i = 0; i < L; ++i) S->lv[i].g = grids[i];
    free(grids);
    for (int i = 0; i < L && !rc; ++i) {
        Level* l = &S->lv[i];
        if ((rc = level_init(S, l))) break;
        if (i + 1 < L) rc = smoother_init(S, l);
        else {
            const int n = l->g.nr * l->g.nt;
            int* nodes = NEWI(n);
            for (int q = 0; q < n; ++q) nodes[q] = q;
            int ntr;
            Trip* tr = assemble_coo(S, l, nodes, n, &ntr);
            rc = env_factor(&l->direct, n, tr, ntr, NULL);
            free(nodes); free(tr);
        }
    }
    const int scratch = S->lv[0].g.nt > S->lv[0].g.nr ? S->lv[0].g.nt : S->lv[0].g.nr;
    S->work = NEWD(scratch);
    if (rc) { solver_free(S); return rc; }
    *out = S;
    return 0;
}

void orc_destroy(void* h) { solver_free((Solver*)h); }
int orc_num_levels(void* h) { return ((Solver*)h)->L; }

static Level* lev(void* h, int level) { return &((Solver*)h)->lv[level]; }

int orc_level_info(void* h, int level, int* nr, int* nt, int* split) {
    Solver* S = (Solver*)h;
    if (level < 0 || level >= S->L) return fail(1, "level out of range");
    *nr = S->lv[level].g.nr; *nt = S->lv[level].g.nt; *split = S->lv[level].g.split;
    return 0;
}

int orc_level_grid(void* h, int level, double* radii, double* angles) {
    const Grid* g = &lev(h, level)->g;
    memcpy(radii, g->r, sizeof(double) * g->nr);
    memcpy(angles, g->th, sizeof(double) * g->nt);
    return 0;
}

int orc_level_coeffs(void* h, int level, double* arr, double* art, double* att,
                     double* det, double* alpha, double* beta) {
    const Level* l = lev(h, level);
    const size_t n = (size_t)l->g.nr * l->g.nt;
    memcpy(arr, l->arr, n * 8); memcpy(art, l->art, n * 8);
    memcpy(att, l->att, n * 8); memcpy(det, l->det, n * 8);
    memcpy(alpha, l->alpha, l->g.nr * 8); memcpy(beta, l->beta, l->g.nr * 8);
    return 0;
}

int orc_row(void* h, int level, int s, int t, int* cols, double* vals, int* count) {
    Row r;
    build_row((Solver*)h, lev(h, level), s, t, 1, &r);
    for (int i = 0; i < r.count; ++i) { cols[i] = r.cols[i]; vals[i] = r.vals[i]; }
    *count = r.count;
    return 0;
}

int orc_apply(void* h, int level, int mode, const double* u, double* y) {
    apply_op((Solver*)h, lev(h, level), mode, u, y);
    return 0;
}

int orc_residual(void* h, int level, int mode, const double* u, const double* f, double* r) {
    residual((Solver*)h, lev(h, level), mode, u, f, r);
    return 0;
}

int orc_smooth(void* h, int level, double* u, const double* f) {
    Solver* S = (Solver*)h;
    if (level >= S->L - 1) return fail(1, "coarsest level has no smoother");
    smooth(S, lev(h, level), u, f);
    return 0;
}

int orc_sweep(void* h, int level, int kind, int parity, double* u, const double* f) {
    Solver* S = (Solver*)h;
    if (level >= S->L - 1) return fail(1, "coarsest level has no smoother");
    if (kind == 0) sweep_circle(S, lev(h, level), parity, u, f, S->work);
    else if (lev(h, level)->g.split < lev(h, level)->g.nr) sweep_radial(S, lev(h, level), parity, u, f);
    return 0;
}

int orc_restrict(void* h, int fine_level, const double* fine, double* coarse) {
    restrict_t(&lev(h, fine_level)->g, &lev(h, fine_level + 1)->g, fine, coarse);
    return 0;
}

int orc_prolongate(void* h, int fine_level, const double* coarse, double* fine, int add) {
    prolongate(&lev(h, fine_level)->g, &lev(h, fine_level + 1)->g, coarse, fine, add);
    return 0;
}

int orc_coarse_solve(void* h, const double* f, double* u) {
    Solver* S = (Solver*)h;
    Level* l = &S->lv[S->L - 1];
    memcpy(u, f, sizeof(double) * l->g.nr * l->g.nt);
    env_solve(&l->direct, u, NULL);
    return 0;
}

/* --- mt19937 + libstdc++ uniform_real_distribution<double>(-1,1) -------- */
typedef struct { unsigned mt[624]; int i; } MT;
static void mt_seed(MT* m, unsigned s) {
    m->mt[0] = s;
    for (int i = 1; i < 624; ++i) m->mt[i] = 1812433253u * (m->mt[i - 1] ^ (m->mt[i - 1] >> 30)) + (unsigned)i;
    m->i = 624;
}
static unsigned mt_next(MT* m) {
    if (m->i >= 624) {
        for (int k = 0; k < 624; ++k) {
            const unsigned y = (m->mt[k] & 0x80000000u) | (m->mt[(k + 1) % 624] & 0x7fffffffu);
            m->mt[k] = m->mt[(k + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        m->i = 0;
    }
    unsigned y = m->mt[m->i++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}
static double mt_uniform(MT* m, double a, double b) {
    const double lo = (double)mt_next(m);
    const double hi = (double)mt_next(m);
    double c = (lo + hi * 4294967296.0) / 18446744073709551616.0;
    if (c >= 1.0) c = nextafter(1.0, 0.0);
    return c * (b - a) + a;
}

int orc_seeded_field(void* h, unsigned seed, double* u) {
    const Grid* g = &lev(h, 0)->g;
    MT m;
    mt_seed(&m, seed);
    for (int s = 0; s < g->nr; ++s)
        for (int t = 0; t < g->nt; ++t) u[gidx(g, s, t)] = mt_uniform(&m, -1.0, 1.0);
    for (int t = 0; t < g->nt; ++t) u[gidx(g, g->nr - 1, t)] = 0.0;
    return 0;
}

/* seeded-RHS solve, ref multigrid.cpp:298-357 with f supplied */
int orc_solve(void* h, const double* f, double* u_out, double* history,
              int* iterations, int* converged, double* mean_reduction, double* seconds) {
    Solver* S = (Solver*)h;
    Level* l0 = &S->lv[0];
    const long n = (long)l0->g.nr * l0->g.nt;
    memcpy(l0->f, f, sizeof(double) * n);
    struct timespec ts0, ts1;
    clock_gettime(CLOCK_MONOTONIC, &ts0);
    memset(l0->u, 0, sizeof(double) * n);
    set_dirichlet_rows(S, l0, l0->u);
    const double r0 = residual_norm(S);
    history[0] = r0;
    int conv = r0 == 0.0 || (S->abs_tol > 0.0 && r0 <= S->abs_tol);
    int it = 0;
    while (!conv && it < S->max_it) {
        cycle(S, 0, S->cycle);
        ++it;
        const double r = residual_norm(S);
        history[it] = r;
        conv = (S->abs_tol > 0.0 && r <= S->abs_tol) || (S->rel_tol > 0.0 && r <= S->rel_tol * r0);
    }
    clock_gettime(CLOCK_MONOTONIC, &ts1);
    *seconds = (ts1.tv_sec - ts0.tv_sec) + 1e-9 * (ts1.tv_nsec - ts0.tv_nsec);
    *iterations = it;
    *converged = conv;
    const double r_end = history[it];
    *mean_reduction = (it > 0 && r0 > 0.0 && r_end > 0.0) ? pow(r_end / r0, 1.0 / it) : 0.0;
    memcpy(u_out, l0->u, sizeof(double) * n);
    return 0;
}

/* MultigridSolver::solve() itself (ref multigrid.cpp:298-357): manufactured
 * RHS (or FMG start), solve loop, exact errors. */
int orc_solve_native(void* h, double* u_out, double* history, int* iterations,
                     int* fine_cycles, int* converged, double* mean_reduction,
                     double* err_weighted, double* err_inf) {
    Solver* S = (Solver*)h;
    Level* l0 = &S->lv[0];
    const long n = (long)l0->g.nr * l0->g.nt;
    int rc;
    S->fmg_run = 0;
    if (S->fmg) {
        if ((rc = fmg_initialize(S))) return rc;
    } else {
        if ((rc = assemble_rhs(S, l0, l0->f))) return rc;
        if (S->ex) {
            if ((rc = assemble_rhs(S, &S->lv[1], S->lv[1].f))) return rc;
            build_extrapolated_rhs(S);
        }
        memset(l0->u, 0, sizeof(double) * n);
        set_dirichlet_rows(S, l0, l0->u);
    }
    const double r0 = residual_norm(S);
    history[0] = r0;
    int conv = r0 == 0.0 || (S->abs_tol > 0.0 && r0 <= S->abs_tol);
    int it = 0;
    while (!conv && it < S->max_it) {
        cycle(S, 0, S->cycle);
        ++it;
        const double r = residual_norm(S);
        history[it] = r;
        conv = (S->abs_tol > 0.0 && r <= S->abs_tol) || (S->rel_tol > 0.0 && r <= S->rel_tol * r0);
    }
    *iterations = it;
    *fine_cycles = it + S->fmg_run;
    *converged = conv;
    const double r_end = history[it];
    *mean_reduction = (it > 0 && r0 > 0.0 && r_end > 0.0) ? pow(r_end / r0, 1.0 / it) : 0.0;
    exact_errors(S, l0->u, err_weighted, err_inf);
    memcpy(u_out, l0->u, sizeof(double) * n);
    return 0;
}

int orc_assemble_rhs(void* h, int level, double* b) {
    Solver* S = (Solver*)h;
    return assemble_rhs(S, &S->lv[level], b);
}

int orc_exact_errors(void* h, const double* u, double* w, double* inf) {
    exact_errors((Solver*)h, u, w, inf);
    return 0;
}
