/* Speculative exact-order L L^T substitution, simulated on the real line
 * factors of a config: chunk composites (fast-mode affine maps) give start
 * values, every chunk restarts W rows early, then fix waves recompute the
 * inconsistent chunks until every chunk starts from its predecessor's end.
 * Prints waves per line and checks the result is bitwise the sequential one. */
#include "../../oracle/polarmg_oracle.c"
#include <math.h>
static unsigned sd = 777;
static double urand(void) { sd = sd * 1664525u + 1013904223u; return ((sd >> 8) / 16777216.0) * 2 - 1; }
static long hist[64], lines_, exact_steps, nodes_, bad;
static int K = 8, W = 8;
/* forward recurrence step at row i from prev value v */
static inline double fstep(const double* b, const double* l, const double* m, int i, double v) {
    return i == 0 ? b[0] / l[0] : (b[i] - m[i - 1] * v) / l[i];
}
static int spec_fwd(int n, const double* b, const double* l, const double* m, double* out) {
    int T = (n + K - 1) / K;
    double* A = malloc(T * 8), *Bc = malloc(T * 8), *yin = malloc((T + 1) * 8);
    for (int t = 0; t < T; ++t) {
        double a_ = 1, bb = 0;
        for (int j = t * K; j < n && j < t * K + K; ++j) {
            double il = 1.0 / l[j], a = j > 0 ? -(m[j - 1] * il) : 0.0;
            bb = a * bb + b[j] * il; a_ = a * a_;
        }
        A[t] = a_; Bc[t] = bb;
    }
    yin[0] = 0; for (int t = 0; t < T; ++t) yin[t + 1] = A[t] * yin[t] + Bc[t];
    /* pass 1: chunk t starts at row max(0,tK-W) from the approximate value yin */
    double* st = malloc(T * 8), *en = malloc(T * 8);
    for (int t = 0; t < T; ++t) {
        int j0 = t * K, s = j0 - W; if (s < 0) s = 0;
        /* approximate value at row s-1: rerun fast from chunk start of s */
        double v;
        { int tc = (s - 1) / K; if (s == 0) v = 0; else { v = yin[tc]; for (int j = tc * K; j <= s - 1; ++j) { double il = 1.0 / l[j]; v = (b[j] - (j ? m[j - 1] : 0) * v) * il; } } }
        for (int j = s; j < j0; ++j) { v = fstep(b, l, m, j, v); exact_steps++; }
        st[t] = v;  /* value at row j0-1 on this trajectory */
        for (int j = j0; j < n && j < j0 + K; ++j) { v = fstep(b, l, m, j, v); out[j] = v; exact_steps++; }
        en[t] = v;
    }
    int waves = 0;
    static int inc[1 << 16];
    for (;;) {
        int any = 0;
        for (int t = 1; t < T; ++t) { inc[t] = st[t] != en[t - 1]; any |= inc[t]; }
        if (!any) break;
        ++waves;
        /* recompute only the first flagged chunk of each run (its predecessor is consistent) */
        for (int t = T - 1; t >= 1; --t) if (inc[t] && !(t > 1 && inc[t - 1])) {
            double v = en[t - 1]; st[t] = v;
            for (int j = t * K; j < n && j < t * K + K; ++j) { v = fstep(b, l, m, j, v); out[j] = v; exact_steps++; }
            en[t] = v;
        }
    }
    free(A); free(Bc); free(yin); free(st); free(en);
    return waves;
}
static void line(int n, const double* l, const double* m) {
    double* b = malloc(n * 8), *y = malloc(n * 8), *o = malloc(n * 8);
    for (int i = 0; i < n; ++i) b[i] = urand();
    y[0] = b[0] / l[0];
    for (int i = 1; i < n; ++i) y[i] = (b[i] - m[i - 1] * y[i - 1]) / l[i];
    int w = spec_fwd(n, b, l, m, o);
    for (int i = 0; i < n; ++i) if (o[i] != y[i]) { bad++; break; }
    hist[w < 63 ? w : 63]++; lines_++; nodes_ += n;
    free(b); free(y); free(o);
}
int main(int argc, char** argv) {
    int cfg = argc > 1 ? atoi(argv[1]) : 1; K = argc > 2 ? atoi(argv[2]) : 8; W = argc > 3 ? atoi(argv[3]) : 8;
    void* h; int rc;
    if (cfg == 1) rc = orc_create(1, 0.3, 0.2, 1, 1, 1.3, 0.5, 0.1, 1.0, 0, 1e-5, 1025, 1024, 0, 0, 1e-12, 0, 0, 0, 1, 1, 0, 0, 200, -1, 1e-10, 0, &h);
    else if (cfg == 3) rc = orc_create(1, 0.3, 0.2, 1, 1, 1.3, 0.5, 0.1, 1.9, 0, 1e-5, 513, 512, 0, 0, 1e-12, 0, 0, 0, 1, 1, 0, 0, 200, -1, 1e-10, 0, &h);
    else rc = orc_create(2, 0.3, 1.4, 1, 1, 1.3, 0.5, 0.1, 1.0, 1, 1e-5, 8, 8, 0, 4, 1e-12, 0, 0, 0, 1, 1, 0, 0, 200, -1, 1e-10, 0, &h);
    if (rc) { printf("create failed %s\n", g_err); return 1; }
    Solver* S = h;
    int maxL = argc > 4 ? atoi(argv[4]) : 3;
    for (int L = 0; L + 1 < S->L && L < maxL; ++L) {
        Level* l = &S->lv[L];
        for (int kind = 0; kind < 2; ++kind) {
            memset(hist, 0, sizeof hist); lines_ = exact_steps = nodes_ = bad = 0;
            if (kind == 0) for (int s = 1; s < l->g.split; ++s) line(l->g.nt, l->cl[s], l->cm[s]);
            else for (int t = 0; t < l->g.nt; ++t) line(l->g.nr - l->g.split, l->rl[t], l->rm[t]);
            printf("L%d %s lines %ld bad %ld exact steps/node %.2f waves:", L, kind ? "radial" : "circle", lines_, bad, (double)exact_steps / nodes_);
            for (int w = 0; w < 12; ++w) printf(" %ld", hist[w]);
            printf("\n");
        }
    }
    return 0;
}
