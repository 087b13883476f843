/* Speculative exact substitution with merge-walkers (device algorithm emulated
 * on the CPU): spec pass (warm-up over the previous chunk from the fast-scan
 * value), chunk-start consistency flags, one walker per run of flagged chunks
 * walking until it merges with the stored trajectory, full verification
 * + re-walk only on conflicts.  Reports the longest walker per line (the
 * sequential latency) and checks bitwise equality with the sequential solve. */
#include "../../oracle/polarmg_oracle.c"
#include <math.h>
static unsigned sd = 777;
static double urand(void) { sd = sd * 1664525u + 1013904223u; return ((sd >> 8) / 16777216.0) * 2 - 1; }
static int K = 8, REV = 0;
static long hist[5000], lines_, bad, rounds_hist[8], conflicts;
static inline double fstep(const double* b, const double* l, const double* m, int i, double v) {
    return i == 0 ? b[0] / l[0] : (b[i] - m[i - 1] * v) / l[i];
}
static void spec(int n, const double* b, const double* l, const double* m, double* Y) {
    int T = (n + K - 1) / K;
    double A[4096], Bc[4096], yin[4097], w[4096];
    int fl[4097];
    for (int t = 0; t < T; ++t) {
        double a_ = 1, bb = 0;
        for (int j = t * K; j < n && j < t * K + K; ++j) {
            double il = 1.0 / l[j], a = j > 0 ? -(m[j - 1] * il) : 0.0;
            bb = a * bb + b[j] * il; a_ = a * a_;
        }
        A[t] = a_; Bc[t] = bb;
    }
    yin[0] = 0; for (int t = 0; t < T; ++t) yin[t + 1] = A[t] * yin[t] + Bc[t];
    for (int t = 0; t < T; ++t) {
        int j0 = t * K;
        double v = t >= 2 ? yin[t - 1] : 0;  /* approx value at row (t-1)K-1 */
        if (t >= 1) for (int j = j0 - K; j < j0; ++j) v = fstep(b, l, m, j, v);
        w[t] = v;
        for (int j = j0; j < n && j < j0 + K; ++j) { v = fstep(b, l, m, j, v); Y[j] = v; }
    }
    fl[T] = 0; fl[0] = 0;
    for (int t = 1; t < T; ++t) fl[t] = w[t] != Y[t * K - 1];
    int maxwalk = 0, round = 0;
    for (;;) {
        int any = 0; for (int t = 1; t < T; ++t) any |= fl[t];
        if (!any) break;
        int conflict = 0;
        int first[4096];
        for (int t = 0; t < T; ++t) first[t] = fl[t] && !(t > 0 && fl[t - 1]);
        for (int ti = 0; ti < T; ++ti) {
            int t = REV ? T - 1 - ti : ti;
            if (!first[t]) continue;
            int j = t * K, steps = 0; double v = Y[j - 1];
            while (j < n) {
                double nv = fstep(b, l, m, j, v); steps++;
                if (nv == Y[j]) {
                    int c = j / K, nx = (c + 1) * K;
                    if (nx < n && fl[c + 1] && fl[c]) { v = Y[nx - 1]; j = nx; continue; }
                    break;
                }
                Y[j] = nv; v = nv; ++j;
                if (j < n && j % K == 0 && first[j / K]) conflict = 1;
            }
            if (steps > maxwalk) maxwalk = steps;
        }
        round++;
        if (!conflict) break;
        conflicts++;
        /* full verification: flag chunks containing an inconsistent row */
        for (int t = 1; t < T; ++t) {
            fl[t] = 0;
            for (int j = t * K; j < n && j < t * K + K; ++j) if (Y[j] != fstep(b, l, m, j, Y[j - 1])) { fl[t] = 1; break; }
        }
        /* walkers start at chunk starts: a chunk with a bad row mid-chunk restarts from its start (correct, a bit more work) */
    }
    rounds_hist[round < 7 ? round : 7]++;
    int bucket = maxwalk < 4999 ? maxwalk : 4999; hist[bucket / 1]++;
}
static void line(int n, const double* l, const double* m) {
    double* b = malloc(n * 8), *y = malloc(n * 8), *o = malloc(n * 8);
    for (int i = 0; i < n; ++i) b[i] = urand();
    y[0] = b[0] / l[0];
    for (int i = 1; i < n; ++i) y[i] = (b[i] - m[i - 1] * y[i - 1]) / l[i];
    spec(n, b, l, m, o);
    for (int i = 0; i < n; ++i) if (o[i] != y[i]) { bad++; break; }
    lines_++;
    free(b); free(y); free(o);
}
int main(int argc, char** argv) {
    int cfg = argc > 1 ? atoi(argv[1]) : 1; K = argc > 2 ? atoi(argv[2]) : 8; REV = argc > 3 ? atoi(argv[3]) : 0;
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
            memset(hist, 0, sizeof hist); memset(rounds_hist, 0, sizeof rounds_hist); lines_ = bad = conflicts = 0;
            if (kind == 0) for (int s = 1; s < l->g.split; ++s) line(l->g.nt, l->cl[s], l->cm[s]);
            else for (int t = 0; t < l->g.nt; ++t) line(l->g.nr - l->g.split, l->rl[t], l->rm[t]);
            long c50 = 0, tot = 0; int p50 = 0, p99 = 0, mx = 0;
            for (int i = 0; i < 5000; ++i) tot += hist[i];
            int p90 = 0; for (int i = 0; i < 5000; ++i) { if (!p90 && c50 + hist[i] >= tot * 9 / 10) p90 = i; c50 += hist[i]; if (!p50 && c50 >= tot / 2) p50 = i; if (!p99 && c50 >= tot * 99 / 100) p99 = i; if (hist[i]) mx = i; }
            printf("L%d %s lines %ld bad %ld conflicts %ld | longest walk p50 %d p90 %d p99 %d max %d%s | rounds:", L, kind ? "radial" : "circle", lines_, bad, conflicts, p50, p90, p99, mx, mx == 4999 ? "+" : "");
            for (int i = 0; i < 5; ++i) printf(" %ld", rounds_hist[i]);
            printf("\n");
        }
    }
    return 0;
}
