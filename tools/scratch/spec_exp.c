/* Experiment: speculative exact-order line solves.  For every smoother line of
 * every level, compare the reference's sequential L L^T substitution with a
 * chunked scheme where chunk t restarts W rows early from a perturbed value
 * and is accepted when its trajectory meets chunk t-1's at the boundary. */
#include "../../oracle/polarmg_oracle.c"
#include <math.h>
static double perturb(double v, double rel, unsigned* s) {
    *s = *s * 1664525u + 1013904223u;
    double r = ((*s >> 8) / 16777216.0) * 2 - 1;
    return v * (1 + rel * r);
}
static long fails_f, fails_b, chunks;
static double maxc_f, maxc_b;
static void line(int n, const double* l, const double* m, int K, int W, double rel, unsigned* seed) {
    double* b = malloc(n * 8), *y = malloc(n * 8), *x = malloc(n * 8);
    for (int i = 0; i < n; ++i) { *seed = *seed * 1664525u + 1013904223u; b[i] = ((*seed >> 8) / 16777216.0) * 2 - 1; }
    y[0] = b[0] / l[0];
    for (int i = 1; i < n; ++i) y[i] = (b[i] - m[i - 1] * y[i - 1]) / l[i];
    x[n - 1] = y[n - 1] / l[n - 1];
    for (int i = n - 2; i >= 0; --i) x[i] = (y[i] - m[i] * x[i + 1]) / l[i];
    for (int i = 1; i < n; ++i) { double c = fabs(m[i - 1] / l[i]); if (c > maxc_f) maxc_f = c; }
    for (int i = 0; i < n - 1; ++i) { double c = fabs(m[i] / l[i]); if (c > maxc_b) maxc_b = c; }
    for (int t0 = K; t0 < n; t0 += K) {
        ++chunks;
        int s = t0 - W; if (s < 1) s = 1;
        double v = perturb(y[s - 1], rel, seed);
        for (int i = s; i < t0; ++i) v = (b[i] - m[i - 1] * v) / l[i];
        if (v != y[t0 - 1]) ++fails_f;
        /* backward: chunk ending at t0-1 (from the top) restarts W rows later */
        int e = t0 - 1 + W; if (e > n - 2) e = n - 2;
        double w = perturb(x[e + 1], rel, seed);
        for (int i = e; i >= t0; --i) w = (y[i] - m[i] * w) / l[i];
        if (w != x[t0]) ++fails_b;
    }
    free(b); free(y); free(x);
}
int main(int argc, char** argv) {
    int cfg = argc > 1 ? atoi(argv[1]) : 1, K = argc > 2 ? atoi(argv[2]) : 8;
    int W = argc > 3 ? atoi(argv[3]) : 8; double rel = argc > 4 ? atof(argv[4]) : 1e-15;
    void* h; int rc;
    if (cfg == 1) rc = orc_create(1, 0.3, 0.2, 1, 1, 1.3, 0.5, 0.1, 1.0, 0, 1e-5, 1025, 1024, 0, 0, 1e-12, 0, 0, 0, 1, 1, 0, 0, 200, -1, 1e-10, 0, &h);
    else if (cfg == 3) rc = orc_create(1, 0.3, 0.2, 1, 1, 1.3, 0.5, 0.1, 1.9, 0, 1e-5, 513, 512, 0, 0, 1e-12, 0, 0, 0, 1, 1, 0, 0, 200, -1, 1e-10, 0, &h);
    else if (cfg == 0) rc = orc_create(0, 0, 0, 1, 0, 1.3, 0.5, 0.1, 1.0, 0, 1e-5, 257, 256, 0, 0, 1e-12, 0, 0, 0, 1, 1, 0, 0, 200, -1, 1e-10, 0, &h);
    else rc = orc_create(2, 0.3, 1.4, 1, 1, 1.3, 0.5, 0.1, 1.0, 1, 1e-5, 8, 8, 0, 4, 1e-12, 0, 0, 0, 1, 1, 0, 0, 200, -1, 1e-10, 0, &h);
    if (rc) { printf("create failed %s\n", g_err); return 1; }
    Solver* S = h;
    unsigned seed = 12345;
    for (int L = 0; L + 1 < S->L; ++L) {
        Level* l = &S->lv[L];
        fails_f = fails_b = chunks = 0; maxc_f = maxc_b = 0;
        long cf = 0, cb = 0, cc = 0;
        for (int s = 1; s < l->g.split; ++s) line(l->g.nt, l->cl[s], l->cm[s], K, W, rel, &seed);
        cf = fails_f; cb = fails_b; cc = chunks; double mcf = maxc_f, mcb = maxc_b;
        fails_f = fails_b = chunks = 0; maxc_f = maxc_b = 0;
        for (int t = 0; t < l->g.nt; ++t) line(l->g.nr - l->g.split, l->rl[t], l->rm[t], K, W, rel, &seed);
        printf("level %d %dx%d split %d | circle chunks %ld fail f %ld b %ld maxc %.4f %.4f | radial chunks %ld fail f %ld b %ld maxc %.4f %.4f\n",
               L, l->g.nr, l->g.nt, l->g.split, cc, cf, cb, mcf, mcb, chunks, fails_f, fails_b, maxc_f, maxc_b);
    }
    return 0;
}
