// FP64 dependent-latency probe: cycles per dependent op and per exact
// substitution step (mul, sub, Markstein division).
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
    double x = a, y = b;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = fma(x, y, a); }
    long long t1 = clock64();
    double z = a;
    for (int i = 0; i < n; ++i) { z = z * y; }
    long long t2 = clock64();
    double q = a, l = 1.0001, r = 1.0 / l, m = -0.5;
    for (int i = 0; i < n; ++i) {
        double aa = b - m * q;
        double q0 = aa * r;
        double e = fma(-l, q0, aa);
        q = fma(e, r, q0);
    }
    long long t3 = clock64();
    double w = a;
    for (int i = 0; i < n; ++i) { w = __drcp_rn(w + 1.0); }
    long long t4 = clock64();
    out[threadIdx.x] = x + z + q + w;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64);
    int n = 100000;
    k<<<1, 32>>>(o, c, 0.999, 0.5, n); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 0.999, 0.5, n); cudaDeviceSynchronize();
    printf("dfma %.2f dmul %.2f subst_step %.2f (dadd+drcp) %.2f cycles\n", (double)c[0] / n,
           (double)c[1] / n, (double)c[2] / n, (double)c[3] / n);
}
