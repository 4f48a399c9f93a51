// Dependent-chain latency of fp64 ops on this GPU (cycles per op), one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double x0, int n) {
    double a = x0, b = x0 * 0.5 + 1.0, c = 1.0000001;
    long long t0, t1;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) { a = a + c; a = a + c; a = a + c; a = a + c; }
    t1 = clock64(); cyc[0] = (t1 - t0); out[0] = a;
    // DMUL chain
    a = x0; t0 = clock64();
    for (int i = 0; i < n; ++i) { a = a * c; a = a * c; a = a * c; a = a * c; }
    t1 = clock64(); cyc[1] = (t1 - t0); out[1] = a;
    // DFMA chain
    a = x0; t0 = clock64();
    for (int i = 0; i < n; ++i) { a = fma(a, c, b); a = fma(a, c, b); a = fma(a, c, b); a = fma(a, c, b); }
    t1 = clock64(); cyc[2] = (t1 - t0); out[2] = a;
    // IEEE reciprocal chain
    a = x0; t0 = clock64();
    for (int i = 0; i < n; ++i) { a = 1.0 / (a + 1.5); a = 1.0 / (a + 1.5); a = 1.0 / (a + 1.5); a = 1.0 / (a + 1.5); }
    t1 = clock64(); cyc[3] = (t1 - t0); out[3] = a;
    // IEEE division chain
    a = x0; t0 = clock64();
    for (int i = 0; i < n; ++i) { a = b / (a + 1.5); a = b / (a + 1.5); a = b / (a + 1.5); a = b / (a + 1.5); }
    t1 = clock64(); cyc[4] = (t1 - t0); out[4] = a;
    // Thomas forward step chain: cp = c * (1/(b - cp*a))
    double cp = 0.1, aa = -0.05, bb = 0.15, cc = 0.03;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) { double r = 1.0 / (bb - cp * aa); cp = cc * r; }
    }
    t1 = clock64(); cyc[5] = (t1 - t0); out[5] = cp;
    // rcp approx (MUFU.RCP64H only) chain
    a = x0; t0 = clock64();
    for (int i = 0; i < n; ++i) { a = __drcp_rn(a + 1.5); a = __drcp_rn(a + 1.5); a = __drcp_rn(a + 1.5); a = __drcp_rn(a + 1.5); }
    t1 = clock64(); cyc[6] = (t1 - t0); out[6] = a;
}
int main() {
    double *o; long long *c; cudaMallocManaged(&o, 64 * 8); cudaMallocManaged(&c, 64 * 8);
    int n = 1000;
    k<<<1, 32>>>(o, c, 1.0, n); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 1.0, n); cudaDeviceSynchronize();
    const char *names[] = {"DADD", "DMUL", "DFMA", "1.0/x (+DADD)", "b/x (+DADD)", "thomas cp step", "__drcp_rn (+DADD)"};
    for (int q = 0; q < 7; ++q) printf("%-20s %.1f cycles/op\n", names[q], (double)c[q] / (4.0 * n));
    return 0;
}
