// Per-level cost of the vadv forward recurrence as used in the kernels, adding parts one at a time.
// 1 CTA per SM x 4 warps (one per SMSP), each thread one column; cycles per level from clock64.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2005_13014_b200/csrc/tma.h"
template <int MODE>
__global__ void __launch_bounds__(128, 1) chain(const double *a_, const double *b_, const double *c_, const double *d_,
                                               double *out, long long *cyc, int K, int tmem_cols) {
    __shared__ uint32_t tb;
    __shared__ double rows[4][5][128];
    const int tid = threadIdx.x, warp = tid >> 5;
    if (MODE >= 3) { if (warp == 0) oec::tmem_alloc(&tb, tmem_cols); oec::tmem_fence_before(); __syncthreads(); oec::tmem_fence_after(); }
    const uint32_t taddr = (MODE >= 3) ? tb + ((uint32_t)(32 * warp) << 16) : 0;
    double a = a_[tid], b = b_[tid], c = c_[tid], dd = d_[tid];
    for (int l = 0; l < 4; ++l) { rows[l][0][tid] = a + l * 1e-3; rows[l][1][tid] = b; rows[l][2][tid] = c; rows[l][3][tid] = dd; rows[l][4][tid] = dd; }
    __syncthreads();
    double cpp = 0, dpp = 0, acc = 0;
    long long t0 = clock64();
    for (int g = 0; g < K / 4; ++g) {
        double ra[4], rb[4], rc[4], rd[4], ru[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            if (MODE >= 2) { ra[l] = rows[l][0][tid]; rb[l] = rows[l][1][tid]; rc[l] = rows[l][2][tid]; rd[l] = rows[l][3][tid]; ru[l] = rows[l][4][tid]; }
            else { ra[l] = a + l * 1e-3; rb[l] = b + g * 1e-9; rc[l] = c; rd[l] = dd; ru[l] = dd; }
        }
        double cpv[4], dpv[4];
        bool okall = true;
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            double r;
            if (MODE == 0) r = 1.0 / (rb[l] - cpp * ra[l]);
            else { bool ok; r = oec::rcp_rn_fast(rb[l] - cpp * ra[l], ok); okall = okall && ok; }
            cpv[l] = rc[l] * r;
            dpv[l] = (rd[l] - dpp * ra[l]) * r;
            cpp = cpv[l];
            dpp = dpv[l];
        }
        if (MODE >= 1 && !__all_sync(0xffffffffu, okall)) acc += 1.0;
        if (MODE >= 3) {
            uint32_t cells[24];
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                cells[6 * l] = __double2loint(cpv[l]); cells[6 * l + 1] = __double2hiint(cpv[l]);
                cells[6 * l + 2] = __double2loint(dpv[l]); cells[6 * l + 3] = __double2hiint(dpv[l]);
                cells[6 * l + 4] = __double2loint(ru[l]); cells[6 * l + 5] = __double2hiint(ru[l]);
            }
            oec::tmem_st16(taddr + (24 * g) % 480, cells);
            oec::tmem_st8(taddr + (24 * g) % 480 + 16, cells + 16);
        } else {
            acc += cpv[0] + dpv[3];
        }
    }
    long long t1 = clock64();
    if (MODE >= 3) { oec::tmem_wait_st(); oec::tmem_fence_before(); __syncthreads(); oec::tmem_fence_after(); if (warp == 0) oec::tmem_dealloc(tb, tmem_cols); }
    out[blockIdx.x * 128 + tid] = cpp + dpp + acc;
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double *a, *b, *c, *d, *o; long long *cy;
    cudaMalloc(&a, 128 * 8); cudaMalloc(&b, 128 * 8); cudaMalloc(&c, 128 * 8); cudaMalloc(&d, 128 * 8); cudaMalloc(&o, 148 * 128 * 8);
    cudaMallocManaged(&cy, 148 * 8);
    double h[128]; for (int q = 0; q < 128; ++q) h[q] = -0.01 - q * 1e-5; cudaMemcpy(a, h, 1024, cudaMemcpyHostToDevice);
    for (int q = 0; q < 128; ++q) h[q] = 0.15 + q * 1e-5; cudaMemcpy(b, h, 1024, cudaMemcpyHostToDevice);
    for (int q = 0; q < 128; ++q) h[q] = 0.012; cudaMemcpy(c, h, 1024, cudaMemcpyHostToDevice);
    for (int q = 0; q < 128; ++q) h[q] = 0.3; cudaMemcpy(d, h, 1024, cudaMemcpyHostToDevice);
    const int K = 8000;
    const char *names[] = {"IEEE 1/x chain (compiler division)", "branch-free rcp + warp vote", "+ rows from smem", "+ TMEM stores"};
    for (int pass = 0; pass < 2; ++pass) {
        chain<0><<<148, 128>>>(a, b, c, d, o, cy, K, 512); cudaDeviceSynchronize();
        if (pass) printf("%-40s %.1f cycles/level\n", names[0], cy[0] / (double)K);
        chain<1><<<148, 128>>>(a, b, c, d, o, cy, K, 512); cudaDeviceSynchronize();
        if (pass) printf("%-40s %.1f cycles/level\n", names[1], cy[0] / (double)K);
        chain<2><<<148, 128>>>(a, b, c, d, o, cy, K, 512); cudaDeviceSynchronize();
        if (pass) printf("%-40s %.1f cycles/level\n", names[2], cy[0] / (double)K);
        chain<3><<<148, 128>>>(a, b, c, d, o, cy, K, 512); cudaDeviceSynchronize();
        if (pass) printf("%-40s %.1f cycles/level  (err %d)\n", names[3], cy[0] / (double)K, (int)cudaGetLastError());
    }
}
