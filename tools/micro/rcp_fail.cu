// find inputs where the branch-free IEEE reciprocal fast path (tma.h rcp_rn_fast) differs from 1.0/x
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2005_13014_b200/csrc/tma.h"
__global__ void k(unsigned long long n, unsigned long long seed, double *bad, int *nbad) {
    for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; t < n; t += (unsigned long long)gridDim.x * blockDim.x) {
        unsigned long long z = (t + 1) * 0x9E3779B97F4A7C15ull ^ seed;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
        if (!(t & 1)) continue;
        double x = __longlong_as_double((long long)z);
        bool ok; double r = oec::rcp_rn_fast(x, ok); double ref = 1.0 / x;
        if (ok && __double_as_longlong(r) != __double_as_longlong(ref) && !(r != r && ref != ref)) {
            int q = atomicAdd(nbad, 1);
            if (q < 64) { bad[3 * q] = x; bad[3 * q + 1] = r; bad[3 * q + 2] = ref; }
        }
    }
}
int main() {
    double *b; int *nb; cudaMallocManaged(&b, 64 * 3 * 8); cudaMallocManaged(&nb, 4); *nb = 0;
    k<<<148 * 8, 256>>>(200000000ull, 12345ull, b, nb); cudaDeviceSynchronize();
    printf("bad %d\n", *nb);
    for (int q = 0; q < *nb && q < 64; ++q) {
        unsigned long long xb; memcpy(&xb, &b[3 * q], 8);
        printf("x=%a (0x%016llx)  fast=%a  ref=%a\n", b[3 * q], xb, b[3 * q + 1], b[3 * q + 2]);
    }
}
