// TMA issue cost of many small 3D boxes: per CTA a ring of S chunks; each chunk = NB boxes of
// (BX i, 8 k, BJ j) doubles from an (i, k, j) tensor, issued by ISS lanes of the producer warp
// (lane l issues boxes l, l+ISS, ...).  Reports GB/s total and per CTA at grid = #SMs.
// Question answered: can vadv feed a CTA from 7 x 5 boxes of 1 KB per chunk (16-column units)
// as fast as from 5 boxes of 8 KB (128-column rows)?
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t *b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(su(b)),
                 "r"(ph)
                 : "memory");
}

__global__ void stream(const __grid_constant__ CUtensorMap m, int nb, int bx, int bj, int iss, int S, int iters, int ni,
                       int nj, int nk) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int box_bytes = bx * 8 * bj * 8;
    const int slot = nb * box_bytes;
    uint64_t *full = (uint64_t *)(sm + S * slot), *empty = full + S;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int nxb = ni / bx, njb = nj / bj, nkb = nk / 8;
    if (warp == 0) {
        for (int n = 0; n < iters; ++n) {
            const int s = n % S;
            if (n >= S) wait(&empty[s], ((n / S) - 1) & 1);
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(slot));
            __syncwarp();
            if (lane < iss) {
                for (int b = lane; b < nb; b += iss) {
                    const int u = (blockIdx.x * 977 + n * nb + b) % (nxb * njb);
                    const int kb = (blockIdx.x + n) % nkb;
                    const int i = (u % nxb) * bx, j = (u / nxb) * bj, k = kb * 8;
                    asm volatile(
                        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
                        "%5}], [%2];" ::"r"(su(sm + s * slot + b * box_bytes)),
                        "l"((uint64_t)&m), "r"(su(&full[s])), "r"(i), "r"(k), "r"(j)
                        : "memory");
                }
            }
        }
    } else if (threadIdx.x == 32) {
        for (int n = 0; n < iters; ++n) {
            const int s = n % S;
            wait(&full[s], (n / S) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])));
        }
    }
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    const int ni = 1024, nk = 80, nj = 1024;  // 671 MB: streams from HBM
    double *buf;
    cudaMalloc(&buf, (size_t)ni * nk * nj * 8);
    cudaMemset(buf, 0, (size_t)ni * nk * nj * 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Cfg {
        int nb, bx, bj, iss, S;
    } cfgs[] = {
        {5, 128, 1, 1, 4},  {5, 128, 1, 5, 4},  {35, 16, 1, 1, 4}, {35, 16, 1, 8, 4},  {35, 16, 1, 32, 4},
        {10, 16, 4, 1, 4},  {10, 16, 4, 10, 4}, {40, 16, 1, 8, 4}, {70, 16, 1, 32, 2}, {35, 16, 1, 8, 5},
        {20, 16, 2, 8, 4},  {14, 16, 4, 8, 2},
    };
    for (auto c : cfgs) {
        CUtensorMap m;
        cuuint64_t dims[3] = {(cuuint64_t)ni, (cuuint64_t)nk, (cuuint64_t)nj};
        cuuint64_t strides[2] = {(cuuint64_t)ni * 8, (cuuint64_t)ni * nk * 8};
        cuuint32_t box[3] = {(cuuint32_t)c.bx, 8, (cuuint32_t)c.bj}, es[3] = {1, 1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int slot = c.nb * c.bx * 8 * c.bj * 8;
        const int smem = c.S * slot + 2 * c.S * 8;
        if (r != CUDA_SUCCESS || smem > 227 * 1024) {
            printf("skip nb=%d box %dx8x%d S=%d (enc %d, smem %d)\n", c.nb, c.bx, c.bj, c.S, (int)r, smem);
            continue;
        }
        for (int grid : {sms, 16}) {
        const int iters = (int)((2048ll << 20) / sms / slot);  // ~2 GB total at the full grid
        stream<<<grid, 64, smem>>>(m, c.nb, c.bx, c.bj, c.iss, c.S, 16, ni, nj, nk);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        stream<<<grid, 64, smem>>>(m, c.nb, c.bx, c.bj, c.iss, c.S, iters, ni, nj, nk);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = (double)grid * iters * slot;
        printf("grid %3d chunk = %2d boxes of %3dx8x%d (%5d B each, %6d B/chunk) S=%d issue lanes %2d: %7.1f GB/s total, %5.1f GB/s per "
               "CTA, %.1f ns per box per CTA (err %d)\n",
               grid, c.nb, c.bx, c.bj, c.bx * 64 * c.bj, slot, c.S, c.iss, bytes / ms / 1e6, bytes / ms / 1e6 / grid,
               ms * 1e6 / ((double)iters * c.nb), (int)cudaGetLastError());
        }
    }
    return 0;
}
