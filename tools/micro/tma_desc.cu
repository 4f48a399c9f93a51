// Does rotating among several tensor-map descriptors slow TMA issue?  One CTA per SM, one producer
// thread issues boxes round-robin over D descriptors (same buffer); also 1D cp.async.bulk rows.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t *b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(su(b)), "r"(ph) : "memory");
}
struct Maps { CUtensorMap m[5]; };
constexpr int S = 8, PER = 5;  // slot = PER boxes of 128x4 doubles (20 KB), like vadv
__global__ void tma_multi(const __grid_constant__ Maps maps, int D, int nrows, int iters, unsigned long long *tstamp) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int box = 4096, slot = PER * box;
    uint64_t *full = (uint64_t *)(sm + S * slot), *empty = full + S;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int n = 0; n < iters; ++n) {
            int s = n % S;
            if (n >= S) wait(&empty[s], ((n / S) - 1) & 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(slot));
            for (int p = 0; p < PER; ++p) {
                int rb = ((blockIdx.x * 7919 + n * 131 + p * 17) % (nrows / 4)) * 4;
                const CUtensorMap *m = &maps.m[p % D];
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                             ::"r"(su(sm + s * slot + p * box)), "l"((uint64_t)m), "r"(su(&full[s])), "r"(0), "r"(rb) : "memory");
            }
        }
    } else if (threadIdx.x == 32) {
        for (int n = 0; n < iters; ++n) {
            int s = n % S;
            wait(&full[s], (n / S) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])));
        }
    }
}
__global__ void bulk_rows(const double *buf, int nrows, int iters) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int row = 1024, slot = PER * 4 * row;
    uint64_t *full = (uint64_t *)(sm + S * slot), *empty = full + S;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int n = 0; n < iters; ++n) {
            int s = n % S;
            if (n >= S) wait(&empty[s], ((n / S) - 1) & 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(slot));
            for (int p = 0; p < PER * 4; ++p) {
                long long rb = ((blockIdx.x * 7919ll + n * 131 + p * 17) % nrows);
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su(sm + s * slot + p * row)), "l"(buf + rb * 128), "r"(row), "r"(su(&full[s])) : "memory");
            }
        }
    } else if (threadIdx.x == 32) {
        for (int n = 0; n < iters; ++n) {
            int s = n % S;
            wait(&full[s], (n / S) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])));
        }
    }
}
int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    const long long ncols = 128, nrows = 4 * 1024 * 1024;
    double *buf;
    cudaMalloc(&buf, ncols * nrows * 8);
    cudaMemset(buf, 0, ncols * nrows * 8);
    Maps maps;
    for (int d = 0; d < 5; ++d) {
        cuuint64_t dims[2] = {(cuuint64_t)ncols, (cuuint64_t)nrows};
        cuuint64_t strides[1] = {(cuuint64_t)ncols * 8};
        cuuint32_t box[2] = {128, 4}, es[2] = {1, 1};
        enc(&maps.m[d], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int smem = S * PER * 4096 + 2 * S * 8;
    cudaFuncSetAttribute(tma_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bulk_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int D : {1, 2, 5})
        for (int grid : {1, 128, sms}) {
            int iters = 2000;
            tma_multi<<<grid, 64, smem>>>(maps, D, (int)nrows, 16, nullptr);
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            tma_multi<<<grid, 64, smem>>>(maps, D, (int)nrows, iters, nullptr);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double bytes = (double)grid * iters * PER * 4096;
            printf("TMA 20KB slots (5 boxes 128x4) D=%d descriptors, grid %3d: %7.1f GB/s total, %6.1f per SM (err %d)\n", D,
                   grid, bytes / ms / 1e6, bytes / ms / 1e6 / grid, (int)cudaGetLastError());
        }
    for (int grid : {1, 128, sms}) {
        int iters = 2000;
        bulk_rows<<<grid, 64, smem>>>(buf, (int)nrows, 16);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        bulk_rows<<<grid, 64, smem>>>(buf, (int)nrows, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double bytes = (double)grid * iters * PER * 4096;
        printf("BULK 20KB slots (20 rows of 1KB),               grid %3d: %7.1f GB/s total, %6.1f per SM (err %d)\n", grid,
               bytes / ms / 1e6, bytes / ms / 1e6 / grid, (int)cudaGetLastError());
    }
    return 0;
}
