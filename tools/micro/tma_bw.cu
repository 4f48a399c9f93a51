// Per-SM streaming throughput: TMA tensor boxes into an smem ring (one producer thread, one
// consumer warp that just re-arms) vs plain coalesced LDG.128, at various grid sizes.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t *b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(su(b)), "r"(ph) : "memory");
}
template <int S>
__global__ void tma_stream(const __grid_constant__ CUtensorMap m, int bx, int by, int rows_total, int iters, int slot_bytes) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = (uint64_t *)(sm + S * slot_bytes), *empty = full + S;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int nrb = rows_total / by;
    if (threadIdx.x == 0) {
        for (int n = 0; n < iters; ++n) {
            int s = n % S;
            if (n >= S) wait(&empty[s], ((n / S) - 1) & 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(slot_bytes));
            int rb = (blockIdx.x * 7919 + n * 131) % nrb;
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                         ::"r"(su(sm + s * slot_bytes)), "l"((uint64_t)&m), "r"(su(&full[s])), "r"(0), "r"(rb * by) : "memory");
        }
    } else if (threadIdx.x == 32) {
        for (int n = 0; n < iters; ++n) {
            int s = n % S;
            wait(&full[s], (n / S) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])));
        }
    }
}
__global__ void ldg_stream(const double4 *src, double *sink, long long n4, int iters_per_thread) {
    long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, stride = (long long)gridDim.x * blockDim.x;
    double acc = 0;
    for (long long t = tid; t < n4; t += stride) { const double2 *p2 = (const double2 *)(src + t); double2 v = __ldg(p2), w = __ldg(p2 + 1); acc += v.x + v.y + w.x + w.y; }
    if (acc == 12345.678) sink[0] = acc;
}
int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    const long long ncols = 128, nrows = 4 * 1024 * 1024;  // 4M rows x 1 KB = 4 GiB
    double *buf;
    cudaMalloc(&buf, ncols * nrows * 8);
    cudaMemset(buf, 0, ncols * nrows * 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int boxes[][2] = {{128, 4}, {128, 8}, {128, 16}, {128, 32}, {64, 16}, {32, 32}};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (auto &b : boxes) {
        CUtensorMap m;
        cuuint64_t dims[2] = {(cuuint64_t)ncols, (cuuint64_t)nrows};
        cuuint64_t strides[1] = {(cuuint64_t)ncols * 8};
        cuuint32_t box[2] = {(cuuint32_t)b[0], (cuuint32_t)b[1]}, es[2] = {1, 1};
        enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        int slot = b[0] * b[1] * 8;
        const int S = 8;
        int smem = S * slot + 2 * S * 8;
        cudaFuncSetAttribute(tma_stream<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        for (int grid : {1, 16, sms / 2, sms}) {
            int iters = (int)((512ll << 20) / sms / slot);  // ~512 MB total at full grid
            if (smem > 227 * 1024) continue;
            tma_stream<S><<<grid, 64, smem>>>(m, b[0], b[1], (int)nrows, 8, slot);
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            tma_stream<S><<<grid, 64, smem>>>(m, b[0], b[1], (int)nrows, iters, slot);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double bytes = (double)grid * iters * slot;
            printf("TMA box %3dx%-3d (%6d B) S=%d grid %3d: %8.1f GB/s total, %6.1f GB/s per SM  (%d)\n", b[0], b[1], slot,
                   S, grid, bytes / ms / 1e6, bytes / ms / 1e6 / grid, (int)cudaGetLastError());
        }
    }
    double *sink;
    cudaMalloc(&sink, 8);
    for (int grid : {1, 16, sms / 2, sms, 4 * sms}) {
        long long n4 = (grid >= sms ? (512ll << 20) : (64ll << 20) * grid / 16 + (8 << 20)) / 32;
        ldg_stream<<<grid, 1024>>>((const double4 *)buf, sink, n4, 0);
        cudaEventRecord(e0);
        ldg_stream<<<grid, 1024>>>((const double4 *)buf, sink, n4, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("LDG.256 1024 thr/CTA grid %3d: %8.1f GB/s total, %6.1f GB/s per CTA\n", grid, n4 * 32.0 / ms / 1e6,
               n4 * 32.0 / ms / 1e6 / grid);
    }
    return 0;
}
