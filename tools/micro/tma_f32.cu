// Which 3D FLOAT32 TMA boxes / coordinates are legal?  argv: esize box0 box1 c0 base_off_bytes
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c1, int bytes, float *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *bar = (uint64_t *)(sm + 64 * 1024);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(bytes));
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                     ::"r"(su(sm)), "l"((uint64_t)&m), "r"(su(bar)), "r"(c0), "r"(c1), "r"(0) : "memory");
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}" ::"r"(su(bar)) : "memory");
        out[0] = ((float *)sm)[0];
    }
}
int main(int argc, char **argv) {
    int es = atoi(argv[1]), b0 = atoi(argv[2]), b1 = atoi(argv[3]), c0 = atoi(argv[4]), off = atoi(argv[5]);
    void *fn; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    char *buf; cudaMalloc(&buf, 1 << 24); cudaMemset(buf, 0, 1 << 24);
    float *out; cudaMalloc(&out, 16);
    const int pitch = 256;  // elements
    cuuint64_t dims[3] = {(cuuint64_t)(pitch - 8), 64, 4};
    cuuint64_t strides[2] = {(cuuint64_t)pitch * es, (cuuint64_t)pitch * 64 * es};
    cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, 1}, ones[3] = {1, 1, 1};
    CUtensorMap m;
    CUresult r = enc(&m, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, buf + 1024 + off, dims,
                     strides, box, ones, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    k<<<1, 32, 80 * 1024>>>(m, c0, -2, b0 * b1 * es, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("es=%d box=(%d,%d) c0=%d off=%d encode=%d -> %s\n", es, b0, b1, c0, off, (int)r, cudaGetErrorString(e));
    return 0;
}
