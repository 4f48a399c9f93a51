// Host side of tma.h: encode a 3D tensor map over an oec_field's allocation.
#include <cudaTypedefs.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "tma.h"

namespace oec {

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_once;

static void load_encode() {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
        g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
}

bool pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("OEC_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

bool make_tmap(const oec_field *f, const int box[3], TMap *out, int l2_promotion) {
    std::call_once(g_once, load_encode);
    if (!g_encode || !f || f->stride[0] != 1) return false;
    if (f->stride[2] == 0) return false;  // k-invariant: not a TMA tensor
    const int esz = f->dtype == OEC_F32 ? 4 : 8;
    const int64_t sj = f->stride[1], sk = f->stride[2];
    if (sj <= 0 || sk <= 0 || (sj * esz % 16) || (sk * esz % 16)) return false;  // strides: 16-byte multiples
    const uintptr_t data = (uintptr_t)f->data;
    const uintptr_t base = data & ~(uintptr_t)15;
    const int ioff = (int)((data - base) / esz);
    const int64_t ni = f->ub[0] - f->lb[0] + ioff, nj = f->ub[1] - f->lb[1], nk = f->ub[2] - f->lb[2];
    const int swap = sk < sj;  // dims ordered by stride
    cuuint64_t dims[3] = {(cuuint64_t)ni, (cuuint64_t)(swap ? nk : nj), (cuuint64_t)(swap ? nj : nk)};
    cuuint64_t strides[2] = {(cuuint64_t)((swap ? sk : sj) * esz), (cuuint64_t)((swap ? sj : sk) * esz)};
    cuuint32_t bx[3] = {(cuuint32_t)box[0], (cuuint32_t)(swap ? box[2] : box[1]), (cuuint32_t)(swap ? box[1] : box[2])};
    cuuint32_t es[3] = {1, 1, 1};
    if (bx[0] * esz % 16 || bx[0] > 256 || bx[1] > 256 || bx[2] > 256) return false;
    memset(out, 0, sizeof *out);
    const CUtensorMapL2promotion promo = l2_promotion >= 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                         : l2_promotion >= 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                               : CU_TENSOR_MAP_L2_PROMOTION_NONE;
    CUresult r = g_encode(&out->map, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)base, dims, strides, bx, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    out->ioff = ioff;
    out->lb0 = (int32_t)f->lb[0];
    out->lb1 = (int32_t)f->lb[1];
    out->lb2 = (int32_t)f->lb[2];
    out->kj_swap = swap;
    return true;
}

// 2D (i, j) tensor map over a k-invariant field (stride[2] == 0), box {box[0], box[1]}; the
// third coordinate of the 3D interface is absent.  Same alignment rules as make_tmap.
bool make_tmap2d(const oec_field *f, const int box[2], TMap *out) {
    std::call_once(g_once, load_encode);
    if (!g_encode || !f || f->stride[0] != 1 || f->stride[2] != 0) return false;
    const int esz = f->dtype == OEC_F32 ? 4 : 8;
    const int64_t sj = f->stride[1];
    if (sj <= 0 || (sj * esz % 16)) return false;
    const uintptr_t data = (uintptr_t)f->data;
    const uintptr_t base = data & ~(uintptr_t)15;
    const int ioff = (int)((data - base) / esz);
    cuuint64_t dims[2] = {(cuuint64_t)(f->ub[0] - f->lb[0] + ioff), (cuuint64_t)(f->ub[1] - f->lb[1])};
    cuuint64_t strides[1] = {(cuuint64_t)(sj * esz)};
    cuuint32_t bx[2] = {(cuuint32_t)box[0], (cuuint32_t)box[1]};
    cuuint32_t es[2] = {1, 1};
    if (bx[0] * esz % 16 || bx[0] > 256 || bx[1] > 256) return false;
    memset(out, 0, sizeof *out);
    CUresult r = g_encode(&out->map, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                          (void *)base, dims, strides, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    out->ioff = ioff;
    out->lb0 = (int32_t)f->lb[0];
    out->lb1 = (int32_t)f->lb[1];
    out->lb2 = 0;
    out->kj_swap = 0;
    return true;
}

}  // namespace oec
