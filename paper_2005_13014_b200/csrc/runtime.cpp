// liboec host runtime: field descriptors, program registry (access extents), validation,
// host staging for the end-to-end path, and dispatch to the sm_100a kernels.
//
// Registry extents are shape inference (§5.2) done once by hand per program:
// the minimal bounding box of every access of every inlined operator.  tests/test_abi_host.py
// checks them against the oracle's brute-force touched-index trace.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "oec_internal.h"

namespace oec {

static thread_local char g_err[1024];
static thread_local int g_launches;

void set_launch_count(int n) { g_launches = n; }

oec_status set_error(oec_status st, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return st;
}

// ---------------------------------------------------------------------------------------------
// program registry
// ---------------------------------------------------------------------------------------------
struct InSpec {
    const char *name;
    int lo[3], hi[3];  // access extent relative to the domain
    int k_invariant;
};
struct ScSpec {
    const char *name;
    double dflt;
};
struct ProgSpec {
    const char *name;
    int n_in, n_out, n_sc;
    InSpec in[9];
    const char *out[3];
    ScSpec sc[2];
};

#define Z3 {0, 0, 0}
static const ProgSpec PROGS[OEC_NPROG] = {
    {"hdiff", 2, 1, 0, {{"in", {-2, -2, 0}, {2, 2, 0}, 0}, {"coeff", Z3, Z3, 0}}, {"out"}, {}},
    {"vadv",
     5,
     1,
     1,
     {{"u_stage", Z3, Z3, 0},
      {"wcon", Z3, {1, 0, 0}, 0},
      {"u_pos", Z3, Z3, 0},
      {"utens", Z3, Z3, 0},
      {"utens_stage_in", Z3, Z3, 0}},
     {"utens_stage_out"},
     {{"dtr_stage", 3.0 / 20.0}}},
    {"uvbke",
     4,
     2,
     1,
     {{"uc", {0, -1, 0}, Z3, 0}, {"vc", {-1, 0, 0}, Z3, 0}, {"cosa", Z3, Z3, 1}, {"rsina", Z3, Z3, 1}},
     {"ub", "vb"},
     {{"dt5", 0.5 * 225.0 / 1000.0}}},
    {"p_grad_c",
     7,
     2,
     1,
     {{"uc", Z3, Z3, 0},
      {"vc", Z3, Z3, 0},
      {"delpc", {-1, -1, 0}, Z3, 0},
      {"pkc", {-1, -1, 0}, {0, 0, 1}, 0},
      {"gz", {-1, -1, 0}, {0, 0, 1}, 0},
      {"rdxc", Z3, Z3, 1},
      {"rdyc", Z3, Z3, 1}},
     {"uc_out", "vc_out"},
     {{"dt2", 0.5 * 225.0 / 1000.0}}},
    {"nh_p_grad",
     8,
     2,
     1,
     {{"u", Z3, Z3, 0},
      {"v", Z3, Z3, 0},
      {"pp", Z3, {1, 1, 1}, 0},
      {"gz", Z3, {1, 1, 1}, 0},
      {"pk3", Z3, {1, 1, 1}, 0},
      {"delp", Z3, {1, 1, 0}, 0},
      {"rdx", Z3, Z3, 1},
      {"rdy", Z3, Z3, 1}},
     {"u_out", "v_out"},
     {{"dt", 225.0 / 1000.0}}},
    {"fvtp2d_qi",
     5,
     2,
     0,
     {{"q", {0, -3, 0}, {0, 3, 0}, 0},
      {"cry", Z3, {0, 1, 0}, 0},
      {"yfx", Z3, {0, 1, 0}, 0},
      {"area", Z3, Z3, 1},
      {"ra_y", Z3, Z3, 0}},
     {"q_i", "fy2"},
     {}},
    {"fvtp2d_qj",
     6,
     3,
     0,
     {{"q", {-3, 0, 0}, {3, 0, 0}, 0},
      {"q_i", {-3, 0, 0}, {2, 0, 0}, 0},
      {"crx", Z3, {1, 0, 0}, 0},
      {"xfx", Z3, {1, 0, 0}, 0},
      {"area", Z3, Z3, 1},
      {"ra_x", Z3, Z3, 0}},
     {"q_j", "fx", "fx2"},
     {}},
    {"fvtp2d_flux",
     7,
     2,
     0,
     {{"q_j", {0, -3, 0}, {0, 2, 0}, 0},
      {"cry", Z3, Z3, 0},
      {"fx", Z3, Z3, 0},
      {"fx2", Z3, Z3, 0},
      {"fy2", Z3, Z3, 0},
      {"mfx", Z3, Z3, 0},
      {"mfy", Z3, Z3, 0}},
     {"fx_out", "fy_out"},
     {}},
    {"fastwaves",
     9,
     2,
     2,
     {{"u_pos", Z3, Z3, 0},
      {"v_pos", Z3, Z3, 0},
      {"u_tens", Z3, Z3, 0},
      {"v_tens", Z3, Z3, 0},
      {"rho", Z3, {1, 1, 0}, 0},
      {"ppuv", {0, 0, -1}, {1, 1, 1}, 0},
      {"fx", Z3, Z3, 1},
      {"wgtfac", Z3, {1, 1, 1}, 0},
      {"hhl", Z3, {1, 1, 1}, 0}},
     {"u_out", "v_out"},
     {{"edadlat", 0.25}, {"dt", 10.0 / 1000.0}}},
};

static int find_prog(const char *name) {
    if (!name) return -1;
    for (int p = 0; p < OEC_NPROG; ++p)
        if (strcmp(PROGS[p].name, name) == 0) return p;
    return -1;
}

// ---------------------------------------------------------------------------------------------
// validation
// ---------------------------------------------------------------------------------------------
static int esize(int32_t dtype) { return dtype == OEC_F32 ? 4 : 8; }

static bool span_bytes(const oec_field *f, uintptr_t *lo, uintptr_t *hi) {
    // byte range [lo, hi) spanned by the allocation of f
    int64_t mn = 0, mx = 0;
    for (int d = 0; d < 3; ++d) {
        int64_t n = f->ub[d] - f->lb[d];
        if (n <= 0) return false;
        int64_t e = (n - 1) * f->stride[d];
        if (e < 0) mn += e; else mx += e;
    }
    const int es = esize(f->dtype);
    *lo = (uintptr_t)f->data + (uintptr_t)(mn * es);
    *hi = (uintptr_t)f->data + (uintptr_t)((mx + 1) * es);
    return true;
}

static oec_status check_field(const oec_field *f, const char *what, int *device, int *dtype) {
    if (!f || !f->data) return set_error(OEC_ERR_ARG, "%s: NULL field or data pointer", what);
    if (f->dtype != OEC_F64 && f->dtype != OEC_F32)
        return set_error(OEC_ERR_DTYPE, "%s: dtype %d is neither OEC_F64 nor OEC_F32", what, f->dtype);
    if (*dtype == -1) *dtype = f->dtype;
    else if (*dtype != f->dtype)
        return set_error(OEC_ERR_DTYPE, "%s: dtype %d differs from the other fields' dtype %d", what, f->dtype, *dtype);
    if (*device == -2) *device = f->device;
    else if (*device != f->device)
        return set_error(OEC_ERR_DTYPE, "%s: device %d differs from the other fields' device %d", what, f->device,
                         *device);
    if (f->stride[0] != 1) return set_error(OEC_ERR_LAYOUT, "%s: stride[0] = %lld, must be 1", what, (long long)f->stride[0]);
    for (int d = 0; d < 3; ++d)
        if (f->ub[d] <= f->lb[d]) return set_error(OEC_ERR_SHAPE, "%s: empty allocation in dim %d", what, d);
    if (((uintptr_t)f->data) % esize(f->dtype))
        return set_error(OEC_ERR_LAYOUT, "%s: data not %d-byte aligned", what, esize(f->dtype));
    return OEC_OK;
}

static bool is_k_invariant(const oec_field *f) { return f->stride[2] == 0 && f->ub[2] - f->lb[2] == 1 && f->lb[2] == 0; }

// make the kernel view; checks every allocated element is reachable with int32 offsets from the origin
template <class V>
static oec_status make_view(const oec_field *f, const char *what, V *v) {
    int64_t sj = f->stride[1], sk = is_k_invariant(f) ? 0 : f->stride[2];
    if (sj > INT32_MAX || sk > INT32_MAX || sj < INT32_MIN || sk < INT32_MIN)
        return set_error(OEC_ERR_LAYOUT, "%s: stride exceeds int32", what);
    int64_t lbk = is_k_invariant(f) ? 0 : f->lb[2];
    int64_t origin_off = -(f->lb[0] + f->lb[1] * sj + lbk * sk);  // element offset of (0,0,0) from data
    for (int c = 0; c < 8; ++c) {
        int64_t i = (c & 1) ? f->ub[0] - 1 : f->lb[0];
        int64_t j = (c & 2) ? f->ub[1] - 1 : f->lb[1];
        int64_t k = (c & 4) ? f->ub[2] - 1 : f->lb[2];
        int64_t off = i + j * sj + k * sk;
        if (off > INT32_MAX || off < INT32_MIN)
            return set_error(OEC_ERR_LAYOUT, "%s: element offsets exceed int32 (field too large for this build)", what);
    }
    v->p = (decltype(v->p))((char *)f->data + origin_off * (int64_t)sizeof(*v->p));
    v->sj = (int32_t)sj;
    v->sk = (int32_t)sk;
    return OEC_OK;
}

// exported to the other translation units (csrc/pipeline.cpp)
template <class V>
oec_status field_view(const oec_field *f, const char *what, V *v) {
    return make_view(f, what, v);
}
template oec_status field_view<FVT<double>>(const oec_field *, const char *, FVT<double> *);
template oec_status field_view<FVT<float>>(const oec_field *, const char *, FVT<float> *);
template oec_status field_view<FOT<double>>(const oec_field *, const char *, FOT<double> *);
template oec_status field_view<FOT<float>>(const oec_field *, const char *, FOT<float> *);
oec_status field_check(const oec_field *f, const char *what, int *device, int *dtype) {
    return check_field(f, what, device, dtype);
}
bool field_span(const oec_field *f, uintptr_t *lo, uintptr_t *hi) { return span_bytes(f, lo, hi); }
bool field_overlap(const oec_field *a, const oec_field *b) {
    uintptr_t alo, ahi, blo, bhi;
    if (!span_bytes(a, &alo, &ahi) || !span_bytes(b, &blo, &bhi)) return false;
    return alo < bhi && blo < ahi;
}

static oec_status check_domain(const int64_t *lo, const int64_t *hi) {
    if (!lo || !hi) return set_error(OEC_ERR_ARG, "NULL domain");
    for (int d = 0; d < 3; ++d) {
        if (hi[d] < lo[d]) return set_error(OEC_ERR_SHAPE, "domain dim %d: ub %lld < lb %lld", d, (long long)hi[d], (long long)lo[d]);
        if (lo[d] < INT32_MIN / 2 || hi[d] > INT32_MAX / 2) return set_error(OEC_ERR_LAYOUT, "domain bounds exceed int32");
    }
    return OEC_OK;
}

static bool domain_empty(const int64_t *lo, const int64_t *hi) {
    return hi[0] <= lo[0] || hi[1] <= lo[1] || hi[2] <= lo[2];
}

static oec_status check_cover(const oec_field *f, const char *what, const int64_t *lo, const int64_t *hi,
                              const int *elo, const int *ehi, int k_inv) {
    if (k_inv && !is_k_invariant(f))
        return set_error(OEC_ERR_SHAPE, "%s: must be a k-invariant (2D) field: lb[2]=0, ub[2]=1, stride[2]=0", what);
    for (int d = 0; d < 3; ++d) {
        if (d == 2 && is_k_invariant(f)) continue;
        int64_t need_lo = lo[d] + elo[d], need_hi = hi[d] + ehi[d];
        if (f->lb[d] > need_lo || f->ub[d] < need_hi)
            return set_error(OEC_ERR_SHAPE,
                             "%s: allocation [%lld,%lld) in dim %d does not cover the accessed range [%lld,%lld) "
                             "(domain + access extent, P:482)",
                             what, (long long)f->lb[d], (long long)f->ub[d], d, (long long)need_lo, (long long)need_hi);
    }
    return OEC_OK;
}

// ---------------------------------------------------------------------------------------------
// host staging (end-to-end path, device == OEC_DEVICE_HOST)
// ---------------------------------------------------------------------------------------------
constexpr int STAGE_SLABS = 8;
struct Staging {
    std::mutex mu;
    std::vector<void *> bufs;
    std::vector<size_t> sizes;
    int device = -1;
    cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of the pipelined host path
    cudaEvent_t ev[2 * STAGE_SLABS] = {};
};
// One staging set per (device, caller stream): host-path calls on different streams run
// concurrently -- e.g. one program's H2D while another's D2H, PCIe being full duplex -- and calls
// on one stream are serialised by its set's mutex.  A set lives for the life of the process
// (its buffers only grow), so a caller should reuse a few streams, not create one per call.
static std::mutex g_stages_mu;
static std::map<std::pair<int, cudaStream_t>, std::unique_ptr<Staging>> g_stages;

static Staging &stage_for(cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_stages_mu);
    auto &p = g_stages[std::make_pair(dev, s)];
    if (!p) {
        p.reset(new Staging);
        p->device = dev;
    }
    return *p;
}

static oec_status stage_buffer(Staging &S, size_t idx, size_t bytes, void **p) {
    if (S.bufs.size() <= idx) {
        S.bufs.resize(idx + 1, nullptr);
        S.sizes.resize(idx + 1, 0);
    }
    if (S.sizes[idx] < bytes) {
        if (S.bufs[idx]) cudaFree(S.bufs[idx]);
        S.bufs[idx] = nullptr;
        S.sizes[idx] = 0;
        cudaError_t e = cudaMalloc(&S.bufs[idx], bytes);
        if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "staging cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
        S.sizes[idx] = bytes;
    }
    *p = S.bufs[idx];
    return OEC_OK;
}

// copy the allocated rows j in [j0, j1) (all i and k) of a host field into its device twin
static cudaError_t h2d_rows(const oec_field *dev, const oec_field *host, int64_t j0, int64_t j1, cudaStream_t s) {
    const int es = esize(host->dtype);
    const int64_t ni = host->ub[0] - host->lb[0], nk = host->ub[2] - host->lb[2], s1 = host->stride[1];
    const int64_t off = (j0 - host->lb[1]) * s1;
    const char *src = (const char *)host->data + off * es;
    char *dst = (char *)dev->data + off * es;
    if (is_k_invariant(host) || nk == 1)  // rows only
        return cudaMemcpy2DAsync(dst, s1 * es, src, s1 * es, ni * es, j1 - j0, cudaMemcpyHostToDevice, s);
    const int64_t s2 = host->stride[2];
    if (s1 >= s2 * nk)  // j outermost (default i, k, j layout): the rows are one contiguous block
        return cudaMemcpyAsync(dst, src, ((j1 - j0 - 1) * s1 + (nk - 1) * s2 + ni) * es, cudaMemcpyHostToDevice, s);
    // k outermost: one 2D copy, a (j1-j0) x pitch block per level
    return cudaMemcpy2DAsync(dst, s2 * es, src, s2 * es, ((j1 - j0 - 1) * s1 + ni) * es, nk, cudaMemcpyHostToDevice, s);
}

// copy the domain box of a strided device field back into the same-layout host field
static cudaError_t d2h_box(const oec_field *host, const oec_field *dev, const int64_t *lo, const int64_t *hi,
                           cudaStream_t s) {
    // the box spans whole rows and planes of a dense i, j, k field: one contiguous copy
    {
        const int64_t ni = host->ub[0] - host->lb[0], nj = host->ub[1] - host->lb[1];
        if (!is_k_invariant(host) && host->stride[1] == ni && host->stride[2] == ni * nj && lo[0] == host->lb[0] &&
            hi[0] == host->ub[0] && lo[1] == host->lb[1] && hi[1] == host->ub[1]) {
            const int es = esize(host->dtype);
            const int64_t off = (lo[2] - host->lb[2]) * host->stride[2];
            return cudaMemcpyAsync((char *)host->data + off * es, (const char *)dev->data + off * es,
                                   (hi[2] - lo[2]) * ni * nj * es, cudaMemcpyDeviceToHost, s);
        }
    }
    // whole dense i rows, k outermost (a j-slab of a numpy-style [k][j][i] field): the box's rows
    // of one level are contiguous -- one 2D copy over the levels (round 1 issued one 2D copy per
    // level: 80 API calls per field and slab, which made the slab pipeline slower than one slab)
    {
        const int64_t ni = host->ub[0] - host->lb[0];
        if (!is_k_invariant(host) && host->stride[1] == ni && host->stride[2] >= ni * (host->ub[1] - host->lb[1]) &&
            dev->stride[1] == ni && dev->stride[2] == host->stride[2] && lo[0] == host->lb[0] && hi[0] == host->ub[0]) {
            const int es = esize(host->dtype);
            const int64_t off = (lo[1] - host->lb[1]) * ni + (lo[2] - host->lb[2]) * host->stride[2];
            return cudaMemcpy2DAsync((char *)host->data + off * es, host->stride[2] * es, (const char *)dev->data + off * es,
                                     dev->stride[2] * es, (hi[1] - lo[1]) * ni * es, hi[2] - lo[2], cudaMemcpyDeviceToHost, s);
        }
    }
    // outer loop over the dimension with the larger stride, 2D copies over the other two
    int outer = (host->stride[2] >= host->stride[1]) ? 2 : 1;
    int mid = 3 - outer;
    const int es = esize(host->dtype);
    int64_t w = (hi[0] - lo[0]) * es;
    for (int64_t o = lo[outer]; o < hi[outer]; ++o) {
        int64_t idx[3] = {lo[0], 0, 0};
        idx[outer] = o;
        idx[mid] = lo[mid];
        int64_t off = (idx[0] - host->lb[0]) + (idx[1] - host->lb[1]) * host->stride[1] +
                      (is_k_invariant(host) ? 0 : (idx[2] - host->lb[2]) * host->stride[2]);
        cudaError_t e = cudaMemcpy2DAsync((char *)host->data + off * es, host->stride[mid] * es,
                                          (char *)dev->data + off * es, dev->stride[mid] * es, w, hi[mid] - lo[mid],
                                          cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// ---------------------------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------------------------
// AUTO's unroll factor per suite program: the paper picks it by empirical tuning; these are
// the fastest of 1 / 2 / 4 measured on B200 at 128x128x80 (bench.py optimization_levels,
// profiles/ncu_summary_r01.md)
static int unroll_of(int p, int variant) {
    if (variant == OEC_VARIANT_AUTO) return (p == OEC_PROG_UVBKE || p == OEC_PROG_FVTP2D_QI) ? 2 : 1;
    return variant == OEC_VARIANT_UNROLL2 ? 2 : variant == OEC_VARIANT_UNROLL4 ? 4 : 1;
}

template <class T>
static oec_status run_device(int p, const oec_field *const *in, oec_field *const *out, const double *sc,
                             const int64_t *lo, const int64_t *hi, int variant, cudaStream_t s) {
    const ProgSpec &P = PROGS[p];
    FVT<T> v_in[9];
    FOT<T> v_out[3];
    constexpr int V16 = 16 / (int)sizeof(T);  // elements per 16 bytes
    bool aligned16 = true;
    for (int q = 0; q < P.n_in; ++q) {
        oec_status st = make_view(in[q], P.in[q].name, &v_in[q]);
        if (st) return st;
        aligned16 = aligned16 && ((uintptr_t)v_in[q].p % 16 == 0) && (v_in[q].sj % V16 == 0) && (v_in[q].sk % V16 == 0);
    }
    for (int q = 0; q < P.n_out; ++q) {
        oec_status st = make_view(out[q], P.out[q], &v_out[q]);
        if (st) return st;
        aligned16 = aligned16 && ((uintptr_t)v_out[q].p % 16 == 0) && (v_out[q].sj % V16 == 0) && (v_out[q].sk % V16 == 0);
    }
    Dom d;
    for (int q = 0; q < 3; ++q) {
        d.lo[q] = (int32_t)lo[q];
        d.hi[q] = (int32_t)hi[q];
    }
    aligned16 = aligned16 && (d.lo[0] % V16 == 0);
    int launches = 0;
    cudaError_t e;
    if (variant == OEC_VARIANT_UNFUSED) {
        if (p == OEC_PROG_HDIFF) e = launch_hdiff_unfused<T>(v_in[0], v_in[1], v_out[0], d, s, &launches);
        else if (p == OEC_PROG_VADV)
            e = launch_vadv_unfused<T>(v_in[0], v_in[1], v_in[2], v_in[3], v_in[4], v_out[0], sc[0], d, s, &launches);
        else e = launch_suite_unfused<T>(p, P.n_in, v_in, v_out, sc, d, s, &launches);
        if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "%s (unfused): %s", P.name, cudaGetErrorString(e));
        g_launches = launches;
        return OEC_OK;
    }
    switch (p) {
    case OEC_PROG_HDIFF: {
        TMap tin, tcf;
        int bin[3], bcf[3];
        hdiff_tma_boxes<T>(d, bin, bcf);
        const bool tma = variant == OEC_VARIANT_AUTO && make_tmap(in[0], bin, &tin, HD_PROMO) && make_tmap(in[1], bcf, &tcf, HD_PROMO);
        e = launch_hdiff<T>(v_in[0], v_in[1], v_out[0], d, variant, aligned16, tma ? &tin : nullptr, tma ? &tcf : nullptr,
                         s, &launches);
        break;
    }
    case OEC_PROG_VADV: {
        // TMA path: u_stage, wcon, u_pos, utens, utens_stage_in (tmaps[0..4])
        TMap tm[5];
        int box[3], bwc[3], bus[3];
        bool fits;
        vadv_tma_boxes<T>(d, box, bwc, bus, &fits);
        bool tma = fits && aligned16 && variant == OEC_VARIANT_AUTO;
#ifndef VA_PROMO
#define VA_PROMO 0  // no L2 sector promotion for vadv's 1 KB rows: 0.68 -> 0.69 at 128^2 (profiles/l2_prefetch_r02.md)
#endif
        for (int q = 0; q < 5 && tma; ++q) tma = make_tmap(in[q], q == 0 ? bus : (q == 1 ? bwc : box), &tm[q], VA_PROMO);
        if constexpr (sizeof(T) == 4)
            e = launch_vadv_f32(v_in[0], v_in[1], v_in[2], v_in[3], v_in[4], v_out[0], sc[0], d, tma ? tm : nullptr, s,
                                &launches);
        else
            e = launch_vadv(v_in[0], v_in[1], v_in[2], v_in[3], v_in[4], v_out[0], sc[0], d, tma ? tm : nullptr, s,
                            &launches);
        break;
    }
    default: {
        // AUTO: the library's compiler (csrc/jit.cpp) on the program's stencil-language text
        // (csrc/programs.cpp), tuned over inline / unrolled / TMA-tiled kernels; the
        // hand-written kernels serve the explicit variants, and AUTO when NVRTC is unavailable
        // (OEC_BUILTIN_JIT=0 forces them).
        static const bool use_jit = !(getenv("OEC_BUILTIN_JIT") && getenv("OEC_BUILTIN_JIT")[0] == '0');
        if (variant == OEC_VARIANT_AUTO && use_jit) {
            if (const char *txt = builtin_program_text(p)) {
                auto J = jit_internal(txt);
                if (J) {
                    oec_status st = J->run(sizeof(T) == 4 ? OEC_F32 : OEC_F64, in, out, sc, lo, hi, OEC_VARIANT_AUTO, s);
                    if (st != OEC_ERR_UNSUPPORTED) return st;  // launches counted by the JIT
                }
            }
        }
        e = launch_suite<T>(p, v_in, v_out, sc, d, unroll_of(p, variant), s, &launches);
        break;
    }
    }
    if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "%s: kernel launch failed: %s", P.name, cudaGetErrorString(e));
    g_launches = launches;
    return OEC_OK;
}

// builtin registry entries as generic descriptors (built once)
static const ProgDesc &builtin_desc(int p) {
    static std::vector<ProgDesc> descs;
    static std::once_flag once;
    std::call_once(once, [] {
        descs.resize(OEC_NPROG);
        for (int q = 0; q < OEC_NPROG; ++q) {
            const ProgSpec &S = PROGS[q];
            ProgDesc &D = descs[q];
            D.name = S.name;
            for (int r = 0; r < S.n_in; ++r) {
                D.in_names.push_back(S.in[r].name);
                D.in_lo.push_back({S.in[r].lo[0], S.in[r].lo[1], S.in[r].lo[2]});
                D.in_hi.push_back({S.in[r].hi[0], S.in[r].hi[1], S.in[r].hi[2]});
                D.in_kinv.push_back(S.in[r].k_invariant);
            }
            for (int r = 0; r < S.n_out; ++r) D.out_names.push_back(S.out[r]);
            for (int r = 0; r < S.n_sc; ++r) {
                D.sc_names.push_back(S.sc[r].name);
                D.sc_dflt.push_back(S.sc[r].dflt);
            }
            D.min_k = q == OEC_PROG_VADV ? 2 : 1;
            D.unroll_ok = q != OEC_PROG_VADV;
            D.run = [q](int dtype, const oec_field *const *in, oec_field *const *out, const double *sc, const int64_t *lo,
                        const int64_t *hi, int variant, cudaStream_t s) {
                return dtype == OEC_F32 ? run_device<float>(q, in, out, sc, lo, hi, variant, s)
                                        : run_device<double>(q, in, out, sc, lo, hi, variant, s);
            };
        }
    });
    return descs[p];
}

// the program named `name`: a builtin, else a program registered with oec_program_create
static std::shared_ptr<const ProgDesc> lookup(const char *name) {
    int p = find_prog(name);
    if (p >= 0) return std::shared_ptr<const ProgDesc>(&builtin_desc(p), [](const ProgDesc *) {});
    return name ? jit_lookup(name) : nullptr;
}

bool builtin_program(const char *name) { return find_prog(name) >= 0; }

static oec_status apply(const ProgDesc &P, const oec_field *const *in, int n_in, oec_field *const *out, int n_out,
                        const double *scalars, int n_sc, const int64_t *lo, const int64_t *hi, int variant,
                        void *stream) {
    const char *pname = P.name.c_str();
    const int P_n_in = (int)P.in_names.size(), P_n_out = (int)P.out_names.size(), P_n_sc = (int)P.sc_names.size();
    g_err[0] = 0;
    g_launches = 0;
    if (n_in != P_n_in || n_out != P_n_out)
        return set_error(OEC_ERR_ARG, "%s: expects %d inputs / %d outputs, got %d / %d", pname, P_n_in, P_n_out, n_in, n_out);
    if (!in || !out) return set_error(OEC_ERR_ARG, "%s: NULL input/output array", pname);
    if (n_sc != 0 && n_sc != P_n_sc) return set_error(OEC_ERR_ARG, "%s: expects %d scalars, got %d", pname, P_n_sc, n_sc);
    if (n_sc && !scalars) return set_error(OEC_ERR_ARG, "%s: NULL scalars", pname);
    if (variant < OEC_VARIANT_AUTO || variant > OEC_VARIANT_TILED)
        return set_error(OEC_ERR_ARG, "%s: unknown variant %d", pname, variant);
    if ((variant == OEC_VARIANT_UNROLL2_K || variant == OEC_VARIANT_UNROLL4_K || variant == OEC_VARIANT_TILED) &&
        !P.kunroll_ok)
        return set_error(OEC_ERR_UNSUPPORTED,
                         "%s: unrolling along k and the tiled variant are implemented for stencil-language programs "
                         "(oec_program_create)", pname);
    if ((variant == OEC_VARIANT_UNROLL2 || variant == OEC_VARIANT_UNROLL4) && !P.unroll_ok)
        return set_error(OEC_ERR_UNSUPPORTED,
                         "%s: stencil unrolling (P:447) does not apply to the vertical solver (independent columns, "
                         "no shared producers for CSE to remove)", pname);
    oec_status st = check_domain(lo, hi);
    if (st) return st;
    int device = -2, dtype = -1;
    for (int q = 0; q < P_n_in; ++q)
        if ((st = check_field(in[q], P.in_names[q].c_str(), &device, &dtype))) return st;
    for (int q = 0; q < P_n_out; ++q)
        if ((st = check_field(out[q], P.out_names[q].c_str(), &device, &dtype))) return st;
    for (int q = 0; q < P_n_out; ++q)
        if (is_k_invariant(out[q]))
            return set_error(OEC_ERR_SHAPE, "%s: output %s must not be k-invariant", pname, P.out_names[q].c_str());
    if (hi[2] - lo[2] < P.min_k)
        return set_error(OEC_ERR_SHAPE, "%s: K = %lld < %d (the k=0 and k=K-1 rows would coincide)", pname,
                         (long long)(hi[2] - lo[2]), P.min_k);
    static const int Z[3] = {0, 0, 0};
    bool empty = domain_empty(lo, hi);
    if (!empty) {
        for (int q = 0; q < P_n_in; ++q)
            if ((st = check_cover(in[q], P.in_names[q].c_str(), lo, hi, P.in_lo[q].data(), P.in_hi[q].data(),
                                  P.in_kinv[q])))
                return st;
        for (int q = 0; q < P_n_out; ++q)
            if ((st = check_cover(out[q], P.out_names[q].c_str(), lo, hi, Z, Z, 0))) return st;
    }
    // aliasing: an output may not overlap any input or another output
    for (int q = 0; q < P_n_out; ++q) {
        uintptr_t a0, a1;
        span_bytes(out[q], &a0, &a1);
        for (int r = 0; r < P_n_in; ++r) {
            uintptr_t b0, b1;
            span_bytes(in[r], &b0, &b1);
            if (a0 < b1 && b0 < a1)
                return set_error(OEC_ERR_ALIAS, "%s: output %s overlaps input %s (P:381 alias-free parameters)", pname,
                                 P.out_names[q].c_str(), P.in_names[r].c_str());
        }
        for (int r = 0; r < q; ++r) {
            uintptr_t b0, b1;
            span_bytes(out[r], &b0, &b1);
            if (a0 < b1 && b0 < a1)
                return set_error(OEC_ERR_ALIAS, "%s: outputs %s and %s overlap", pname, P.out_names[q].c_str(),
                                 P.out_names[r].c_str());
        }
    }
    std::vector<double> sc(P_n_sc + 1);
    for (int q = 0; q < P_n_sc; ++q) sc[q] = n_sc ? scalars[q] : P.sc_dflt[q];
    if (empty) return OEC_OK;
    cudaStream_t s = (cudaStream_t)stream;

    if (device >= 0) return P.run(dtype, in, out, sc.data(), lo, hi, variant, s);
    if (device != OEC_DEVICE_HOST) return set_error(OEC_ERR_ARG, "%s: invalid device %d", pname, device);

    // ---- end-to-end path: stage host fields through cached device buffers, pipelined over j-slabs
    // (grid points are independent given their inputs' access extents): the H2D copy of
    // slab s+1 (copy stream), the kernel on slab s (the caller's stream) and the D2H copy of slab
    // s-1 (a third stream) overlap -- PCIe is full duplex.  Each input row is copied once, in the
    // first slab that needs it; the call returns when the outputs are back in host memory.
    Staging &S = stage_for(s);  // the device twins live on the caller's current device
    std::lock_guard<std::mutex> lock(S.mu);
    std::vector<oec_field> din(P_n_in), dout(P_n_out);
    std::vector<const oec_field *> pin(P_n_in);
    std::vector<oec_field *> pout(P_n_out);
    size_t slot = 0, total = 0;
    for (int q = 0; q < P_n_in; ++q) {
        uintptr_t b0, b1;
        span_bytes(in[q], &b0, &b1);
        void *dptr;
        if ((st = stage_buffer(S, slot++, b1 - b0, &dptr))) return st;
        din[q] = *in[q];
        din[q].device = S.device;
        din[q].data = (char *)dptr + ((uintptr_t)in[q]->data - b0);
        pin[q] = &din[q];
        total += b1 - b0;
    }
    for (int q = 0; q < P_n_out; ++q) {
        uintptr_t b0, b1;
        span_bytes(out[q], &b0, &b1);
        void *dptr;
        if ((st = stage_buffer(S, slot++, b1 - b0, &dptr))) return st;
        dout[q] = *out[q];
        dout[q].device = S.device;
        dout[q].data = (char *)dptr + ((uintptr_t)out[q]->data - b0);
        pout[q] = &dout[q];
    }
    if (!S.h2d) {
        cudaStreamCreateWithFlags(&S.h2d, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&S.d2h, cudaStreamNonBlocking);
        for (int e = 0; e < 2 * STAGE_SLABS; ++e) cudaEventCreateWithFlags(&S.ev[e], cudaEventDisableTiming);
    }
    const int64_t nj = hi[1] - lo[1];
    static int max_slabs = -1;
    if (max_slabs < 0) {
        const char *ev = getenv("OEC_STAGE_SLABS");
        // default 2 (round 2): with the slab's D2H as one 2D copy (round 1 issued one per level,
        // which made 2 slabs slower than 1), the 128x128x80 step is 1.85 ms with 1 slab, 1.79 with
        // 2 or 3, 1.80 with 4 (profiles/r02/e2e_slabs_r02.txt)
        max_slabs = ev ? std::max(1, std::min(STAGE_SLABS, atoi(ev))) : 2;
    }
    const int ns = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(max_slabs, nj / 4),
                                                                  (int64_t)(total >> 22)));  // >= ~4 MB per slab
    std::vector<int64_t> next_row(P_n_in);  // first allocated row not yet copied, per input
    for (int q = 0; q < P_n_in; ++q) {
        next_row[q] = in[q]->lb[1];
        const bool rows_ok = in[q]->stride[1] > 0 && (is_k_invariant(in[q]) || in[q]->stride[2] > 0);
        if (!rows_ok) {  // unusual strides: the whole allocation up front
            uintptr_t b0, b1;
            span_bytes(in[q], &b0, &b1);
            cudaError_t e0 = cudaMemcpyAsync((char *)din[q].data - ((uintptr_t)in[q]->data - b0), (const void *)b0,
                                             b1 - b0, cudaMemcpyHostToDevice, S.h2d);
            if (e0 != cudaSuccess) return set_error(OEC_ERR_CUDA, "H2D copy of %s: %s", P.in_names[q].c_str(),
                                                    cudaGetErrorString(e0));
            next_row[q] = in[q]->ub[1];
        }
    }
    int launches = 0;
    cudaError_t e = cudaSuccess;
    for (int sl = 0; sl < ns && e == cudaSuccess; ++sl) {
        int64_t slo[3] = {lo[0], lo[1] + nj * sl / ns, lo[2]}, shi[3] = {hi[0], lo[1] + nj * (sl + 1) / ns, hi[2]};
        for (int q = 0; q < P_n_in && e == cudaSuccess; ++q) {  // rows this slab needs, not copied yet
            int64_t need = sl == ns - 1 ? in[q]->ub[1] : std::min<int64_t>(in[q]->ub[1], shi[1] + P.in_hi[q][1]);
            if (need > next_row[q]) e = h2d_rows(&din[q], in[q], next_row[q], need, S.h2d);
            next_row[q] = std::max(next_row[q], need);
        }
        if (e != cudaSuccess) break;
        cudaEventRecord(S.ev[2 * sl], S.h2d);
        cudaStreamWaitEvent(s, S.ev[2 * sl], 0);
        if ((st = P.run(dtype, pin.data(), pout.data(), sc.data(), slo, shi, variant, s))) return st;
        launches += g_launches;
        cudaEventRecord(S.ev[2 * sl + 1], s);
        cudaStreamWaitEvent(S.d2h, S.ev[2 * sl + 1], 0);
        for (int q = 0; q < P_n_out && e == cudaSuccess; ++q) e = d2h_box(out[q], &dout[q], slo, shi, S.d2h);
    }
    if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "%s: host staging copy: %s", pname, cudaGetErrorString(e));
    e = cudaStreamSynchronize(S.d2h);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "%s: %s", pname, cudaGetErrorString(e));
    g_launches = launches;
    return OEC_OK;
}

}  // namespace oec

using namespace oec;

extern "C" {

int32_t oec_abi_version(void) { return OEC_ABI_VERSION; }

const char *oec_build_info(void) {
    return "liboec: sm_100a, fp64 + f32, --fmad=false; kernels: hdiff (TMA ring, rolling-j, naive/unrolled, unfused, "
           "fused-exchange pipeline), vadv (TMEM c'/d' f64+f32, TMA smem, one thread per column, unfused), suite "
           "(stencil-language JIT: inline/unrolled/TMA-tiled, tuned; hand-written inlined/unrolled/unfused), halo "
           "(pack/unpack, NCCL send/recv)";
}

const char *oec_last_error(void) { return g_err; }

int32_t oec_last_launch_count(void) { return g_launches; }

oec_status oec_field_create(const int64_t domain[3], const int32_t halo_lo[3], const int32_t halo_hi[3], int32_t dtype,
                            int32_t device, const int32_t order[3], int32_t k_invariant, oec_field *out) {
    g_err[0] = 0;
    if (!domain || !halo_lo || !halo_hi || !out) return set_error(OEC_ERR_ARG, "oec_field_create: NULL argument");
    if (dtype != OEC_F64 && dtype != OEC_F32) return set_error(OEC_ERR_DTYPE, "oec_field_create: dtype %d unsupported", dtype);
    const int es = esize(dtype), pad = 128 / es;  // i = 0 is 128-byte aligned; pitch 128-byte multiple
    if (device < 0) return set_error(OEC_ERR_ARG, "oec_field_create: device %d must be a CUDA ordinal", device);
    for (int d = 0; d < 3; ++d)
        if (domain[d] < 1 || halo_lo[d] < 0 || halo_hi[d] < 0)
            return set_error(OEC_ERR_ARG, "oec_field_create: domain >= 1 and halos >= 0 required");
    if (halo_lo[0] > pad)
        return set_error(OEC_ERR_ARG, "oec_field_create: i halo_lo %d > %d (the left pad)", halo_lo[0], pad);
    if (k_invariant && (domain[2] != 1 || halo_lo[2] || halo_hi[2]))
        return set_error(OEC_ERR_ARG, "oec_field_create: k_invariant requires domain[2] == 1 and no k halo");
    int ord[3] = {0, 2, 1};
    if (order) {
        bool seen[3] = {false, false, false};
        for (int d = 0; d < 3; ++d) {
            if (order[d] < 0 || order[d] > 2 || seen[order[d]])
                return set_error(OEC_ERR_ARG, "oec_field_create: order is not a permutation");
            seen[order[d]] = true;
            ord[d] = order[d];
        }
        if (ord[0] != 0) return set_error(OEC_ERR_LAYOUT, "oec_field_create: i must be the fastest dimension");
    }
    // i: 128-byte left pad (i = 0 is 128-byte aligned), pitch a multiple of 128 bytes
    int64_t n[3];
    n[0] = pad + domain[0] + halo_hi[0];
    n[0] = (n[0] + pad - 1) / pad * pad;
    n[1] = domain[1] + halo_lo[1] + halo_hi[1];
    n[2] = domain[2] + halo_lo[2] + halo_hi[2];
    int64_t stride[3];
    stride[ord[0]] = 1;
    stride[ord[1]] = n[ord[0]];
    stride[ord[2]] = n[ord[0]] * n[ord[1]];
    size_t bytes = (size_t)(n[0] * n[1] * n[2]) * es;
    int prev;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    void *base = nullptr;
    cudaError_t e = cudaMalloc(&base, bytes);
    if (e == cudaSuccess) e = cudaMemset(base, 0, bytes);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "oec_field_create: %s", cudaGetErrorString(e));
    memset(out, 0, sizeof *out);
    out->lb[0] = -halo_lo[0];
    out->lb[1] = -halo_lo[1];
    out->lb[2] = -halo_lo[2];
    out->ub[0] = domain[0] + halo_hi[0];
    out->ub[1] = domain[1] + halo_hi[1];
    out->ub[2] = domain[2] + halo_hi[2];
    out->stride[0] = 1;
    out->stride[1] = stride[1];
    out->stride[2] = k_invariant ? 0 : stride[2];
    // data points at (lb0, lb1, lb2): the row starts pad - halo_lo[0] elements into the pad
    out->data = (char *)base + (pad - halo_lo[0]) * es;
    out->dtype = dtype;
    out->device = device;
    out->owned = 1;
    return OEC_OK;
}

oec_status oec_field_wrap(void *data, const int64_t lb[3], const int64_t ub[3], const int64_t stride[3], int32_t dtype,
                          int32_t device, oec_field *out) {
    g_err[0] = 0;
    if (!data || !lb || !ub || !stride || !out) return set_error(OEC_ERR_ARG, "oec_field_wrap: NULL argument");
    if (dtype != OEC_F64 && dtype != OEC_F32) return set_error(OEC_ERR_DTYPE, "oec_field_wrap: dtype %d unsupported", dtype);
    if (stride[0] != 1) return set_error(OEC_ERR_LAYOUT, "oec_field_wrap: stride[0] must be 1");
    for (int d = 0; d < 3; ++d)
        if (ub[d] <= lb[d]) return set_error(OEC_ERR_ARG, "oec_field_wrap: empty range in dim %d", d);
    if (stride[2] == 0 && !(lb[2] == 0 && ub[2] == 1))
        return set_error(OEC_ERR_LAYOUT, "oec_field_wrap: stride[2] == 0 requires lb[2]=0, ub[2]=1");
    memset(out, 0, sizeof *out);
    out->data = data;
    for (int d = 0; d < 3; ++d) {
        out->lb[d] = lb[d];
        out->ub[d] = ub[d];
        out->stride[d] = stride[d];
    }
    out->dtype = dtype;
    out->device = device;
    out->owned = 0;
    return OEC_OK;
}

oec_status oec_field_destroy(oec_field *f) {
    g_err[0] = 0;
    if (!f) return set_error(OEC_ERR_ARG, "oec_field_destroy: NULL");
    if (f->owned && f->data) {
        const int es = esize(f->dtype), pad = 128 / es;
        void *base = (char *)f->data - (pad + f->lb[0]) * es;
        int prev;
        cudaGetDevice(&prev);
        cudaSetDevice(f->device);
        cudaError_t e = cudaFree(base);
        cudaSetDevice(prev);
        if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "oec_field_destroy: %s", cudaGetErrorString(e));
    }
    memset(f, 0, sizeof *f);
    return OEC_OK;
}

oec_status oec_program_info(const char *program, int32_t *n_inputs, int32_t *n_outputs, int32_t *n_scalars) {
    g_err[0] = 0;
    auto P = lookup(program);
    if (!P) return set_error(OEC_ERR_ARG, "unknown program '%s'", program ? program : "(null)");
    if (n_inputs) *n_inputs = (int32_t)P->in_names.size();
    if (n_outputs) *n_outputs = (int32_t)P->out_names.size();
    if (n_scalars) *n_scalars = (int32_t)P->sc_names.size();
    return OEC_OK;
}

// names returned by the queries below are valid while the program stays registered (builtins: always)
oec_status oec_program_input(const char *program, int32_t idx, const char **name, int64_t lo[3], int64_t hi[3],
                             int32_t *k_invariant) {
    g_err[0] = 0;
    auto P = lookup(program);
    if (!P) return set_error(OEC_ERR_ARG, "unknown program '%s'", program ? program : "(null)");
    if (idx < 0 || idx >= (int)P->in_names.size()) return set_error(OEC_ERR_ARG, "%s: input index %d out of range", program, idx);
    if (name) *name = P->in_names[idx].c_str();
    for (int d = 0; d < 3; ++d) {
        if (lo) lo[d] = P->in_lo[idx][d];
        if (hi) hi[d] = P->in_hi[idx][d];
    }
    if (k_invariant) *k_invariant = P->in_kinv[idx];
    return OEC_OK;
}

oec_status oec_program_extent(const char *program, int32_t input_idx, int64_t lo[3], int64_t hi[3]) {
    return oec_program_input(program, input_idx, nullptr, lo, hi, nullptr);
}

oec_status oec_program_output(const char *program, int32_t idx, const char **name) {
    g_err[0] = 0;
    auto P = lookup(program);
    if (!P) return set_error(OEC_ERR_ARG, "unknown program '%s'", program ? program : "(null)");
    if (idx < 0 || idx >= (int)P->out_names.size()) return set_error(OEC_ERR_ARG, "%s: output index %d out of range", program, idx);
    if (name) *name = P->out_names[idx].c_str();
    return OEC_OK;
}

oec_status oec_program_scalar(const char *program, int32_t idx, const char **name, double *default_value) {
    g_err[0] = 0;
    auto P = lookup(program);
    if (!P) return set_error(OEC_ERR_ARG, "unknown program '%s'", program ? program : "(null)");
    if (idx < 0 || idx >= (int)P->sc_names.size()) return set_error(OEC_ERR_ARG, "%s: scalar index %d out of range", program, idx);
    if (name) *name = P->sc_names[idx].c_str();
    if (default_value) *default_value = P->sc_dflt[idx];
    return OEC_OK;
}

oec_status oec_hdiff_variant(const oec_field *in, const oec_field *coeff, oec_field *out, const int64_t dom_lb[3],
                             const int64_t dom_ub[3], int32_t variant, void *stream) {
    const oec_field *ins[2] = {in, coeff};
    oec_field *outs[1] = {out};
    return apply(builtin_desc(OEC_PROG_HDIFF), ins, 2, outs, 1, nullptr, 0, dom_lb, dom_ub, variant, stream);
}

oec_status oec_hdiff(const oec_field *in, const oec_field *coeff, oec_field *out, const int64_t dom_lb[3],
                     const int64_t dom_ub[3], void *stream) {
    return oec_hdiff_variant(in, coeff, out, dom_lb, dom_ub, OEC_VARIANT_AUTO, stream);
}

oec_status oec_vadv(const oec_field *u_stage, const oec_field *wcon, const oec_field *u_pos, const oec_field *utens,
                    const oec_field *utens_stage_in, oec_field *utens_stage_out, double dtr_stage,
                    const int64_t dom_lb[3], const int64_t dom_ub[3], void *stream) {
    const oec_field *ins[5] = {u_stage, wcon, u_pos, utens, utens_stage_in};
    oec_field *outs[1] = {utens_stage_out};
    return apply(builtin_desc(OEC_PROG_VADV), ins, 5, outs, 1, &dtr_stage, 1, dom_lb, dom_ub, OEC_VARIANT_AUTO, stream);
}

oec_status oec_apply_program(const char *program, const oec_field *const *inputs, int32_t n_inputs,
                             oec_field *const *outputs, int32_t n_outputs, const double *scalars, int32_t n_scalars,
                             const int64_t dom_lb[3], const int64_t dom_ub[3], int32_t variant, void *stream) {
    g_err[0] = 0;
    auto P = lookup(program);
    if (!P) return set_error(OEC_ERR_ARG, "unknown program '%s'", program ? program : "(null)");
    return apply(*P, inputs, n_inputs, outputs, n_outputs, scalars, n_scalars, dom_lb, dom_ub, variant, stream);
}

}  // extern "C"
