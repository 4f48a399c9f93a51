// The paper's "original" optimisation level (§7.3) for the remaining suite
// programs: every stencil.apply of the program (oracle/suite.py lists them, Table II's "apply
// ops" column) is its own kernel, and every intermediate is materialised in HBM over the box shape
// inference gives it (demand-driven bounding boxes, §5.2).  Outputs whose producer box
// equals the domain are written straight into the caller's field; the others (fvtp2d fy2 / fx2,
// which later operators also read outside the domain) are computed into a temporary and stored
// to the output on the domain (stencil.store).  Same operation order as the fused kernels
// (csrc/suite.cu) and the oracle, --fmad=false: bit-identical results.
#include <mutex>

#include "oec_internal.h"

namespace oec {
namespace {

template <class T>
__device__ __forceinline__ T A(const FVT<T> &f, int i, int j, int k) { return __ldg(f.p + (i + j * f.sj + k * f.sk)); }

constexpr int NSLOT = 16;
template <class T>
struct SArgs {
    FVT<T> f[NSLOT];  // inputs (registry order), then temporaries
    FOT<T> o[2];      // this operator's results
    T sc[2];
    Dom box;
};

template <class T, void (*F)(const FVT<T> *, const T *, int, int, int, T *), int NR>
__global__ void __launch_bounds__(128) stage_kernel(const __grid_constant__ SArgs<T> a) {
    const int i = a.box.lo[0] + blockIdx.x * 32 + threadIdx.x;
    const int j = a.box.lo[1] + blockIdx.y * 4 + threadIdx.y;
    const int k = a.box.lo[2] + blockIdx.z;
    if (i >= a.box.hi[0] || j >= a.box.hi[1]) return;
    T r[NR];
    F(a.f, a.sc, i, j, k, r);
#pragma unroll
    for (int q = 0; q < NR; ++q) a.o[q].p[i + j * a.o[q].sj + k * a.o[q].sk] = r[q];
}

typedef cudaError_t (*StageLaunch)(const void *, dim3, cudaStream_t);  // args: const SArgs<T> *
template <class T, void (*F)(const FVT<T> *, const T *, int, int, int, T *), int NR>
cudaError_t launch_stage(const void *a, dim3 grid, cudaStream_t s) {
    stage_kernel<T, F, NR><<<grid, dim3(32, 4, 1), 0, s>>>(*static_cast<const SArgs<T> *>(a));
    return cudaGetLastError();
}

// ---- uvbke: slots uc 0, vc 1, cosa 2, rsina 3 ---------------------------------------------
template <class T>
__device__ void uv_ub(const FVT<T> *f, const T *sc, int i, int j, int k, T *r) {
    r[0] = (sc[0] * ((A(f[0], i, j - 1, k) + A(f[0], i, j, k)) - (A(f[1], i - 1, j, k) + A(f[1], i, j, k)) * A(f[2], i, j, k))) *
           A(f[3], i, j, k);
}
template <class T>
__device__ void uv_vb(const FVT<T> *f, const T *sc, int i, int j, int k, T *r) {
    r[0] = (sc[0] * ((A(f[1], i - 1, j, k) + A(f[1], i, j, k)) - (A(f[0], i, j - 1, k) + A(f[0], i, j, k)) * A(f[2], i, j, k))) *
           A(f[3], i, j, k);
}

// ---- p_grad_c: uc 0, vc 1, delpc 2, pkc 3, gz 4, rdxc 5, rdyc 6; temp wk 7 ------------------
template <class T>
__device__ void pg_wk(const FVT<T> *f, const T *, int i, int j, int k, T *r) { r[0] = A(f[2], i, j, k); }
template <class T>
__device__ void pg_uc(const FVT<T> *f, const T *sc, int i, int j, int k, T *r) {
    const FVT<T> &gz = f[4], &pkc = f[3], &wk = f[7];
    const T t = (A(gz, i - 1, j, k + 1) - A(gz, i, j, k)) * (A(pkc, i, j, k + 1) - A(pkc, i - 1, j, k)) +
                     (A(gz, i - 1, j, k) - A(gz, i, j, k + 1)) * (A(pkc, i - 1, j, k + 1) - A(pkc, i, j, k));
    r[0] = A(f[0], i, j, k) + ((sc[0] * A(f[5], i, j, k)) / (A(wk, i - 1, j, k) + A(wk, i, j, k))) * t;
}
template <class T>
__device__ void pg_vc(const FVT<T> *f, const T *sc, int i, int j, int k, T *r) {
    const FVT<T> &gz = f[4], &pkc = f[3], &wk = f[7];
    const T t = (A(gz, i, j - 1, k + 1) - A(gz, i, j, k)) * (A(pkc, i, j, k + 1) - A(pkc, i, j - 1, k)) +
                     (A(gz, i, j - 1, k) - A(gz, i, j, k + 1)) * (A(pkc, i, j - 1, k + 1) - A(pkc, i, j, k));
    r[0] = A(f[1], i, j, k) + ((sc[0] * A(f[6], i, j, k)) / (A(wk, i, j - 1, k) + A(wk, i, j, k))) * t;
}

// ---- nh_p_grad: u 0, v 1, pp 2, gz 3, pk3 4, delp 5, rdx 6, rdy 7; temps wk 8, du 9, dv 10 --
template <class T>
__device__ void nh_wk(const FVT<T> *f, const T *, int i, int j, int k, T *r) {
    r[0] = A(f[4], i, j, k + 1) - A(f[4], i, j, k);
}
template <class T, int DI, int DJ>
__device__ __forceinline__ T nh_grad(const FVT<T> &gz, const FVT<T> &p, int i, int j, int k) {
    return (A(gz, i, j, k + 1) - A(gz, i + DI, j + DJ, k)) * (A(p, i + DI, j + DJ, k + 1) - A(p, i, j, k)) +
           (A(gz, i, j, k) - A(gz, i + DI, j + DJ, k + 1)) * (A(p, i, j, k + 1) - A(p, i + DI, j + DJ, k));
}
template <class T>
__device__ void nh_du(const FVT<T> *f, const T *sc, int i, int j, int k, T *r) {
    r[0] = (sc[0] / (A(f[8], i, j, k) + A(f[8], i + 1, j, k))) * nh_grad<T, 1, 0>(f[3], f[4], i, j, k);
}
template <class T>
__device__ void nh_dv(const FVT<T> *f, const T *sc, int i, int j, int k, T *r) {
    r[0] = (sc[0] / (A(f[8], i, j, k) + A(f[8], i, j + 1, k))) * nh_grad<T, 0, 1>(f[3], f[4], i, j, k);
}
template <class T>
__device__ void nh_u(const FVT<T> *f, const T *sc, int i, int j, int k, T *r) {
    r[0] = ((A(f[0], i, j, k) + A(f[9], i, j, k)) +
            (sc[0] / (A(f[5], i, j, k) + A(f[5], i + 1, j, k))) * nh_grad<T, 1, 0>(f[3], f[2], i, j, k)) *
           A(f[6], i, j, k);
}
template <class T>
__device__ void nh_v(const FVT<T> *f, const T *sc, int i, int j, int k, T *r) {
    r[0] = ((A(f[1], i, j, k) + A(f[10], i, j, k)) +
            (sc[0] / (A(f[5], i, j, k) + A(f[5], i, j + 1, k))) * nh_grad<T, 0, 1>(f[3], f[2], i, j, k)) *
           A(f[7], i, j, k);
}

// ---- PPM operators (al, (bl, br), flux) along (DI, DJ) on slots Q (field), C (Courant), AL, BL, BR
constexpr double P1 = 7.0 / 12.0;
constexpr double P2 = -1.0 / 12.0;
template <class T, int Q, int DI, int DJ>
__device__ void ppm_al(const FVT<T> *f, const T *, int i, int j, int k, T *r) {
    const FVT<T> &q = f[Q];
    r[0] = T(P1) * (A(q, i - DI, j - DJ, k) + A(q, i, j, k)) + T(P2) * (A(q, i - 2 * DI, j - 2 * DJ, k) + A(q, i + DI, j + DJ, k));
}
template <class T, int Q, int AL, int DI, int DJ>
__device__ void ppm_blbr(const FVT<T> *f, const T *, int i, int j, int k, T *r) {
    const T qq = A(f[Q], i, j, k);
    r[0] = A(f[AL], i, j, k) - qq;
    r[1] = A(f[AL], i + DI, j + DJ, k) - qq;
}
template <class T, int Q, int C, int BL, int BR, int DI, int DJ>
__device__ void ppm_flux(const FVT<T> *f, const T *, int i, int j, int k, T *r) {
    const T c = A(f[C], i, j, k);
    if (c > T(0.0)) {
        const T blm = A(f[BL], i - DI, j - DJ, k), brm = A(f[BR], i - DI, j - DJ, k);
        r[0] = A(f[Q], i - DI, j - DJ, k) + (T(1.0) - c) * (brm - c * (blm + brm));
    } else {
        const T bl = A(f[BL], i, j, k), br = A(f[BR], i, j, k);
        r[0] = A(f[Q], i, j, k) + (T(1.0) + c) * (bl + c * (bl + br));
    }
}
template <class T, int X, int F2>
__device__ void mul2(const FVT<T> *f, const T *, int i, int j, int k, T *r) {
    r[0] = A(f[X], i, j, k) * A(f[F2], i, j, k);
}
// q_new = ((q area + g) - g[+1]) / ra   (fvtp2d_qi: g = fyy, +1 in j; fvtp2d_qj: g = fx1, +1 in i)
template <class T, int Q, int AREA, int G, int RA, int DI, int DJ>
__device__ void fv_update(const FVT<T> *f, const T *, int i, int j, int k, T *r) {
    r[0] = ((A(f[Q], i, j, k) * A(f[AREA], i, j, k) + A(f[G], i, j, k)) - A(f[G], i + DI, j + DJ, k)) / A(f[RA], i, j, k);
}
// fvtp2d_flux outputs: (0.5 (a + b)) m
template <class T, int X, int Y, int M>
__device__ void fv_avg(const FVT<T> *f, const T *, int i, int j, int k, T *r) {
    r[0] = (T(0.5) * (A(f[X], i, j, k) + A(f[Y], i, j, k))) * A(f[M], i, j, k);
}

// ---- fastwaves: u_pos 0, v_pos 1, u_tens 2, v_tens 3, rho 4, ppuv 5, fx 6, wgtfac 7, hhl 8;
//      temps ppgk 9, ppgc 10, ppgu 11, ppgv 12 ------------------------------------------------
template <class T>
__device__ void fw_ppgk(const FVT<T> *f, const T *, int i, int j, int k, T *r) {
    const T w = A(f[7], i, j, k);
    r[0] = w * A(f[5], i, j, k) + (T(1.0) - w) * A(f[5], i, j, k - 1);
}
template <class T>
__device__ void fw_ppgc(const FVT<T> *f, const T *, int i, int j, int k, T *r) {
    r[0] = A(f[9], i, j, k + 1) - A(f[9], i, j, k);
}
template <class T, int DI, int DJ>
__device__ void fw_ppg(const FVT<T> *f, const T *, int i, int j, int k, T *r) {
    const FVT<T> &pp = f[5], &pc = f[10], &h = f[8];
    const T h0 = A(h, i, j, k), h1 = A(h, i, j, k + 1), hE = A(h, i + DI, j + DJ, k), hE1 = A(h, i + DI, j + DJ, k + 1);
    r[0] = (A(pp, i + DI, j + DJ, k) - A(pp, i, j, k)) +
           (((A(pc, i + DI, j + DJ, k) + A(pc, i, j, k)) * T(0.5)) * ((h1 + h0) - (hE1 + hE))) / ((h1 - h0) + (hE1 - hE));
}
template <class T>
__device__ void fw_u(const FVT<T> *f, const T *sc, int i, int j, int k, T *r) {
    r[0] = A(f[0], i, j, k) +
           (A(f[2], i, j, k) - ((A(f[11], i, j, k) * T(2.0)) * A(f[6], i, j, k)) / (A(f[4], i + 1, j, k) + A(f[4], i, j, k))) * sc[1];
}
template <class T>
__device__ void fw_v(const FVT<T> *f, const T *sc, int i, int j, int k, T *r) {
    r[0] = A(f[1], i, j, k) +
           (A(f[3], i, j, k) - ((A(f[12], i, j, k) * T(2.0)) * sc[0]) / (A(f[4], i, j + 1, k) + A(f[4], i, j, k))) * sc[1];
}

// ---------------------------------------------------------------------------------------------
// host tables.  A result slot >= OUT means the caller's output (slot - OUT) written directly.
// Temporary boxes are offsets from the domain bounds: [lo + blo, hi + bhi), derived by
// demand-driven bounding boxes over the operators' accesses; the fused registry's
// input extents already bound every input read of these boxes (bbox(T) + o = bbox(T + o)).
// ---------------------------------------------------------------------------------------------
constexpr int OUT = 100;
struct TmpDef {
    int slot, blo[3], bhi[3];
};
struct StageDef {
    StageLaunch fn;
    int nres, res[2];
    int blo[3], bhi[3];  // the operator's own box (offsets from the domain)
};
struct UProg {
    int n_tmp;
    TmpDef tmp[10];
    int n_stage;
    StageDef st[9];
    int out_src[3];  // slot holding output q (temporary -> stored on the domain) or OUT + q
};

#define Z3 {0, 0, 0}
template <class T>
const UProg *uprog(int p) {
    static const UProg uvbke = {0, {}, 2,
        {{launch_stage<T, uv_ub<T>, 1>, 1, {OUT + 0}, Z3, Z3}, {launch_stage<T, uv_vb<T>, 1>, 1, {OUT + 1}, Z3, Z3}},
        {OUT + 0, OUT + 1}};
    static const UProg p_grad_c = {1, {{7, {-1, -1, 0}, Z3}}, 3,
        {{launch_stage<T, pg_wk<T>, 1>, 1, {7}, {-1, -1, 0}, Z3},
         {launch_stage<T, pg_uc<T>, 1>, 1, {OUT + 0}, Z3, Z3},
         {launch_stage<T, pg_vc<T>, 1>, 1, {OUT + 1}, Z3, Z3}},
        {OUT + 0, OUT + 1}};
    static const UProg nh_p_grad = {3, {{8, Z3, {1, 1, 0}}, {9, Z3, Z3}, {10, Z3, Z3}}, 5,
        {{launch_stage<T, nh_wk<T>, 1>, 1, {8}, Z3, {1, 1, 0}},
         {launch_stage<T, nh_du<T>, 1>, 1, {9}, Z3, Z3},
         {launch_stage<T, nh_dv<T>, 1>, 1, {10}, Z3, Z3},
         {launch_stage<T, nh_u<T>, 1>, 1, {OUT + 0}, Z3, Z3},
         {launch_stage<T, nh_v<T>, 1>, 1, {OUT + 1}, Z3, Z3}},
        {OUT + 0, OUT + 1}};
    // fvtp2d_qi: q 0, cry 1, yfx 2, area 3, ra_y 4; al 5, bl 6, br 7, fy2 8, fyy 9
    static const UProg fvtp2d_qi = {5,
        {{5, {0, -1, 0}, {0, 2, 0}}, {6, {0, -1, 0}, {0, 1, 0}}, {7, {0, -1, 0}, {0, 1, 0}}, {8, Z3, {0, 1, 0}},
         {9, Z3, {0, 1, 0}}},
        5,
        {{launch_stage<T, ppm_al<T, 0, 0, 1>, 1>, 1, {5}, {0, -1, 0}, {0, 2, 0}},
         {launch_stage<T, ppm_blbr<T, 0, 5, 0, 1>, 2>, 2, {6, 7}, {0, -1, 0}, {0, 1, 0}},
         {launch_stage<T, ppm_flux<T, 0, 1, 6, 7, 0, 1>, 1>, 1, {8}, Z3, {0, 1, 0}},
         {launch_stage<T, mul2<T, 2, 8>, 1>, 1, {9}, Z3, {0, 1, 0}},
         {launch_stage<T, fv_update<T, 0, 3, 9, 4, 0, 1>, 1>, 1, {OUT + 0}, Z3, Z3}},
        {OUT + 0, 8}};
    // fvtp2d_qj: q 0, q_i 1, crx 2, xfx 3, area 4, ra_x 5; al 6, bl 7, br 8, (fx -> out 1),
    //            al2 10, bl2 11, br2 12, fx2 13, fx1 14
    static const UProg fvtp2d_qj = {8,
        {{6, {-1, 0, 0}, {1, 0, 0}}, {7, {-1, 0, 0}, Z3}, {8, {-1, 0, 0}, Z3}, {10, {-1, 0, 0}, {2, 0, 0}},
         {11, {-1, 0, 0}, {1, 0, 0}}, {12, {-1, 0, 0}, {1, 0, 0}}, {13, Z3, {1, 0, 0}}, {14, Z3, {1, 0, 0}}},
        8,
        {{launch_stage<T, ppm_al<T, 1, 1, 0>, 1>, 1, {6}, {-1, 0, 0}, {1, 0, 0}},
         {launch_stage<T, ppm_blbr<T, 1, 6, 1, 0>, 2>, 2, {7, 8}, {-1, 0, 0}, Z3},
         {launch_stage<T, ppm_flux<T, 1, 2, 7, 8, 1, 0>, 1>, 1, {OUT + 1}, Z3, Z3},
         {launch_stage<T, ppm_al<T, 0, 1, 0>, 1>, 1, {10}, {-1, 0, 0}, {2, 0, 0}},
         {launch_stage<T, ppm_blbr<T, 0, 10, 1, 0>, 2>, 2, {11, 12}, {-1, 0, 0}, {1, 0, 0}},
         {launch_stage<T, ppm_flux<T, 0, 2, 11, 12, 1, 0>, 1>, 1, {13}, Z3, {1, 0, 0}},
         {launch_stage<T, mul2<T, 3, 13>, 1>, 1, {14}, Z3, {1, 0, 0}},
         {launch_stage<T, fv_update<T, 0, 4, 14, 5, 1, 0>, 1>, 1, {OUT + 0}, Z3, Z3}},
        {OUT + 0, OUT + 1, 13}};
    // fvtp2d_flux: q_j 0, cry 1, fx 2, fx2 3, fy2 4, mfx 5, mfy 6; al 7, bl 8, br 9, fy 10
    static const UProg fvtp2d_flux = {4,
        {{7, {0, -1, 0}, {0, 1, 0}}, {8, {0, -1, 0}, Z3}, {9, {0, -1, 0}, Z3}, {10, Z3, Z3}},
        5,
        {{launch_stage<T, ppm_al<T, 0, 0, 1>, 1>, 1, {7}, {0, -1, 0}, {0, 1, 0}},
         {launch_stage<T, ppm_blbr<T, 0, 7, 0, 1>, 2>, 2, {8, 9}, {0, -1, 0}, Z3},
         {launch_stage<T, ppm_flux<T, 0, 1, 8, 9, 0, 1>, 1>, 1, {10}, Z3, Z3},
         {launch_stage<T, fv_avg<T, 2, 3, 5>, 1>, 1, {OUT + 0}, Z3, Z3},
         {launch_stage<T, fv_avg<T, 10, 4, 6>, 1>, 1, {OUT + 1}, Z3, Z3}},
        {OUT + 0, OUT + 1}};
    static const UProg fastwaves = {4,
        {{9, Z3, {1, 1, 1}}, {10, Z3, {1, 1, 0}}, {11, Z3, Z3}, {12, Z3, Z3}},
        6,
        {{launch_stage<T, fw_ppgk<T>, 1>, 1, {9}, Z3, {1, 1, 1}},
         {launch_stage<T, fw_ppgc<T>, 1>, 1, {10}, Z3, {1, 1, 0}},
         {launch_stage<T, fw_ppg<T, 1, 0>, 1>, 1, {11}, Z3, Z3},
         {launch_stage<T, fw_ppg<T, 0, 1>, 1>, 1, {12}, Z3, Z3},
         {launch_stage<T, fw_u<T>, 1>, 1, {OUT + 0}, Z3, Z3},
         {launch_stage<T, fw_v<T>, 1>, 1, {OUT + 1}, Z3, Z3}},
        {OUT + 0, OUT + 1}};
    switch (p) {
    case OEC_PROG_UVBKE: return &uvbke;
    case OEC_PROG_P_GRAD_C: return &p_grad_c;
    case OEC_PROG_NH_P_GRAD: return &nh_p_grad;
    case OEC_PROG_FVTP2D_QI: return &fvtp2d_qi;
    case OEC_PROG_FVTP2D_QJ: return &fvtp2d_qj;
    case OEC_PROG_FVTP2D_FLUX: return &fvtp2d_flux;
    case OEC_PROG_FASTWAVES: return &fastwaves;
    default: return nullptr;
    }
}
#undef Z3

struct Workspace {
    std::mutex mu;
    void *p = nullptr;
    size_t n = 0;  // bytes
};
Workspace g_ws;

}  // namespace

int suite_unfused_stages(int program_id) {
    const UProg *u = uprog<double>(program_id);
    return u ? u->n_stage : 0;
}

template <class T>
cudaError_t launch_suite_unfused(int program_id, int n_in, const FVT<T> *in, const FOT<T> *out, const double *scalars,
                                 const Dom &d, cudaStream_t s, int *launches) {
    const UProg *u = uprog<T>(program_id);
    if (!u) return cudaErrorInvalidValue;
    // temporaries: dense boxes, i pitch rounded to an even element count
    Dom tb[NSLOT];
    size_t off[NSLOT], total = 0;
    int ni[NSLOT], nj[NSLOT];
    for (int t = 0; t < u->n_tmp; ++t) {
        const TmpDef &td = u->tmp[t];
        for (int q = 0; q < 3; ++q) {
            tb[td.slot].lo[q] = d.lo[q] + td.blo[q];
            tb[td.slot].hi[q] = d.hi[q] + td.bhi[q];
        }
        ni[td.slot] = (tb[td.slot].hi[0] - tb[td.slot].lo[0] + 1) & ~1;
        nj[td.slot] = tb[td.slot].hi[1] - tb[td.slot].lo[1];
        off[td.slot] = total;
        total += (size_t)ni[td.slot] * nj[td.slot] * (tb[td.slot].hi[2] - tb[td.slot].lo[2]);
    }
    if ((long long)total > INT32_MAX) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> lock(g_ws.mu);
    if (g_ws.n < total * sizeof(T)) {
        if (g_ws.p) cudaFree(g_ws.p);
        g_ws.p = nullptr;
        g_ws.n = 0;
        cudaError_t e = cudaMalloc(&g_ws.p, total * sizeof(T));
        if (e != cudaSuccess) return e;
        g_ws.n = total * sizeof(T);
    }
    SArgs<T> a;
    for (int q = 0; q < NSLOT; ++q) a.f[q] = FVT<T>{nullptr, 0, 0};
    for (int q = 0; q < n_in; ++q) a.f[q] = in[q];
    FOT<T> tmp_o[NSLOT];
    for (int t = 0; t < u->n_tmp; ++t) {
        const int sl = u->tmp[t].slot;
        const int32_t sj = ni[sl], sk = ni[sl] * nj[sl];
        T *origin = (T *)g_ws.p + off[sl] - ((long long)tb[sl].lo[0] + (long long)tb[sl].lo[1] * sj + (long long)tb[sl].lo[2] * sk);
        a.f[sl] = FVT<T>{origin, sj, sk};
        tmp_o[sl] = FOT<T>{origin, sj, sk};
    }
    a.sc[0] = (T)scalars[0];
    a.sc[1] = (T)scalars[1];
    for (int st = 0; st < u->n_stage; ++st) {
        const StageDef &S = u->st[st];
        for (int r = 0; r < S.nres; ++r) a.o[r] = S.res[r] >= OUT ? out[S.res[r] - OUT] : tmp_o[S.res[r]];
        for (int q = 0; q < 3; ++q) {
            a.box.lo[q] = d.lo[q] + S.blo[q];
            a.box.hi[q] = d.hi[q] + S.bhi[q];
        }
        dim3 grid((a.box.hi[0] - a.box.lo[0] + 31) / 32, (a.box.hi[1] - a.box.lo[1] + 3) / 4, a.box.hi[2] - a.box.lo[2]);
        cudaError_t e = S.fn(&a, grid, s);
        ++*launches;
        if (e != cudaSuccess) return e;
    }
    // stencil.store of outputs held in temporaries
    for (int q = 0; q < 3; ++q) {
        const int src = u->out_src[q];
        if (src == 0 || src >= OUT) continue;
        Box b;
        for (int c = 0; c < 3; ++c) {
            b.lo[c] = d.lo[c];
            b.hi[c] = d.hi[c];
        }
        cudaError_t e = launch_box_copy(a.f[src], out[q], b, s, launches);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template cudaError_t launch_suite_unfused<double>(int, int, const FV *, const FO *, const double *, const Dom &,
                                                  cudaStream_t, int *);
template cudaError_t launch_suite_unfused<float>(int, int, const FVf *, const FOf *, const double *, const Dom &,
                                                 cudaStream_t, int *);

}  // namespace oec
