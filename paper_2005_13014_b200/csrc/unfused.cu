// The paper's "original" optimisation level (§7.3: "Optimization level one applies
// no optimizing transformations"): every stencil operator of the program is its own kernel and
// every intermediate is materialised in HBM over the range shape inference gives it (§5.2,
// P:480-482).  Selected with OEC_VARIANT_UNFUSED; exists to measure what stencil inlining buys on
// B200 (the paper's Fig. 11 experiment), not for speed.  Same operation order as the fused
// kernels and the oracle, so the results are bit-identical.
#include <mutex>

#include "oec_internal.h"

namespace oec {
namespace {

// dense temporary over a box [lo, hi): element (i,j,k) at p[(i-lo0) + ni*((j-lo1) + nj*(k-lo2))]
template <class T>
struct Tmp {
    T *p;
    int lo0, lo1, lo2, ni, nj;
    __device__ __forceinline__ T &at(int i, int j, int k) const {
        return p[(i - lo0) + (long long)ni * ((j - lo1) + (long long)nj * (k - lo2))];
    }
};

template <class T>
__device__ __forceinline__ T ld(const FVT<T> &f, int i, int j, int k) { return __ldg(f.p + (i + j * f.sj + k * f.sk)); }

// ---- hdiff: lap -> flx, fly -> out --------------------------------------------------------
template <class T>
__global__ void k_lap(FVT<T> in, Tmp<T> lap, int i1, int j1, int k1) {
    const int i = lap.lo0 + blockIdx.x * blockDim.x + threadIdx.x, j = lap.lo1 + blockIdx.y, k = lap.lo2 + blockIdx.z;
    if (i >= i1 || j >= j1 || k >= k1) return;
    lap.at(i, j, k) = ((ld(in, i - 1, j, k) + ld(in, i + 1, j, k)) + (ld(in, i, j - 1, k) + ld(in, i, j + 1, k))) -
                      T(4.0) * ld(in, i, j, k);
}
template <class T>
__global__ void k_flx(FVT<T> in, Tmp<T> lap, Tmp<T> flx, int i1, int j1, int k1) {
    const int i = flx.lo0 + blockIdx.x * blockDim.x + threadIdx.x, j = flx.lo1 + blockIdx.y, k = flx.lo2 + blockIdx.z;
    if (i >= i1 || j >= j1 || k >= k1) return;
    const T f = lap.at(i + 1, j, k) - lap.at(i, j, k);
    flx.at(i, j, k) = (f * (ld(in, i + 1, j, k) - ld(in, i, j, k)) > T(0.0)) ? T(0.0) : f;
}
template <class T>
__global__ void k_fly(FVT<T> in, Tmp<T> lap, Tmp<T> fly, int i1, int j1, int k1) {
    const int i = fly.lo0 + blockIdx.x * blockDim.x + threadIdx.x, j = fly.lo1 + blockIdx.y, k = fly.lo2 + blockIdx.z;
    if (i >= i1 || j >= j1 || k >= k1) return;
    const T g = lap.at(i, j + 1, k) - lap.at(i, j, k);
    fly.at(i, j, k) = (g * (ld(in, i, j + 1, k) - ld(in, i, j, k)) > T(0.0)) ? T(0.0) : g;
}
template <class T>
__global__ void k_hout(FVT<T> in, FVT<T> coeff, Tmp<T> flx, Tmp<T> fly, FOT<T> out, Dom d) {
    const int i = d.lo[0] + blockIdx.x * blockDim.x + threadIdx.x, j = d.lo[1] + blockIdx.y, k = d.lo[2] + blockIdx.z;
    if (i >= d.hi[0]) return;
    out.p[i + j * out.sj + k * out.sk] =
        ld(in, i, j, k) -
        ld(coeff, i, j, k) * ((flx.at(i, j, k) - flx.at(i - 1, j, k)) + (fly.at(i, j, k) - fly.at(i, j - 1, k)));
}

// ---- vadv: coefficients -> forward sweep -> backward sweep -> output ----------------------
constexpr double BET_M = 0.5, BET_P = 0.5;

template <class T>
__global__ void k_vcoef(FVT<T> us, FVT<T> wc, FVT<T> up, FVT<T> ut, FVT<T> usi, T dtr, Dom d, Tmp<T> A, Tmp<T> B, Tmp<T> Cc, Tmp<T> D) {
    const int i = d.lo[0] + blockIdx.x * blockDim.x + threadIdx.x, j = d.lo[1] + blockIdx.y, k = d.lo[2] + blockIdx.z;
    if (i >= d.hi[0]) return;
    const int k0 = d.lo[2], kN = d.hi[2] - 1;
    T a, b, c, corr;
    if (k == k0) {
        const T gcv = T(0.25) * (ld(wc, i + 1, j, k + 1) + ld(wc, i, j, k + 1));
        const T cs = gcv * T(BET_M);
        a = T(0.0);
        c = gcv * T(BET_P);
        b = dtr - c;
        corr = -cs * (ld(us, i, j, k + 1) - ld(us, i, j, k));
    } else if (k == kN) {
        const T gav = T(-0.25) * (ld(wc, i + 1, j, k) + ld(wc, i, j, k));
        const T as = gav * T(BET_M);
        a = gav * T(BET_P);
        c = T(0.0);
        b = dtr - a;
        corr = -as * (ld(us, i, j, k - 1) - ld(us, i, j, k));
    } else {
        const T gav = T(-0.25) * (ld(wc, i + 1, j, k) + ld(wc, i, j, k));
        const T gcv = T(0.25) * (ld(wc, i + 1, j, k + 1) + ld(wc, i, j, k + 1));
        const T as = gav * T(BET_M), cs = gcv * T(BET_M);
        a = gav * T(BET_P);
        c = gcv * T(BET_P);
        b = (dtr - a) - c;
        corr = (-as * (ld(us, i, j, k - 1) - ld(us, i, j, k))) - cs * (ld(us, i, j, k + 1) - ld(us, i, j, k));
    }
    A.at(i, j, k) = a;
    B.at(i, j, k) = b;
    Cc.at(i, j, k) = c;
    D.at(i, j, k) = ((dtr * ld(up, i, j, k) + ld(ut, i, j, k)) + ld(usi, i, j, k)) + corr;
}
template <class T>
__global__ void k_vfwd(Dom d, Tmp<T> A, Tmp<T> B, Tmp<T> Cc, Tmp<T> D, Tmp<T> CP, Tmp<T> DP) {
    const int i = d.lo[0] + blockIdx.x * blockDim.x + threadIdx.x, j = d.lo[1] + blockIdx.y;
    if (i >= d.hi[0]) return;
    const int k0 = d.lo[2];
    T r = T(1.0) / B.at(i, j, k0);
    CP.at(i, j, k0) = Cc.at(i, j, k0) * r;
    DP.at(i, j, k0) = D.at(i, j, k0) * r;
    for (int k = k0 + 1; k < d.hi[2]; ++k) {
        r = T(1.0) / (B.at(i, j, k) - CP.at(i, j, k - 1) * A.at(i, j, k));
        CP.at(i, j, k) = Cc.at(i, j, k) * r;
        DP.at(i, j, k) = (D.at(i, j, k) - DP.at(i, j, k - 1) * A.at(i, j, k)) * r;
    }
}
template <class T>
__global__ void k_vbwd(Dom d, Tmp<T> CP, Tmp<T> DP, Tmp<T> X) {
    const int i = d.lo[0] + blockIdx.x * blockDim.x + threadIdx.x, j = d.lo[1] + blockIdx.y;
    if (i >= d.hi[0]) return;
    const int kN = d.hi[2] - 1;
    X.at(i, j, kN) = DP.at(i, j, kN);
    for (int k = kN - 1; k >= d.lo[2]; --k) X.at(i, j, k) = DP.at(i, j, k) - CP.at(i, j, k) * X.at(i, j, k + 1);
}
template <class T>
__global__ void k_vout(FVT<T> up, T dtr, Dom d, Tmp<T> X, FOT<T> out) {
    const int i = d.lo[0] + blockIdx.x * blockDim.x + threadIdx.x, j = d.lo[1] + blockIdx.y, k = d.lo[2] + blockIdx.z;
    if (i >= d.hi[0]) return;
    out.p[i + j * out.sj + k * out.sk] = dtr * (X.at(i, j, k) - ld(up, i, j, k));
}

struct Workspace {
    std::mutex mu;
    void *p = nullptr;
    size_t n = 0;  // bytes
};
Workspace g_ws;

template <class T>
cudaError_t workspace(size_t elems, T **p) {
    std::lock_guard<std::mutex> lock(g_ws.mu);
    if (g_ws.n < elems * sizeof(T)) {
        if (g_ws.p) cudaFree(g_ws.p);
        g_ws.p = nullptr;
        g_ws.n = 0;
        cudaError_t e = cudaMalloc(&g_ws.p, elems * sizeof(T));
        if (e != cudaSuccess) return e;
        g_ws.n = elems * sizeof(T);
    }
    *p = (T *)g_ws.p;
    return cudaSuccess;
}

template <class T>
Tmp<T> make_tmp(T *&cursor, int lo0, int lo1, int lo2, int hi0, int hi1, int hi2) {
    Tmp<T> t{cursor, lo0, lo1, lo2, hi0 - lo0, hi1 - lo1};
    cursor += (size_t)(hi0 - lo0) * (hi1 - lo1) * (hi2 - lo2);
    return t;
}

dim3 grid_box(int lo0, int lo1, int lo2, int hi0, int hi1, int hi2) {
    return dim3((hi0 - lo0 + 127) / 128, hi1 - lo1, hi2 - lo2);
}

}  // namespace

template <class T>
cudaError_t launch_hdiff_unfused(const FVT<T> &in, const FVT<T> &coeff, const FOT<T> &out, const Dom &d, cudaStream_t s,
                                 int *launches) {
    const int *lo = d.lo, *hi = d.hi;
    const size_t nl = (size_t)(hi[0] - lo[0] + 2) * (hi[1] - lo[1] + 2) * (hi[2] - lo[2]);
    const size_t nx = (size_t)(hi[0] - lo[0] + 1) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
    const size_t ny = (size_t)(hi[0] - lo[0]) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2]);
    T *w;
    cudaError_t e = workspace(nl + nx + ny, &w);
    if (e != cudaSuccess) return e;
    Tmp<T> lap = make_tmp(w, lo[0] - 1, lo[1] - 1, lo[2], hi[0] + 1, hi[1] + 1, hi[2]);
    Tmp<T> flx = make_tmp(w, lo[0] - 1, lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp<T> fly = make_tmp(w, lo[0], lo[1] - 1, lo[2], hi[0], hi[1], hi[2]);
    k_lap<<<grid_box(lo[0] - 1, lo[1] - 1, lo[2], hi[0] + 1, hi[1] + 1, hi[2]), 128, 0, s>>>(in, lap, hi[0] + 1, hi[1] + 1,
                                                                                          hi[2]);
    k_flx<<<grid_box(lo[0] - 1, lo[1], lo[2], hi[0], hi[1], hi[2]), 128, 0, s>>>(in, lap, flx, hi[0], hi[1], hi[2]);
    k_fly<<<grid_box(lo[0], lo[1] - 1, lo[2], hi[0], hi[1], hi[2]), 128, 0, s>>>(in, lap, fly, hi[0], hi[1], hi[2]);
    k_hout<<<grid_box(lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]), 128, 0, s>>>(in, coeff, flx, fly, out, d);
    *launches += 4;
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_vadv_unfused(const FVT<T> &us, const FVT<T> &wc, const FVT<T> &up, const FVT<T> &ut, const FVT<T> &usi, const FOT<T> &out,
                                double dtr, const Dom &d, cudaStream_t s, int *launches) {
    const int *lo = d.lo, *hi = d.hi;
    const size_t n = (size_t)(hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
    T *w;
    cudaError_t e = workspace(7 * n, &w);
    if (e != cudaSuccess) return e;
    Tmp<T> A = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp<T> B = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp<T> Cc = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp<T> D = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp<T> CP = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp<T> DP = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp<T> X = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    const dim3 g3 = grid_box(lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    const dim3 g2(g3.x, g3.y, 1);
    k_vcoef<<<g3, 128, 0, s>>>(us, wc, up, ut, usi, (T)dtr, d, A, B, Cc, D);
    k_vfwd<<<g2, 128, 0, s>>>(d, A, B, Cc, D, CP, DP);
    k_vbwd<<<g2, 128, 0, s>>>(d, CP, DP, X);
    k_vout<<<g3, 128, 0, s>>>(up, (T)dtr, d, X, out);
    *launches += 4;
    return cudaGetLastError();
}

template cudaError_t launch_hdiff_unfused<double>(const FV &, const FV &, const FO &, const Dom &, cudaStream_t, int *);
template cudaError_t launch_hdiff_unfused<float>(const FVf &, const FVf &, const FOf &, const Dom &, cudaStream_t, int *);
template cudaError_t launch_vadv_unfused<double>(const FV &, const FV &, const FV &, const FV &, const FV &, const FO &,
                                                 double, const Dom &, cudaStream_t, int *);
template cudaError_t launch_vadv_unfused<float>(const FVf &, const FVf &, const FVf &, const FVf &, const FVf &,
                                                const FOf &, double, const Dom &, cudaStream_t, int *);

}  // namespace oec
