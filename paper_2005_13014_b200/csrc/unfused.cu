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
struct Tmp {
    double *p;
    int lo0, lo1, lo2, ni, nj;
    __device__ __forceinline__ double &at(int i, int j, int k) const {
        return p[(i - lo0) + (long long)ni * ((j - lo1) + (long long)nj * (k - lo2))];
    }
};

__device__ __forceinline__ double ld(const FV &f, int i, int j, int k) { return __ldg(f.p + (i + j * f.sj + k * f.sk)); }

// ---- hdiff: lap -> flx, fly -> out --------------------------------------------------------
__global__ void k_lap(FV in, Tmp lap, int i1, int j1, int k1) {
    const int i = lap.lo0 + blockIdx.x * blockDim.x + threadIdx.x, j = lap.lo1 + blockIdx.y, k = lap.lo2 + blockIdx.z;
    if (i >= i1 || j >= j1 || k >= k1) return;
    lap.at(i, j, k) = ((ld(in, i - 1, j, k) + ld(in, i + 1, j, k)) + (ld(in, i, j - 1, k) + ld(in, i, j + 1, k))) -
                      4.0 * ld(in, i, j, k);
}
__global__ void k_flx(FV in, Tmp lap, Tmp flx, int i1, int j1, int k1) {
    const int i = flx.lo0 + blockIdx.x * blockDim.x + threadIdx.x, j = flx.lo1 + blockIdx.y, k = flx.lo2 + blockIdx.z;
    if (i >= i1 || j >= j1 || k >= k1) return;
    const double f = lap.at(i + 1, j, k) - lap.at(i, j, k);
    flx.at(i, j, k) = (f * (ld(in, i + 1, j, k) - ld(in, i, j, k)) > 0.0) ? 0.0 : f;
}
__global__ void k_fly(FV in, Tmp lap, Tmp fly, int i1, int j1, int k1) {
    const int i = fly.lo0 + blockIdx.x * blockDim.x + threadIdx.x, j = fly.lo1 + blockIdx.y, k = fly.lo2 + blockIdx.z;
    if (i >= i1 || j >= j1 || k >= k1) return;
    const double g = lap.at(i, j + 1, k) - lap.at(i, j, k);
    fly.at(i, j, k) = (g * (ld(in, i, j + 1, k) - ld(in, i, j, k)) > 0.0) ? 0.0 : g;
}
__global__ void k_hout(FV in, FV coeff, Tmp flx, Tmp fly, FO out, Dom d) {
    const int i = d.lo[0] + blockIdx.x * blockDim.x + threadIdx.x, j = d.lo[1] + blockIdx.y, k = d.lo[2] + blockIdx.z;
    if (i >= d.hi[0]) return;
    out.p[i + j * out.sj + k * out.sk] =
        ld(in, i, j, k) -
        ld(coeff, i, j, k) * ((flx.at(i, j, k) - flx.at(i - 1, j, k)) + (fly.at(i, j, k) - fly.at(i, j - 1, k)));
}

// ---- vadv: coefficients -> forward sweep -> backward sweep -> output ----------------------
constexpr double BET_M = 0.5, BET_P = 0.5;

__global__ void k_vcoef(FV us, FV wc, FV up, FV ut, FV usi, double dtr, Dom d, Tmp A, Tmp B, Tmp Cc, Tmp D) {
    const int i = d.lo[0] + blockIdx.x * blockDim.x + threadIdx.x, j = d.lo[1] + blockIdx.y, k = d.lo[2] + blockIdx.z;
    if (i >= d.hi[0]) return;
    const int k0 = d.lo[2], kN = d.hi[2] - 1;
    double a, b, c, corr;
    if (k == k0) {
        const double gcv = 0.25 * (ld(wc, i + 1, j, k + 1) + ld(wc, i, j, k + 1));
        const double cs = gcv * BET_M;
        a = 0.0;
        c = gcv * BET_P;
        b = dtr - c;
        corr = -cs * (ld(us, i, j, k + 1) - ld(us, i, j, k));
    } else if (k == kN) {
        const double gav = -0.25 * (ld(wc, i + 1, j, k) + ld(wc, i, j, k));
        const double as = gav * BET_M;
        a = gav * BET_P;
        c = 0.0;
        b = dtr - a;
        corr = -as * (ld(us, i, j, k - 1) - ld(us, i, j, k));
    } else {
        const double gav = -0.25 * (ld(wc, i + 1, j, k) + ld(wc, i, j, k));
        const double gcv = 0.25 * (ld(wc, i + 1, j, k + 1) + ld(wc, i, j, k + 1));
        const double as = gav * BET_M, cs = gcv * BET_M;
        a = gav * BET_P;
        c = gcv * BET_P;
        b = (dtr - a) - c;
        corr = (-as * (ld(us, i, j, k - 1) - ld(us, i, j, k))) - cs * (ld(us, i, j, k + 1) - ld(us, i, j, k));
    }
    A.at(i, j, k) = a;
    B.at(i, j, k) = b;
    Cc.at(i, j, k) = c;
    D.at(i, j, k) = ((dtr * ld(up, i, j, k) + ld(ut, i, j, k)) + ld(usi, i, j, k)) + corr;
}
__global__ void k_vfwd(Dom d, Tmp A, Tmp B, Tmp Cc, Tmp D, Tmp CP, Tmp DP) {
    const int i = d.lo[0] + blockIdx.x * blockDim.x + threadIdx.x, j = d.lo[1] + blockIdx.y;
    if (i >= d.hi[0]) return;
    const int k0 = d.lo[2];
    double r = 1.0 / B.at(i, j, k0);
    CP.at(i, j, k0) = Cc.at(i, j, k0) * r;
    DP.at(i, j, k0) = D.at(i, j, k0) * r;
    for (int k = k0 + 1; k < d.hi[2]; ++k) {
        r = 1.0 / (B.at(i, j, k) - CP.at(i, j, k - 1) * A.at(i, j, k));
        CP.at(i, j, k) = Cc.at(i, j, k) * r;
        DP.at(i, j, k) = (D.at(i, j, k) - DP.at(i, j, k - 1) * A.at(i, j, k)) * r;
    }
}
__global__ void k_vbwd(Dom d, Tmp CP, Tmp DP, Tmp X) {
    const int i = d.lo[0] + blockIdx.x * blockDim.x + threadIdx.x, j = d.lo[1] + blockIdx.y;
    if (i >= d.hi[0]) return;
    const int kN = d.hi[2] - 1;
    X.at(i, j, kN) = DP.at(i, j, kN);
    for (int k = kN - 1; k >= d.lo[2]; --k) X.at(i, j, k) = DP.at(i, j, k) - CP.at(i, j, k) * X.at(i, j, k + 1);
}
__global__ void k_vout(FV up, double dtr, Dom d, Tmp X, FO out) {
    const int i = d.lo[0] + blockIdx.x * blockDim.x + threadIdx.x, j = d.lo[1] + blockIdx.y, k = d.lo[2] + blockIdx.z;
    if (i >= d.hi[0]) return;
    out.p[i + j * out.sj + k * out.sk] = dtr * (X.at(i, j, k) - ld(up, i, j, k));
}

struct Workspace {
    std::mutex mu;
    double *p = nullptr;
    size_t n = 0;
};
Workspace g_ws;

cudaError_t workspace(size_t elems, double **p) {
    std::lock_guard<std::mutex> lock(g_ws.mu);
    if (g_ws.n < elems) {
        if (g_ws.p) cudaFree(g_ws.p);
        g_ws.p = nullptr;
        g_ws.n = 0;
        cudaError_t e = cudaMalloc(&g_ws.p, elems * sizeof(double));
        if (e != cudaSuccess) return e;
        g_ws.n = elems;
    }
    *p = g_ws.p;
    return cudaSuccess;
}

Tmp make_tmp(double *&cursor, int lo0, int lo1, int lo2, int hi0, int hi1, int hi2) {
    Tmp t{cursor, lo0, lo1, lo2, hi0 - lo0, hi1 - lo1};
    cursor += (size_t)(hi0 - lo0) * (hi1 - lo1) * (hi2 - lo2);
    return t;
}

dim3 grid_box(int lo0, int lo1, int lo2, int hi0, int hi1, int hi2) {
    return dim3((hi0 - lo0 + 127) / 128, hi1 - lo1, hi2 - lo2);
}

}  // namespace

cudaError_t launch_hdiff_unfused(const FV &in, const FV &coeff, const FO &out, const Dom &d, cudaStream_t s,
                                 int *launches) {
    const int *lo = d.lo, *hi = d.hi;
    const size_t nl = (size_t)(hi[0] - lo[0] + 2) * (hi[1] - lo[1] + 2) * (hi[2] - lo[2]);
    const size_t nx = (size_t)(hi[0] - lo[0] + 1) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
    const size_t ny = (size_t)(hi[0] - lo[0]) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2]);
    double *w;
    cudaError_t e = workspace(nl + nx + ny, &w);
    if (e != cudaSuccess) return e;
    Tmp lap = make_tmp(w, lo[0] - 1, lo[1] - 1, lo[2], hi[0] + 1, hi[1] + 1, hi[2]);
    Tmp flx = make_tmp(w, lo[0] - 1, lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp fly = make_tmp(w, lo[0], lo[1] - 1, lo[2], hi[0], hi[1], hi[2]);
    k_lap<<<grid_box(lo[0] - 1, lo[1] - 1, lo[2], hi[0] + 1, hi[1] + 1, hi[2]), 128, 0, s>>>(in, lap, hi[0] + 1, hi[1] + 1,
                                                                                          hi[2]);
    k_flx<<<grid_box(lo[0] - 1, lo[1], lo[2], hi[0], hi[1], hi[2]), 128, 0, s>>>(in, lap, flx, hi[0], hi[1], hi[2]);
    k_fly<<<grid_box(lo[0], lo[1] - 1, lo[2], hi[0], hi[1], hi[2]), 128, 0, s>>>(in, lap, fly, hi[0], hi[1], hi[2]);
    k_hout<<<grid_box(lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]), 128, 0, s>>>(in, coeff, flx, fly, out, d);
    *launches += 4;
    return cudaGetLastError();
}

cudaError_t launch_vadv_unfused(const FV &us, const FV &wc, const FV &up, const FV &ut, const FV &usi, const FO &out,
                                double dtr, const Dom &d, cudaStream_t s, int *launches) {
    const int *lo = d.lo, *hi = d.hi;
    const size_t n = (size_t)(hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
    double *w;
    cudaError_t e = workspace(7 * n, &w);
    if (e != cudaSuccess) return e;
    Tmp A = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp B = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp Cc = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp D = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp CP = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp DP = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    Tmp X = make_tmp(w, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    const dim3 g3 = grid_box(lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]);
    const dim3 g2(g3.x, g3.y, 1);
    k_vcoef<<<g3, 128, 0, s>>>(us, wc, up, ut, usi, dtr, d, A, B, Cc, D);
    k_vfwd<<<g2, 128, 0, s>>>(d, A, B, Cc, D, CP, DP);
    k_vbwd<<<g2, 128, 0, s>>>(d, CP, DP, X);
    k_vout<<<g3, 128, 0, s>>>(up, dtr, d, X, out);
    *launches += 4;
    return cudaGetLastError();
}

}  // namespace oec
