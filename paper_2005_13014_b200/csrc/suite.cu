// The remaining benchmark stencil programs (Table II, + fastwaves), each fused into ONE
// kernel: every producer is inlined at every offset its consumers access (stencil inlining)
// and evaluated in registers, one thread per grid point, no shared memory, no synchronisation --
// the paper's execution model.  Definitions and operation order: DESIGN.md R12-R17
// (the CPU oracle writes the same definitions in oracle/suite.py; no code is shared).  --fmad=false
// keeps every + - * / separately rounded, so results are bit-identical to the oracle.
#include "oec_internal.h"

namespace oec {
namespace {

struct Pt {
    int i, j, k;
};

template <class T>
__device__ __forceinline__ T A(const FVT<T> &f, int i, int j, int k) { return __ldg(f.p + (i + j * f.sj + k * f.sk)); }
// point functions return their outputs in r[]; the kernel stores them after all loads of its levels
#define OUT(o, v) (r[o] = (v))

// ---------------------------------------------------------------------------------------------
// uvbke:  ub = (dt5 ((uc[j-1] + uc) - (vc[i-1] + vc) cosa)) rsina ;  vb analogous
// ---------------------------------------------------------------------------------------------
template <class T>
__device__ __forceinline__ void uvbke_pt(const FVT<T> *in, const T *sc, int i, int j, int k, T *r) {
    const FVT<T> &uc = in[0], &vc = in[1], &cosa = in[2], &rsina = in[3];
    const T dt5 = sc[0];
    const T u2 = A(uc, i, j - 1, k) + A(uc, i, j, k);
    const T v2 = A(vc, i - 1, j, k) + A(vc, i, j, k);
    const T ca = A(cosa, i, j, k), rs = A(rsina, i, j, k);
    OUT(0, (dt5 * (u2 - v2 * ca)) * rs);
    OUT(1, (dt5 * (v2 - u2 * ca)) * rs);
}

// ---------------------------------------------------------------------------------------------
// p_grad_c (wk = delpc):
//   uc' = uc + ((dt2 rdxc) / (wk[i-1] + wk)) * ((gz[i-1,k+1] - gz)(pkc[k+1] - pkc[i-1])
//                                                + (gz[i-1] - gz[k+1])(pkc[i-1,k+1] - pkc))
// ---------------------------------------------------------------------------------------------
template <class T>
__device__ __forceinline__ void p_grad_c_pt(const FVT<T> *in, const T *sc, int i, int j, int k, T *r) {
    const FVT<T> &uc = in[0], &vc = in[1], &delpc = in[2], &pkc = in[3], &gz = in[4], &rdxc = in[5], &rdyc = in[6];
    const T dt2 = sc[0];
    const T gz0 = A(gz, i, j, k), gz1 = A(gz, i, j, k + 1), pk0 = A(pkc, i, j, k), pk1 = A(pkc, i, j, k + 1);
    const T wk = A(delpc, i, j, k);
    {
        const T t = (A(gz, i - 1, j, k + 1) - gz0) * (pk1 - A(pkc, i - 1, j, k)) +
                         (A(gz, i - 1, j, k) - gz1) * (A(pkc, i - 1, j, k + 1) - pk0);
        OUT(0, A(uc, i, j, k) + ((dt2 * A(rdxc, i, j, k)) / (A(delpc, i - 1, j, k) + wk)) * t);
    }
    {
        const T t = (A(gz, i, j - 1, k + 1) - gz0) * (pk1 - A(pkc, i, j - 1, k)) +
                         (A(gz, i, j - 1, k) - gz1) * (A(pkc, i, j - 1, k + 1) - pk0);
        OUT(1, A(vc, i, j, k) + ((dt2 * A(rdyc, i, j, k)) / (A(delpc, i, j - 1, k) + wk)) * t);
    }
}

// ---------------------------------------------------------------------------------------------
// nh_p_grad:  wk = pk3[k+1] - pk3
//   du = (dt / (wk + wk[i+1])) ((gz[k+1] - gz[i+1])(pk3[i+1,k+1] - pk3) + (gz - gz[i+1,k+1])(pk3[k+1] - pk3[i+1]))
//   u' = ((u + du) + (dt / (delp + delp[i+1])) ((gz[k+1] - gz[i+1])(pp[i+1,k+1] - pp)
//                                                + (gz - gz[i+1,k+1])(pp[k+1] - pp[i+1]))) rdx
// ---------------------------------------------------------------------------------------------
template <class T>
__device__ __forceinline__ void nh_p_grad_pt(const FVT<T> *in, const T *sc, int i, int j, int k, T *r) {
    const FVT<T> &u = in[0], &v = in[1], &pp = in[2], &gz = in[3], &pk3 = in[4], &delp = in[5], &rdx = in[6], &rdy = in[7];
    const T dt = sc[0];
    const T gz0 = A(gz, i, j, k), gz1 = A(gz, i, j, k + 1);
    const T pk0 = A(pk3, i, j, k), pk1 = A(pk3, i, j, k + 1);
    const T pp0 = A(pp, i, j, k), pp1 = A(pp, i, j, k + 1);
    const T wk = pk1 - pk0;
    const T dl = A(delp, i, j, k);
    {  // i direction
        const T gzE = A(gz, i + 1, j, k), gzE1 = A(gz, i + 1, j, k + 1);
        const T pkE = A(pk3, i + 1, j, k), pkE1 = A(pk3, i + 1, j, k + 1);
        const T wkE = pkE1 - pkE;
        const T du = (dt / (wk + wkE)) * ((gz1 - gzE) * (pkE1 - pk0) + (gz0 - gzE1) * (pk1 - pkE));
        const T nh = (dt / (dl + A(delp, i + 1, j, k))) *
                          ((gz1 - gzE) * (A(pp, i + 1, j, k + 1) - pp0) + (gz0 - gzE1) * (pp1 - A(pp, i + 1, j, k)));
        OUT(0, ((A(u, i, j, k) + du) + nh) * A(rdx, i, j, k));
    }
    {  // j direction
        const T gzN = A(gz, i, j + 1, k), gzN1 = A(gz, i, j + 1, k + 1);
        const T pkN = A(pk3, i, j + 1, k), pkN1 = A(pk3, i, j + 1, k + 1);
        const T wkN = pkN1 - pkN;
        const T dv = (dt / (wk + wkN)) * ((gz1 - gzN) * (pkN1 - pk0) + (gz0 - gzN1) * (pk1 - pkN));
        const T nh = (dt / (dl + A(delp, i, j + 1, k))) *
                          ((gz1 - gzN) * (A(pp, i, j + 1, k + 1) - pp0) + (gz0 - gzN1) * (pp1 - A(pp, i, j + 1, k)));
        OUT(1, ((A(v, i, j, k) + dv) + nh) * A(rdy, i, j, k));
    }
}

// ---------------------------------------------------------------------------------------------
// PPM flux through the low face of cell p along direction (di, dj):
//   al(p) = p1 (q[p-1] + q[p]) + p2 (q[p-2] + q[p+1]);  bl(p) = al(p) - q(p);  br(p) = al(p+1) - q(p)
//   flux = c > 0 ? q[p-1] + (1 - c)(br[p-1] - c (bl[p-1] + br[p-1])) : q + (1 + c)(bl + c (bl + br))
// ---------------------------------------------------------------------------------------------
constexpr double P1 = 7.0 / 12.0;
constexpr double P2 = -1.0 / 12.0;

template <class T>
__device__ __forceinline__ T ppm_flux(const FVT<T> &q, T c, int i, int j, int k, int di, int dj) {
    // q at p-3 .. p+2
    const T qm3 = A(q, i - 3 * di, j - 3 * dj, k), qm2 = A(q, i - 2 * di, j - 2 * dj, k);
    const T qm1 = A(q, i - di, j - dj, k), q0 = A(q, i, j, k);
    const T qp1 = A(q, i + di, j + dj, k), qp2 = A(q, i + 2 * di, j + 2 * dj, k);
    const T al_m1 = T(P1) * (qm2 + qm1) + T(P2) * (qm3 + q0);  // al(p-1)
    const T al_0 = T(P1) * (qm1 + q0) + T(P2) * (qm2 + qp1);   // al(p)
    const T al_p1 = T(P1) * (q0 + qp1) + T(P2) * (qm1 + qp2);  // al(p+1)
    if (c > T(0.0)) {
        const T blm = al_m1 - qm1, brm = al_0 - qm1;
        return qm1 + (T(1.0) - c) * (brm - c * (blm + brm));
    } else {
        const T bl = al_0 - q0, br = al_p1 - q0;
        return q0 + (T(1.0) + c) * (bl + c * (bl + br));
    }
}

// fvtp2d_qi: fy2 = flux_y(q, cry); fyy = yfx fy2; q_i = ((q area + fyy) - fyy[j+1]) / ra_y
template <class T>
__device__ __forceinline__ void fvtp2d_qi_pt(const FVT<T> *in, const T *, int i, int j, int k, T *r) {
    const FVT<T> &q = in[0], &cry = in[1], &yfx = in[2], &area = in[3], &ra_y = in[4];
    const T fy2 = ppm_flux(q, A(cry, i, j, k), i, j, k, 0, 1);
    const T fy2n = ppm_flux(q, A(cry, i, j + 1, k), i, j + 1, k, 0, 1);
    const T fyy = A(yfx, i, j, k) * fy2, fyyn = A(yfx, i, j + 1, k) * fy2n;
    OUT(0, ((A(q, i, j, k) * A(area, i, j, k) + fyy) - fyyn) / A(ra_y, i, j, k));
    OUT(1, fy2);
}

// fvtp2d_qj: fx = flux_x(q_i, crx); fx2 = flux_x(q, crx); fx1 = xfx fx2; q_j = ((q area + fx1) - fx1[i+1]) / ra_x
template <class T>
__device__ __forceinline__ void fvtp2d_qj_pt(const FVT<T> *in, const T *, int i, int j, int k, T *r) {
    const FVT<T> &q = in[0], &q_i = in[1], &crx = in[2], &xfx = in[3], &area = in[4], &ra_x = in[5];
    const T c0 = A(crx, i, j, k), c1 = A(crx, i + 1, j, k);
    const T fx = ppm_flux(q_i, c0, i, j, k, 1, 0);
    const T fx2 = ppm_flux(q, c0, i, j, k, 1, 0);
    const T fx2n = ppm_flux(q, c1, i + 1, j, k, 1, 0);
    const T fx1 = A(xfx, i, j, k) * fx2, fx1n = A(xfx, i + 1, j, k) * fx2n;
    OUT(0, ((A(q, i, j, k) * A(area, i, j, k) + fx1) - fx1n) / A(ra_x, i, j, k));
    OUT(1, fx);
    OUT(2, fx2);
}

// fvtp2d_flux: fy = flux_y(q_j, cry); fx_out = (0.5 (fx + fx2)) mfx; fy_out = (0.5 (fy + fy2)) mfy
template <class T>
__device__ __forceinline__ void fvtp2d_flux_pt(const FVT<T> *in, const T *, int i, int j, int k, T *r) {
    const FVT<T> &q_j = in[0], &cry = in[1], &fx = in[2], &fx2 = in[3], &fy2 = in[4], &mfx = in[5], &mfy = in[6];
    const T fy = ppm_flux(q_j, A(cry, i, j, k), i, j, k, 0, 1);
    OUT(0, (T(0.5) * (A(fx, i, j, k) + A(fx2, i, j, k))) * A(mfx, i, j, k));
    OUT(1, (T(0.5) * (fy + A(fy2, i, j, k))) * A(mfy, i, j, k));
}

// ---------------------------------------------------------------------------------------------
// fastwaves:
//   ppgk = wgtfac ppuv + (1 - wgtfac) ppuv[k-1];  ppgc = ppgk[k+1] - ppgk
//   ppgu = (ppuv[i+1] - ppuv) + ((((ppgc[i+1] + ppgc) 0.5) ((hhl[k+1] + hhl) - (hhl[i+1,k+1] + hhl[i+1])))
//                               / ((hhl[k+1] - hhl) + (hhl[i+1,k+1] - hhl[i+1])))
//   u_out = u_pos + (u_tens - ((ppgu 2) fx) / (rho[i+1] + rho)) dt ;  v: j, edadlat
// ---------------------------------------------------------------------------------------------
template <class T>
__device__ __forceinline__ T fw_ppgc(const FVT<T> &ppuv, const FVT<T> &wgt, int i, int j, int k) {
    const T w0 = A(wgt, i, j, k), w1 = A(wgt, i, j, k + 1);
    const T pm = A(ppuv, i, j, k - 1), p0 = A(ppuv, i, j, k), p1 = A(ppuv, i, j, k + 1);
    const T g0 = w0 * p0 + (T(1.0) - w0) * pm;
    const T g1 = w1 * p1 + (T(1.0) - w1) * p0;
    return g1 - g0;
}

template <class T>
__device__ __forceinline__ void fastwaves_pt(const FVT<T> *in, const T *sc, int i, int j, int k, T *r) {
    const FVT<T> &u_pos = in[0], &v_pos = in[1], &u_tens = in[2], &v_tens = in[3], &rho = in[4], &ppuv = in[5], &fx = in[6],
             &wgt = in[7], &hhl = in[8];
    const T edadlat = sc[0], dt = sc[1];
    const T pc = fw_ppgc(ppuv, wgt, i, j, k);
    const T p0 = A(ppuv, i, j, k), h0 = A(hhl, i, j, k), h1 = A(hhl, i, j, k + 1), r0 = A(rho, i, j, k);
    {
        const T hE = A(hhl, i + 1, j, k), hE1 = A(hhl, i + 1, j, k + 1);
        const T ppgu = (A(ppuv, i + 1, j, k) - p0) +
                            (((fw_ppgc(ppuv, wgt, i + 1, j, k) + pc) * T(0.5)) * ((h1 + h0) - (hE1 + hE))) /
                                ((h1 - h0) + (hE1 - hE));
        OUT(0,
          A(u_pos, i, j, k) + (A(u_tens, i, j, k) - ((ppgu * T(2.0)) * A(fx, i, j, k)) / (A(rho, i + 1, j, k) + r0)) * dt);
    }
    {
        const T hN = A(hhl, i, j + 1, k), hN1 = A(hhl, i, j + 1, k + 1);
        const T ppgv = (A(ppuv, i, j + 1, k) - p0) +
                            (((fw_ppgc(ppuv, wgt, i, j + 1, k) + pc) * T(0.5)) * ((h1 + h0) - (hN1 + hN))) /
                                ((h1 - h0) + (hN1 - hN));
        OUT(1,
          A(v_pos, i, j, k) + (A(v_tens, i, j, k) - ((ppgv * T(2.0)) * edadlat) / (A(rho, i, j + 1, k) + r0)) * dt);
    }
}

// ---------------------------------------------------------------------------------------------
template <class T>
struct SuiteArgs {
    FVT<T> in[9];
    FOT<T> out[3];
    T sc[2];
    Dom d;
};

#ifndef SU_BX
#define SU_BX 32
#endif
#ifndef SU_BY
#define SU_BY 4
#endif
#ifndef SU_KC
#define SU_KC 1
#endif

// One thread computes KC consecutive levels and UJ consecutive rows of one i (stencil unrolling
// along j: the operator is replicated per row, and the compiler's common-subexpression
// elimination removes the loads and producer evaluations the rows share).  Every load is issued
// before any store (outputs are kept in registers), so the loads overlap.
template <class T, void (*F)(const FVT<T> *, const T *, int, int, int, T *), int NO, int KC, int UJ>
__global__ void __launch_bounds__(SU_BX * SU_BY) suite_kernel(const __grid_constant__ SuiteArgs<T> a) {
    const int i = a.d.lo[0] + blockIdx.x * SU_BX + threadIdx.x;
    const int j = a.d.lo[1] + (blockIdx.y * SU_BY + threadIdx.y) * UJ;
    const int k0 = a.d.lo[2] + blockIdx.z * KC;
    griddep_wait();  // PDL: inputs may be the previous kernel's outputs
    if (i >= a.d.hi[0] || j >= a.d.hi[1]) {
        griddep_launch_dependents();
        return;
    }
    T r[KC][UJ][NO];
#pragma unroll
    for (int kk = 0; kk < KC; ++kk)
#pragma unroll
        for (int u = 0; u < UJ; ++u) F(a.in, a.sc, i, min(j + u, a.d.hi[1] - 1), min(k0 + kk, a.d.hi[2] - 1), r[kk][u]);
#pragma unroll
    for (int kk = 0; kk < KC; ++kk)
#pragma unroll
        for (int u = 0; u < UJ; ++u)
            if (k0 + kk < a.d.hi[2] && j + u < a.d.hi[1]) {
#pragma unroll
                for (int o = 0; o < NO; ++o)
                    a.out[o].p[i + (j + u) * a.out[o].sj + (k0 + kk) * a.out[o].sk] = r[kk][u][o];
            }
    griddep_launch_dependents();  // late: dependents launched early would idle in griddepcontrol.wait
}

template <class T, int UJ>
cudaError_t launch_suite_u(int program_id, const SuiteArgs<T> &a, cudaStream_t s) {
    constexpr int KC = SU_KC;
    const Dom &d = a.d;
    dim3 block(SU_BX, SU_BY, 1);
    dim3 grid((d.hi[0] - d.lo[0] + SU_BX - 1) / SU_BX, (d.hi[1] - d.lo[1] + SU_BY * UJ - 1) / (SU_BY * UJ),
              (d.hi[2] - d.lo[2] + KC - 1) / KC);
    switch (program_id) {
    case OEC_PROG_UVBKE: return launch_pdl(suite_kernel<T, uvbke_pt<T>, 2, KC, UJ>, grid, block, 0, s, a);
    case OEC_PROG_P_GRAD_C: return launch_pdl(suite_kernel<T, p_grad_c_pt<T>, 2, KC, UJ>, grid, block, 0, s, a);
    case OEC_PROG_NH_P_GRAD: return launch_pdl(suite_kernel<T, nh_p_grad_pt<T>, 2, KC, UJ>, grid, block, 0, s, a);
    case OEC_PROG_FVTP2D_QI: return launch_pdl(suite_kernel<T, fvtp2d_qi_pt<T>, 2, KC, UJ>, grid, block, 0, s, a);
    case OEC_PROG_FVTP2D_QJ: return launch_pdl(suite_kernel<T, fvtp2d_qj_pt<T>, 3, KC, UJ>, grid, block, 0, s, a);
    case OEC_PROG_FVTP2D_FLUX: return launch_pdl(suite_kernel<T, fvtp2d_flux_pt<T>, 2, KC, UJ>, grid, block, 0, s, a);
    case OEC_PROG_FASTWAVES: return launch_pdl(suite_kernel<T, fastwaves_pt<T>, 2, KC, UJ>, grid, block, 0, s, a);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace

template <class T>
cudaError_t launch_suite(int program_id, const FVT<T> *in, const FOT<T> *out, const double *scalars, const Dom &d,
                         int unroll, cudaStream_t s, int *launches) {
    SuiteArgs<T> a;
    for (int q = 0; q < 9; ++q) a.in[q] = in[q];
    for (int q = 0; q < 3; ++q) a.out[q] = out[q];
    a.sc[0] = (T)scalars[0];
    a.sc[1] = (T)scalars[1];
    a.d = d;
    cudaError_t e = unroll == 4 ? launch_suite_u<T, 4>(program_id, a, s)
                  : unroll == 2 ? launch_suite_u<T, 2>(program_id, a, s)
                                : launch_suite_u<T, 1>(program_id, a, s);
    ++*launches;
    return e != cudaSuccess ? e : cudaGetLastError();
}

template cudaError_t launch_suite<double>(int, const FV *, const FO *, const double *, const Dom &, int, cudaStream_t,
                                          int *);
template cudaError_t launch_suite<float>(int, const FVf *, const FOf *, const double *, const Dom &, int, cudaStream_t,
                                         int *);

}  // namespace oec
