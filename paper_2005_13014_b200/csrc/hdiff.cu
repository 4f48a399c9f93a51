// hdiff -- COSMO horizontal diffusion, fused into one pass over HBM (stencil inlining, P:431;
// "we do not need to store and load any temporary buffer").  Definition: include/oec.h,
// DESIGN.md readings R1-R6.  Built with --fmad=false: every + - * below rounds separately, in the
// parenthesised order of the definition, so results equal the CPU oracle bit for bit.
//
// Three kernels:
//  * hdiff_tma    -- default B200 design: persistent CTAs of NW
//                    independent warps; each warp owns an S-deep ring of shared-memory slots fed by
//                    TMA (cp.async.bulk.tensor, mbarrier complete_tx).  A work item is a W x JB tile
//                    of one k-plane: one TMA box of `in` ((W+2LP) x (JB+4), halo included, OOB
//                    zero-filled) and one of `coeff` (W x JB).  The warp walks the tile along j,
//                    each lane reading its V columns plus the 2-wide halo straight from shared
//                    memory (16-byte LDS, conflict-free) and rolling lap/flx/fly in registers.
//                    The bytes in flight live in the TMA ring, not in registers, so ~S items per
//                    warp are always streaming from HBM while the warp computes.
//  * hdiff_naive  -- the paper's execution model: one thread per grid point, every
//                    producer inlined and recomputed, all temporaries in registers, no shared
//                    memory, no synchronisation.  13 `in` loads per point go through L1.
//  * hdiff_roll   -- B200 design: a warp owns a W = 32*V wide i-segment
//                    of one k-plane and walks a chunk of JB rows along j.  Each `in` row is loaded
//                    once (coalesced, 16-byte vectors when aligned) plus a 2-wide halo on each side,
//                    extended to i-2..i+V+1 per lane with warp shuffles, and rolled through
//                    registers: lap, flx and fly are recomputed per lane from registers (no L1
//                    re-reads, no shared memory, no barriers).  P rows of `in` and `coeff` are kept
//                    in flight per warp (software prefetch) for memory-level parallelism.
#include <algorithm>

#include "oec_internal.h"
#include "tma.h"

// Two tile configurations (measured sweeps in profiles/ncu_summary_r01.md): small domains want
// many short tiles per SM (V=2: 64 columns, JB=4 rows, 12 warps x 2 slots); large domains want
// wide 2-row tiles (V=4: 128 columns) -- more independent warps in flight per SM.
#ifndef HD_V
#define HD_V 2
#endif
#ifndef HD_JB
#define HD_JB 4
#endif
#ifndef HD_S
#define HD_S 2
#endif
#ifndef HD_NW
#define HD_NW 12
#endif
#ifndef HDL_V
#define HDL_V 4
#endif
#ifndef HDL_JB
#define HDL_JB 2
#endif
#ifndef HDL_S
#define HDL_S 2
#endif
#ifndef HDL_NW
#define HDL_NW 12
#endif
// f32: V doubled so a tile row is as many bytes as in f64 (the TMA box is <= 256 elements
// wide: 32 V + 8 <= 256 -> V <= 7; V % 4 == 0 for 16-byte shared-memory loads)
#ifndef HF_V
#define HF_V 4
#endif
#ifndef HF_JB
#define HF_JB 4
#endif
#ifndef HF_S
#define HF_S 2
#endif
#ifndef HF_NW
#define HF_NW 12
#endif
#ifndef HFL_V
#define HFL_V 4
#endif
#ifndef HFL_JB
#define HFL_JB 2
#endif
#ifndef HFL_S
#define HFL_S 2
#endif
#ifndef HFL_NW
#define HFL_NW 8  // round 2: two 8-warp CTAs per SM, f32 1024^2 210.6 -> 197.4 us (f64 keeps 12: 381.6 vs 393.1)
#endif
#ifndef HD_PF
#define HD_PF 1  // tiles per warp prefetched into L2 before griddepcontrol.wait (round 2: 1 beats 2 by 1.5% at 128^2, profiles/r02/hdiff_cfg_r02.md)
#endif
// tiny domains (<= HD_TINY_POINTS, e.g. 128x128x80): the same tiles in CTAs of HD_TNW warps, two
// per SM (16 warps instead of 12; an SM starts a CTA of the next launch as soon as one of its two
// finishes): 128^2 x 80 f64 6.76 -> 6.57 us, f32 4.65 -> 4.38; 256x256x60 keeps 12-warp CTAs
// (16.2 vs 16.7 us; profiles/r02/hdiff_nw_r02.md)
#ifndef HF_PF
#define HF_PF HD_PF  // f32
#endif
#ifndef HD_TNW
#define HD_TNW 8
#endif
#ifndef HF_TNW
#define HF_TNW 8
#endif
#ifndef HD_TINY_POINTS
#define HD_TINY_POINTS (2ll << 20)
#endif
#ifndef HD_LARGE_POINTS
#define HD_LARGE_POINTS (8ll << 20)  // measured: the small tiles win up to 256^2 x 80 (0.79 -> 0.83)
#endif

#ifdef HD_TRACE
// debug timeline of CTA 0 and CTA gridDim-1: [cta(0/1)][warp][event]: 0 start, 1+2n item n data ready, 2+2n item n done
__device__ unsigned long long g_htrace[2][8][64];
extern "C" int oec_debug_hdiff_trace(unsigned long long *out) {
    return (int)cudaMemcpyFromSymbol(out, g_htrace, sizeof(g_htrace));
}
#define HTRACE(ev)                                                                                         \
    do {                                                                                                   \
        const int c_ = blockIdx.x == 0 ? 0 : (blockIdx.x == gridDim.x - 1 ? 1 : -1);                        \
        if (c_ >= 0 && (threadIdx.x & 31) == 0 && (ev) < 64) {                                             \
            unsigned long long t_;                                                                         \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                          \
            g_htrace[c_][threadIdx.x >> 5][ev] = t_;                                                        \
        }                                                                                                  \
    } while (0)
#else
#define HTRACE(ev) \
    do {           \
    } while (0)
#endif

namespace oec {
namespace {

template <class T>
__device__ __forceinline__ T ld(const FVT<T> &f, int i, int j, int k) { return __ldg(f.p + (i + j * f.sj + k * f.sk)); }

template <class T>
__device__ __forceinline__ T lap_pt(T c, T w, T e, T s, T n) {
    // lap(i,j) = ((in(i-1,j) + in(i+1,j)) + (in(i,j-1) + in(i,j+1))) - 4 in(i,j)
    return ((w + e) + (s + n)) - T(4.0) * c;
}
template <class T>
__device__ __forceinline__ T limit(T f, T din) { return (f * din > T(0.0)) ? T(0.0) : f; }

// ---------------------------------------------------------------------------------------------
// paper execution model
// ---------------------------------------------------------------------------------------------
// UJ > 1: stencil unrolling along j: one thread updates UJ consecutive rows; the
// Laplacians and loads the rows share are computed once (common-subexpression elimination).
template <class T, int UJ>
__global__ void __launch_bounds__(128) hdiff_naive(FVT<T> in, FVT<T> coeff, FOT<T> out, Dom d) {
    const int i = d.lo[0] + blockIdx.x * 32 + threadIdx.x;
    const int j0 = d.lo[1] + (blockIdx.y * 4 + threadIdx.y) * UJ;
    const int k = d.lo[2] + blockIdx.z;
    if (i >= d.hi[0] || j0 >= d.hi[1]) return;
    auto L = [&](int a, int b) {
        return lap_pt(ld(in, a, b, k), ld(in, a - 1, b, k), ld(in, a + 1, b, k), ld(in, a, b - 1, k), ld(in, a, b + 1, k));
    };
    T r[UJ];
#pragma unroll
    for (int u = 0; u < UJ; ++u) {
        const int j = min(j0 + u, d.hi[1] - 1);
        const T c0 = ld(in, i, j, k);
        const T l0 = L(i, j), le = L(i + 1, j), lw = L(i - 1, j), ln = L(i, j + 1), ls = L(i, j - 1);
        const T flx = limit(le - l0, ld(in, i + 1, j, k) - c0);
        const T flxm = limit(l0 - lw, c0 - ld(in, i - 1, j, k));
        const T fly = limit(ln - l0, ld(in, i, j + 1, k) - c0);
        const T flym = limit(l0 - ls, c0 - ld(in, i, j - 1, k));
        r[u] = c0 - ld(coeff, i, j, k) * ((flx - flxm) + (fly - flym));
    }
#pragma unroll
    for (int u = 0; u < UJ; ++u)
        if (j0 + u < d.hi[1]) out.p[i + (j0 + u) * out.sj + k * out.sk] = r[u];
}

// ---------------------------------------------------------------------------------------------
// rolling kernel
// ---------------------------------------------------------------------------------------------
template <class T, int V>
struct Vec {  // generic: scalar accesses
    static __device__ __forceinline__ void load(const T *p, T *v) {
#pragma unroll
        for (int x = 0; x < V; ++x) v[x] = __ldg(p + x);
    }
    static __device__ __forceinline__ void store(T *p, const T *v) {
#pragma unroll
        for (int x = 0; x < V; ++x) p[x] = v[x];
    }
};
template <>
struct Vec<double, 2> {
    static __device__ __forceinline__ void load(const double *p, double *v) {
        double2 t = __ldg(reinterpret_cast<const double2 *>(p));
        v[0] = t.x;
        v[1] = t.y;
    }
    static __device__ __forceinline__ void store(double *p, const double *v) {
        *reinterpret_cast<double2 *>(p) = make_double2(v[0], v[1]);
    }
};
template <>
struct Vec<double, 4> {
    static __device__ __forceinline__ void load(const double *p, double *v) {
        Vec<double, 2>::load(p, v);
        Vec<double, 2>::load(p + 2, v + 2);
    }
    static __device__ __forceinline__ void store(double *p, const double *v) {
        Vec<double, 2>::store(p, v);
        Vec<double, 2>::store(p + 2, v + 2);
    }
};
template <>
struct Vec<float, 4> {
    static __device__ __forceinline__ void load(const float *p, float *v) {
        float4 t = __ldg(reinterpret_cast<const float4 *>(p));
        v[0] = t.x;
        v[1] = t.y;
        v[2] = t.z;
        v[3] = t.w;
    }
    static __device__ __forceinline__ void store(float *p, const float *v) {
        *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <>
struct Vec<float, 8> {
    static __device__ __forceinline__ void load(const float *p, float *v) {
        Vec<float, 4>::load(p, v);
        Vec<float, 4>::load(p + 4, v + 4);
    }
    static __device__ __forceinline__ void store(float *p, const float *v) {
        Vec<float, 4>::store(p, v);
        Vec<float, 4>::store(p + 4, v + 4);
    }
};

// raw row as loaded: V own values + (lane 0) 2 left-halo values + (lane 31) 2 right-halo values
template <class T, int V>
struct RawRow {
    T v[V];
    T h[2];
};

template <class T, int V>
__device__ __forceinline__ void load_row(const T *rowp, int i_own, int lane, int i_end_in, int ib, RawRow<T, V> &r) {
    // rowp: pointer to element (0, j, k); i_own = ib + lane*V; valid `in` columns: i < i_end_in
    if (i_own + V <= i_end_in) {
        Vec<T, V>::load(rowp + i_own, r.v);
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v) r.v[v] = (i_own + v < i_end_in) ? __ldg(rowp + i_own + v) : T(0.0);
    }
    r.h[0] = r.h[1] = T(0.0);
    if (lane == 0) {
        r.h[0] = __ldg(rowp + ib - 2);
        r.h[1] = __ldg(rowp + ib - 1);
    } else if (lane == 31) {
        const int ir = ib + 32 * V;
        if (ir < i_end_in) r.h[0] = __ldg(rowp + ir);
        if (ir + 1 < i_end_in) r.h[1] = __ldg(rowp + ir + 1);
    }
}

// extended row: e[x + 2] = in(i_own + x), x in [-2, V+1]
template <class T, int V>
__device__ __forceinline__ void extend(const RawRow<T, V> &r, int lane, T *e) {
    constexpr unsigned FULL = 0xffffffffu;
#pragma unroll
    for (int v = 0; v < V; ++v) e[v + 2] = r.v[v];
    T l1, l2, r1, r2;
    if (V >= 2) {
        l2 = __shfl_up_sync(FULL, r.v[V - 2 < 0 ? 0 : V - 2], 1);
        l1 = __shfl_up_sync(FULL, r.v[V - 1], 1);
        r1 = __shfl_down_sync(FULL, r.v[0], 1);
        r2 = __shfl_down_sync(FULL, r.v[V >= 2 ? 1 : 0], 1);
    } else {
        l2 = __shfl_up_sync(FULL, r.v[0], 2);
        l1 = __shfl_up_sync(FULL, r.v[0], 1);
        r1 = __shfl_down_sync(FULL, r.v[0], 1);
        r2 = __shfl_down_sync(FULL, r.v[0], 2);
    }
    if (V == 1) {  // lanes 1 and 30 take the halo values held by lanes 0 and 31
        const T hl = __shfl_sync(FULL, r.h[1], 0);
        const T hr = __shfl_sync(FULL, r.h[0], 31);
        if (lane == 1) l2 = hl;
        if (lane == 30) r2 = hr;
    }
    if (lane == 0) {
        l2 = r.h[0];
        l1 = r.h[1];
    }
    if (lane == 31) {
        r1 = r.h[0];
        r2 = r.h[1];
    }
    e[0] = l2;
    e[1] = l1;
    e[V + 2] = r1;
    e[V + 3] = r2;
}

template <class T, int V, int JB, int P>
__global__ void __launch_bounds__(128) hdiff_roll(FVT<T> in, FVT<T> coeff, FOT<T> out, Dom d, int nseg, int nchunk) {
    constexpr int W = 32 * V;
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int seg = warp % nseg;
    const int chunk = (warp / nseg) % nchunk;
    const int k = d.lo[2] + warp / (nseg * nchunk);
    if (k >= d.hi[2]) return;  // whole warp exits together
    const int ib = d.lo[0] + seg * W;
    const int i_own = ib + lane * V;
    const int i_end_in = d.hi[0] + 2;  // `in` columns needed: [ib-2, min(ib+W, hi0)+2)
    const int j0 = d.lo[1] + chunk * JB;
    const int j1 = min(j0 + JB, d.hi[1]);
    const T *in_k = in.p + k * in.sk;
    const T *cf_k = coeff.p + k * coeff.sk;
    T *out_k = out.p + k * out.sk;

    T E0[V + 4], E1[V + 4], E2[V + 4];  // in rows j, j+1, j+2 (extended)
    T Lj[V + 2];                        // lap row j at i_own-1 .. i_own+V
    T FYm[V];                           // fly(j-1) at own points

    // ---- warm-up: rows j0-2 .. j0+1 ----
    {
        RawRow<T, V> r;
        T Em2[V + 4], Em1[V + 4];
        load_row<T, V>(in_k + (j0 - 2) * in.sj, i_own, lane, i_end_in, ib, r);
        extend<T, V>(r, lane, Em2);
        load_row<T, V>(in_k + (j0 - 1) * in.sj, i_own, lane, i_end_in, ib, r);
        extend<T, V>(r, lane, Em1);
        load_row<T, V>(in_k + j0 * in.sj, i_own, lane, i_end_in, ib, r);
        extend<T, V>(r, lane, E0);
        load_row<T, V>(in_k + (j0 + 1) * in.sj, i_own, lane, i_end_in, ib, r);
        extend<T, V>(r, lane, E1);
        T Lm[V];  // lap(j0-1) at own points
#pragma unroll
        for (int x = 0; x < V; ++x) Lm[x] = lap_pt(Em1[x + 2], Em1[x + 1], Em1[x + 3], Em2[x + 2], E0[x + 2]);
#pragma unroll
        for (int y = 0; y < V + 2; ++y)  // lap(j0) at i_own + y - 1
            Lj[y] = lap_pt(E0[y + 1], E0[y], E0[y + 2], Em1[y + 1], E1[y + 1]);
#pragma unroll
        for (int x = 0; x < V; ++x) FYm[x] = limit(Lj[x + 1] - Lm[x], E0[x + 2] - Em1[x + 2]);
    }

    // ---- prefetch ring: slot s holds in row (j+2) and coeff row j for step j = j0 + s (mod P) ----
    RawRow<T, V> ring_in[P];
    T ring_cf[P][V];
    const bool own_valid = i_own < d.hi[0];
#pragma unroll
    for (int s = 0; s < P; ++s) {
        const int j = j0 + s;
        if (j < j1) {
            load_row<T, V>(in_k + (j + 2) * in.sj, i_own, lane, i_end_in, ib, ring_in[s]);
            if (own_valid) {
                if (i_own + V <= d.hi[0]) Vec<T, V>::load(cf_k + j * coeff.sj + i_own, ring_cf[s]);
                else {
#pragma unroll
                    for (int v = 0; v < V; ++v) ring_cf[s][v] = (i_own + v < d.hi[0]) ? __ldg(cf_k + j * coeff.sj + i_own + v) : T(0.0);
                }
            }
        }
    }

    for (int jb = j0; jb < j1; jb += P) {
#pragma unroll
        for (int s = 0; s < P; ++s) {
            const int j = jb + s;
            if (j < j1) {  // warp-uniform
                extend<T, V>(ring_in[s], lane, E2);
                T cf[V];
#pragma unroll
                for (int v = 0; v < V; ++v) cf[v] = ring_cf[s][v];
                // refill this slot with step j + P
                const int jn = j + P;
                if (jn < j1) {
                    load_row<T, V>(in_k + (jn + 2) * in.sj, i_own, lane, i_end_in, ib, ring_in[s]);
                    if (own_valid) {
                        if (i_own + V <= d.hi[0]) Vec<T, V>::load(cf_k + jn * coeff.sj + i_own, ring_cf[s]);
                        else {
#pragma unroll
                            for (int v = 0; v < V; ++v)
                                ring_cf[s][v] = (i_own + v < d.hi[0]) ? __ldg(cf_k + jn * coeff.sj + i_own + v) : T(0.0);
                        }
                    }
                }
                // lap(j+1) at i_own-1 .. i_own+V
                T L1[V + 2];
#pragma unroll
                for (int y = 0; y < V + 2; ++y) L1[y] = lap_pt(E1[y + 1], E1[y], E1[y + 2], E0[y + 1], E2[y + 1]);
                // flx(j) at i_own-1 .. i_own+V-1:  FX[y] <-> i_own + y - 1
                T FX[V + 1];
#pragma unroll
                for (int y = 0; y < V + 1; ++y) FX[y] = limit(Lj[y + 1] - Lj[y], E0[y + 2] - E0[y + 1]);
                // fly(j) at own points
                T FY[V];
#pragma unroll
                for (int x = 0; x < V; ++x) FY[x] = limit(L1[x + 1] - Lj[x + 1], E1[x + 2] - E0[x + 2]);
                T o[V];
#pragma unroll
                for (int x = 0; x < V; ++x) o[x] = E0[x + 2] - cf[x] * ((FX[x + 1] - FX[x]) + (FY[x] - FYm[x]));
                if (own_valid) {
                    T *op = out_k + j * out.sj + i_own;
                    if (i_own + V <= d.hi[0]) Vec<T, V>::store(op, o);
                    else {
#pragma unroll
                        for (int v = 0; v < V; ++v)
                            if (i_own + v < d.hi[0]) op[v] = o[v];
                    }
                }
                // roll
#pragma unroll
                for (int y = 0; y < V + 4; ++y) {
                    E0[y] = E1[y];
                    E1[y] = E2[y];
                }
#pragma unroll
                for (int y = 0; y < V + 2; ++y) Lj[y] = L1[y];
#pragma unroll
                for (int x = 0; x < V; ++x) FYm[x] = FY[x];
            }
        }
    }
}

// ---------------------------------------------------------------------------------------------
// TMA-fed kernel
// ---------------------------------------------------------------------------------------------
// The `in` box starts LP columns left of the tile: TMA needs the inner start coordinate on a 16-byte
// boundary (measured: tools/micro/tma_f32.cu -- an f32 box starting 8 bytes off a 16-byte boundary
// faults with an illegal instruction), so LP = 16 bytes of elements (2 f64, 4 f32) >= the 2-wide
// halo, and a row is RW = W + 2 LP elements (a 16-byte multiple).
template <class T, int V, int JB, int S, int NW>
struct TmaCfg {
    static constexpr int W = 32 * V;
    static constexpr int LP = 16 / (int)sizeof(T);
    static constexpr int RW = W + 2 * LP;
    static constexpr int IN_ELEMS = (JB + 4) * RW;
    static constexpr int IN_BYTES = IN_ELEMS * (int)sizeof(T);
    static constexpr int CF_BYTES = JB * W * (int)sizeof(T);
    static constexpr int IN_PAD = (IN_BYTES + 127) / 128 * 128;
    static constexpr int CF_PAD = (CF_BYTES + 127) / 128 * 128;
    static constexpr int SLOT = IN_PAD + CF_PAD;
    static constexpr int SMEM = NW * S * SLOT + NW * S * 8;
};

template <class T, int V, int LP>
__device__ __forceinline__ void lds_row(const T *row, int lane, T *e) {
    // e[x] = row[lane*V + (LP-2) + x], x in [0, V+4)  (row element y <-> i = ib - LP + y); widest aligned LDS
    const T *p = row + lane * V;
    if constexpr (sizeof(T) == 4 && V % 4 == 0) {  // LP = 4: 16-byte loads of V+8 elements, shifted by 2
        T t[V + 8];
#pragma unroll
        for (int x = 0; x < V + 8; x += 4) {
            const float4 q = *reinterpret_cast<const float4 *>(p + x);
            t[x] = q.x;
            t[x + 1] = q.y;
            t[x + 2] = q.z;
            t[x + 3] = q.w;
        }
#pragma unroll
        for (int x = 0; x < V + 4; ++x) e[x] = t[x + 2];
    } else if constexpr (sizeof(T) == 8 && V % 2 == 0) {  // LP = 2: 16-byte loads, no shift
#pragma unroll
        for (int x = 0; x < V + 4; x += 2) {
            const double2 q = *reinterpret_cast<const double2 *>(p + x);
            e[x] = q.x;
            e[x + 1] = q.y;
        }
    } else {
#pragma unroll
        for (int x = 0; x < V + 4; ++x) e[x] = p[(LP - 2) + x];
    }
}

// One W x JB tile from shared memory: rows 0..JB+3 of `tin` are j0-2 .. j0+JB+1 (each RW wide,
// element y <-> i = ib-LP+y), `tcf` holds coeff rows j0 .. j0+JB-1 (W wide).  FULL: all JB rows are
// in the domain -> the row loop is fully unrolled without checks (registers renamed, no moves).
template <class T, int V, int JB, int LP, bool FULL>
__device__ __forceinline__ void hdiff_tile(const T *tin, const T *tcf, T *out_k, int sj, int j0,
                                           int nrows, int i_own, int hi0, int lane) {
    constexpr int W = 32 * V;
    constexpr int RW = W + 2 * LP;
    const bool own_valid = i_own < hi0;
    const bool own_full = i_own + V <= hi0;
    const bool warp_full = __all_sync(0xffffffffu, own_full);
    T E0[V + 4], E1[V + 4], E2[V + 4], Lj[V + 2], FYm[V];
    {
        T Em2[V + 4], Em1[V + 4], Lm[V];
        lds_row<T, V, LP>(tin + 0 * RW, lane, Em2);
        lds_row<T, V, LP>(tin + 1 * RW, lane, Em1);
        lds_row<T, V, LP>(tin + 2 * RW, lane, E0);
        lds_row<T, V, LP>(tin + 3 * RW, lane, E1);
#pragma unroll
        for (int x = 0; x < V; ++x) Lm[x] = lap_pt(Em1[x + 2], Em1[x + 1], Em1[x + 3], Em2[x + 2], E0[x + 2]);
#pragma unroll
        for (int y = 0; y < V + 2; ++y) Lj[y] = lap_pt(E0[y + 1], E0[y], E0[y + 2], Em1[y + 1], E1[y + 1]);
#pragma unroll
        for (int x = 0; x < V; ++x) FYm[x] = limit(Lj[x + 1] - Lm[x], E0[x + 2] - Em1[x + 2]);
    }
#pragma unroll
    for (int r = 0; r < JB; ++r) {
        if (!FULL && r >= nrows) break;  // warp-uniform
        lds_row<T, V, LP>(tin + (r + 4) * RW, lane, E2);
        T L1[V + 2], FX[V + 1], FY[V], o[V];
#pragma unroll
        for (int y = 0; y < V + 2; ++y) L1[y] = lap_pt(E1[y + 1], E1[y], E1[y + 2], E0[y + 1], E2[y + 1]);
#pragma unroll
        for (int y = 0; y < V + 1; ++y) FX[y] = limit(Lj[y + 1] - Lj[y], E0[y + 2] - E0[y + 1]);
#pragma unroll
        for (int x = 0; x < V; ++x) FY[x] = limit(L1[x + 1] - Lj[x + 1], E1[x + 2] - E0[x + 2]);
        const T *cfr = tcf + r * W + lane * V;
#pragma unroll
        for (int x = 0; x < V; ++x) o[x] = E0[x + 2] - cfr[x] * ((FX[x + 1] - FX[x]) + (FY[x] - FYm[x]));
        T *op = out_k + (j0 + r) * sj + i_own;
        if (warp_full) Vec<T, V>::store(op, o);  // warp-uniform: no per-lane branch
        else if (own_full) Vec<T, V>::store(op, o);
        else if (own_valid) {
#pragma unroll
            for (int v = 0; v < V; ++v)
                if (i_own + v < hi0) op[v] = o[v];
        }
#pragma unroll
        for (int y = 0; y < V + 4; ++y) {
            E0[y] = E1[y];
            E1[y] = E2[y];
        }
#pragma unroll
        for (int y = 0; y < V + 2; ++y) Lj[y] = L1[y];
#pragma unroll
        for (int x = 0; x < V; ++x) FYm[x] = FY[x];
    }
}

template <class T, int V, int JB, int S, int NW>
__global__ void __launch_bounds__(NW * 32, 1) hdiff_tma(const __grid_constant__ TMap m_in, const __grid_constant__ TMap m_cf,
                                                     FOT<T> out, Dom d, int nseg, int nchunk, int nitems) {
    using C = TmaCfg<T, V, JB, S, NW>;
    constexpr int W = C::W;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *wbase = smem + warp * S * C::SLOT;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + NW * S * C::SLOT) + warp * S;
    const int gw = blockIdx.x * NW + warp, nwt = gridDim.x * NW;

    auto in_s = [&](int s) { return reinterpret_cast<T *>(wbase + s * C::SLOT); };
    auto cf_s = [&](int s) { return reinterpret_cast<T *>(wbase + s * C::SLOT + C::IN_PAD); };
    auto decode = [&](int item, int &ib, int &j0, int &k) {
        const int seg = item % nseg, chunk = (item / nseg) % nchunk;
        k = d.lo[2] + item / (nseg * nchunk);
        ib = d.lo[0] + seg * W;
        j0 = d.lo[1] + chunk * JB;
    };
    auto issue = [&](int item, int s) {
        int ib, j0, k;
        decode(item, ib, j0, k);
        mbar_expect_tx(&bars[s], C::IN_BYTES + C::CF_BYTES);
        tma_load_ijk(in_s(s), m_in, &bars[s], ib - C::LP, j0 - 2, k);
        tma_load_ijk(cf_s(s), m_cf, &bars[s], ib, j0, k);
    };

    HTRACE(0);
    griddep_launch_dependents();
    if (lane == 0) {
        prefetch_tmap(&m_in.map);
        prefetch_tmap(&m_cf.map);
#pragma unroll
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
#pragma unroll
        for (int s = 0; s < (sizeof(T) == 8 ? HD_PF : HF_PF); ++s)  // warm L2 with the first tiles during the previous kernel's drain
            if (gw + s * nwt < nitems) {
                int ib, j0, k;
                decode(gw + s * nwt, ib, j0, k);
                tma_prefetch_ijk(m_in, ib - C::LP, j0 - 2, k);
                tma_prefetch_ijk(m_cf, ib, j0, k);
            }
    }
    griddep_wait();  // inputs may be the previous kernel's outputs
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (gw + s * nwt < nitems) issue(gw + s * nwt, s);
    }
    __syncwarp();

    int n = 0;
    for (int item = gw; item < nitems; item += nwt, ++n) {
        const int s = n % S;
        int ib, j0, k;
        decode(item, ib, j0, k);
        const int nrows = min(JB, d.hi[1] - j0);
        const int i_own = ib + lane * V;
        T *out_k = out.p + k * out.sk;
        mbar_wait(&bars[s], (n / S) & 1);
        HTRACE(1 + 2 * n);
        if (nrows == JB)
            hdiff_tile<T, V, JB, C::LP, true>(in_s(s), cf_s(s), out_k, out.sj, j0, JB, i_own, d.hi[0], lane);
        else
            hdiff_tile<T, V, JB, C::LP, false>(in_s(s), cf_s(s), out_k, out.sj, j0, nrows, i_own, d.hi[0], lane);
        __syncwarp();
        HTRACE(2 + 2 * n);
        if (lane == 0) {
            const int nxt = item + S * nwt;
            if (nxt < nitems) {
                fence_proxy_async();  // our generic-proxy reads of slot s precede the TMA refill
                issue(nxt, s);
            }
        }
    }
}

template <class T, int V, int JB, int S, int NW>
cudaError_t launch_tma(const TMap &tin, const TMap &tcf, const FOT<T> &out, const Dom &d, cudaStream_t st, int *launches) {
    using C = TmaCfg<T, V, JB, S, NW>;
    const int ni = d.hi[0] - d.lo[0], nj = d.hi[1] - d.lo[1], nk = d.hi[2] - d.lo[2];
    const int nseg = (ni + C::W - 1) / C::W, nchunk = (nj + JB - 1) / JB;
    const long long nitems = (long long)nseg * nchunk * nk;
    if (nitems > INT32_MAX) return cudaErrorInvalidValue;
    static bool configured = false;
    static int blocks_per_sm = 1, sms = 148;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(hdiff_tma<T, V, JB, S, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        int dev;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, hdiff_tma<T, V, JB, S, NW>, NW * 32, C::SMEM);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
        configured = true;
    }
    long long blocks = std::min<long long>((nitems + NW - 1) / NW, (long long)sms * blocks_per_sm);
    cudaError_t e = launch_pdl(hdiff_tma<T, V, JB, S, NW>, dim3((unsigned)blocks), dim3(NW * 32), C::SMEM, st, tin, tcf, out,
                               d, nseg, nchunk, (int)nitems);
    ++*launches;
    return e != cudaSuccess ? e : cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// multi-step hdiff with the halo exchange fused in (north_star (3))
// ---------------------------------------------------------------------------------------------
// One launch = one time step t of x_{t+1} = hdiff(x_t) on this rank's sub-domain, x_t in buffer
// t % 2.  t lives in the signal pad (device memory), so a captured CUDA graph of N launches runs N
// steps.  Work items are ordered interior first: an interior tile's 13-point diamond never leaves
// our sub-domain (or reaches only the caller's global outer halo), so it streams through the TMA
// ring exactly as hdiff_tma and needs nothing from the neighbours.  Boundary tiles come last: the
// warp waits (once) until every neighbour has completed step t-1, then assembles the tile in
// shared memory with plain loads -- our cells from our field, the neighbours' cells straight from
// THEIR fields (peer memory over NVLink, or the same device) -- and runs the same tile code.  No
// halo is copied, no exchange kernel or NCCL call exists, and the transfer overlaps the interior.
// Step counting without a returning atomic: every CTA, once its warps are done, adds its share
// w_b of 2^20 (the shares of a grid sum to exactly 2^20, whatever its size) to our FINISHED word
// (relaxed: read by our next step after griddepcontrol.wait, i.e. after this grid completed, so
// t = FINISHED >> 20) and to each neighbour's word for us (red.release.sys: the neighbour's
// boundary tiles of step t+1 wait until it reaches (t+1) << 20).  Safety: a neighbour's step t+1
// overwrites the buffer we read at step t only in its boundary tiles, which wait for our "step t
// done".  (Round 1 counted CTAs with acq_rel atomics and let the last one publish: the returning
// atomics of 148 CTAs on one word cost 0.85 us per step at 128^2.)
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_gpu(unsigned long long *p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
constexpr int PIPE_STEP_SHIFT = 20;  // one completed step = 2^20 in a FINISHED / neighbour word

// "step done" counting: acq_rel atomics (PTX release is cumulative over everything that
// happens-before it, acquire makes the other arrivals' prior accesses visible to the last one)
__device__ __forceinline__ unsigned atom_add_acqrel_cta_shared(unsigned *p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned long long atom_add_relaxed_gpu(unsigned long long *p, unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
    return old;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
}
#ifndef PIPE_WAIT_NS
#define PIPE_WAIT_NS 20000000000ull
#endif

template <class T>
__device__ __forceinline__ T pipe_cell(const PipeArgs<T> &a, int b, int i, int j, int k) {
    // value of x_t at (i, j, k), local coordinates, whoever owns it; cells beyond the 2-wide halo
    // are never used by the tile arithmetic (0)
    const int ni = a.d.hi[0], nj = a.d.hi[1];
    if (i < -2 || i >= ni + 2 || j < -2 || j >= nj + 2) return T(0);
    const int si = i < 0 ? 0 : (i >= ni ? 2 : 1), sj = j < 0 ? 0 : (j >= nj ? 2 : 1);
    const int dir = si * 3 + sj;
    if (dir != 4 && a.nb[dir].exists) {
        const PeerNb<T> &n = a.nb[dir];
        return __ldcg(n.x[b] + ((i - n.oi) + (j - n.oj) * n.sj + k * n.sk));  // peer: bypass L1
    }
    if (i < a.alo[0] || i >= a.ahi[0] || j < a.alo[1] || j >= a.ahi[1]) return T(0);
    return a.x[b].p[i + j * a.x[b].sj + k * a.x[b].sk];
}

template <class T, int V, int JB, int S, int NW>
__global__ void __launch_bounds__(NW * 32, 1) hdiff_pipe(const __grid_constant__ TMap m0, const __grid_constant__ TMap m1,
                                                      const __grid_constant__ TMap m_cf,
                                                      const __grid_constant__ PipeArgs<T> a) {
    using C = TmaCfg<T, V, JB, S, NW>;
    constexpr int W = C::W;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *wbase = smem + warp * S * C::SLOT;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + NW * S * C::SLOT) + warp * S;
    unsigned *warps_done = reinterpret_cast<unsigned *>(reinterpret_cast<uint64_t *>(smem + NW * S * C::SLOT) + NW * S);
    const int gw = blockIdx.x * NW + warp, nwt = gridDim.x * NW;
    bool any_nb = false;
#pragma unroll
    for (int dd = 0; dd < 9; ++dd) any_nb = any_nb || (a.nb[dd].exists != 0);
    // programmatic dependent launch: descriptor prefetch and barrier setup overlap the previous
    // step's drain; the step counter and x_t are read only after the previous grid completed
    if (lane == 0) {
        prefetch_tmap(&m0.map);
        prefetch_tmap(&m1.map);
        prefetch_tmap(&m_cf.map);
    }
    if (threadIdx.x == 0) *warps_done = 0;
    unsigned long long tg = 0;  // the guessed step t (lane 0)
    if (lane == 0) {
        // warm L2 with the first interior tiles during the previous kernel's drain: coefficients,
        // and x_t of the GUESSED step t.  The guess reads the pad before griddepcontrol.wait, so
        // it may be stale; it selects what to prefetch and which buffer the first tiles are
        // requested from -- the step t read after the wait decides.  If this pipeline's previous
        // step is still draining (this CTA only got an SM because one of its CTAs exited, having
        // added its share), FINISHED is between two multiples of 2^20: rounding up gives t.
        static_assert(PIPE_PAD_FINISHED % 2 == 0 && PIPE_PAD_FLIP == PIPE_PAD_FINISHED + 1, "pad layout");
        unsigned long long fin, flip;
        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(fin), "=l"(flip) : "l"(a.pad + PIPE_PAD_FINISHED));
        tg = (fin + (1ull << PIPE_STEP_SHIFT) - 1) >> PIPE_STEP_SHIFT;
        tg ^= flip & 1;
        const TMap &mg = (tg & 1) ? m1 : m0;
        const int ns = a.sb - a.sa, nc = a.cb - a.ca;
        for (int q = 0; q < S; ++q) {
            const int item = gw + q * nwt;
            if (item < a.n_int) {
                const int ib = (a.sa + item % ns) * W, j0 = (a.ca + (item / ns) % nc) * JB, k = item / (ns * nc);
                tma_prefetch_ijk(m_cf, ib, j0, k);
                tma_prefetch_ijk(mg, ib - C::LP, j0 - 2, k);
            }
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    griddep_launch_dependents();
    griddep_wait();
    const int gb = (int)(__shfl_sync(0xffffffffu, tg, 0) & 1);  // guessed parity

    auto in_s = [&](int s) { return reinterpret_cast<T *>(wbase + s * C::SLOT); };
    auto cf_s = [&](int s) { return reinterpret_cast<T *>(wbase + s * C::SLOT + C::IN_PAD); };
    const int ns_int = a.sb - a.sa, nc_int = a.cb - a.ca;
    auto decode_int = [&](int item, int &ib, int &j0, int &k) {
        ib = (a.sa + item % ns_int) * W;
        j0 = (a.ca + (item / ns_int) % nc_int) * JB;
        k = item / (ns_int * nc_int);
    };
    auto issue_from = [&](const TMap &mx, int item, int s) {
        int ib, j0, k;
        decode_int(item, ib, j0, k);
        mbar_expect_tx(&bars[s], C::IN_BYTES + C::CF_BYTES);
        tma_load_ijk(in_s(s), mx, &bars[s], ib - C::LP, j0 - 2, k);
        tma_load_ijk(cf_s(s), m_cf, &bars[s], ib, j0, k);
    };
    // ---- interior tiles: the TMA ring of hdiff_tma.  The first S tiles are requested from the
    // GUESSED x_t right after griddepcontrol.wait, while the step counter is read (an L2 round
    // trip otherwise on the critical path); a wrong guess (never in steady state) drains those
    // loads and requests the tiles again from the right buffer, the ring's phases shifted by one.
    const int n_int = a.n_int;
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (gw + s * nwt < n_int) issue_from(gb ? m1 : m0, gw + s * nwt, s);
    }
    const unsigned long long t =
        *reinterpret_cast<volatile const unsigned long long *>(a.pad + PIPE_PAD_FINISHED) >> PIPE_STEP_SHIFT;
    const int b = (int)(t & 1);
    const TMap &m_in = b ? m1 : m0;
    const FOT<T> out = a.y[b ^ 1];
    const int nk = a.d.hi[2];
    auto issue = [&](int item, int s) { issue_from(m_in, item, s); };
    int poff = 0;
    if (b != gb) {
        if (lane == 0) {
            atom_add_relaxed_gpu(a.pad + PIPE_PAD_MISGUESS, 1ull);
#pragma unroll
            for (int s = 0; s < S; ++s)
                if (gw + s * nwt < n_int) {
                    mbar_wait(&bars[s], 0);
                    issue(gw + s * nwt, s);
                }
        }
        poff = 1;
    }
    __syncwarp();
    int n = 0;
    for (int item = gw; item < n_int; item += nwt, ++n) {
        const int s = n % S;
        int ib, j0, k;
        decode_int(item, ib, j0, k);
        const int nrows = min(JB, a.d.hi[1] - j0);
        const int i_own = ib + lane * V;
        T *out_k = out.p + k * out.sk;
        mbar_wait(&bars[s], ((n / S) + poff) & 1);
        if (nrows == JB)
            hdiff_tile<T, V, JB, C::LP, true>(in_s(s), cf_s(s), out_k, out.sj, j0, JB, i_own, a.d.hi[0], lane);
        else
            hdiff_tile<T, V, JB, C::LP, false>(in_s(s), cf_s(s), out_k, out.sj, j0, nrows, i_own, a.d.hi[0], lane);
        __syncwarp();
        if (lane == 0) {
            const int nxt = item + S * nwt;
            if (nxt < n_int) {
                fence_proxy_async();
                issue(nxt, s);
            }
        }
    }
    // ---- boundary tiles: neighbours' cells read from their memory once they finished step t-1
    const int per_plane = a.nseg * a.nchunk - ns_int * nc_int;
    const int nb_items = a.n_items - n_int;
    bool ready = false;
    fence_proxy_async();  // slot 0 was last written by TMA (async proxy); now generic stores
    T *tin = in_s(0), *tcf = cf_s(0);
    for (int item = gw; item < nb_items; item += nwt) {
        if (!ready) {
            if (lane == 0) {
                // a neighbour that never runs step t-1 (a caller bug) must not hang the GPU:
                // give up after PIPE_WAIT_NS with a device trap (the launch reports an error)
                const unsigned long long t0 = globaltimer_ns();
                for (int dd = 0; dd < 9; ++dd)
                    if (a.nb[dd].exists)
                        while (ld_acquire_sys(a.pad + dd) < (t << PIPE_STEP_SHIFT)) {
                            __nanosleep(64);
                            if (globaltimer_ns() - t0 > PIPE_WAIT_NS) __trap();
                        }
            }
            __syncwarp();
            ready = true;
        }
        // boundary item -> (seg, chunk, k): per k-plane, chunk rows below the interior band (all
        // segments), the band (segments outside [sa, sb)), the rows above (all segments)
        const int k = item / per_plane;
        int r = item % per_plane, seg, chunk;
        const int mid = a.nseg - ns_int;
        if (r < a.ca * a.nseg) {
            chunk = r / a.nseg;
            seg = r % a.nseg;
        } else if ((r -= a.ca * a.nseg) < nc_int * mid) {
            chunk = a.ca + r / mid;
            const int q = r % mid;
            seg = q < a.sa ? q : a.sb + (q - a.sa);
        } else {
            r -= nc_int * mid;
            chunk = a.cb + r / a.nseg;
            seg = r % a.nseg;
        }
        const int ib = seg * W, j0 = chunk * JB;
        for (int e = lane; e < (JB + 4) * C::RW; e += 32) {
            const int rr = e / C::RW, y = e % C::RW;
            tin[e] = pipe_cell(a, b, ib - C::LP + y, j0 - 2 + rr, k);
        }
        for (int e = lane; e < JB * W; e += 32) {
            const int rr = e / W, x = e % W;
            const int i = ib + x, j = j0 + rr;
            tcf[e] = (i < a.d.hi[0] && j < a.d.hi[1]) ? a.cf.p[i + j * a.cf.sj + k * a.cf.sk] : T(0);
        }
        __syncwarp();
        const int nrows = min(JB, a.d.hi[1] - j0);
        T *out_k = out.p + k * out.sk;
        if (nrows == JB)
            hdiff_tile<T, V, JB, C::LP, true>(tin, tcf, out_k, out.sj, j0, JB, ib + lane * V, a.d.hi[0], lane);
        else
            hdiff_tile<T, V, JB, C::LP, false>(tin, tcf, out_k, out.sj, j0, nrows, ib + lane * V, a.d.hi[0], lane);
        __syncwarp();
    }
    (void)nk;
    // ---- publish "step t done" (our outputs written, our reads of the neighbours' x_t finished)
    // without a CTA barrier: each warp arrives on a per-CTA shared counter (acq_rel, CTA scope, so
    // the last warp's release below is cumulative over every warp's accesses); the CTA's last warp
    // adds the CTA's share -- fire and forget, no round trip
    __syncwarp();
    if (lane == 0 && atom_add_acqrel_cta_shared(warps_done, 1u) == NW - 1) {
        const unsigned G = gridDim.x, unit = 1u << PIPE_STEP_SHIFT;
        const unsigned long long w = unit / G + (blockIdx.x < unit % G ? 1u : 0u);
        for (int dd = 0; dd < 9; ++dd)
            if (a.nb[dd].exists) red_release_sys(a.nb[dd].flag, w);
        red_relaxed_gpu(a.pad + PIPE_PAD_FINISHED, w);
    }
    (void)any_nb;
}

template <class T, int V, int JB, int S, int NW>
cudaError_t launch_pipe(const TMap &m0, const TMap &m1, const TMap &mcf, const PipeArgs<T> &a, int nsteps, cudaStream_t st,
                        int *launches) {
    using C = TmaCfg<T, V, JB, S, NW>;
    static bool configured = false;
    static int blocks_per_sm = 1, sms = 148;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(hdiff_pipe<T, V, JB, S, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM + 16);
        if (e != cudaSuccess) return e;
        int dev;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, hdiff_pipe<T, V, JB, S, NW>, NW * 32, C::SMEM + 16);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
        configured = true;
    }
    const long long blocks = std::max(1ll, std::min<long long>((a.n_items + NW - 1) / NW, (long long)sms * blocks_per_sm));
    for (int s = 0; s < nsteps; ++s) {
        cudaError_t e = launch_pdl(hdiff_pipe<T, V, JB, S, NW>, dim3((unsigned)blocks), dim3(NW * 32), C::SMEM + 16, st, m0,
                                   m1, mcf, a);
        ++*launches;
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <class T, int V, int JB, int P>
cudaError_t launch_roll(const FVT<T> &in, const FVT<T> &coeff, const FOT<T> &out, const Dom &d, cudaStream_t s, int *launches) {
    constexpr int W = 32 * V;
    const int ni = d.hi[0] - d.lo[0], nj = d.hi[1] - d.lo[1], nk = d.hi[2] - d.lo[2];
    const int nseg = (ni + W - 1) / W, nchunk = (nj + JB - 1) / JB;
    const long long warps = (long long)nseg * nchunk * nk;
    const int threads = 128;
    const long long blocks = (warps * 32 + threads - 1) / threads;
    hdiff_roll<T, V, JB, P><<<(unsigned)blocks, threads, 0, s>>>(in, coeff, out, d, nseg, nchunk);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace

static bool hdiff_large(const Dom &d) {
    return (long long)(d.hi[0] - d.lo[0]) * (d.hi[1] - d.lo[1]) * (d.hi[2] - d.lo[2]) >= HD_LARGE_POINTS;
}
static bool hdiff_tiny(const Dom &d) {
    return (long long)(d.hi[0] - d.lo[0]) * (d.hi[1] - d.lo[1]) * (d.hi[2] - d.lo[2]) <= HD_TINY_POINTS;
}

// tile configuration per element type: f32 tiles have the same bytes per row as f64 (V doubled)
template <class T>
struct HdCfg;
template <>
struct HdCfg<double> {
    static constexpr int V = HD_V, JB = HD_JB, S = HD_S, NW = HD_NW, TNW = HD_TNW;
    static constexpr int LV = HDL_V, LJB = HDL_JB, LS = HDL_S, LNW = HDL_NW;
    static constexpr int RV = 2;  // rolling kernel vector width when 16-byte aligned
};
template <>
struct HdCfg<float> {
    static constexpr int V = HF_V, JB = HF_JB, S = HF_S, NW = HF_NW, TNW = HF_TNW;
    static constexpr int LV = HFL_V, LJB = HFL_JB, LS = HFL_S, LNW = HFL_NW;
    static constexpr int RV = 4;
};

template <class T>
void hdiff_tma_boxes(const Dom &d, int box_in[3], int box_cf[3]) {
    using C = HdCfg<T>;
    const bool L = hdiff_large(d);
    const int V = L ? C::LV : C::V, JB = L ? C::LJB : C::JB;
    box_in[0] = 32 * V + 2 * (16 / (int)sizeof(T));  // TmaCfg::RW
    box_in[1] = JB + 4;
    box_in[2] = 1;
    box_cf[0] = 32 * V;
    box_cf[1] = JB;
    box_cf[2] = 1;
}

// aligned16: every field pointer, stride and the domain's i origin allow 16-byte vector accesses
template <class T>
cudaError_t launch_hdiff(const FVT<T> &in, const FVT<T> &coeff, const FOT<T> &out, const Dom &d, int variant,
                         bool aligned16, const TMap *tin, const TMap *tcf, cudaStream_t s, int *launches) {
    using C = HdCfg<T>;
    if (variant == OEC_VARIANT_NAIVE || variant == OEC_VARIANT_UNROLL2 || variant == OEC_VARIANT_UNROLL4) {
        const int uj = variant == OEC_VARIANT_UNROLL4 ? 4 : variant == OEC_VARIANT_UNROLL2 ? 2 : 1;
        dim3 block(32, 4, 1);
        dim3 grid((d.hi[0] - d.lo[0] + 31) / 32, (d.hi[1] - d.lo[1] + 4 * uj - 1) / (4 * uj), d.hi[2] - d.lo[2]);
        if (uj == 4) hdiff_naive<T, 4><<<grid, block, 0, s>>>(in, coeff, out, d);
        else if (uj == 2) hdiff_naive<T, 2><<<grid, block, 0, s>>>(in, coeff, out, d);
        else hdiff_naive<T, 1><<<grid, block, 0, s>>>(in, coeff, out, d);
        ++*launches;
        return cudaGetLastError();
    }
    if (tin && tcf && aligned16) {
        if (hdiff_large(d)) return launch_tma<T, C::LV, C::LJB, C::LS, C::LNW>(*tin, *tcf, out, d, s, launches);
        if (hdiff_tiny(d)) return launch_tma<T, C::V, C::JB, C::S, C::TNW>(*tin, *tcf, out, d, s, launches);
        return launch_tma<T, C::V, C::JB, C::S, C::NW>(*tin, *tcf, out, d, s, launches);
    }
    if (aligned16) return launch_roll<T, C::RV, 16, 4>(in, coeff, out, d, s, launches);
    return launch_roll<T, 1, 16, 4>(in, coeff, out, d, s, launches);
}

template <class T>
void hdiff_pipe_boxes(const Dom &d, int box_in[3], int box_cf[3], int *tile_w, int *tile_jb) {
    using C = HdCfg<T>;
    const bool L = hdiff_large(d);
    hdiff_tma_boxes<T>(d, box_in, box_cf);
    *tile_w = 32 * (L ? C::LV : C::V);
    *tile_jb = L ? C::LJB : C::JB;
}

template <class T>
cudaError_t launch_hdiff_pipe(const TMap &m0, const TMap &m1, const TMap &mcf, PipeArgs<T> &a, int nsteps,
                              cudaStream_t s, int *launches) {
    using C = HdCfg<T>;
    if (hdiff_large(a.d)) return launch_pipe<T, C::LV, C::LJB, C::LS, C::LNW>(m0, m1, mcf, a, nsteps, s, launches);
    return launch_pipe<T, C::V, C::JB, C::S, C::NW>(m0, m1, mcf, a, nsteps, s, launches);
}

template void hdiff_pipe_boxes<double>(const Dom &, int *, int *, int *, int *);
template void hdiff_pipe_boxes<float>(const Dom &, int *, int *, int *, int *);
template cudaError_t launch_hdiff_pipe<double>(const TMap &, const TMap &, const TMap &, PipeArgs<double> &, int,
                                               cudaStream_t, int *);
template cudaError_t launch_hdiff_pipe<float>(const TMap &, const TMap &, const TMap &, PipeArgs<float> &, int,
                                              cudaStream_t, int *);
template void hdiff_tma_boxes<double>(const Dom &, int *, int *);
template void hdiff_tma_boxes<float>(const Dom &, int *, int *);
template cudaError_t launch_hdiff<double>(const FV &, const FV &, const FO &, const Dom &, int, bool, const TMap *,
                                          const TMap *, cudaStream_t, int *);
template cudaError_t launch_hdiff<float>(const FVf &, const FVf &, const FOf &, const Dom &, int, bool, const TMap *,
                                         const TMap *, cudaStream_t, int *);

}  // namespace oec
