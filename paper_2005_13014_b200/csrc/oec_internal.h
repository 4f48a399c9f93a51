// Internal declarations of liboec (not part of the ABI; see include/oec.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <array>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../../include/oec.h"
#include "tma.h"

namespace oec {

// A field as the kernels see it: a pointer to the ORIGIN element (0,0,0) -- possibly outside
// the allocation, only ever dereferenced at validated in-range offsets -- and 32-bit element
// strides (the host checks every reachable offset fits in int32; "integer index
// computations are a significant performance bottleneck").
// T = double (OEC_F64) or float (OEC_F32, the paper's f32 runs).
template <class T>
struct FVT {
    const T *p;
    int32_t sj, sk;  // sk == 0 for k-invariant fields
};
template <class T>
struct FOT {
    T *p;
    int32_t sj, sk;
};
using FV = FVT<double>;
using FO = FOT<double>;
using FVf = FVT<float>;
using FOf = FOT<float>;

// Domain of one launch: [lo, hi) in absolute coordinates.
struct Dom {
    int32_t lo[3], hi[3];
};

// launchers (return cudaGetLastError() of their launches); `launches` is incremented per launch.
// Templates are instantiated for T = double and T = float; scalars arrive as double and are
// rounded to T once.
template <class T>
cudaError_t launch_hdiff(const FVT<T> &in, const FVT<T> &coeff, const FOT<T> &out, const Dom &d, int variant,
                         bool aligned16, const TMap *tin, const TMap *tcf, cudaStream_t s, int *launches);
template <class T>
void hdiff_tma_boxes(const Dom &d, int box_in[3], int box_cf[3]);
cudaError_t launch_vadv(const FV &u_stage, const FV &wcon, const FV &u_pos, const FV &utens, const FV &usi,
                        const FO &out, double dtr, const Dom &d, const TMap *tmaps, cudaStream_t s, int *launches);
// f32 vadv: the TMA / shared-memory solver (vadv_tma<float>) when tmaps is given, else one thread
// per column (vadv_kernel<float>)
cudaError_t launch_vadv_f32(const FVf &u_stage, const FVf &wcon, const FVf &u_pos, const FVf &utens, const FVf &usi,
                            const FOf &out, double dtr, const Dom &d, const TMap *tmaps, cudaStream_t s, int *launches);
template <class T>
void vadv_tma_boxes(const Dom &d, int box[3], int box_wc[3], int box_us[3], bool *fits);
// the paper's "original" level: one kernel per operator, temporaries in HBM (csrc/unfused.cu)
template <class T>
cudaError_t launch_hdiff_unfused(const FVT<T> &in, const FVT<T> &coeff, const FOT<T> &out, const Dom &d,
                                 cudaStream_t s, int *launches);
template <class T>
cudaError_t launch_vadv_unfused(const FVT<T> &us, const FVT<T> &wc, const FVT<T> &up, const FVT<T> &ut,
                                const FVT<T> &usi, const FOT<T> &out, double dtr, const Dom &d, cudaStream_t s,
                                int *launches);
// suite: inputs / outputs in registry order; `unroll` = points per thread along j (1, 2, 4)
template <class T>
cudaError_t launch_suite(int program_id, const FVT<T> *in, const FOT<T> *out, const double *scalars, const Dom &d,
                         int unroll, cudaStream_t s, int *launches);
// suite "original" level: one kernel per stencil.apply, temporaries in HBM (csrc/suite_unfused.cu)
template <class T>
cudaError_t launch_suite_unfused(int program_id, int n_in, const FVT<T> *in, const FOT<T> *out,
                                 const double *scalars, const Dom &d, cudaStream_t s, int *launches);
int suite_unfused_stages(int program_id);

// box copies for halo exchange: [lo, hi) box (absolute coords) between fields / packed buffers
struct Box {
    int32_t lo[3], hi[3];
};
template <class T>
cudaError_t launch_pack(const FVT<T> &src, const Box &b, T *buf, cudaStream_t s, int *launches);
template <class T>
cudaError_t launch_unpack(const T *buf, const Box &b, const FOT<T> &dst, cudaStream_t s, int *launches);
template <class T>
cudaError_t launch_box_copy(const FVT<T> &src, const FOT<T> &dst, const Box &b, cudaStream_t s, int *launches);

// ---- multi-step hdiff with the halo exchange fused into the kernel:
// boundary tiles read the neighbours' interior rows straight from their memory (NVLink peer
// pointers, or plain pointers when the sub-domains share a device); csrc/pipeline.cpp.
// Directions: index si*3 + sj with si, sj in {0: low side, 1: inside, 2: high side}; 4 = self.
template <class T>
struct PeerNb {
    const T *x[2];             // the neighbour's x0 / x1, origin pointers (its local (0,0,0))
    int32_t sj, sk;            // its strides (x0 and x1 alike)
    int32_t oi, oj;            // its local origin in OUR local coordinates
    unsigned long long *flag;  // the slot of the neighbour's signal pad we write when a step is done
    int32_t exists, pad_;
};
// signal pad words (device memory of the rank that owns the pipeline)
// PIPE_PAD_MISGUESS: warps that requested their first tiles from the wrong x_t (diagnostics);
// PIPE_PAD_FLIP != 0: the kernel inverts its guess (tests of the recovery path; 0 from creation)
// Words 0-8: steps completed by the neighbour in direction d, 2^20 per step; FINISHED: our own
// steps, 2^20 per step (each CTA adds its share; hdiff.cu).  (FINISHED and FLIP share one 16-byte
// load: FINISHED even.)  Word 9 is unused.
enum { PIPE_PAD_STEP = 9, PIPE_PAD_FINISHED = 10, PIPE_PAD_FLIP = 11, PIPE_PAD_MISGUESS = 12, PIPE_PAD_WORDS = 16 };
template <class T>
struct PipeArgs {
    PeerNb<T> nb[9];
    FVT<T> x[2];
    FOT<T> y[2];       // the same memory as x[0], x[1], writable
    FVT<T> cf;
    int32_t alo[2], ahi[2];     // allocated i, j range of x0/x1 (local coordinates)
    unsigned long long *pad;    // our signal pad: [d] = steps completed by the neighbour in direction d
    Dom d;                      // [0, N) local domain
    int32_t nseg, nchunk;       // tiles per k-plane
    int32_t sa, sb, ca, cb;     // interior tiles (their halo never leaves our sub-domain or the global halo)
    int32_t n_int, n_items;
};
template <class T>
cudaError_t launch_hdiff_pipe(const TMap &m0, const TMap &m1, const TMap &mcf, PipeArgs<T> &a, int nsteps,
                              cudaStream_t s, int *launches);
// TMA boxes of the pipeline kernel (same tile configuration rule as hdiff)
template <class T>
void hdiff_pipe_boxes(const Dom &d, int box_in[3], int box_cf[3], int *tile_w, int *tile_jb);

// oec_decomp_create's block split: rank's sub-domain [lo, hi) of global domain g (csrc/halo.cu)
void subdomain(const int64_t g[3], int px, int py, int rank, int64_t lo[3], int64_t hi[3]);

// field validation shared with runtime.cpp: kernel views (int32 offsets checked), dtype/device
// agreement (device/dtype start at -2/-1), byte-range overlap
template <class V>
oec_status field_view(const oec_field *f, const char *what, V *v);
oec_status field_check(const oec_field *f, const char *what, int *device, int *dtype);
bool field_overlap(const oec_field *a, const oec_field *b);
// byte range [lo, hi) of a field's allocation (false for an empty field)
bool field_span(const oec_field *f, uintptr_t *lo, uintptr_t *hi);

// error plumbing; launch count reported by oec_last_launch_count
oec_status set_error(oec_status st, const char *fmt, ...);
void set_launch_count(int n);

// A program as the validation / host-staging layer (runtime.cpp apply) sees it: a builtin
// registry entry or a program compiled from stencil-language text (csrc/jit.cpp).  Extents are
// the shape-inference result relative to the domain.
struct ProgDesc {
    std::string name;
    std::vector<std::string> in_names, out_names, sc_names;
    std::vector<std::array<int, 3>> in_lo, in_hi;
    std::vector<int> in_kinv;
    std::vector<double> sc_dflt;
    int min_k = 1;          // smallest K the program accepts (vadv: 2)
    bool unroll_ok = true;    // OEC_VARIANT_UNROLL2/4 meaningful
    bool kunroll_ok = false;  // OEC_VARIANT_UNROLL2_K/4_K implemented (stencil-language programs)
    // device runner: called with validated device fields (registry order) and complete scalars
    std::function<oec_status(int dtype, const oec_field *const *in, oec_field *const *out, const double *sc,
                             const int64_t *lo, const int64_t *hi, int variant, cudaStream_t s)>
        run;
};
// JIT registry (csrc/jit.cpp): the program registered under `name`, or null
std::shared_ptr<const ProgDesc> jit_lookup(const char *name);
// a program compiled from library-internal text (not visible by name), cached per text; null
// (with the error set) if it does not parse
std::shared_ptr<const ProgDesc> jit_internal(const char *source);
// stencil-language text of a builtin suite program (csrc/programs.cpp), or null
const char *builtin_program_text(int program_id);
// true for the hand-written programs of the builtin registry (runtime.cpp)
bool builtin_program(const char *name);

}  // namespace oec

// program ids (registry order in runtime.cpp)
enum {
    OEC_PROG_HDIFF = 0,
    OEC_PROG_VADV = 1,
    OEC_PROG_UVBKE = 2,
    OEC_PROG_P_GRAD_C = 3,
    OEC_PROG_NH_P_GRAD = 4,
    OEC_PROG_FVTP2D_QI = 5,
    OEC_PROG_FVTP2D_QJ = 6,
    OEC_PROG_FVTP2D_FLUX = 7,
    OEC_PROG_FASTWAVES = 8,
    OEC_NPROG = 9
};
