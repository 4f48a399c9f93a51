/*
 * oec.h -- C ABI of liboec, the B200-native hot path of the Open Earth Compiler paper
 * (arXiv 2005.13014, "PAPER.md" below): fused fp64 (and f32) stencil programs on 3D fields with
 * halos.
 *
 * A STENCIL PROGRAM "loads the data from the input arrays, implements the stencil operators
 * inline, and stores the results to the output arrays" (§4.4).  Every entry
 * point below applies one such program, fused into a single pass over HBM (stencil inlining,
 * §5.1; "we do not need to store and load any temporary buffer, and all inputs of the
 * stencil program are only loaded once", §7.3), to a caller-given domain.
 *
 * ---------------------------------------------------------------------------------------------
 * Conventions (apply to every call)
 * ---------------------------------------------------------------------------------------------
 * Coordinates.  Absolute integer (i, j, k) coordinates whose origin is the lower bound of the
 *   computation domain the fields were made for ("The origin denotes the lower bound of the
 *   computation domain and has all coordinates set to zero", §4.2).  Ranges are
 *   [lb, ub): inclusive lower, exclusive upper bound.  i is the fastest dimension.
 * Fields.  An oec_field describes (does not own, unless `owned`) a strided fp64 or f32 array over its
 *   ALLOCATED range [lb, ub): element (i,j,k) lives at
 *     data + (i-lb[0])*stride[0] + (j-lb[1])*stride[1] + (k-lb[2])*stride[2]   (elements).
 *   stride[0] must be 1.  A k-invariant ("2D metric") field has lb[2] = 0, ub[2] = 1 and
 *   stride[2] = 0 and is broadcast along k.
 * Domain.  dom_lb/dom_ub select the points computed; outputs are written ONLY there (the
 *   stencil.store range).  Output halos and padding are never written.
 * Extents.  Each input must cover the domain grown by that program's access extent (shape
 *   inference, §5.2: "verify the input array is large enough"); see
 *   oec_program_input().  Otherwise OEC_ERR_SHAPE.  There is no boundary condition: input
 *   halos are caller data (operators compute "all elements ... except for some constant-width
 *   boundary").
 * Aliasing.  "All stencil program parameters have to be alias-free and are either loaded from
 *   or stored to as a unit".  An output whose bytes overlap any input or another
 *   output -> OEC_ERR_ALIAS.
 * Memory / ownership.  device >= 0: `data` is device memory of that CUDA ordinal; the call
 *   validates synchronously and ENQUEUES the kernel(s) on `stream` (a cudaStream_t passed as
 *   void*, NULL = legacy default stream); it never synchronises.  device == OEC_DEVICE_HOST:
 *   `data` is host memory (pinned or pageable); the library stages it through a cached device
 *   workspace on the current device: H2D copies of the inputs, the kernel, D2H copies of the
 *   outputs' domain, then it synchronises `stream` before returning (the end-to-end path).
 *   All fields of one call must be on the same side.
 * Numerics.  IEEE fp64 -- or binary32 when the fields are OEC_F32 ("single-precision (f32) and
 *   double-precision (f64)", §7.1) -- round-to-nearest-even, no contraction into FMA,
 *   expression order of the program definitions in DESIGN.md: results are bit-identical to the
 *   CPU oracle of the same precision.  All fields of one call share one dtype; scalars are
 *   passed as double and rounded once to the fields' precision.
 * Errors.  Every call returns an oec_status; OEC_OK = 0.  No exception crosses the ABI.  The
 *   message of the last failing call on this thread is oec_last_error().  Launch failures are
 *   OEC_ERR_CUDA; asynchronous device faults surface at the caller's next synchronisation.
 * Threading.  Calls are thread-safe; state is per-thread (last error) or per object (decomp).
 */
#ifndef OEC_H
#define OEC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OEC_ABI_VERSION 1
#define OEC_DEVICE_HOST (-1)

typedef enum {
    OEC_OK = 0,
    OEC_ERR_ARG = 1,         /* NULL pointer, bad enum, unknown program, wrong arg count     */
    OEC_ERR_SHAPE = 2,       /* allocation does not cover domain + extent, K < 2 (vadv), ... */
    OEC_ERR_ALIAS = 3,       /* an output overlaps an input or another output         */
    OEC_ERR_DTYPE = 4,       /* unknown dtype, mixed dtypes, or mixed devices                */
    OEC_ERR_CUDA = 5,        /* CUDA runtime error (launch, allocation, copy)                */
    OEC_ERR_NCCL = 6,        /* NCCL error or NCCL not loadable                               */
    OEC_ERR_UNSUPPORTED = 7, /* valid request this build does not implement                  */
    OEC_ERR_LAYOUT = 8       /* stride[0] != 1, misaligned data, offsets overflow int32      */
} oec_status;

/* Element types (P:556 evaluates every benchmark in both). */
typedef enum { OEC_F64 = 0, OEC_F32 = 1 } oec_dtype;

/* Kernel variants of oec_apply_program / oec_hdiff_variant: the paper's optimisation levels
   (§7.3: original, inline, inline+unroll(2), inline+unroll(4)) plus the tuned
   B200 kernels.  All variants produce bit-identical results.                                   */
typedef enum {
    OEC_VARIANT_AUTO = 0,    /* fastest B200 kernel (default)                                   */
    OEC_VARIANT_UNFUSED = 1, /* "original": one kernel per stencil.apply, every
                                intermediate materialised in HBM over its inferred range
                                (P:480-482); uses a library-owned device workspace, grown on
                                first use -- call once outside stream capture                  */
    OEC_VARIANT_NAIVE = 2,   /* "inline" in the paper's execution model: one thread per point
                                (vadv: per column, sequential in k), every producer inlined and
                                recomputed, registers only, no synchronisation  */
    OEC_VARIANT_UNROLL2 = 3, /* "inline+unroll(2)": NAIVE with stencil unrolling by 2 along j
                                (P:447-454): one thread updates two rows, shared loads and
                                producer evaluations computed once.  Not for vadv
                                (OEC_ERR_UNSUPPORTED: unrolling does not apply to the column
                                solver)                                                        */
    OEC_VARIANT_UNROLL4 = 4, /* "inline+unroll(4)": as UNROLL2 with factor 4                    */
    OEC_VARIANT_UNROLL2_K = 5, /* inline + unroll by 2 along k ("the unrolling pass supports all
                                unroll dimensions"): stencil-language programs only
                                (oec_program_create); builtins: OEC_ERR_UNSUPPORTED            */
    OEC_VARIANT_UNROLL4_K = 6, /* as UNROLL2_K with factor 4                                    */
    OEC_VARIANT_TILED = 7    /* B200 tiling for stencil-language programs: persistent CTAs, each
                                3D input's tile + access extent staged into a shared-memory ring
                                by TMA, the inlined expression reads shared memory; inputs must
                                be TMA-describable (oec_field_create layout) else
                                OEC_ERR_LAYOUT; builtins: OEC_ERR_UNSUPPORTED                    */
} oec_variant;

typedef struct oec_field {
    void *data;        /* element (lb[0], lb[1], lb[2]); device or host memory (see `device`) */
    int64_t lb[3];     /* allocated range, absolute coordinates (origin = domain lower bound)  */
    int64_t ub[3];
    int64_t stride[3]; /* elements; stride[0] == 1; stride[2] == 0 for k-invariant fields      */
    int32_t dtype;     /* oec_dtype                                                            */
    int32_t device;    /* CUDA ordinal, or OEC_DEVICE_HOST                                     */
    int32_t owned;     /* 1: allocated by oec_field_create, freed by oec_field_destroy         */
    int32_t reserved;
} oec_field;

/* ABI version (OEC_ABI_VERSION) and a static build-info string. */
int32_t oec_abi_version(void);
const char *oec_build_info(void);

/* Message for the last non-OK status returned on this thread ("" if none). */
const char *oec_last_error(void);

/* Allocate a device field covering [-halo_lo, domain + halo_hi) per dim (a0 of SURVEY §8(a)).
 *   domain[3]    interior extent (Ni, Nj, Nk), each >= 1 (k: >= 1; use Nk = 1, halo 0 and
 *                k_invariant = 1 for 2D metric fields)
 *   halo_lo/hi   halo widths per dim, 0 <= h <= 16 in i (f32: 32; the left pad), any >= 0 in j, k
 *   order        NULL = default {0, 2, 1}: i fastest, then k, then j (a j-slab halo is one
 *                contiguous block); or a permutation of {0,1,2}
 *                listing dims fastest -> slowest (order[0] must be 0)
 *   k_invariant  1: 2D field broadcast along k (requires domain[2] == 1, halo k == 0)
 *   dtype        OEC_F64 or OEC_F32
 * Layout: i rows start 128 bytes (16 f64 / 32 f32 elements) left of i = 0 so that i = 0 is
 * 128-byte aligned; the row pitch is a multiple of 128 bytes; halo_lo[0] may not exceed that pad.
 * Memory is cudaMalloc'ed on `device` and zeroed.
 * out->owned = 1.  Errors: OEC_ERR_ARG (NULL/invalid), OEC_ERR_CUDA (allocation). */
oec_status oec_field_create(const int64_t domain[3], const int32_t halo_lo[3], const int32_t halo_hi[3],
                            int32_t dtype, int32_t device, const int32_t order[3], int32_t k_invariant,
                            oec_field *out);

/* Describe caller-owned memory (e.g. a torch tensor) as a field; out->owned = 0.  No copy, no
 * allocation.  Errors: OEC_ERR_ARG, OEC_ERR_LAYOUT (stride[0] != 1, stride[2] == 0 without
 * ub[2]-lb[2] == 1). */
oec_status oec_field_wrap(void *data, const int64_t lb[3], const int64_t ub[3], const int64_t stride[3],
                          int32_t dtype, int32_t device, oec_field *out);

/* Free the memory of an owned field (no-op for borrowed ones) and clear the descriptor. */
oec_status oec_field_destroy(oec_field *f);

/* ----------------------------------------------------------------------------------------- */
/* Program registry: names, argument order and access extents (a1, shape inference P:480).     */
/* ----------------------------------------------------------------------------------------- */
/* Programs: "hdiff", "vadv", "uvbke", "p_grad_c", "nh_p_grad", "fvtp2d_qi", "fvtp2d_qj",
 * "fvtp2d_flux", "fastwaves" (Table II P:575-580 + north_star).  n_* may be NULL. */
oec_status oec_program_info(const char *program, int32_t *n_inputs, int32_t *n_outputs, int32_t *n_scalars);

/* Input `idx` of `program`: its name (static string), its access extent relative to the
 * domain -- the input must cover [dom_lb + lo, dom_ub + hi) -- and whether it is a k-invariant
 * (2D) field.  lo[d] <= 0 <= hi[d].  (vadv's wcon: lo = {0,0,0}, hi = {1,0,0}.) */
oec_status oec_program_input(const char *program, int32_t idx, const char **name, int64_t lo[3], int64_t hi[3],
                             int32_t *k_invariant);

/* a1 as SURVEY §8(b) names it: the access extent [lo, hi) of input `input_idx` relative to the
 * domain (shape inference) -- the same lo / hi as oec_program_input. */
oec_status oec_program_extent(const char *program, int32_t input_idx, int64_t lo[3], int64_t hi[3]);

/* Name of output `idx` / scalar `idx` (static strings). */
oec_status oec_program_output(const char *program, int32_t idx, const char **name);
oec_status oec_program_scalar(const char *program, int32_t idx, const char **name, double *default_value);

/* ----------------------------------------------------------------------------------------- */
/* The hot path.                                                                              */
/* ----------------------------------------------------------------------------------------- */

/* hdiff -- COSMO horizontal diffusion (north_star; PAPER.md has no definition, R1-R6):
 *   lap = ((in[i-1]+in[i+1]) + (in[j-1]+in[j+1])) - 4 in
 *   flx = f*(in[i+1]-in) > 0 ? 0 : f,  f = lap[i+1]-lap        (flux limiter, select)
 *   fly = g*(in[j+1]-in) > 0 ? 0 : g,  g = lap[j+1]-lap
 *   out = in - coeff*((flx - flx[i-1]) + (fly - fly[j-1]))
 * in: extent i,j in [-2,+2], k 0 (13-point diamond); coeff: the output point only.
 * One fused kernel; lap/flx/fly never touch HBM. */
oec_status oec_hdiff(const oec_field *in, const oec_field *coeff, oec_field *out, const int64_t dom_lb[3],
                     const int64_t dom_ub[3], void *stream);

/* Same with an explicit oec_variant. */
oec_status oec_hdiff_variant(const oec_field *in, const oec_field *coeff, oec_field *out, const int64_t dom_lb[3],
                             const int64_t dom_ub[3], int32_t variant, void *stream);

/* vadv -- vertical advection: per column (i,j) the tridiagonal system
 *   a_k x_{k-1} + b_k x_k + c_k x_{k+1} = d_k,  k = dom_lb[2] .. dom_ub[2]-1,
 * solved by the Thomas algorithm ("Some use the Thomas algorithm to perform implicit
 * integration in the vertical direction"); coefficients from u_stage and wcon
 * (BET_M = BET_P = 0.5), d from u_pos, utens, utens_stage_in; out = dtr_stage*(x - u_pos).
 * Full definition: DESIGN.md R7-R11.  wcon extent i in [0,+1]; all others the point only.
 * K = dom_ub[2]-dom_lb[2] >= 2 else OEC_ERR_SHAPE.  One fused kernel; c', d' stay on chip. */
oec_status oec_vadv(const oec_field *u_stage, const oec_field *wcon, const oec_field *u_pos, const oec_field *utens,
                    const oec_field *utens_stage_in, oec_field *utens_stage_out, double dtr_stage,
                    const int64_t dom_lb[3], const int64_t dom_ub[3], void *stream);

/* Apply any registered program (incl. hdiff and vadv).  inputs/outputs in registry order
 * (oec_program_input/output), scalars in registry order (NULL/n_scalars = 0: defaults).
 * variant: oec_variant.  Errors as above; OEC_ERR_ARG for wrong counts / unknown program. */
oec_status oec_apply_program(const char *program, const oec_field *const *inputs, int32_t n_inputs,
                             oec_field *const *outputs, int32_t n_outputs, const double *scalars, int32_t n_scalars,
                             const int64_t dom_lb[3], const int64_t dom_ub[3], int32_t variant, void *stream);

/* Number of kernel launches the last successful oec_* compute call on this thread enqueued
 * (bench.py's gpu_launches count). */
int32_t oec_last_launch_count(void);

/* ----------------------------------------------------------------------------------------- */
/* Stencil programs from text: shape inference, inlining, unrolling and size-specialised JIT   */
/* (§4 the stencil dialect, §5.1 inlining P:431 and unrolling    */
/* P:447, §5.2 shape inference P:480-482, size specialization P:338).                          */
/* ----------------------------------------------------------------------------------------- */
/* The stencil language mirrors the dialect's program structure:
 *
 *   program NAME                       # a stencil program
 *   input  NAME [: ij | : ijk]         # stencil.load of an input array; ij = k-invariant (2D)
 *   scalar NAME [= NUMBER]             # a scalar parameter (default value)
 *   output NAME                        # an output array
 *   apply  R1[, R2 ...] {              # stencil.apply defining results R1, R2, ...
 *       LOCAL = EXPR                   #   scalar values inside the operator (SSA)
 *       return EXPR[, EXPR ...]        #   stencil.return, one value per result
 *   }
 *   apply  R = EXPR                    # short form of a one-result operator
 *   store  R -> OUTPUT                 # stencil.store of a result over the domain
 *   end                                # optional
 *
 *   EXPR: NUMBER | SCALAR | LOCAL | NAME | NAME[di, dj, dk] (stencil.access of an input or an
 *   EARLIER result at a constant offset; NAME alone = [0, 0, 0]) | - EXPR | EXPR (+ - * /)
 *   EXPR | select(COND, EXPR, EXPR) (loop.if / select) | min(a, b) := b < a ? b : a |
 *   max(a, b) := b > a ? b : a | abs(EXPR) | sqrt(EXPR) | ( EXPR ).
 *   COND: EXPR (< > <= >= == !=) EXPR | COND && COND | COND || COND | ! COND | ( COND ).
 *   Precedence (low -> high): ||, &&, comparisons, + -, * /, unary; binary operators associate
 *   to the left, so `a + b + c` is `(a + b) + c`: the evaluation order of every program is fixed
 *   by its text, and results are bit-identical to any evaluator that follows it.  `#` starts a
 *   comment; `;` and newlines are whitespace.
 * Semantics: IEEE arithmetic in the fields' precision (f64, or binary32 with every literal and
 * scalar rounded once), no contraction, correctly rounded / and sqrt.  An operator reads inputs
 * and EARLIER results only (the def-use graph is acyclic); outputs are never read and
 * inputs never stored.  Operators no output depends on are dead.
 * Shape inference gives each input its access extent (oec_program_input): the
 * union over its readers of their iteration domains grown by the access offsets, where an
 * operator's iteration domain is the bounding box of what its own readers need and a stored
 * result is needed on the domain.
 *
 * Variants (oec_apply_program): NAIVE = inline, one generated kernel, one thread per
 * point, every operator recomputed at every offset its readers use, each (operator, offset) and
 * (input, offset) evaluated once per thread (CSE); UNROLL2 / UNROLL4 = inline + unroll along
 * j, UNROLL2_K / UNROLL4_K along k; TILED = the B200 execution model (TMA-staged
 * input boxes in a shared-memory ring, persistent CTAs); UNFUSED = the original level, one
 * kernel per live operator over its inferred domain, temporaries in a library device workspace
 * (single stream at a time); AUTO = empirical tuning: the first call of a specialisation
 * times inline, the unrolled variants and four tiled configurations on the caller's stream
 * (synchronising it; every candidate writes the same bits) and caches the fastest.  Inside a
 * stream capture AUTO never tunes or compiles: it runs the inline kernel if already compiled,
 * else returns OEC_ERR_UNSUPPORTED.  The builtin suite programs' AUTO uses this compiler on their
 * stencil-language definitions (and their hand-written kernels when it returns
 * OEC_ERR_UNSUPPORTED).
 * Kernels are generated with the domain size and all strides as constants, compiled by
 * NVRTC for sm_100a on first use of a (program, dtype, variant, size, strides, device) and
 * cached for the life of the process; the first call of a specialisation must not be inside a
 * CUDA graph capture.  NVRTC is loaded at run time (libnvrtc.so.12): OEC_ERR_UNSUPPORTED if
 * absent. */

/* Parse, verify and shape-infer `source`; register the program under its `program NAME` so that
 * oec_program_info / _input / _output / _scalar and oec_apply_program accept the name.
 * *name (may be NULL): the registered name, valid until oec_program_destroy.  Errors:
 * OEC_ERR_ARG with "line L:C: message" for syntax / type / definition errors, a name that is a
 * builtin program or already registered. */
oec_status oec_program_create(const char *source, const char **name);

/* Unregister a program created by oec_program_create (its cached kernels stay loaded; launches
 * already enqueued are unaffected).  OEC_ERR_ARG for builtins and unknown names. */
oec_status oec_program_destroy(const char *program);

/* The CUDA source oec_apply_program would compile for these fields / domain / variant (no launch,
 * no device memory touched: descriptors may hold any pointers of any device value).  source may
 * be NULL; at most capacity-1 bytes are written plus a NUL; *length = the full source length.
 * compile != 0: also compile it with NVRTC for sm_100a (host only, no GPU needed) and report the
 * cubin size in *cubin_bytes (0 otherwise).  Errors: OEC_ERR_ARG (not a registered text
 * program, counts, variant), field errors as oec_apply_program, OEC_ERR_CUDA with the NVRTC log
 * on a compile error, OEC_ERR_UNSUPPORTED without NVRTC. */
oec_status oec_program_generate(const char *program, const oec_field *const *inputs, int32_t n_inputs,
                                oec_field *const *outputs, int32_t n_outputs, const int64_t dom_lb[3],
                                const int64_t dom_ub[3], int32_t variant, int32_t compile, char *source,
                                int64_t capacity, int64_t *length, int64_t *cubin_bytes);

/* ----------------------------------------------------------------------------------------- */
/* Horizontal domain decomposition + halo exchange (a8; north_star (3)).  Not in PAPER.md. */
/* ----------------------------------------------------------------------------------------- */
typedef struct oec_decomp oec_decomp; /* opaque */

/* One halo message of a rank: copy the box [lo, hi) of a field between this rank and `peer`
 * (send: from our interior; recv: into our halo).  Boxes are absolute GLOBAL coordinates. */
typedef struct oec_halo_msg {
    int32_t peer;   /* rank                                                 */
    int32_t is_send;/* 1 = send our box to peer, 0 = receive peer's into it */
    int32_t phase;  /* 0 = i-phase, 1 = j-phase (corners ride in phase 1)    */
    int32_t tag;
    int64_t lo[3];
    int64_t hi[3];
} oec_halo_msg;

/* Split global_domain over px * py ranks (i split px ways, j split py ways, k never split --
 * the vadv recurrence is sequential in k); rank r sits at (r % px, r / px).  Blocks differ in
 * size by at most one cell.  local_lb/ub (may be NULL): this rank's sub-domain in GLOBAL
 * coordinates.  nccl_comm: an ncclComm_t (e.g. torch ProcessGroupNCCL._comm_ptr()) used by
 * oec_halo_exchange, or NULL for plan-only use (oec_decomp_plan).  The library resolves NCCL
 * from the process (the copy torch already loaded) at the first exchange. */
oec_status oec_decomp_create(const int64_t global_domain[3], int32_t px, int32_t py, int32_t rank, void *nccl_comm,
                             oec_decomp **out, int64_t local_lb[3], int64_t local_ub[3]);

/* The messages rank `rank` exchanges for a halo of widths width_lo/width_hi (i, j; k ignored)
 * around its sub-domain, in execution order: phase 0 (i-neighbours, j-range of the interior)
 * then phase 1 (j-neighbours, i-range INCLUDING the i-halo, so corners are filled).  Non-periodic
 * global boundary: nothing is exchanged across it.  *n_msgs = the number of messages; at most
 * `capacity` are written to `msgs` (msgs may be NULL to query the count). */
oec_status oec_decomp_plan(const oec_decomp *d, const int32_t width_lo[3], const int32_t width_hi[3],
                           oec_halo_msg *msgs, int32_t capacity, int32_t *n_msgs);

/* Exchange the halos of n device fields with the neighbouring ranks over NCCL (send/recv
 * groups over NVLink/NVSwitch), enqueued on `stream`.  Each field is described in the rank's
 * LOCAL coordinates (origin = the rank's sub-domain lower bound local_lb, exactly like a
 * single-GPU field of that sub-domain) and must cover the sub-domain grown by the widths.
 * Boxes are packed/unpacked by liboec kernels around the NCCL calls (j-slab rows, px == 1, are
 * sent from / received into the field itself).  Errors: OEC_ERR_NCCL when no communicator /
 * NCCL unavailable, OEC_ERR_SHAPE when a field does not cover the halo or a width exceeds a
 * neighbour's sub-domain (two hops would be needed). */
oec_status oec_halo_exchange(oec_decomp *d, oec_field *const *fields, int32_t n, const int32_t width_lo[3],
                             const int32_t width_hi[3], void *stream);

/* Same exchange executed on ONE device between sub-domain fields of all ranks
 * (fields[r * n + f] = field f of rank r, in rank r's local coordinates): device-to-device box
 * copies driven by the same plan, phase 0 for all ranks before phase 1.
 * Used to test decomposition logic on a single GPU. */
oec_status oec_halo_exchange_local(const int64_t global_domain[3], int32_t px, int32_t py, oec_field *const *fields,
                                   int32_t n, const int32_t width_lo[3], const int32_t width_hi[3], void *stream);

/* As oec_halo_exchange_local on a global domain that is periodic in i (periodic[0] != 0) and/or
 * j (periodic[1] != 0); periodic may be NULL (= neither). */
oec_status oec_halo_exchange_local_periodic(const int64_t global_domain[3], int32_t px, int32_t py,
                                            const int32_t periodic[2], oec_field *const *fields, int32_t n,
                                            const int32_t width_lo[3], const int32_t width_hi[3], void *stream);

/* Make the global domain of d periodic in i and/or j (default: neither; not in PAPER.md -- a
 * global latitude-longitude grid wraps in i).  The first and last rank of a rank-grid row
 * (column) become neighbours -- with px == 1 (py == 1) the rank exchanges with ITSELF, which is
 * how the NCCL transport is exercised on one GPU.  Receive boxes then lie outside [0, global
 * domain) in the receiver's frame (oec_decomp_plan) and equal the sender's box modulo the
 * period.  Periodic i with non-periodic j: the i-exchange also carries the global outer j-halo
 * rows (caller data), so the corners beyond a periodic i edge hold the wrapped columns' values.  NCCL pairs a rank's messages to one peer in issue order: oec_halo_exchange issues
 * them by (peer, tag, field) on both sides.  Errors: OEC_ERR_ARG (NULL d). */
oec_status oec_decomp_set_periodic(oec_decomp *d, int32_t periodic_i, int32_t periodic_j);

oec_status oec_decomp_destroy(oec_decomp *d);

/* ----------------------------------------------------------------------------------------- */
/* Multi-step hdiff with the halo exchange fused into the kernel (SURVEY §8(f) rank 2;         */
/* north_star (3): "halo exchange via NCCL or P2P over NVLink overlapped with interior          */
/* compute").  Not in PAPER.md (single GPU, one application per run).                          */
/* ----------------------------------------------------------------------------------------- */
/* A pipeline advances x_{t+1} = hdiff(x_t, coeff) on one rank's sub-domain of a px x py
 * decomposition (oec_decomp_create's split) for any number of steps without host round trips:
 * x_t lives in x0 (t even) or x1 (t odd).  Each step is ONE kernel: tiles whose 13-point diamond
 * stays inside the sub-domain stream through the TMA ring first; the boundary tiles then read
 * the neighbours' cells of x_t directly from the neighbours' x0/x1 (device pointers valid on this
 * device: NVLink peer memory imported with oec_ipc_import, or plain pointers when the sub-domains
 * share a device), after the neighbours have signalled (each of their CTAs adds its share of
 * 2^20 with red.release.sys into this rank's signal pad; no returning atomic) that step t-1 is
 * complete.  No halo is copied and there is no exchange launch; the
 * transfer overlaps the interior tiles.  The step counter t lives in device memory, so a CUDA
 * graph of captured oec_hdiff_pipeline_run calls advances on every replay.
 *
 * Semantics (R19, R23): the global domain is non-periodic; cells outside it are the
 * caller's global outer halo, which is CONSTANT over the steps: x0 and x1 must hold the same
 * values there (e.g. x1 created as a copy of x0).  After n steps the result equals n
 * applications of oec_hdiff on the global domain, each followed by copying the outer halo of x0
 * into the new field -- bit for bit.
 *
 * Fields, in the rank's LOCAL coordinates (origin = local_lb of oec_decomp_create):
 *   x0, x1   device fields covering the sub-domain grown by 2 in i and j (all of k); identical
 *            lb/ub/strides; TMA-describable (oec_field_create layout); x0, x1, coeff alias-free
 *   coeff    covers the sub-domain
 * Every sub-domain must be >= 2 wide in each split dimension.  Neighbours may stall this rank
 * (it waits for them); all ranks must run the same number of steps.
 * Errors: OEC_ERR_ARG (bad grid/rank, NULL), OEC_ERR_SHAPE (coverage), OEC_ERR_DTYPE,
 * OEC_ERR_LAYOUT (not TMA-describable), OEC_ERR_ALIAS, OEC_ERR_CUDA. */
typedef struct oec_hdiff_pipeline oec_hdiff_pipeline; /* opaque */

oec_status oec_hdiff_pipeline_create(const int64_t global_domain[3], int32_t px, int32_t py, int32_t rank,
                                     const oec_field *coeff, const oec_field *x0, const oec_field *x1,
                                     oec_hdiff_pipeline **out);

/* This rank's signal pad (library-owned device memory the neighbours write into; 128 bytes):
 * export it to the other processes with oec_ipc_export. */
oec_status oec_hdiff_pipeline_signal_pad(const oec_hdiff_pipeline *p, void **pad, int64_t *bytes);

/* Register neighbour `peer_rank` (one of the up to 8 ranks adjacent to this one, corners
 * included): its x0/x1 descriptors in ITS local coordinates with `data` valid on this device,
 * and its signal pad.  OEC_ERR_ARG if peer_rank is not adjacent. */
oec_status oec_hdiff_pipeline_set_peer(oec_hdiff_pipeline *p, int32_t peer_rank, const oec_field *peer_x0,
                                       const oec_field *peer_x1, void *peer_signal_pad);

/* Enqueue nsteps steps (nsteps kernels) on `stream`; all adjacent ranks must have been
 * registered.  Asynchronous. */
oec_status oec_hdiff_pipeline_run(oec_hdiff_pipeline *p, int32_t nsteps, void *stream);

/* Steps completed so far (synchronous read of the device counter; x_t is in x0 iff t is even). */
oec_status oec_hdiff_pipeline_steps(const oec_hdiff_pipeline *p, int64_t *steps);

oec_status oec_hdiff_pipeline_destroy(oec_hdiff_pipeline *p);

/* CUDA IPC for peer memory between the processes of one node (one process per GPU):
 * oec_ipc_export writes a 64-byte handle of the cudaMalloc allocation containing dev_ptr plus the
 * byte offset of dev_ptr in it; oec_ipc_import maps it in this process (peer access over NVLink
 * enabled) and returns the pointer; oec_ipc_close unmaps it.  Handles of one process cannot be
 * imported by the same process (use the pointer directly). */
#define OEC_IPC_HANDLE_BYTES 64
oec_status oec_ipc_export(const void *dev_ptr, void *handle, int64_t *offset);
oec_status oec_ipc_import(const void *handle, int64_t offset, void **dev_ptr);
oec_status oec_ipc_close(void *dev_ptr);

/* ----------------------------------------------------------------------------------------- */
/* Self-test (used by the GPU test suite).                                                    */
/* ----------------------------------------------------------------------------------------- */
/* The vadv kernel computes the fp64 reciprocal with the branch-free instruction sequence of the
 * CUDA IEEE fast path and falls back to 1.0/x where that path does not apply.  This runs it on n
 * pseudo-random doubles (seeded) on the current device and reports how many it checked (fast
 * path applicable) and how many differed bitwise from 1.0/x (must be 0).  Synchronous. */
oec_status oec_selftest_rcp(unsigned long long n, unsigned long long seed, unsigned long long *mismatches,
                            unsigned long long *checked);

/* The f32 vadv kernel's branch-free binary32 reciprocal (seed + one fused Newton step) checked
 * against 1.0f / x on EVERY 32-bit pattern for which it claims to apply (normal x with exponent
 * field in [2, 252]).  Synchronous. */
oec_status oec_selftest_rcp32(unsigned long long *mismatches, unsigned long long *checked);

#ifdef __cplusplus
}
#endif
#endif /* OEC_H */
