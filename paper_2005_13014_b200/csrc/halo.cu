// Horizontal domain decomposition and halo exchange (north_star (3)).
// Not in PAPER.md (single GPU).  k is never split (the vadv recurrence is sequential in k).
//
// Plan: phase 0 exchanges i-halos over the interior j-range; phase 1 exchanges j-halos over the
// i-range INCLUDING the i-halo, so the (+-1,+-1) corner cells hdiff's diamond reads arrive in
// two hops.  Transport: NCCL send/recv groups (the communicator torch created; NCCL resolved from
// the process at run time, so liboec carries no link dependence on it), strided boxes packed and
// unpacked by the kernels below.  `oec_halo_exchange_local` runs the same plan between sub-domain
// fields that all live on one device (device-to-device box copies) to test the logic on one GPU.
#include <dlfcn.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "oec_internal.h"

struct oec_decomp {
    int64_t gdom[3];
    int32_t px, py, rank, ri, rj;
    int64_t lo[3], hi[3];
    void *comm;
    int32_t periodic[2];  // i, j: the global domain wraps around (oec_decomp_set_periodic)
};

namespace oec {
namespace {

// box kernels: x threads along i, grid.y over j, grid.z over k (grid-stride in every dimension);
// no per-element integer division
template <class T>
__global__ void pack_kernel(FVT<T> src, Box b, T *buf) {
    const int ni = b.hi[0] - b.lo[0], nj = b.hi[1] - b.lo[1], nk = b.hi[2] - b.lo[2];
    for (int k = blockIdx.z; k < nk; k += gridDim.z)
        for (int j = blockIdx.y; j < nj; j += gridDim.y) {
            const T *row = src.p + (b.lo[1] + j) * (long long)src.sj + (b.lo[2] + k) * (long long)src.sk + b.lo[0];
            T *dst = buf + ((long long)k * nj + j) * ni;
            for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ni; i += gridDim.x * blockDim.x) dst[i] = row[i];
        }
}
template <class T>
__global__ void unpack_kernel(const T *buf, Box b, FOT<T> dst) {
    const int ni = b.hi[0] - b.lo[0], nj = b.hi[1] - b.lo[1], nk = b.hi[2] - b.lo[2];
    for (int k = blockIdx.z; k < nk; k += gridDim.z)
        for (int j = blockIdx.y; j < nj; j += gridDim.y) {
            T *row = dst.p + (b.lo[1] + j) * (long long)dst.sj + (b.lo[2] + k) * (long long)dst.sk + b.lo[0];
            const T *src = buf + ((long long)k * nj + j) * ni;
            for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ni; i += gridDim.x * blockDim.x) row[i] = src[i];
        }
}
template <class T>
__global__ void box_copy_kernel(FVT<T> src, FOT<T> dst, Box b) {
    const int ni = b.hi[0] - b.lo[0], nj = b.hi[1] - b.lo[1], nk = b.hi[2] - b.lo[2];
    for (int k = blockIdx.z; k < nk; k += gridDim.z)
        for (int j = blockIdx.y; j < nj; j += gridDim.y) {
            const long long j_ = b.lo[1] + j, k_ = b.lo[2] + k;
            const T *r = src.p + j_ * src.sj + k_ * src.sk + b.lo[0];
            T *w = dst.p + j_ * dst.sj + k_ * dst.sk + b.lo[0];
            for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ni; i += gridDim.x * blockDim.x) w[i] = r[i];
        }
}

long long box_volume(const Box &b) {
    return (long long)(b.hi[0] - b.lo[0]) * (b.hi[1] - b.lo[1]) * (b.hi[2] - b.lo[2]);
}
// threads along i (up to 256), rows over y/z, at most ~16 CTAs per SM in total
void grid_for(const Box &b, dim3 *g, dim3 *t) {
    const int ni = b.hi[0] - b.lo[0], nj = b.hi[1] - b.lo[1], nk = b.hi[2] - b.lo[2];
    t->x = ni >= 256 ? 256 : ni >= 128 ? 128 : ni >= 64 ? 64 : 32;
    g->x = (unsigned)std::min(8, (ni + (int)t->x - 1) / (int)t->x);
    g->y = (unsigned)std::min(nj, 65535);
    g->z = (unsigned)std::max(1, std::min(nk, std::max(1, 148 * 16 / (int)(g->x * g->y))));
    g->z = std::min<unsigned>(g->z, 65535);
}

}  // namespace

template <class T>
cudaError_t launch_pack(const FVT<T> &src, const Box &b, T *buf, cudaStream_t s, int *launches) {
    if (box_volume(b) <= 0) return cudaSuccess;
    dim3 g, t;
    grid_for(b, &g, &t);
    pack_kernel<<<g, t, 0, s>>>(src, b, buf);
    ++*launches;
    return cudaGetLastError();
}
template <class T>
cudaError_t launch_unpack(const T *buf, const Box &b, const FOT<T> &dst, cudaStream_t s, int *launches) {
    if (box_volume(b) <= 0) return cudaSuccess;
    dim3 g, t;
    grid_for(b, &g, &t);
    unpack_kernel<<<g, t, 0, s>>>(buf, b, dst);
    ++*launches;
    return cudaGetLastError();
}
template <class T>
cudaError_t launch_box_copy(const FVT<T> &src, const FOT<T> &dst, const Box &b, cudaStream_t s, int *launches) {
    if (box_volume(b) <= 0) return cudaSuccess;
    dim3 g, t;
    grid_for(b, &g, &t);
    box_copy_kernel<<<g, t, 0, s>>>(src, dst, b);
    ++*launches;
    return cudaGetLastError();
}
template cudaError_t launch_pack<double>(const FV &, const Box &, double *, cudaStream_t, int *);
template cudaError_t launch_pack<float>(const FVf &, const Box &, float *, cudaStream_t, int *);
template cudaError_t launch_unpack<double>(const double *, const Box &, const FO &, cudaStream_t, int *);
template cudaError_t launch_unpack<float>(const float *, const Box &, const FOf &, cudaStream_t, int *);
template cudaError_t launch_box_copy<double>(const FV &, const FO &, const Box &, cudaStream_t, int *);
template cudaError_t launch_box_copy<float>(const FVf &, const FOf &, const Box &, cudaStream_t, int *);

static int64_t block_start(int64_t n, int p, int r) { return r * (n / p) + std::min<int64_t>(r, n % p); }

void subdomain(const int64_t g[3], int px, int py, int rank, int64_t lo[3], int64_t hi[3]) {
    const int ri = rank % px, rj = rank / px;
    lo[0] = block_start(g[0], px, ri);
    hi[0] = block_start(g[0], px, ri + 1);
    lo[1] = block_start(g[1], py, rj);
    hi[1] = block_start(g[1], py, rj + 1);
    lo[2] = 0;
    hi[2] = g[2];
}

namespace {

// messages of `rank` in execution order (see oec.h oec_decomp_plan).  per_i / per_j: periodic
// global domain in i / j -- the first and last rank of a row (column) of the rank grid are
// neighbours (the same rank when px (py) == 1); receive boxes then lie outside [0, g) in the
// receiver's frame and equal the sender's box modulo the period.
std::vector<oec_halo_msg> make_plan(const int64_t g[3], int px, int py, int rank, const int32_t wlo[3],
                                    const int32_t whi[3], bool per_i = false, bool per_j = false) {
    std::vector<oec_halo_msg> m;
    int64_t lo[3], hi[3];
    subdomain(g, px, py, rank, lo, hi);
    const int ri = rank % px, rj = rank / px;
    auto add = [&](int peer, int is_send, int phase, int tag, int64_t a0, int64_t a1, int64_t b0, int64_t b1) {
        oec_halo_msg x;
        x.peer = peer;
        x.is_send = is_send;
        x.phase = phase;
        x.tag = tag;
        x.lo[0] = a0;
        x.hi[0] = a1;
        x.lo[1] = b0;
        x.hi[1] = b1;
        x.lo[2] = 0;
        x.hi[2] = g[2];
        if (a1 > a0 && b1 > b0) m.push_back(x);
    };
    // phase 0: i-neighbours, interior j-range. tags: 0 = towards -i, 1 = towards +i, 2 = -j, 3 = +j
    const int left = ri > 0 ? rank - 1 : per_i ? rank + px - 1 : -1;
    const int right = ri < px - 1 ? rank + 1 : per_i ? rank - px + 1 : -1;
    const int down = rj > 0 ? rank - px : per_j ? rank + (py - 1) * px : -1;
    const int up = rj < py - 1 ? rank + px : per_j ? rank - (py - 1) * px : -1;
    // phase-0 rows: the interior j-range; with a periodic i and a NON-periodic j, also the global
    // outer j-halo rows at the domain's j edges (caller data on every rank): the corner cells
    // beyond a periodic i edge are the wrapped columns' caller data, held by the i-neighbour
    const int64_t j0 = lo[1] - (per_i && !per_j && rj == 0 ? wlo[1] : 0);
    const int64_t j1 = hi[1] + (per_i && !per_j && rj == py - 1 ? whi[1] : 0);
    if (left >= 0) {  // left neighbour: it needs our first whi[0] columns, we need its last wlo[0]
        add(left, 1, 0, 0, lo[0], lo[0] + whi[0], j0, j1);
        add(left, 0, 0, 1, lo[0] - wlo[0], lo[0], j0, j1);
    }
    if (right >= 0) {
        add(right, 1, 0, 1, hi[0] - wlo[0], hi[0], j0, j1);
        add(right, 0, 0, 0, hi[0], hi[0] + whi[0], j0, j1);
    }
    // phase 1: j-neighbours, i-range including the i-halo (corners)
    const int64_t i0 = lo[0] - wlo[0], i1 = hi[0] + whi[0];
    if (down >= 0) {
        add(down, 1, 1, 2, i0, i1, lo[1], lo[1] + whi[1]);
        add(down, 0, 1, 3, i0, i1, lo[1] - wlo[1], lo[1]);
    }
    if (up >= 0) {
        add(up, 1, 1, 3, i0, i1, hi[1] - wlo[1], hi[1]);
        add(up, 0, 1, 2, i0, i1, hi[1], hi[1] + whi[1]);
    }
    return m;
}

// ---- NCCL, resolved from the process at run time ----
typedef int (*nccl_sendrecv_t)(const void *, size_t, int, int, void *, cudaStream_t);
typedef int (*nccl_recv_t)(void *, size_t, int, int, void *, cudaStream_t);
typedef int (*nccl_group_t)(void);
typedef const char *(*nccl_errstr_t)(int);
struct Nccl {
    bool tried = false, ok = false;
    nccl_sendrecv_t send = nullptr;
    nccl_recv_t recv = nullptr;
    nccl_group_t gstart = nullptr, gend = nullptr;
    nccl_errstr_t errstr = nullptr;
};
Nccl g_nccl;
std::mutex g_nccl_mu;
constexpr int NCCL_FLOAT32 = 7, NCCL_FLOAT64 = 8;

bool load_nccl() {
    std::lock_guard<std::mutex> lock(g_nccl_mu);
    if (g_nccl.tried) return g_nccl.ok;
    g_nccl.tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_LAZY | RTLD_NOLOAD);  // the copy torch already loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_LAZY);
    if (!h) return false;
    g_nccl.send = (nccl_sendrecv_t)dlsym(h, "ncclSend");
    g_nccl.recv = (nccl_recv_t)dlsym(h, "ncclRecv");
    g_nccl.gstart = (nccl_group_t)dlsym(h, "ncclGroupStart");
    g_nccl.gend = (nccl_group_t)dlsym(h, "ncclGroupEnd");
    g_nccl.errstr = (nccl_errstr_t)dlsym(h, "ncclGetErrorString");
    g_nccl.ok = g_nccl.send && g_nccl.recv && g_nccl.gstart && g_nccl.gend;
    return g_nccl.ok;
}

bool is_kinv(const oec_field *f) { return f->stride[2] == 0 && f->ub[2] - f->lb[2] == 1 && f->lb[2] == 0; }

template <class T>
oec_status view_of(const oec_field *f, FVT<T> *v) {
    if (!f || !f->data) return set_error(OEC_ERR_ARG, "halo: NULL field");
    if (f->dtype != (sizeof(T) == 8 ? OEC_F64 : OEC_F32))
        return set_error(OEC_ERR_DTYPE, "halo: all fields of one call must share one dtype");
    if (f->stride[0] != 1) return set_error(OEC_ERR_LAYOUT, "halo: stride[0] != 1");
    const int64_t sj = f->stride[1], sk = is_kinv(f) ? 0 : f->stride[2];
    const int64_t lbk = is_kinv(f) ? 0 : f->lb[2];
    const int64_t far = (f->ub[0] - f->lb[0]) + (f->ub[1] - f->lb[1]) * sj + (f->ub[2] - f->lb[2]) * sk;
    if (far > INT32_MAX || sj > INT32_MAX || sk > INT32_MAX) return set_error(OEC_ERR_LAYOUT, "halo: offsets exceed int32");
    v->p = (const T *)((const char *)f->data - (f->lb[0] + f->lb[1] * sj + lbk * sk) * (int64_t)sizeof(T));
    v->sj = (int32_t)sj;
    v->sk = (int32_t)sk;
    return OEC_OK;
}

// the box of message m for field f, in the field's rank-LOCAL coordinates (origin = the owning
// rank's sub-domain lower bound `org`): the plan's i/j box shifted by -org, the field's k range
oec_status field_box(const oec_field *f, const oec_halo_msg &m, const int64_t org[3], Box *b) {
    b->lo[0] = (int32_t)(m.lo[0] - org[0]);
    b->hi[0] = (int32_t)(m.hi[0] - org[0]);
    b->lo[1] = (int32_t)(m.lo[1] - org[1]);
    b->hi[1] = (int32_t)(m.hi[1] - org[1]);
    b->lo[2] = (int32_t)f->lb[2];
    b->hi[2] = (int32_t)f->ub[2];
    for (int d = 0; d < 2; ++d)
        if (b->lo[d] < f->lb[d] || b->hi[d] > f->ub[d])
            return set_error(OEC_ERR_SHAPE, "halo: field allocation [%lld,%lld) in dim %d does not cover box [%d,%d)",
                             (long long)f->lb[d], (long long)f->ub[d], d, b->lo[d], b->hi[d]);
    return OEC_OK;
}

oec_status check_widths(const int32_t *wlo, const int32_t *whi) {
    if (!wlo || !whi) return set_error(OEC_ERR_ARG, "halo: NULL widths");
    for (int d = 0; d < 3; ++d)
        if (wlo[d] < 0 || whi[d] < 0) return set_error(OEC_ERR_ARG, "halo: negative width");
    return OEC_OK;
}

// every box a rank sends must lie in its own sub-domain along the exchanged dimension (i in
// phase 0, j in phase 1): a halo wider than the neighbour's sub-domain would need two hops
oec_status check_plan(const int64_t g[3], int px, int py, int rank, const std::vector<oec_halo_msg> &plan) {
    int64_t lo[3], hi[3];
    subdomain(g, px, py, rank, lo, hi);
    for (const auto &m : plan) {
        const int dim = m.phase;
        if (m.is_send && (m.lo[dim] < lo[dim] || m.hi[dim] > hi[dim]))
            return set_error(OEC_ERR_SHAPE, "halo: width exceeds rank %d's sub-domain [%lld,%lld) in dim %d", rank,
                             (long long)lo[dim], (long long)hi[dim], dim);
    }
    return OEC_OK;
}

// One (message, field) buffer of a rank.  DIRECT: with a j-slab decomposition (px == 1) and a
// field whose j rows are the slowest dimension (the default i,k,j order, or a k-invariant
// field), the message's box -- whole j rows, all k, the i range including the i-halo -- lies in
// ONE contiguous span of the field: it is sent from / received into the field itself (no pack,
// no kernel).  The span also covers the row padding and any i-halo cells beyond the exchanged
// width in those rows; with px == 1 those are the global outer halo of the same global rows,
// which the sender holds as caller data, so the receiver gets the values it would hold anyway.
// All ranks must pass fields with the same i / k allocation and strides (oec_field_create gives
// that for equal i / k extents and halos), so both sides compute the same span length.
// STAGED: other boxes are packed into (unpacked from) a stream-ordered staging buffer.
template <class T>
struct MsgBuf {
    oec_halo_msg m;
    int field;
    Box box;       // the field-local box
    bool direct;
    size_t count;  // elements on the wire
    size_t off;    // STAGED: element offset in the rank's staging buffer
    T *ptr;        // DIRECT: first element of the span; STAGED: set once staging is allocated
};

template <class T>
bool span_of(const oec_field *f, const FVT<T> &v, const Box &b, int px, int phase, T **p, size_t *count) {
    if (px != 1 || phase != 1) return false;  // phase 0 (periodic i) boxes are not whole rows
    const bool kinv = is_kinv(f);
    const int64_t ni = f->ub[0] - f->lb[0], nk = f->ub[2] - f->lb[2];
    const int64_t sj = f->stride[1], sk = kinv ? 0 : f->stride[2];
    const bool rows_slowest = kinv ? sj >= ni : (sk >= ni && sj >= sk * nk);
    if (!rows_slowest || b.hi[0] <= b.lo[0] || b.hi[1] <= b.lo[1] || b.hi[2] <= b.lo[2]) return false;
    const int64_t first = b.lo[0] + (int64_t)b.lo[1] * sj + (int64_t)b.lo[2] * sk;
    const int64_t last = (b.hi[0] - 1) + (int64_t)(b.hi[1] - 1) * sj + (int64_t)(b.hi[2] - 1) * sk;
    *p = (T *)v.p + first;
    *count = (size_t)(last - first + 1);
    return true;
}

// the buffers of one rank's plan for n fields; *staged = elements of staging it needs
template <class T>
oec_status rank_buffers(const std::vector<oec_halo_msg> &plan, oec_field *const *fields, int32_t n, const int64_t org[3],
                        int px, std::vector<MsgBuf<T>> *out, size_t *staged) {
    out->clear();
    *staged = 0;
    for (size_t q = 0; q < plan.size(); ++q)
        for (int f = 0; f < n; ++f) {
            MsgBuf<T> mb;
            mb.m = plan[q];
            mb.field = f;
            FVT<T> v;
            oec_status st = view_of(fields[f], &v);
            if (st || (st = field_box(fields[f], plan[q], org, &mb.box))) return st;
            mb.direct = span_of(fields[f], v, mb.box, px, plan[q].phase, &mb.ptr, &mb.count);
            if (!mb.direct) {
                mb.count = (size_t)box_volume(mb.box);
                mb.off = *staged;
                mb.ptr = nullptr;
                *staged += mb.count;
            }
            out->push_back(mb);
        }
    return OEC_OK;
}

template <class T>
cudaError_t pack_phase(std::vector<MsgBuf<T>> &bufs, oec_field *const *fields, int phase, bool send, cudaStream_t s,
                       int *launches) {
    for (auto &mb : bufs) {
        if (mb.m.phase != phase || mb.direct || (mb.m.is_send != 0) != send) continue;
        FVT<T> v;
        view_of(fields[mb.field], &v);
        cudaError_t e = send ? launch_pack(v, mb.box, mb.ptr, s, launches)
                             : launch_unpack((const T *)mb.ptr, mb.box, FOT<T>{(T *)v.p, v.sj, v.sk}, s, launches);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace

template <class T>
oec_status halo_exchange_impl(oec_decomp *d, oec_field *const *fields, int32_t n, const int32_t width_lo[3],
                              const int32_t width_hi[3], void *stream) {
    oec_status st = check_widths(width_lo, width_hi);
    if (st) return st;
    auto plan = make_plan(d->gdom, d->px, d->py, d->rank, width_lo, width_hi, d->periodic[0], d->periodic[1]);
    if ((st = check_plan(d->gdom, d->px, d->py, d->rank, plan))) return st;
    set_launch_count(0);
    if (plan.empty() || n == 0) return OEC_OK;
    if (!d->comm) return set_error(OEC_ERR_NCCL, "oec_halo_exchange: decomposition has no NCCL communicator");
    if (!load_nccl()) return set_error(OEC_ERR_NCCL, "oec_halo_exchange: libnccl.so.2 not loadable in this process");
    for (int f = 0; f < n; ++f)
        if (!fields[f] || fields[f]->device < 0) return set_error(OEC_ERR_ARG, "oec_halo_exchange: fields must be device memory");
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<MsgBuf<T>> bufs;
    size_t staged = 0;
    if ((st = rank_buffers(plan, fields, n, d->lo, d->px, &bufs, &staged))) return st;
    // staging: stream-ordered (allocated and freed on the caller's stream): concurrent exchanges on
    // other streams and CUDA graphs (graph memory nodes) each get their own; on the fields' device
    T *stage = nullptr;
    if (staged) {
        cudaError_t e = cudaMallocAsync((void **)&stage, staged * sizeof(T), s);
        if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "halo staging: %s", cudaGetErrorString(e));
        for (auto &mb : bufs)
            if (!mb.direct) mb.ptr = stage + mb.off;
    }
    constexpr int NCCL_DT = sizeof(T) == 8 ? NCCL_FLOAT64 : NCCL_FLOAT32;
    // NCCL matches the sends and receives between two ranks in issue order (no tags): issue each
    // peer's messages by (tag, field) on both sides -- with a periodic domain a peer can be both
    // neighbours (px == 2) or this rank itself (px == 1), so plan order alone would not match
    std::vector<size_t> order(bufs.size());
    for (size_t q = 0; q < order.size(); ++q) order[q] = q;
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        const MsgBuf<T> &x = bufs[a], &y = bufs[b];
        if (x.m.peer != y.m.peer) return x.m.peer < y.m.peer;
        if (x.m.tag != y.m.tag) return x.m.tag < y.m.tag;
        return x.field < y.field;
    });
    int launches = 0;
    oec_status result = OEC_OK;
    for (int phase = 0; phase < 2 && result == OEC_OK; ++phase) {
        cudaError_t e = pack_phase(bufs, fields, phase, true, s, &launches);
        if (e != cudaSuccess) {
            result = set_error(OEC_ERR_CUDA, "halo pack: %s", cudaGetErrorString(e));
            break;
        }
        int r = g_nccl.gstart();
        for (size_t q : order) {
            const MsgBuf<T> &mb = bufs[q];
            if (r != 0) break;
            if (mb.m.phase != phase) continue;
            r = mb.m.is_send ? g_nccl.send(mb.ptr, mb.count, NCCL_DT, mb.m.peer, d->comm, s)
                             : g_nccl.recv(mb.ptr, mb.count, NCCL_DT, mb.m.peer, d->comm, s);
        }
        int r2 = g_nccl.gend();
        if (r || r2) {
            result = set_error(OEC_ERR_NCCL, "oec_halo_exchange: NCCL error %d (%s)", r ? r : r2,
                               g_nccl.errstr ? g_nccl.errstr(r ? r : r2) : "?");
            break;
        }
        if ((e = pack_phase(bufs, fields, phase, false, s, &launches)) != cudaSuccess)
            result = set_error(OEC_ERR_CUDA, "halo unpack: %s", cudaGetErrorString(e));
    }
    if (stage) cudaFreeAsync(stage, s);
    if (result == OEC_OK) set_launch_count(launches);
    return result;
}

// The same plans, buffers, pack / unpack kernels and direct spans on ONE device: the transport is
// a device-to-device copy from the sender's buffer (its staging or its field span) into the
// receiver's, in place of ncclSend / ncclRecv.  Tests the whole exchange but the NCCL calls.
template <class T>
oec_status halo_exchange_local_impl(const int64_t global_domain[3], int32_t px, int32_t py, const int32_t *periodic,
                                    oec_field *const *fields, int32_t n, const int32_t width_lo[3],
                                    const int32_t width_hi[3], void *stream) {
    oec_status st = check_widths(width_lo, width_hi);
    if (st) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const int R = px * py;
    std::vector<std::vector<MsgBuf<T>>> bufs(R);
    std::vector<size_t> staged(R);
    size_t total = 0;
    for (int r = 0; r < R; ++r) {
        int64_t org[3], tmp[3];
        subdomain(global_domain, px, py, r, org, tmp);
        auto plan = make_plan(global_domain, px, py, r, width_lo, width_hi, periodic && periodic[0], periodic && periodic[1]);
        if ((st = check_plan(global_domain, px, py, r, plan))) return st;
        if ((st = rank_buffers(plan, fields + (size_t)r * n, n, org, px, &bufs[r], &staged[r]))) return st;
        total += staged[r];
    }
    T *stage = nullptr;
    if (total) {
        cudaError_t e = cudaMallocAsync((void **)&stage, total * sizeof(T), s);
        if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "halo staging: %s", cudaGetErrorString(e));
    }
    size_t base = 0;
    for (int r = 0; r < R; ++r) {
        for (auto &mb : bufs[r])
            if (!mb.direct) mb.ptr = stage + base + mb.off;
        base += staged[r];
    }
    int launches = 0;
    oec_status result = OEC_OK;
    for (int phase = 0; phase < 2 && result == OEC_OK; ++phase) {
        cudaError_t e = cudaSuccess;
        for (int r = 0; r < R && e == cudaSuccess; ++r) e = pack_phase(bufs[r], fields + (size_t)r * n, phase, true, s, &launches);
        for (int r = 0; r < R && e == cudaSuccess && result == OEC_OK; ++r)
            for (auto &rv : bufs[r]) {
                if (rv.m.phase != phase || rv.m.is_send) continue;
                const MsgBuf<T> *sd = nullptr;  // the peer's matching send: same phase, tag and field
                for (auto &x : bufs[rv.m.peer])
                    if (x.m.is_send && x.m.peer == r && x.m.phase == phase && x.m.tag == rv.m.tag && x.field == rv.field) sd = &x;
                if (!sd || sd->count != rv.count) {
                    result = set_error(OEC_ERR_SHAPE, "oec_halo_exchange_local: rank %d's message from %d does not match "
                                       "the sender's (%zu vs %zu elements)", r, rv.m.peer, rv.count, sd ? sd->count : 0);
                    break;
                }
                e = cudaMemcpyAsync(rv.ptr, sd->ptr, rv.count * sizeof(T), cudaMemcpyDeviceToDevice, s);
                if (e != cudaSuccess) break;
            }
        for (int r = 0; r < R && e == cudaSuccess; ++r) e = pack_phase(bufs[r], fields + (size_t)r * n, phase, false, s, &launches);
        if (e != cudaSuccess && result == OEC_OK) result = set_error(OEC_ERR_CUDA, "halo copy: %s", cudaGetErrorString(e));
    }
    if (stage) cudaFreeAsync(stage, s);
    if (result == OEC_OK) set_launch_count(launches);
    return result;
}

}  // namespace oec

using namespace oec;

extern "C" {

oec_status oec_decomp_create(const int64_t global_domain[3], int32_t px, int32_t py, int32_t rank, void *nccl_comm,
                             oec_decomp **out, int64_t local_lb[3], int64_t local_ub[3]) {
    if (!global_domain || !out) return set_error(OEC_ERR_ARG, "oec_decomp_create: NULL argument");
    if (px < 1 || py < 1 || rank < 0 || rank >= px * py)
        return set_error(OEC_ERR_ARG, "oec_decomp_create: bad grid %dx%d / rank %d", px, py, rank);
    if (global_domain[0] < px || global_domain[1] < py || global_domain[2] < 1)
        return set_error(OEC_ERR_SHAPE, "oec_decomp_create: domain smaller than the rank grid");
    oec_decomp *d = new oec_decomp;
    memcpy(d->gdom, global_domain, sizeof d->gdom);
    d->px = px;
    d->py = py;
    d->rank = rank;
    d->ri = rank % px;
    d->rj = rank / px;
    d->comm = nccl_comm;
    d->periodic[0] = d->periodic[1] = 0;
    subdomain(global_domain, px, py, rank, d->lo, d->hi);
    if (local_lb) memcpy(local_lb, d->lo, sizeof d->lo);
    if (local_ub) memcpy(local_ub, d->hi, sizeof d->hi);
    *out = d;
    return OEC_OK;
}

oec_status oec_decomp_set_periodic(oec_decomp *d, int32_t periodic_i, int32_t periodic_j) {
    if (!d) return set_error(OEC_ERR_ARG, "oec_decomp_set_periodic: NULL decomposition");
    d->periodic[0] = periodic_i != 0;
    d->periodic[1] = periodic_j != 0;
    return OEC_OK;
}

oec_status oec_decomp_destroy(oec_decomp *d) {
    delete d;
    return OEC_OK;
}

oec_status oec_decomp_plan(const oec_decomp *d, const int32_t width_lo[3], const int32_t width_hi[3],
                           oec_halo_msg *msgs, int32_t capacity, int32_t *n_msgs) {
    if (!d || !n_msgs) return set_error(OEC_ERR_ARG, "oec_decomp_plan: NULL argument");
    oec_status st = check_widths(width_lo, width_hi);
    if (st) return st;
    auto m = make_plan(d->gdom, d->px, d->py, d->rank, width_lo, width_hi, d->periodic[0], d->periodic[1]);
    *n_msgs = (int32_t)m.size();
    for (int32_t q = 0; q < (int32_t)m.size() && q < capacity && msgs; ++q) msgs[q] = m[q];
    return OEC_OK;
}

oec_status oec_halo_exchange(oec_decomp *d, oec_field *const *fields, int32_t n, const int32_t width_lo[3],
                             const int32_t width_hi[3], void *stream) {
    if (!d || (!fields && n > 0) || n < 0) return set_error(OEC_ERR_ARG, "oec_halo_exchange: bad arguments");
    if (n > 0 && !fields[0]) return set_error(OEC_ERR_ARG, "oec_halo_exchange: NULL field");
    if (n > 0 && fields[0]->dtype == OEC_F32) return halo_exchange_impl<float>(d, fields, n, width_lo, width_hi, stream);
    return halo_exchange_impl<double>(d, fields, n, width_lo, width_hi, stream);
}

oec_status oec_halo_exchange_local_periodic(const int64_t global_domain[3], int32_t px, int32_t py,
                                            const int32_t periodic[2], oec_field *const *fields, int32_t n,
                                            const int32_t width_lo[3], const int32_t width_hi[3], void *stream) {
    if (!global_domain || !fields || n < 1 || px < 1 || py < 1 || !fields[0])
        return set_error(OEC_ERR_ARG, "oec_halo_exchange_local: bad arguments");
    if (fields[0]->dtype == OEC_F32)
        return halo_exchange_local_impl<float>(global_domain, px, py, periodic, fields, n, width_lo, width_hi, stream);
    return halo_exchange_local_impl<double>(global_domain, px, py, periodic, fields, n, width_lo, width_hi, stream);
}

oec_status oec_halo_exchange_local(const int64_t global_domain[3], int32_t px, int32_t py, oec_field *const *fields,
                                   int32_t n, const int32_t width_lo[3], const int32_t width_hi[3], void *stream) {
    return oec_halo_exchange_local_periodic(global_domain, px, py, nullptr, fields, n, width_lo, width_hi, stream);
}

}  // extern "C"
