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

#include <mutex>
#include <vector>

#include "oec_internal.h"

struct oec_decomp {
    int64_t gdom[3];
    int32_t px, py, rank, ri, rj;
    int64_t lo[3], hi[3];
    void *comm;
};

namespace oec {
namespace {

template <class T>
__global__ void pack_kernel(FVT<T> src, Box b, T *buf) {
    const long long ni = b.hi[0] - b.lo[0], nj = b.hi[1] - b.lo[1], nk = b.hi[2] - b.lo[2];
    const long long n = ni * nj * nk;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
        const int i = b.lo[0] + (int)(t % ni), j = b.lo[1] + (int)((t / ni) % nj), k = b.lo[2] + (int)(t / (ni * nj));
        buf[t] = src.p[i + j * src.sj + k * src.sk];
    }
}
template <class T>
__global__ void unpack_kernel(const T *buf, Box b, FOT<T> dst) {
    const long long ni = b.hi[0] - b.lo[0], nj = b.hi[1] - b.lo[1], nk = b.hi[2] - b.lo[2];
    const long long n = ni * nj * nk;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
        const int i = b.lo[0] + (int)(t % ni), j = b.lo[1] + (int)((t / ni) % nj), k = b.lo[2] + (int)(t / (ni * nj));
        dst.p[i + j * dst.sj + k * dst.sk] = buf[t];
    }
}
template <class T>
__global__ void box_copy_kernel(FVT<T> src, FOT<T> dst, Box b) {
    const long long ni = b.hi[0] - b.lo[0], nj = b.hi[1] - b.lo[1], nk = b.hi[2] - b.lo[2];
    const long long n = ni * nj * nk;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
        const int i = b.lo[0] + (int)(t % ni), j = b.lo[1] + (int)((t / ni) % nj), k = b.lo[2] + (int)(t / (ni * nj));
        dst.p[i + j * dst.sj + k * dst.sk] = src.p[i + j * src.sj + k * src.sk];
    }
}

long long box_volume(const Box &b) {
    return (long long)(b.hi[0] - b.lo[0]) * (b.hi[1] - b.lo[1]) * (b.hi[2] - b.lo[2]);
}
unsigned grid_for(long long n) {
    long long g = (n + 255) / 256;
    return (unsigned)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

template <class T>
cudaError_t launch_pack(const FVT<T> &src, const Box &b, T *buf, cudaStream_t s, int *launches) {
    if (box_volume(b) <= 0) return cudaSuccess;
    pack_kernel<<<grid_for(box_volume(b)), 256, 0, s>>>(src, b, buf);
    ++*launches;
    return cudaGetLastError();
}
template <class T>
cudaError_t launch_unpack(const T *buf, const Box &b, const FOT<T> &dst, cudaStream_t s, int *launches) {
    if (box_volume(b) <= 0) return cudaSuccess;
    unpack_kernel<<<grid_for(box_volume(b)), 256, 0, s>>>(buf, b, dst);
    ++*launches;
    return cudaGetLastError();
}
template <class T>
cudaError_t launch_box_copy(const FVT<T> &src, const FOT<T> &dst, const Box &b, cudaStream_t s, int *launches) {
    if (box_volume(b) <= 0) return cudaSuccess;
    box_copy_kernel<<<grid_for(box_volume(b)), 256, 0, s>>>(src, dst, b);
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

// messages of `rank` in execution order (see oec.h oec_decomp_plan)
std::vector<oec_halo_msg> make_plan(const int64_t g[3], int px, int py, int rank, const int32_t wlo[3],
                                    const int32_t whi[3]) {
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
    if (ri > 0) {  // left neighbour: it needs our first whi[0] columns, we need its last wlo[0]
        add(rank - 1, 1, 0, 0, lo[0], lo[0] + whi[0], lo[1], hi[1]);
        add(rank - 1, 0, 0, 1, lo[0] - wlo[0], lo[0], lo[1], hi[1]);
    }
    if (ri < px - 1) {
        add(rank + 1, 1, 0, 1, hi[0] - wlo[0], hi[0], lo[1], hi[1]);
        add(rank + 1, 0, 0, 0, hi[0], hi[0] + whi[0], lo[1], hi[1]);
    }
    // phase 1: j-neighbours, i-range including the i-halo (corners)
    const int64_t i0 = lo[0] - wlo[0], i1 = hi[0] + whi[0];
    if (rj > 0) {
        add(rank - px, 1, 1, 2, i0, i1, lo[1], lo[1] + whi[1]);
        add(rank - px, 0, 1, 3, i0, i1, lo[1] - wlo[1], lo[1]);
    }
    if (rj < py - 1) {
        add(rank + px, 1, 1, 3, i0, i1, hi[1] - wlo[1], hi[1]);
        add(rank + px, 0, 1, 2, i0, i1, hi[1], hi[1] + whi[1]);
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

// staging for packed messages
struct Stage {
    std::mutex mu;
    void *p = nullptr;
    size_t n = 0;  // bytes
};
Stage g_hstage;

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

}  // namespace

template <class T>
oec_status halo_exchange_impl(oec_decomp *d, oec_field *const *fields, int32_t n, const int32_t width_lo[3],
                              const int32_t width_hi[3], void *stream) {
    oec_status st = check_widths(width_lo, width_hi);
    if (st) return st;
    auto plan = make_plan(d->gdom, d->px, d->py, d->rank, width_lo, width_hi);
    set_launch_count(0);
    if (plan.empty() || n == 0) return OEC_OK;
    if (!d->comm) return set_error(OEC_ERR_NCCL, "oec_halo_exchange: decomposition has no NCCL communicator");
    if (!load_nccl()) return set_error(OEC_ERR_NCCL, "oec_halo_exchange: libnccl.so.2 not loadable in this process");
    cudaStream_t s = (cudaStream_t)stream;
    // staging: one slot per (message, field)
    std::vector<Box> boxes(plan.size() * n);
    std::vector<FVT<T>> views(n);
    size_t total = 0;
    for (int f = 0; f < n; ++f) {
        if (fields[f]->device < 0) return set_error(OEC_ERR_ARG, "oec_halo_exchange: fields must be device memory");
        if ((st = view_of(fields[f], &views[f]))) return st;
        for (size_t q = 0; q < plan.size(); ++q) {
            if ((st = field_box(fields[f], plan[q], d->lo, &boxes[q * n + f]))) return st;
            total += (size_t)box_volume(boxes[q * n + f]);
        }
    }
    std::lock_guard<std::mutex> lock(g_hstage.mu);
    if (g_hstage.n < total * sizeof(T)) {
        if (g_hstage.p) cudaFree(g_hstage.p);
        g_hstage.p = nullptr;
        g_hstage.n = 0;
        cudaError_t e = cudaMalloc(&g_hstage.p, total * sizeof(T));
        if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "halo staging: %s", cudaGetErrorString(e));
        g_hstage.n = total * sizeof(T);
    }
    std::vector<T *> bufs(plan.size() * n);
    size_t off = 0;
    for (size_t t = 0; t < bufs.size(); ++t) {
        bufs[t] = (T *)g_hstage.p + off;
        off += (size_t)box_volume(boxes[t]);
    }
    constexpr int NCCL_DT = sizeof(T) == 8 ? NCCL_FLOAT64 : NCCL_FLOAT32;
    int launches = 0;
    for (int phase = 0; phase < 2; ++phase) {
        for (size_t q = 0; q < plan.size(); ++q)
            if (plan[q].phase == phase && plan[q].is_send)
                for (int f = 0; f < n; ++f) {
                    cudaError_t e = launch_pack(views[f], boxes[q * n + f], bufs[q * n + f], s, &launches);
                    if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "halo pack: %s", cudaGetErrorString(e));
                }
        int r = g_nccl.gstart();
        for (size_t q = 0; q < plan.size() && r == 0; ++q) {
            if (plan[q].phase != phase) continue;
            for (int f = 0; f < n && r == 0; ++f) {
                const size_t cnt = (size_t)box_volume(boxes[q * n + f]);
                r = plan[q].is_send ? g_nccl.send(bufs[q * n + f], cnt, NCCL_DT, plan[q].peer, d->comm, s)
                                    : g_nccl.recv(bufs[q * n + f], cnt, NCCL_DT, plan[q].peer, d->comm, s);
            }
        }
        int r2 = g_nccl.gend();
        if (r || r2)
            return set_error(OEC_ERR_NCCL, "oec_halo_exchange: NCCL error %d (%s)", r ? r : r2,
                             g_nccl.errstr ? g_nccl.errstr(r ? r : r2) : "?");
        for (size_t q = 0; q < plan.size(); ++q)
            if (plan[q].phase == phase && !plan[q].is_send)
                for (int f = 0; f < n; ++f) {
                    FOT<T> o{(T *)views[f].p, views[f].sj, views[f].sk};
                    cudaError_t e = launch_unpack(bufs[q * n + f], boxes[q * n + f], o, s, &launches);
                    if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "halo unpack: %s", cudaGetErrorString(e));
                }
    }
    set_launch_count(launches);
    return OEC_OK;
}

template <class T>
oec_status halo_exchange_local_impl(const int64_t global_domain[3], int32_t px, int32_t py, oec_field *const *fields,
                                    int32_t n, const int32_t width_lo[3], const int32_t width_hi[3], void *stream) {
    oec_status st = check_widths(width_lo, width_hi);
    if (st) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const int R = px * py;
    int launches = 0;
    for (int phase = 0; phase < 2; ++phase) {
        for (int r = 0; r < R; ++r) {
            auto plan = make_plan(global_domain, px, py, r, width_lo, width_hi);
            for (auto &m : plan) {
                if (m.phase != phase || m.is_send) continue;
                for (int f = 0; f < n; ++f) {
                    const oec_field *src = fields[m.peer * n + f];
                    oec_field *dst = fields[r * n + f];
                    int64_t org_d[3], org_s[3], tmp[3];
                    subdomain(global_domain, px, py, r, org_d, tmp);
                    subdomain(global_domain, px, py, m.peer, org_s, tmp);
                    FVT<T> vs, vd;
                    Box bd, bs;
                    if ((st = view_of(src, &vs)) || (st = view_of(dst, &vd)) || (st = field_box(dst, m, org_d, &bd)) ||
                        (st = field_box(src, m, org_s, &bs)))
                        return st;
                    // shift the source origin so that the destination's local box indexes it
                    vs.p += (int64_t)(bs.lo[0] - bd.lo[0]) + (int64_t)(bs.lo[1] - bd.lo[1]) * vs.sj;
                    FOT<T> o{(T *)vd.p, vd.sj, vd.sk};
                    cudaError_t e = launch_box_copy(vs, o, bd, s, &launches);
                    if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "halo copy: %s", cudaGetErrorString(e));
                }
            }
        }
    }
    set_launch_count(launches);
    return OEC_OK;
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
    subdomain(global_domain, px, py, rank, d->lo, d->hi);
    if (local_lb) memcpy(local_lb, d->lo, sizeof d->lo);
    if (local_ub) memcpy(local_ub, d->hi, sizeof d->hi);
    *out = d;
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
    auto m = make_plan(d->gdom, d->px, d->py, d->rank, width_lo, width_hi);
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

oec_status oec_halo_exchange_local(const int64_t global_domain[3], int32_t px, int32_t py, oec_field *const *fields,
                                   int32_t n, const int32_t width_lo[3], const int32_t width_hi[3], void *stream) {
    if (!global_domain || !fields || n < 1 || px < 1 || py < 1 || !fields[0])
        return set_error(OEC_ERR_ARG, "oec_halo_exchange_local: bad arguments");
    if (fields[0]->dtype == OEC_F32)
        return halo_exchange_local_impl<float>(global_domain, px, py, fields, n, width_lo, width_hi, stream);
    return halo_exchange_local_impl<double>(global_domain, px, py, fields, n, width_lo, width_hi, stream);
}

}  // extern "C"
