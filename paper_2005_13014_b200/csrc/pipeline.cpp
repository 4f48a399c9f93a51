// Multi-step hdiff with the halo exchange fused into the kernel (include/oec.h
// "oec_hdiff_pipeline"; north_star (3)).  Host side: validation, the
// neighbour table (8 directions, corners included -- hdiff's diamond reads the (+-1, +-1)
// cells), the signal pad, and CUDA IPC for peer memory between processes.  The kernel is
// hdiff_pipe in csrc/hdiff.cu.
#include <cudaTypedefs.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "oec_internal.h"

using namespace oec;

struct oec_hdiff_pipeline {
    int64_t gdom[3];
    int32_t px, py, rank, ri, rj;
    int64_t glo[3], ghi[3];  // this rank's sub-domain, global coordinates
    int32_t dtype, device;
    oec_field x[2], coeff;
    unsigned long long *pad;  // PIPE_PAD_WORDS words, device memory
    struct Nb {
        int32_t exists, set, rank;
        int64_t glo[3], ghi[3];
        oec_field x[2];
        unsigned long long *pad;
    } nb[9];
    TMap m[2], mcf;
    Dom d;
    int tile_w, tile_jb;
};

namespace {

template <class T>
oec_status run_impl(oec_hdiff_pipeline *p, int32_t nsteps, cudaStream_t s) {
    PipeArgs<T> a;
    memset(&a, 0, sizeof a);
    oec_status st;
    for (int b = 0; b < 2; ++b) {
        if ((st = field_view(&p->x[b], b ? "x1" : "x0", &a.x[b]))) return st;
        if ((st = field_view(&p->x[b], b ? "x1" : "x0", &a.y[b]))) return st;
    }
    if ((st = field_view(&p->coeff, "coeff", &a.cf))) return st;
    for (int dd = 0; dd < 9; ++dd) {
        const auto &n = p->nb[dd];
        if (!n.exists) continue;
        if (!n.set) return set_error(OEC_ERR_ARG, "oec_hdiff_pipeline_run: neighbour rank %d not registered", n.rank);
        PeerNb<T> &q = a.nb[dd];
        FVT<T> v[2];
        for (int b = 0; b < 2; ++b) {
            if ((st = field_view(&n.x[b], "peer field", &v[b]))) return st;
            q.x[b] = v[b].p;
        }
        q.sj = v[0].sj;
        q.sk = v[0].sk;
        q.oi = (int32_t)(n.glo[0] - p->glo[0]);
        q.oj = (int32_t)(n.glo[1] - p->glo[1]);
        q.flag = n.pad + (8 - dd);  // from the neighbour we sit in direction 8 - dd
        q.exists = 1;
    }
    for (int q = 0; q < 2; ++q) {
        a.alo[q] = (int32_t)p->x[0].lb[q];
        a.ahi[q] = (int32_t)p->x[0].ub[q];
    }
    a.pad = p->pad;
    a.d = p->d;
    const int W = p->tile_w, JB = p->tile_jb;
    const int ni = p->d.hi[0], nj = p->d.hi[1], nk = p->d.hi[2];
    const bool lo_i = p->nb[0 * 3 + 1].exists, hi_i = p->nb[2 * 3 + 1].exists;
    const bool lo_j = p->nb[1 * 3 + 0].exists, hi_j = p->nb[1 * 3 + 2].exists;
    a.nseg = (ni + W - 1) / W;
    a.nchunk = (nj + JB - 1) / JB;
    // interior tiles: rows/columns [ib-2, ib+W+2) x [j0-2, j0+JB+2) stay inside the sub-domain on
    // every side that has a neighbour (the global outer halo is our own caller data)
    a.sa = lo_i ? 1 : 0;
    a.sb = hi_i ? std::max(0, (ni - 2) / W) : a.nseg;
    a.ca = lo_j ? (2 + JB - 1) / JB : 0;
    a.cb = hi_j ? std::max(0, (nj - 2) / JB) : a.nchunk;
    a.sb = std::min(std::max(a.sb, a.sa), a.nseg);
    a.cb = std::min(std::max(a.cb, a.ca), a.nchunk);
    if (a.sa > a.nseg) a.sa = a.sb = a.nseg;
    if (a.ca > a.nchunk) a.ca = a.cb = a.nchunk;
    const long long n_int = (long long)(a.sb - a.sa) * (a.cb - a.ca) * nk;
    const long long n_items = (long long)a.nseg * a.nchunk * nk;
    if (n_items > INT32_MAX) return set_error(OEC_ERR_LAYOUT, "oec_hdiff_pipeline_run: too many tiles");
    a.n_int = (int32_t)n_int;
    a.n_items = (int32_t)n_items;
    int launches = 0;
    cudaError_t e = launch_hdiff_pipe<T>(p->m[0], p->m[1], p->mcf, a, nsteps, s, &launches);
    set_launch_count(launches);
    if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "oec_hdiff_pipeline_run: %s", cudaGetErrorString(e));
    return OEC_OK;
}

bool covers(const oec_field *f, const int64_t lo[3], const int64_t hi[3]) {
    for (int d = 0; d < 3; ++d)
        if (f->lb[d] > lo[d] || f->ub[d] < hi[d]) return false;
    return true;
}

// CUDA IPC: imported base pointers by the pointer handed out
std::mutex g_ipc_mu;
std::map<uintptr_t, void *> g_ipc;

PFN_cuMemGetAddressRange_v3020 g_range = nullptr;
std::once_flag g_range_once;

}  // namespace

extern "C" {

oec_status oec_hdiff_pipeline_create(const int64_t global_domain[3], int32_t px, int32_t py, int32_t rank,
                                     const oec_field *coeff, const oec_field *x0, const oec_field *x1,
                                     oec_hdiff_pipeline **out) {
    if (!global_domain || !coeff || !x0 || !x1 || !out) return set_error(OEC_ERR_ARG, "oec_hdiff_pipeline_create: NULL argument");
    *out = nullptr;
    if (px < 1 || py < 1 || rank < 0 || rank >= px * py)
        return set_error(OEC_ERR_ARG, "oec_hdiff_pipeline_create: bad grid %dx%d / rank %d", px, py, rank);
    if (global_domain[0] < 2 * px || global_domain[1] < 2 * py || global_domain[2] < 1)
        return set_error(OEC_ERR_SHAPE, "oec_hdiff_pipeline_create: every sub-domain must be >= 2 wide in i and j");
    int dev = -2, dt = -1;
    oec_status st;
    if ((st = field_check(x0, "x0", &dev, &dt)) || (st = field_check(x1, "x1", &dev, &dt)) ||
        (st = field_check(coeff, "coeff", &dev, &dt)))
        return st;
    if (dev < 0) return set_error(OEC_ERR_ARG, "oec_hdiff_pipeline_create: fields must be device fields");
    if (field_overlap(x0, x1) || field_overlap(x0, coeff) || field_overlap(x1, coeff))
        return set_error(OEC_ERR_ALIAS, "oec_hdiff_pipeline_create: x0, x1 and coeff must not overlap (P:381)");
    for (int d = 0; d < 3; ++d)
        if (x0->lb[d] != x1->lb[d] || x0->ub[d] != x1->ub[d] || x0->stride[d] != x1->stride[d])
            return set_error(OEC_ERR_LAYOUT, "oec_hdiff_pipeline_create: x1 must have x0's lb/ub/strides");
    oec_hdiff_pipeline *p = new oec_hdiff_pipeline;
    memset(p, 0, sizeof *p);
    memcpy(p->gdom, global_domain, sizeof p->gdom);
    p->px = px;
    p->py = py;
    p->rank = rank;
    p->ri = rank % px;
    p->rj = rank / px;
    subdomain(global_domain, px, py, rank, p->glo, p->ghi);
    const int64_t n[3] = {p->ghi[0] - p->glo[0], p->ghi[1] - p->glo[1], p->ghi[2] - p->glo[2]};
    const int64_t zero[3] = {0, 0, 0}, need_lo[3] = {-2, -2, 0}, need_hi[3] = {n[0] + 2, n[1] + 2, n[2]};
    if (!covers(x0, need_lo, need_hi)) {
        delete p;
        return set_error(OEC_ERR_SHAPE, "oec_hdiff_pipeline_create: x0/x1 must cover the sub-domain [0,%lld)x[0,%lld)x[0,%lld) grown by 2 in i, j",
                         (long long)n[0], (long long)n[1], (long long)n[2]);
    }
    if (!covers(coeff, zero, n) || coeff->stride[2] == 0) {
        delete p;
        return set_error(OEC_ERR_SHAPE, "oec_hdiff_pipeline_create: coeff must cover the sub-domain (3D field)");
    }
    p->dtype = dt;
    p->device = dev;
    p->x[0] = *x0;
    p->x[1] = *x1;
    p->coeff = *coeff;
    p->x[0].owned = p->x[1].owned = p->coeff.owned = 0;
    for (int q = 0; q < 3; ++q) {
        p->d.lo[q] = 0;
        p->d.hi[q] = (int32_t)n[q];
    }
    int bin[3], bcf[3];
    if (dt == OEC_F32) hdiff_pipe_boxes<float>(p->d, bin, bcf, &p->tile_w, &p->tile_jb);
    else hdiff_pipe_boxes<double>(p->d, bin, bcf, &p->tile_w, &p->tile_jb);
    const int64_t esz = dt == OEC_F32 ? 4 : 8;
    bool ok = make_tmap(x0, bin, &p->m[0], HD_PROMO) && make_tmap(x1, bin, &p->m[1], HD_PROMO) &&
              make_tmap(coeff, bcf, &p->mcf, HD_PROMO);
    for (const oec_field *f : {x0, x1}) {  // i = 0 of every row on a 16-byte boundary (vector stores)
        const uintptr_t i0 = (uintptr_t)f->data + (uintptr_t)(-f->lb[0] * esz);
        ok = ok && i0 % 16 == 0 && (f->stride[1] * esz) % 16 == 0 && (f->stride[2] * esz) % 16 == 0;
    }
    if (!ok) {
        delete p;
        return set_error(OEC_ERR_LAYOUT, "oec_hdiff_pipeline_create: x0/x1/coeff must be TMA-describable with a 16-byte "
                                         "aligned origin and pitches (oec_field_create layout)");
    }
    for (int si = 0; si < 3; ++si)
        for (int sj = 0; sj < 3; ++sj) {
            auto &nb = p->nb[si * 3 + sj];
            const int qi = p->ri + si - 1, qj = p->rj + sj - 1;
            if ((si == 1 && sj == 1) || qi < 0 || qi >= px || qj < 0 || qj >= py) continue;
            nb.exists = 1;
            nb.rank = qj * px + qi;
            subdomain(global_domain, px, py, nb.rank, nb.glo, nb.ghi);
        }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
    cudaError_t e = cudaMalloc((void **)&p->pad, PIPE_PAD_WORDS * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(p->pad, 0, PIPE_PAD_WORDS * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
        if (p->pad) cudaFree(p->pad);
        delete p;
        return set_error(OEC_ERR_CUDA, "oec_hdiff_pipeline_create: %s", cudaGetErrorString(e));
    }
    *out = p;
    return OEC_OK;
}

oec_status oec_hdiff_pipeline_signal_pad(const oec_hdiff_pipeline *p, void **pad, int64_t *bytes) {
    if (!p) return set_error(OEC_ERR_ARG, "oec_hdiff_pipeline_signal_pad: NULL pipeline");
    if (pad) *pad = p->pad;
    if (bytes) *bytes = PIPE_PAD_WORDS * sizeof(unsigned long long);
    return OEC_OK;
}

oec_status oec_hdiff_pipeline_set_peer(oec_hdiff_pipeline *p, int32_t peer_rank, const oec_field *peer_x0,
                                       const oec_field *peer_x1, void *peer_signal_pad) {
    if (!p || !peer_x0 || !peer_x1 || !peer_signal_pad)
        return set_error(OEC_ERR_ARG, "oec_hdiff_pipeline_set_peer: NULL argument");
    int dd = -1;
    for (int q = 0; q < 9; ++q)
        if (p->nb[q].exists && p->nb[q].rank == peer_rank) dd = q;
    if (dd < 0) return set_error(OEC_ERR_ARG, "oec_hdiff_pipeline_set_peer: rank %d is not adjacent to rank %d", peer_rank, p->rank);
    auto &nb = p->nb[dd];
    int dev = -2, dt = p->dtype;
    oec_status st;
    if ((st = field_check(peer_x0, "peer x0", &dev, &dt)) || (st = field_check(peer_x1, "peer x1", &dev, &dt))) return st;
    const int64_t zero[3] = {0, 0, 0};
    const int64_t n[3] = {nb.ghi[0] - nb.glo[0], nb.ghi[1] - nb.glo[1], nb.ghi[2] - nb.glo[2]};
    if (!covers(peer_x0, zero, n) || !covers(peer_x1, zero, n))
        return set_error(OEC_ERR_SHAPE, "oec_hdiff_pipeline_set_peer: rank %d's fields do not cover its sub-domain", peer_rank);
    for (int d = 0; d < 3; ++d)
        if (peer_x0->stride[d] != peer_x1->stride[d] || peer_x0->lb[d] != peer_x1->lb[d])
            return set_error(OEC_ERR_LAYOUT, "oec_hdiff_pipeline_set_peer: x1 must have x0's layout");
    nb.x[0] = *peer_x0;
    nb.x[1] = *peer_x1;
    nb.x[0].owned = nb.x[1].owned = 0;
    nb.pad = (unsigned long long *)peer_signal_pad;
    nb.set = 1;
    return OEC_OK;
}

oec_status oec_hdiff_pipeline_run(oec_hdiff_pipeline *p, int32_t nsteps, void *stream) {
    if (!p || nsteps < 0) return set_error(OEC_ERR_ARG, "oec_hdiff_pipeline_run: bad arguments");
    if (nsteps == 0) {
        set_launch_count(0);
        return OEC_OK;
    }
    if (p->dtype == OEC_F32) return run_impl<float>(p, nsteps, (cudaStream_t)stream);
    return run_impl<double>(p, nsteps, (cudaStream_t)stream);
}

oec_status oec_hdiff_pipeline_steps(const oec_hdiff_pipeline *p, int64_t *steps) {
    if (!p || !steps) return set_error(OEC_ERR_ARG, "oec_hdiff_pipeline_steps: NULL argument");
    unsigned long long v = 0;
    cudaError_t e = cudaMemcpy(&v, p->pad + PIPE_PAD_FINISHED, sizeof v, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "oec_hdiff_pipeline_steps: %s", cudaGetErrorString(e));
    *steps = (int64_t)(v >> 20);  // one step = 2^20 (hdiff.cu PIPE_STEP_SHIFT)
    return OEC_OK;
}

oec_status oec_hdiff_pipeline_destroy(oec_hdiff_pipeline *p) {
    if (!p) return OEC_OK;
    if (p->pad) cudaFree(p->pad);
    delete p;
    return OEC_OK;
}

oec_status oec_ipc_export(const void *dev_ptr, void *handle, int64_t *offset) {
    if (!dev_ptr || !handle || !offset) return set_error(OEC_ERR_ARG, "oec_ipc_export: NULL argument");
    std::call_once(g_range_once, [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_range = (PFN_cuMemGetAddressRange_v3020)fn;
    });
    if (!g_range) return set_error(OEC_ERR_CUDA, "oec_ipc_export: cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (g_range(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS)
        return set_error(OEC_ERR_ARG, "oec_ipc_export: %p is not device memory", dev_ptr);
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void *)base);
    if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "oec_ipc_export: %s", cudaGetErrorString(e));
    static_assert(sizeof h == OEC_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(handle, &h, sizeof h);
    *offset = (int64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
    return OEC_OK;
}

oec_status oec_ipc_import(const void *handle, int64_t offset, void **dev_ptr) {
    if (!handle || !dev_ptr || offset < 0) return set_error(OEC_ERR_ARG, "oec_ipc_import: bad arguments");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    void *base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "oec_ipc_import: %s", cudaGetErrorString(e));
    *dev_ptr = (char *)base + offset;
    std::lock_guard<std::mutex> g(g_ipc_mu);
    g_ipc[(uintptr_t)*dev_ptr] = base;
    return OEC_OK;
}

oec_status oec_ipc_close(void *dev_ptr) {
    void *base = nullptr;
    {
        std::lock_guard<std::mutex> g(g_ipc_mu);
        auto it = g_ipc.find((uintptr_t)dev_ptr);
        if (it == g_ipc.end()) return set_error(OEC_ERR_ARG, "oec_ipc_close: %p was not imported", dev_ptr);
        base = it->second;
        g_ipc.erase(it);
    }
    cudaError_t e = cudaIpcCloseMemHandle(base);
    if (e != cudaSuccess) return set_error(OEC_ERR_CUDA, "oec_ipc_close: %s", cudaGetErrorString(e));
    return OEC_OK;
}

}  // extern "C"
