"""Periodic decompositions on the GPU (include/oec.h oec_decomp_set_periodic) -- and through them the
NCCL transport of oec_halo_exchange on ONE device: with one rank periodic in i and j the rank is
its own neighbour, so ncclSend / ncclRecv (a world-size-1 NCCL communicator from torch) carry every
halo message, packed boxes (phase 0) and direct j-row spans (phase 1) alike.

Reference: the global field whose halo cells are filled by wrapping the interior (the definition
of a periodic domain), run through the oracle; the exchanged sub-domains through liboec must give
the same outputs bit for bit."""
import os
import socket

import numpy as np
import pytest

import synth
from gpu_util import run_oracle
from synth import HostField

pytestmark = pytest.mark.gpu


def wrapped(host, spec, gdom, per):
    """Copy of the global inputs with every halo cell of a periodic dimension replaced by the
    interior cell it wraps to (index mod the global extent)."""
    out = {}
    for s in spec.inputs:
        g = host[s.name]
        jj = np.arange(g.lb[1], g.ub[1])
        ii = np.arange(g.lb[0], g.ub[0])
        sj = np.where(per[1], np.mod(jj, gdom[1]), jj) - g.lb[1]
        si = np.where(per[0], np.mod(ii, gdom[0]), ii) - g.lb[0]
        out[s.name] = HostField(np.ascontiguousarray(g.data[:, sj][:, :, si]), g.lb, g.ub, g.k_invariant)
    return out


def rank_fields(oec, torch, host, spec, gdom, lo, hi, per, order=None):
    """One rank's fields: its own interior, the global outer halo of NON-periodic dimensions
    (caller data); every other halo cell NaN until the exchange fills it."""
    ldom = tuple(hi[d] - lo[d] for d in range(3))
    out = {}
    for s in spec.inputs:
        g = host[s.name]
        f = oec.oec_field_create(ldom if not s.k_invariant else (ldom[0], ldom[1], 1), s.halo_lo, s.halo_hi,
                                 order=order, k_invariant=s.k_invariant)
        v = f.view()
        v.fill_(float("nan"))
        gl = [max(f.lb[d] + lo[d], g.lb[d]) for d in range(2)]
        gh = [min(f.ub[d] + lo[d], g.ub[d]) for d in range(2)]
        src = g.data[:, gl[1] - g.lb[1]:gh[1] - g.lb[1], gl[0] - g.lb[0]:gh[0] - g.lb[0]].copy()
        jj, ii = np.meshgrid(np.arange(gl[1], gh[1]), np.arange(gl[0], gh[0]), indexing="ij")
        own = (ii >= lo[0]) & (ii < hi[0]) & (jj >= lo[1]) & (jj < hi[1])
        out_i = (ii < 0) | (ii >= gdom[0])
        out_j = (jj < 0) | (jj >= gdom[1])
        caller = (out_i & (not per[0])) | (out_j & (not per[1]))
        src[:, ~(own | caller)] = np.nan
        v[:, gl[1] - lo[1] - f.lb[1]:gh[1] - lo[1] - f.lb[1], gl[0] - lo[0] - f.lb[0]:gh[0] - lo[0] - f.lb[0]] = \
            torch.from_numpy(src)
        out[s.name] = f
    return out


def exchange_groups(spec):
    """Inputs grouped by their halo widths (each exchanged with its own access extent)."""
    groups = {}
    for s in spec.inputs:
        w = ((s.halo_lo[0], s.halo_lo[1], 0), (s.halo_hi[0], s.halo_hi[1], 0))
        if w != ((0, 0, 0), (0, 0, 0)):
            groups.setdefault(w, []).append(s.name)
    return groups


@pytest.mark.parametrize("px,py,per", [
    (1, 1, (True, True)), (2, 2, (True, True)), (3, 1, (True, False)), (1, 3, (False, True)), (2, 1, (True, True)),
])
@pytest.mark.parametrize("program", ["hdiff", "fvtp2d_qi", "nh_p_grad"])
def test_local_periodic_exchange(program, px, py, per):
    import torch

    from paper_2005_13014_b200 import oec

    gdom = (37, 26, 3)
    host = synth.make_inputs(program, gdom, seed=41)
    spec = synth.PROGRAMS[program]
    decs = [oec.oec_decomp_create(gdom, px, py, r) for r in range(px * py)]
    fields = [rank_fields(oec, torch, host, spec, gdom, d.local_lb, d.local_ub, per) for d in decs]
    for (wlo, whi), names in exchange_groups(spec).items():
        flat = [fields[r][nm] for r in range(len(decs)) for nm in names]
        oec.oec_halo_exchange_local(gdom, px, py, flat, len(names), wlo, whi, periodic=per)
    ref = run_oracle(program, wrapped(host, spec, gdom, per), gdom)
    sc = [v for _, v in spec.scalars]
    for r, dec in enumerate(decs):
        lo, hi = dec.local_lb, dec.local_ub
        ldom = tuple(hi[d] - lo[d] for d in range(3))
        outs = [oec.empty_like_domain(ldom) for _ in spec.outputs]
        oec.oec_apply_program(program, [fields[r][s.name] for s in spec.inputs], outs, sc, (0, 0, 0), ldom)
        torch.cuda.synchronize()
        for name, o in zip(spec.outputs, outs):
            assert np.array_equal(o.download(), ref[name][:, lo[1]:hi[1], lo[0]:hi[0]]), (program, name, r)


def test_periodic_width_wider_than_subdomain_is_rejected():
    import torch

    from paper_2005_13014_b200 import oec

    gdom = (9, 8, 2)
    host = synth.make_inputs("hdiff", gdom, seed=1)
    spec = synth.PROGRAMS["hdiff"]
    decs = [oec.oec_decomp_create(gdom, 9, 1, r) for r in range(9)]  # 1-cell sub-domains, halo 2
    fields = [rank_fields(oec, torch, host, spec, gdom, d.local_lb, d.local_ub, (True, False)) for d in decs]
    with pytest.raises(RuntimeError, match="exceeds"):
        oec.oec_halo_exchange_local(gdom, 9, 1, [f["in"] for f in fields], 1, (2, 2, 0), (2, 2, 0),
                                    periodic=(True, False))


# ---------------------------------------------------------------------------------------------
# the NCCL transport: one rank, periodic in i and j -> every message is an ncclSend / ncclRecv to
# itself (world-size-1 communicator created by torch), in a child process so the process group
# does not outlive the test
# ---------------------------------------------------------------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _nccl_worker(port, program, gdom, per, order, graph, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist

        from paper_2005_13014_b200 import oec

        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1)
        dist.all_reduce(torch.ones(1, device="cuda"))  # the communicator exists from here on
        comm = dist.distributed_c10d._get_default_group()._get_backend(torch.device("cuda", 0))._comm_ptr()
        host = synth.make_inputs(program, gdom, seed=43)
        spec = synth.PROGRAMS[program]
        dec = oec.oec_decomp_create(gdom, 1, 1, 0, comm)
        oec.oec_decomp_set_periodic(dec, *per)
        f = rank_fields(oec, torch, host, spec, gdom, dec.local_lb, dec.local_ub, per, order)
        st = torch.cuda.Stream()
        groups = exchange_groups(spec)

        def exchange():
            for (wlo, whi), names in groups.items():
                oec.oec_halo_exchange(dec, [f[nm] for nm in names], wlo, whi, st)

        if graph:  # NCCL send/recv and the stream-ordered staging inside a CUDA graph
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                exchange()
            g.replay()
        else:
            exchange()
        st.synchronize()
        ref = run_oracle(program, wrapped(host, spec, gdom, per), gdom)
        outs = [oec.empty_like_domain(gdom) for _ in spec.outputs]
        oec.oec_apply_program(program, [f[s.name] for s in spec.inputs], outs, [v for _, v in spec.scalars],
                              (0, 0, 0), gdom)
        torch.cuda.synchronize()
        ok = all(np.array_equal(o.download(), ref[n]) for n, o in zip(spec.outputs, outs))
        # every cell of the exchanged fields (own interior, halo) is the wrapped global value
        wh = wrapped(host, spec, gdom, per)
        halo_ok = True
        for names in groups.values():
            for nm in names:
                g, fl = wh[nm], f[nm]
                sl = tuple(slice(fl.lb[d] - g.lb[d], fl.ub[d] - g.lb[d]) for d in (2, 1, 0))
                halo_ok &= bool(np.array_equal(fl.download(), g.data[sl]))
        dist.destroy_process_group()
        q.put((ok, halo_ok, ""))
    except Exception as e:  # surface the failure in the parent
        q.put((False, False, repr(e)))


@pytest.mark.parametrize("program,per,order,graph", [
    ("hdiff", (True, True), None, False),       # i: packed boxes over NCCL; j: direct row spans
    ("hdiff", (True, True), (0, 1, 2), False),  # i,j,k layout: every box packed
    ("hdiff", (False, True), None, True),       # j only, inside a CUDA graph
    ("fvtp2d_flux", (True, True), None, False),
    ("vadv", (True, False), None, False),       # wcon's +1 i-halo
])
def test_nccl_self_exchange(program, per, order, graph):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), program, (40, 21, 5), per, order, graph, q))
    p.start()
    ok, halo_ok, err = q.get(timeout=300)
    p.join(timeout=60)
    assert ok and halo_ok, (program, per, order, err)
