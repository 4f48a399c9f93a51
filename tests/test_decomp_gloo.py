"""Multi-process (gloo, CPU) test of the horizontal decomposition and the halo-exchange PLAN that
liboec executes over NCCL on GPUs (include/oec.h oec_decomp_*).

Each rank owns a sub-domain (oec_decomp_create), fills its interior (and any global outer halo,
which is caller data) from the global seeded input, leaves the inter-rank halo as NaN, executes
oec_decomp_plan's messages with torch.distributed send/recv (phase 0 then phase 1, corners in two
hops), runs the oracle on its sub-domain in rank-local coordinates, and compares with the global
oracle: the decomposed result must be bitwise identical, corners included.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import capi
from synth import HostField


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _box_slices(f: HostField, lo, hi):
    return tuple(slice(lo[d] - f.lb[d], hi[d] - f.lb[d]) for d in (2, 1, 0))


def _local_field(g: HostField, org, lo_local, hi_local, fill=np.nan):
    """Rank-local field over [lo_local, hi_local) (local coords, origin = org in global coords),
    with every cell that lies OUTSIDE the global domain interior copied from the global field (the
    global outer halo is caller data); cells inside the global domain but outside the rank's own
    sub-domain stay `fill` until the exchange delivers them."""
    shape = tuple(hi_local[d] - lo_local[d] for d in (2, 1, 0))
    data = np.full(shape, fill)
    loc = HostField(data, tuple(lo_local), tuple(hi_local), g.k_invariant)
    return loc


def _wrapped(host, gdom, per):
    """Global inputs with the halo cells of periodic dimensions replaced by the interior cells they
    wrap to (the definition of a periodic domain)."""
    out = {}
    for name, g in host.items():
        sj = np.arange(g.lb[1], g.ub[1])
        si = np.arange(g.lb[0], g.ub[0])
        sj = (np.mod(sj, gdom[1]) if per[1] else sj) - g.lb[1]
        si = (np.mod(si, gdom[0]) if per[0] else si) - g.lb[0]
        out[name] = HostField(np.ascontiguousarray(g.data[:, sj][:, :, si]), g.lb, g.ub, g.k_invariant)
    return out


def _worker(rank, world, port, program, gdom, px, py, wlo, whi, q, per=(False, False)):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2005_13014_b200 import oec

        dec = oec.oec_decomp_create(gdom, px, py, rank)
        oec.oec_decomp_set_periodic(dec, *per)
        lo, hi = dec.local_lb, dec.local_ub
        ldom = tuple(hi[d] - lo[d] for d in range(3))
        host = synth.make_inputs(program, gdom, seed=3)
        spec = synth.PROGRAMS[program]
        local = {}
        for s in spec.inputs:
            g = host[s.name]
            llo = (-s.halo_lo[0], -s.halo_lo[1], g.lb[2])
            lhi = (ldom[0] + s.halo_hi[0], ldom[1] + s.halo_hi[1], g.ub[2])
            f = _local_field(g, lo, llo, lhi)
            # fill: own interior + the global outer halo (caller data); inter-rank halo stays NaN
            for k in range(llo[2], lhi[2]):
                for jj in range(llo[1], lhi[1]):
                    for ii in range(llo[0], lhi[0]):
                        gi, gj = ii + lo[0], jj + lo[1]
                        own = 0 <= ii < ldom[0] and 0 <= jj < ldom[1]
                        outside = (not per[0] and not 0 <= gi < gdom[0]) or (not per[1] and not 0 <= gj < gdom[1])
                        if own or outside:
                            f.data[k - llo[2], jj - llo[1], ii - llo[0]] = g.data[k - g.lb[2], gj - g.lb[1], gi - g.lb[0]]
            local[s.name] = f
        # execute the plan: phase 0, then phase 1 (corners ride in phase 1)
        plan = oec.oec_decomp_plan(dec, wlo, whi)
        # exchange the fields whose halo covers the exchange widths (hdiff: `in`; vadv with an i-split: wcon)
        halo_fields = [s.name for s in spec.inputs if not s.k_invariant
                       and all(s.halo_lo[d] >= wlo[d] and s.halo_hi[d] >= whi[d] for d in (0, 1))]
        # (tagged by plan tag and field: with a periodic domain one peer can be both neighbours;
        # messages to this rank itself are copied locally)
        for phase in (0, 1):
            reqs, recvs, own = [], [], {}
            for m in plan:
                if m["phase"] != phase:
                    continue
                for fi, name in enumerate(halo_fields):
                    f = local[name]
                    blo = (m["lo"][0] - lo[0], m["lo"][1] - lo[1], f.lb[2])
                    bhi = (m["hi"][0] - lo[0], m["hi"][1] - lo[1], f.ub[2])
                    sl = _box_slices(f, blo, bhi)
                    tag = 16 * m["tag"] + fi
                    if m["is_send"] and m["peer"] == rank:
                        own[tag] = np.ascontiguousarray(f.data[sl])
                    elif m["is_send"]:
                        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(f.data[sl])), m["peer"], tag=tag))
                    else:
                        buf = torch.empty(f.data[sl].shape, dtype=torch.float64)
                        if m["peer"] != rank:
                            reqs.append(dist.irecv(buf, m["peer"], tag=tag))
                        recvs.append((f, sl, buf, tag, m["peer"] == rank))
            for r in reqs:
                r.wait()
            for f, sl, buf, tag, self_msg in recvs:
                f.data[sl] = own[tag] if self_msg else buf.numpy()
        # no NaN may remain in what the program reads
        sc = synth.scalars(program)
        out = HostField(np.full((ldom[2], ldom[1], ldom[0]), np.nan), (0, 0, 0), ldom)
        if program == "hdiff":
            capi.hdiff(local["in"], local["coeff"], out, (0, 0, 0), ldom)
        else:
            capi.vadv(local, out, sc["dtr_stage"], (0, 0, 0), ldom)
        gout = HostField(np.full((gdom[2], gdom[1], gdom[0]), np.nan), (0, 0, 0), gdom)
        host = _wrapped(host, gdom, per)
        if program == "hdiff":
            capi.hdiff(host["in"], host["coeff"], gout, (0, 0, 0), gdom)
        else:
            capi.vadv(host, gout, sc["dtr_stage"], (0, 0, 0), gdom)
        ref = gout.data[:, lo[1]:hi[1], lo[0]:hi[0]]
        q.put((rank, bool(np.array_equal(out.data, ref)), int(np.isnan(out.data).sum())))
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("program,gdom,px,py,w", [
    ("hdiff", (12, 14, 2), 1, 2, ((2, 2, 0), (2, 2, 0))),
    ("hdiff", (13, 11, 2), 2, 2, ((2, 2, 0), (2, 2, 0))),
    ("hdiff", (17, 6, 1), 4, 1, ((2, 2, 0), (2, 2, 0))),
    ("vadv", (14, 5, 6), 2, 1, ((0, 0, 0), (1, 0, 0))),
])
def test_decomposed_equals_global(program, gdom, px, py, w):
    _run(program, gdom, px, py, w, (False, False))


@pytest.mark.parametrize("program,gdom,px,py,w,per", [
    ("hdiff", (12, 10, 2), 2, 1, ((2, 2, 0), (2, 2, 0)), (True, True)),  # the same peer on both sides in i
    ("hdiff", (13, 11, 2), 2, 2, ((2, 2, 0), (2, 2, 0)), (True, True)),
    ("vadv", (14, 5, 6), 2, 1, ((0, 0, 0), (1, 0, 0)), (True, False)),
    ("hdiff", (13, 9, 2), 3, 1, ((2, 2, 0), (2, 2, 0)), (True, False)),  # corners beyond the periodic i edge
])
def test_periodic_decomposed_equals_wrapped_global(program, gdom, px, py, w, per):
    # periodic domain (oec_decomp_set_periodic): the result equals the oracle on the global field
    # whose halo is the wrapped interior
    _run(program, gdom, px, py, w, per)


def _run(program, gdom, px, py, w, per):
    world = px * py
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, program, gdom, px, py, w[0], w[1], q, per))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, info in sorted(res, key=lambda x: x[0]):
        assert ok, (rank, info)
