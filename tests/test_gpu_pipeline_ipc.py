"""The fused-exchange hdiff pipeline across PROCESSES (one process per rank, as on the 8-GPU box):
each process owns its sub-domain's fields, exports them and its signal pad with CUDA IPC
(oec_ipc_export), the handles travel over a gloo process group, every process imports its
neighbours' memory (oec_ipc_import) and registers it with its pipeline, and the steps run with the
halo read straight from the neighbours' allocations inside the kernel.  gpurun has one GPU, so all
processes share cuda:0 (CUDA IPC works between processes on one device; on the box the same calls
map NVLink peer memory).  After T steps every rank must equal T oracle applications of hdiff on the
global domain, bit for bit (R23)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, gdom, px, py, T, dtype_name, results):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    import torch
    import torch.distributed as dist

    import synth
    from oracle import capi
    from paper_2005_13014_b200 import oec

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dtype = np.dtype(dtype_name)
        host = synth.make_inputs("hdiff", gdom, seed=5, dtype=dtype)
        dec = oec.oec_decomp_create(gdom, px, py, rank)
        lo, hi = dec.local_lb, dec.local_ub
        ldom = tuple(hi[d] - lo[d] for d in range(3))
        x0 = oec.oec_field_create(ldom, (2, 2, 0), (2, 2, 0), dtype=dtype)
        x1 = oec.oec_field_create(ldom, (2, 2, 0), (2, 2, 0), dtype=dtype)
        g = host["in"]
        sub = g.data[:, lo[1] - 2 - g.lb[1]:hi[1] + 2 - g.lb[1], lo[0] - 2 - g.lb[0]:hi[0] + 2 - g.lb[0]]
        v0 = x0.view()
        v0.fill_(float("nan"))
        i0, j0 = -2 - x0.lb[0], -2 - x0.lb[1]
        v0[:, j0:j0 + sub.shape[1], i0:i0 + sub.shape[2]] = torch.from_numpy(np.ascontiguousarray(sub))
        x1.view().copy_(v0)
        c = host["coeff"]
        csub = c.data[:, lo[1] - c.lb[1]:hi[1] - c.lb[1], lo[0] - c.lb[0]:hi[0] - c.lb[0]]
        cf = oec.oec_field_create(ldom, (0, 0, 0), (0, 0, 0), dtype=dtype)
        cf.view()[:, -cf.lb[1]:-cf.lb[1] + csub.shape[1], -cf.lb[0]:-cf.lb[0] + csub.shape[2]] = torch.from_numpy(
            np.ascontiguousarray(csub))
        pipe = oec.HdiffPipeline(gdom, px, py, rank, cf, x0, x1)
        torch.cuda.synchronize()
        pad, _ = pipe.signal_pad()
        mine = dict(x0=oec.oec_ipc_export(x0.desc.data), x1=oec.oec_ipc_export(x1.desc.data),
                    pad=oec.oec_ipc_export(pad), desc=oec.field_descriptor(x0))
        everyone = [None] * world
        dist.all_gather_object(everyone, mine)
        imported = []
        ri, rj = rank % px, rank // px
        for dj in (-1, 0, 1):
            for di in (-1, 0, 1):
                qi, qj = ri + di, rj + dj
                if (di, dj) == (0, 0) or not (0 <= qi < px and 0 <= qj < py):
                    continue
                q = qj * px + qi
                Q = everyone[q]
                p0 = oec.oec_ipc_import(*Q["x0"])
                p1 = oec.oec_ipc_import(*Q["x1"])
                pp = oec.oec_ipc_import(*Q["pad"])
                imported += [p0, p1, pp]
                pipe.set_peer(q, oec.field_at(p0, Q["desc"], 0), oec.field_at(p1, Q["desc"], 0), pp)
        dist.barrier()
        pipe.run(T)
        torch.cuda.synchronize()
        dist.barrier()  # every rank done before anyone unmaps peer memory
        # oracle: T global applications, the outer halo held constant
        x = host["in"]
        for _ in range(T):
            o = x.copy()
            capi.hdiff(x, host["coeff"], o, (0, 0, 0), gdom, capi.HDIFF_UNFUSED, 0)
            x = o
        got = (x0, x1)[T % 2].download()
        gsub = got[:, -x0.lb[1]:-x0.lb[1] + ldom[1], -x0.lb[0]:-x0.lb[0] + ldom[0]]
        want = x.data[:, lo[1] - x.lb[1]:hi[1] - x.lb[1], lo[0] - x.lb[0]:hi[0] - x.lb[0]]
        u = np.uint64 if dtype == np.float64 else np.uint32
        nbad = int(np.count_nonzero(gsub.view(u) != want.view(u)))
        steps = pipe.steps()
        for p in imported:
            oec.oec_ipc_close(p)
        dist.barrier()
        results[rank] = (nbad, steps, int(gsub.size))
    except Exception as e:  # reported to the parent
        results[rank] = ("error", repr(e))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("gdom,px,py,T,dtype", [
    ((96, 64, 3), 2, 1, 3, "float64"),
    ((70, 90, 2), 1, 2, 4, "float64"),
    ((80, 60, 2), 2, 2, 3, "float64"),
    ((64, 40, 2), 2, 1, 3, "float32"),
])
def test_pipeline_ipc_across_processes(gdom, px, py, T, dtype):
    import torch.multiprocessing as mp

    world = px * py
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        results = m.dict()
        port = _free_port()
        procs = [ctx.Process(target=_rank_main, args=(r, world, port, gdom, px, py, T, dtype, results))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=240)
        for p in procs:
            if p.is_alive():
                p.kill()
        res = dict(results)
    assert len(res) == world, res
    for r, v in res.items():
        assert v[0] != "error", (r, v)
        nbad, steps, n = v
        assert steps == T and n > 0 and nbad == 0, (r, v)
