"""GPU tests of oec_hdiff_pipeline: multi-step hdiff with the halo exchange fused into the kernel
(SURVEY §8(f) rank 2).  All ranks' sub-domains live on cuda:0 and their pipelines are given each
other's fields directly (the same kernel reads NVLink peer memory when the pointers come from
oec_ipc_import).  After T steps every rank's sub-domain must equal T applications of the oracle's
hdiff on the global domain, the global outer halo held constant (R23), bit for bit.

Launch order matters on ONE device: a step of rank r waits for its neighbours' previous step,
so the steps are enqueued round-robin (step t of every rank, then step t+1); enqueuing all steps
of one rank first would wait for kernels queued behind it (the kernel traps after 20 s)."""
import numpy as np
import pytest

import synth
from oracle import capi
from synth import HostField

pytestmark = pytest.mark.gpu


def oracle_steps(host, gdom, T):
    """T applications of the oracle hdiff on the global domain; the outer halo stays the caller's."""
    x = host["in"]
    for _ in range(T):
        o = x.copy()  # keeps the outer halo; the domain is overwritten
        capi.hdiff(x, host["coeff"], o, (0, 0, 0), gdom, capi.HDIFF_UNFUSED, 0)
        x = o
    return x


def build_ranks(host, gdom, px, py, dtype):
    from paper_2005_13014_b200 import oec

    import torch

    ranks = []
    for r in range(px * py):
        dec = oec.oec_decomp_create(gdom, px, py, r)
        lo, hi = dec.local_lb, dec.local_ub
        ldom = tuple(hi[d] - lo[d] for d in range(3))
        g = host["in"]
        x0 = oec.oec_field_create(ldom, (2, 2, 0), (2, 2, 0), dtype=dtype)
        x1 = oec.oec_field_create(ldom, (2, 2, 0), (2, 2, 0), dtype=dtype)
        sub = g.data[:, lo[1] - 2 - g.lb[1]:hi[1] + 2 - g.lb[1], lo[0] - 2 - g.lb[0]:hi[0] + 2 - g.lb[0]]
        v0, v1 = x0.view(), x1.view()
        v0.fill_(float("nan"))  # padding outside [-2, n+2) must never be read
        i0, j0 = -2 - x0.lb[0], -2 - x0.lb[1]  # view index of local (-2, -2)
        v0[:, j0:j0 + sub.shape[1], i0:i0 + sub.shape[2]] = torch.from_numpy(np.ascontiguousarray(sub))
        v1.copy_(v0)
        c = host["coeff"]
        csub = c.data[:, lo[1] - c.lb[1]:hi[1] - c.lb[1], lo[0] - c.lb[0]:hi[0] - c.lb[0]]
        cf = oec.oec_field_create(ldom, (0, 0, 0), (0, 0, 0), dtype=dtype)
        cv = cf.view()
        ci0, cj0 = -cf.lb[0], -cf.lb[1]
        cv[:, cj0:cj0 + csub.shape[1], ci0:ci0 + csub.shape[2]] = torch.from_numpy(np.ascontiguousarray(csub))
        pipe = oec.HdiffPipeline(gdom, px, py, r, cf, x0, x1)
        ranks.append(dict(lo=lo, hi=hi, x=(x0, x1), cf=cf, pipe=pipe))
    for r, R in enumerate(ranks):
        ri, rj = r % px, r // px
        for dj in (-1, 0, 1):
            for di in (-1, 0, 1):
                qi, qj = ri + di, rj + dj
                if (di, dj) == (0, 0) or not (0 <= qi < px and 0 <= qj < py):
                    continue
                q = qj * px + qi
                Q = ranks[q]
                R["pipe"].set_peer(q, Q["x"][0], Q["x"][1], Q["pipe"].signal_pad()[0])
    return ranks


def check(ranks, ref, T):
    for R in ranks:
        x = R["x"][T % 2]
        lo, hi = R["lo"], R["hi"]
        got = x.download()  # [k][j][i] over the local allocation
        li = -x.lb[0]
        lj = -x.lb[1]
        g = got[:, lj:lj + hi[1] - lo[1], li:li + hi[0] - lo[0]]
        want = ref.data[:, lo[1] - ref.lb[1]:hi[1] - ref.lb[1], lo[0] - ref.lb[0]:hi[0] - ref.lb[0]]
        assert g.shape == want.shape
        nbad = int(np.count_nonzero(g.view(np.uint64 if g.dtype == np.float64 else np.uint32)
                                    != want.view(np.uint64 if want.dtype == np.float64 else np.uint32)))
        assert nbad == 0, f"rank box {lo}..{hi}: {nbad} of {g.size} differ bitwise"
        assert R["pipe"].steps() == T


@pytest.mark.parametrize("gdom,px,py,T", [
    ((70, 45, 3), 1, 1, 3),
    ((150, 40, 3), 2, 1, 3),
    ((64, 90, 4), 1, 2, 4),
    ((131, 77, 3), 2, 2, 3),
    ((200, 50, 2), 3, 2, 5),
    ((33, 20, 2), 4, 1, 3),      # narrow sub-domains: every tile is a boundary tile
    ((9, 8, 2), 2, 2, 2),        # sub-domains of 4-5 cells
    ((4096, 1100, 4), 2, 1, 2),  # > 8M points per rank: the large tile configuration
])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_pipeline_matches_oracle_steps(gdom, px, py, T, dtype):
    import torch

    host = synth.make_inputs("hdiff", gdom, seed=11, dtype=dtype)
    ref = oracle_steps(host, gdom, T)
    ranks = build_ranks(host, gdom, px, py, dtype)
    for _ in range(T):
        for R in ranks:
            R["pipe"].run(1)
    torch.cuda.synchronize()
    check(ranks, ref, T)


def test_pipeline_graph_replay():
    """A captured round (one step of every rank) replayed T times advances T steps (the step
    counter lives on the device)."""
    import torch

    gdom, px, py, T = (131, 77, 3), 2, 2, 4
    host = synth.make_inputs("hdiff", gdom, seed=3)
    ref = oracle_steps(host, gdom, T)
    ranks = build_ranks(host, gdom, px, py, np.float64)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for R in ranks:
                R["pipe"].run(1)
    for _ in range(T):
        g.replay()
    torch.cuda.synchronize()
    check(ranks, ref, T)


def test_pipeline_single_rank_many_steps():
    """px = py = 1: run(T) in one call (no neighbours to wait for)."""
    import torch

    gdom, T = (96, 64, 5), 7
    host = synth.make_inputs("hdiff", gdom, seed=5)
    ref = oracle_steps(host, gdom, T)
    ranks = build_ranks(host, gdom, 1, 1, np.float64)
    ranks[0]["pipe"].run(T)
    torch.cuda.synchronize()
    check(ranks, ref, T)


def _pad_word(pipe, w):
    """Word w of a pipeline's device signal pad (diagnostic counters, csrc/oec_internal.h)."""
    import torch

    from paper_2005_13014_b200 import oec

    ptr, nbytes = pipe.signal_pad()
    arr = oec._CudaArray(ptr, (nbytes // 8,), (8,), pipe, "<u8")
    return int(torch.as_tensor(arr, device="cuda:0")[w].item())


def _set_pad_word(pipe, w, v):
    import torch

    from paper_2005_13014_b200 import oec

    ptr, nbytes = pipe.signal_pad()
    arr = oec._CudaArray(ptr, (nbytes // 8,), (8,), pipe, "<u8")
    torch.as_tensor(arr, device="cuda:0")[w] = v


@pytest.mark.parametrize("gdom,T", [((64, 4, 1), 5), ((150, 37, 3), 4), ((256, 256, 8), 3)])
def test_pipeline_wrong_step_guess_recovers(gdom, T):
    """The first tiles of a step are requested from the x_t of a GUESSED step before the step
    counter is read; a wrong guess drains those loads and requests them again from the right
    buffer.  Pad word 11 (a test hook) inverts every guess: the results must be unaffected and
    pad word 12 must count the re-requests."""
    import torch

    host = synth.make_inputs("hdiff", gdom, seed=21)
    ref = oracle_steps(host, gdom, T)
    ranks = build_ranks(host, gdom, 1, 1, np.float64)
    _set_pad_word(ranks[0]["pipe"], 11, 1)
    torch.cuda.synchronize()
    ranks[0]["pipe"].run(T)
    torch.cuda.synchronize()
    check(ranks, ref, T)
    assert _pad_word(ranks[0]["pipe"], 12) >= T


def test_pipeline_errors():
    from paper_2005_13014_b200 import oec

    gdom = (40, 30, 2)
    host = synth.make_inputs("hdiff", gdom, seed=1)
    ranks = build_ranks(host, gdom, 1, 1, np.float64)
    # unregistered neighbour
    dec = oec.oec_decomp_create(gdom, 2, 1, 0)
    ldom = tuple(dec.local_ub[d] - dec.local_lb[d] for d in range(3))
    x0 = oec.oec_field_create(ldom, (2, 2, 0), (2, 2, 0))
    x1 = oec.oec_field_create(ldom, (2, 2, 0), (2, 2, 0))
    cf = oec.oec_field_create(ldom, (0, 0, 0), (0, 0, 0))
    p = oec.HdiffPipeline(gdom, 2, 1, 0, cf, x0, x1)
    with pytest.raises(oec.OecError) as e:
        p.run(1)
    assert e.value.status == 1
    # not adjacent (rank 0 of 1x1 has no neighbours)
    with pytest.raises(oec.OecError) as e:
        ranks[0]["pipe"].set_peer(1, x0, x1, p.signal_pad()[0])
    assert e.value.status == 1
    # halo too small
    y0 = oec.oec_field_create(ldom, (1, 2, 0), (2, 2, 0))
    y1 = oec.oec_field_create(ldom, (1, 2, 0), (2, 2, 0))
    with pytest.raises(oec.OecError) as e:
        oec.HdiffPipeline(gdom, 2, 1, 0, cf, y0, y1)
    assert e.value.status == 2
    # aliasing
    with pytest.raises(oec.OecError) as e:
        oec.HdiffPipeline(gdom, 2, 1, 0, cf, x0, x0)
    assert e.value.status == 3


def test_ipc_export_roundtrip_offsets():
    """oec_ipc_export reports the byte offset of an interior pointer in its allocation (the
    import side needs another process: tests/test_gpu_pipeline_ipc.py)."""
    from paper_2005_13014_b200 import oec

    f = oec.oec_field_create((64, 8, 2), (0, 0, 0), (0, 0, 0))
    h, off = oec.oec_ipc_export(f.desc.data)
    assert len(h) == 64 and 0 <= off < 4096  # the library may place data after a small pad
    h2, off2 = oec.oec_ipc_export(f.desc.data + 8 * 40)
    assert off2 == off + 320 and h2 == h
