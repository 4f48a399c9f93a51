"""Dependent launches: every launch reads what the previous launch wrote.

The kernels start before their predecessor ends (programmatic dependent launch), warm L2 with their
first tiles/chunks before `griddepcontrol.wait`, and vadv's single-wave grids release the next
launch late while that launch's early CTAs prefetch the first chunks of every block (DESIGN.md
§7.1, §7.2).  None of that may let a launch see its input before the previous launch finished
writing it: T chained steps on one stream -- eagerly and replayed from a CUDA graph, the bench's
mode -- must equal T oracle applications bit for bit.  Fields ping-pong between two allocations
(an output never aliases an input of the same launch).

Power check (round 2): a mutation build without `griddepcontrol.wait` (`-DOEC_MUTATE_NO_GRIDDEP_WAIT`,
csrc/tma.h) fails 4 of these tests -- the graph-replayed vadv chains at 128^2, 64^2 and 33x31x5 and
the hdiff chain at 200x70x9 (126000 of 126000 points differ); eager launches are separated by the
Python call overhead and pass.  The product build passes all of them."""
import numpy as np
import pytest

import synth
from gpu_util import compare, run_oracle
from synth import HostField

pytestmark = pytest.mark.gpu

T = 5


def _oracle_chain(program, host, domain, chained):
    """T applications of the oracle, the output of step t feeding input `chained` of step t+1
    (its halo, if any, stays the caller's initial data)."""
    h = dict(host)
    out_name = synth.PROGRAMS[program].outputs[0]
    for _ in range(T):
        r = run_oracle(program, h, domain)[out_name]
        f = h[chained].copy()
        lb = f.lb
        f.data[-lb[2]:-lb[2] + domain[2], -lb[1]:-lb[1] + domain[1], -lb[0]:-lb[0] + domain[0]] = r
        h[chained] = f
    return r


def _gpu_chain(program, host, domain, chained, graph, dtype=np.float64):
    import torch

    from paper_2005_13014_b200 import oec

    spec = synth.PROGRAMS[program]
    fixed = {s.name: oec.field_from_host(host[s.name]) for s in spec.inputs if s.name != chained}
    # both ping-pong fields start as the chained input (halo included: caller data, never written)
    ab = [oec.field_from_host(host[chained]), oec.field_from_host(host[chained])]
    sc = [v for _, v in spec.scalars]

    def step(t):
        src, dst = ab[t % 2], ab[(t + 1) % 2]
        ins = [src if s.name == chained else fixed[s.name] for s in spec.inputs]
        oec.oec_apply_program(program, ins, [dst], sc, (0, 0, 0), domain, 0, torch.cuda.current_stream().cuda_stream)

    if graph:
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        # first call outside the capture (one-time setup: tensor maps, function attributes)
        warm = [oec.field_from_host(host[chained]), oec.empty_like_domain(domain, dtype=dtype)]
        ins = [warm[0] if s_.name == chained else fixed[s_.name] for s_ in spec.inputs]
        oec.oec_apply_program(program, ins, [warm[1]], sc, (0, 0, 0), domain, 0, None)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for t in range(T):
                step(t)
        g.replay()
    else:
        for t in range(T):
            step(t)
    torch.cuda.synchronize()
    f = ab[T % 2]
    d = f.download()
    lb = f.lb
    return d[-lb[2]:-lb[2] + domain[2], -lb[1]:-lb[1] + domain[1], -lb[0]:-lb[0] + domain[0]]


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("domain", [(128, 128, 80), (64, 64, 80), (256, 256, 60), (33, 31, 5)])
def test_vadv_chain(domain, graph):
    # u_stage of step t+1 = utens_stage_out of step t: read at k and k+1 from the TMA ring and by
    # the L2 prefetches (128^2 and 64^2: the late-trigger grid; 256^2 x 60: persistent blocks)
    host = synth.make_inputs("vadv", domain, seed=7)
    g = _gpu_chain("vadv", host, domain, "u_stage", graph)
    r = _oracle_chain("vadv", host, domain, "u_stage")
    c = compare(g, r)
    assert c["n_bitdiff"] == 0 and not np.isnan(g).any(), (domain, graph, c)


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("domain", [(128, 128, 80), (200, 70, 9)])
def test_hdiff_chain(domain, graph):
    # in of step t+1 = out of step t on the domain (the 2-wide halo keeps the caller's data)
    host = synth.make_inputs("hdiff", domain, seed=8)
    g = _gpu_chain("hdiff", host, domain, "in", graph)
    r = _oracle_chain("hdiff", host, domain, "in")
    c = compare(g, r)
    assert c["n_bitdiff"] == 0 and not np.isnan(g).any(), (domain, graph, c)


@pytest.mark.parametrize("graph", [False, True])
def test_hdiff_vadv_alternating(graph):
    # hdiff and vadv alternate and feed each other: hdiff's out is vadv's u_stage, vadv's output is
    # the next hdiff's in (domain part; the halo stays the initial data)
    import torch

    from paper_2005_13014_b200 import oec

    domain = (128, 128, 80)
    hh = synth.make_inputs("hdiff", domain, seed=9)
    hv = synth.make_inputs("vadv", domain, seed=9)
    vs = synth.PROGRAMS["vadv"]
    x = oec.field_from_host(hh["in"])  # hdiff input, halo 2
    cf = oec.field_from_host(hh["coeff"])
    u = oec.empty_like_domain(domain)  # hdiff out = vadv u_stage
    fixed = {s.name: oec.field_from_host(hv[s.name]) for s in vs.inputs if s.name != "u_stage"}
    y = oec.empty_like_domain(domain)  # vadv out
    dtr = [v for _, v in vs.scalars]

    def launch():
        st = torch.cuda.current_stream().cuda_stream
        for _ in range(3):
            oec.oec_apply_program("hdiff", [x, cf], [u], None, (0, 0, 0), domain, 0, st)
            oec.oec_apply_program("vadv", [u if s.name == "u_stage" else fixed[s.name] for s in vs.inputs], [y], dtr,
                                  (0, 0, 0), domain, 0, st)
            # next hdiff input: the domain of x <- y (halo untouched), a device copy on the stream
            x.view()[:, 2:-2, 2:-2].copy_(y.view())

    if graph:
        launch_once = oec.field_from_host(hh["in"])  # warm-up on throwaway fields
        oec.oec_apply_program("hdiff", [launch_once, cf], [oec.empty_like_domain(domain)], None, (0, 0, 0), domain, 0, None)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=torch.cuda.Stream()):
            launch()
        g.replay()
    else:
        launch()
    torch.cuda.synchronize()

    h = dict(hh)
    v = dict(hv)
    for _ in range(3):
        uo = run_oracle("hdiff", h, domain)["out"]
        v["u_stage"] = HostField(uo.copy(), (0, 0, 0), domain)
        yo = run_oracle("vadv", v, domain)["utens_stage_out"]
        f = h["in"].copy()
        f.data[:, 2:-2, 2:-2] = yo
        h["in"] = f
    assert compare(y.download(), yo)["n_bitdiff"] == 0, graph


@pytest.mark.parametrize("program,chained", [("hdiff", "in"), ("vadv", "u_stage")])
def test_f32_chain(program, chained):
    # binary32: hdiff's 8-warp tier and vadv_sp<float> in graph-replayed chains
    domain = (128, 128, 80)
    host = synth.make_inputs(program, domain, seed=10, dtype=np.float32)
    g = _gpu_chain(program, host, domain, chained, True, dtype=np.float32)
    r = _oracle_chain(program, host, domain, chained)
    c = compare(g, r)
    assert c["n_bitdiff"] == 0 and not np.isnan(g).any(), (program, c)
