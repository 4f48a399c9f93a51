"""GPU test of the decomposition + halo exchange executed by liboec's kernels on ONE device
(oec_halo_exchange_local: every rank's sub-domain fields live on cuda:0 and the plan's boxes are
moved by device-to-device copy kernels).  Decomposed GPU hdiff / vadv must equal the global GPU
result and the oracle bit for bit, corners included (SURVEY §8(c) "decomposed GPU == 1-GPU")."""
import numpy as np
import pytest

import synth
from gpu_util import run_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("program,gdom,px,py,w", [
    ("hdiff", (70, 66, 5), 1, 4, ((2, 2, 0), (2, 2, 0))),
    ("hdiff", (67, 45, 3), 2, 2, ((2, 2, 0), (2, 2, 0))),
    ("hdiff", (129, 40, 4), 4, 2, ((2, 2, 0), (2, 2, 0))),
    ("vadv", (130, 20, 12), 2, 1, ((0, 0, 0), (1, 0, 0))),
])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_local_exchange_matches_global(program, gdom, px, py, w, dtype):
    import torch

    from paper_2005_13014_b200 import oec

    wlo, whi = w
    host = synth.make_inputs(program, gdom, seed=9, dtype=dtype)
    spec = synth.PROGRAMS[program]
    R = px * py
    decs = [oec.oec_decomp_create(gdom, px, py, r) for r in range(R)]
    exch = [s for s in spec.inputs if all(s.halo_lo[d] >= wlo[d] and s.halo_hi[d] >= whi[d] for d in (0, 1))]
    fields, outs = [], []
    for r, dec in enumerate(decs):
        lo, hi = dec.local_lb, dec.local_ub
        ldom = tuple(hi[d] - lo[d] for d in range(3))
        rank_fields = {}
        for s in spec.inputs:
            g = host[s.name]
            f = oec.oec_field_create(ldom, s.halo_lo, s.halo_hi, dtype=dtype)
            v = f.view()  # [k][j][i] over the local allocation
            v.fill_(float("nan"))
            # own interior + global outer halo (caller data) from the global field
            gl = [max(f.lb[d] + lo[d], g.lb[d]) for d in range(2)]
            gh = [min(f.ub[d] + lo[d], g.ub[d]) for d in range(2)]
            src = g.data[:, gl[1] - g.lb[1]:gh[1] - g.lb[1], gl[0] - g.lb[0]:gh[0] - g.lb[0]].copy()
            jj, ii = np.meshgrid(np.arange(gl[1], gh[1]), np.arange(gl[0], gh[0]), indexing="ij")
            own = (ii >= lo[0]) & (ii < hi[0]) & (jj >= lo[1]) & (jj < hi[1])
            outside = (ii < 0) | (ii >= gdom[0]) | (jj < 0) | (jj >= gdom[1])
            src[:, ~(own | outside)] = np.nan
            v[:, gl[1] - lo[1] - f.lb[1]:gh[1] - lo[1] - f.lb[1], gl[0] - lo[0] - f.lb[0]:gh[0] - lo[0] - f.lb[0]] = \
                torch.from_numpy(src)
            rank_fields[s.name] = f
        fields.append(rank_fields)
    flat = [fields[r][s.name] for r in range(R) for s in exch]
    oec.oec_halo_exchange_local(gdom, px, py, flat, len(exch), wlo, whi)
    sc = [v for _, v in spec.scalars]
    for r, dec in enumerate(decs):
        ldom = tuple(dec.local_ub[d] - dec.local_lb[d] for d in range(3))
        out = oec.empty_like_domain(ldom, dtype=dtype)
        oec.oec_apply_program(program, [fields[r][s.name] for s in spec.inputs], [out], sc, (0, 0, 0), ldom)
        outs.append(out)
    torch.cuda.synchronize()
    ref = run_oracle(program, host, gdom)[spec.outputs[0]]
    for r, dec in enumerate(decs):
        lo, hi = dec.local_lb, dec.local_ub
        got = outs[r].download()
        assert np.array_equal(got, ref[:, lo[1]:hi[1], lo[0]:hi[0]]), (program, r)


def _rank_fields(oec, torch, host, spec, gdom, lo, hi, dtype, order):
    """Sub-domain fields of one rank: own interior + global outer halo from the global field, NaN
    in the halo cells that the exchange must fill."""
    ldom = tuple(hi[d] - lo[d] for d in range(3))
    out = {}
    for s in spec.inputs:
        g = host[s.name]
        f = oec.oec_field_create(ldom if not s.k_invariant else (ldom[0], ldom[1], 1), s.halo_lo, s.halo_hi,
                                 dtype=dtype, order=order, k_invariant=s.k_invariant)
        v = f.view()
        v.fill_(float("nan"))
        gl = [max(f.lb[d] + lo[d], g.lb[d]) for d in range(2)]
        gh = [min(f.ub[d] + lo[d], g.ub[d]) for d in range(2)]
        src = g.data[:, gl[1] - g.lb[1]:gh[1] - g.lb[1], gl[0] - g.lb[0]:gh[0] - g.lb[0]].copy()
        jj, ii = np.meshgrid(np.arange(gl[1], gh[1]), np.arange(gl[0], gh[0]), indexing="ij")
        own = (ii >= lo[0]) & (ii < hi[0]) & (jj >= lo[1]) & (jj < hi[1])
        outside = (ii < 0) | (ii >= gdom[0]) | (jj < 0) | (jj >= gdom[1])
        src[:, ~(own | outside)] = np.nan
        v[:, gl[1] - lo[1] - f.lb[1]:gh[1] - lo[1] - f.lb[1], gl[0] - lo[0] - f.lb[0]:gh[0] - lo[0] - f.lb[0]] = \
            torch.from_numpy(src)
        out[s.name] = f
    return out


@pytest.mark.parametrize("order", [None, (0, 1, 2)])  # i,k,j: direct spans (no pack); i,j,k: packed boxes
@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
def test_local_exchange_per_input_extents(program, order):
    # j-slabs (the bench's decomposition): every input's halo exchanged with ITS OWN access extent
    # (k-invariant metric fields included), as bench.py --config c3 / c5 does per program; then the
    # program on each rank's sub-domain == the global oracle, bit for bit
    import torch

    from paper_2005_13014_b200 import oec

    gdom, px, py = (40, 23, 4), 1, 3
    host = synth.make_inputs(program, gdom, seed=17)
    spec = synth.PROGRAMS[program]
    decs = [oec.oec_decomp_create(gdom, px, py, r) for r in range(px * py)]
    fields = [_rank_fields(oec, torch, host, spec, gdom, d.local_lb, d.local_ub, np.float64, order) for d in decs]
    groups = {}
    for s in spec.inputs:
        w = ((0, s.halo_lo[1], 0), (0, s.halo_hi[1], 0))
        if w != ((0, 0, 0), (0, 0, 0)):
            groups.setdefault(w, []).append(s.name)
    for (wlo, whi), names in groups.items():
        flat = [fields[r][nm] for r in range(len(decs)) for nm in names]
        oec.oec_halo_exchange_local(gdom, px, py, flat, len(names), wlo, whi)
    ref = run_oracle(program, host, gdom)
    sc = [v for _, v in spec.scalars]
    for r, dec in enumerate(decs):
        lo, hi = dec.local_lb, dec.local_ub
        ldom = tuple(hi[d] - lo[d] for d in range(3))
        outs = [oec.empty_like_domain(ldom) for _ in spec.outputs]
        oec.oec_apply_program(program, [fields[r][s.name] for s in spec.inputs], outs, sc, (0, 0, 0), ldom)
        torch.cuda.synchronize()
        for name, o in zip(spec.outputs, outs):
            assert np.array_equal(o.download(), ref[name][:, lo[1]:hi[1], lo[0]:hi[0]]), (program, name, r, order)


def test_local_exchange_inside_cuda_graph():
    # the exchange's stream-ordered staging is capturable: a graph replay exchanges again
    import torch

    from paper_2005_13014_b200 import oec

    gdom, px, py = (35, 30, 3), 2, 2  # 2x2: packed boxes (staging) in both phases
    host = synth.make_inputs("hdiff", gdom, seed=18)
    spec = synth.PROGRAMS["hdiff"]
    decs = [oec.oec_decomp_create(gdom, px, py, r) for r in range(px * py)]
    fields = [_rank_fields(oec, torch, host, spec, gdom, d.local_lb, d.local_ub, np.float64, None) for d in decs]
    flat = [fields[r]["in"] for r in range(len(decs))]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        oec.oec_halo_exchange_local(gdom, px, py, flat, 1, (2, 2, 0), (2, 2, 0))
    g.replay()
    torch.cuda.synchronize()
    ref = run_oracle("hdiff", host, gdom)["out"]
    for r, dec in enumerate(decs):
        lo, hi = dec.local_lb, dec.local_ub
        ldom = tuple(hi[d] - lo[d] for d in range(3))
        out = oec.empty_like_domain(ldom)
        oec.oec_hdiff(fields[r]["in"], fields[r]["coeff"], out, (0, 0, 0), ldom)
        torch.cuda.synchronize()
        assert np.array_equal(out.download(), ref[:, lo[1]:hi[1], lo[0]:hi[0]]), r
