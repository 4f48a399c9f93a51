"""Helpers shared by the GPU parity tests: run a program through the C-ABI on the GPU, run the
oracle on the same seeded inputs, compare element by element."""
from __future__ import annotations

import numpy as np

import synth
from oracle import capi
from oracle import stencil as st
from oracle import suite
from synth import HostField

SENTINEL = 12345.0


def run_gpu(program, host, domain, order=None, dom_lb=(0, 0, 0), dom_ub=None, variant=0, out_halo=(0, 0, 0),
            scalars=None, stream=None):
    """Upload `host` inputs into library-created fields (oec_field_create), allocate outputs over
    the domain grown by out_halo filled with SENTINEL, apply, return {output: HostField}."""
    import torch

    from paper_2005_13014_b200 import oec

    dom_ub = dom_ub or domain
    spec = synth.PROGRAMS[program]
    ins = [oec.field_from_host(host[s.name], order=order) for s in spec.inputs]
    dt = host[spec.inputs[0].name].data.dtype
    outs = [oec.oec_field_create(domain, out_halo, out_halo, order=order, dtype=dt).fill(SENTINEL) for _ in spec.outputs]
    sc = scalars if scalars is not None else [v for _, v in spec.scalars]
    oec.oec_apply_program(program, ins, outs, sc, dom_lb, dom_ub, variant, stream)
    torch.cuda.synchronize()
    res = {}
    for name, f in zip(spec.outputs, outs):
        res[name] = HostField(f.download(), f.lb, f.ub)
    return res


def run_oracle(program, host, domain, dom_lb=(0, 0, 0), dom_ub=None, scalars=None, nthreads=0):
    """Oracle outputs over the domain (arrays [k][j][i] covering [dom_lb, dom_ub))."""
    dom_ub = dom_ub or domain
    ni, nj, nk = (dom_ub[d] - dom_lb[d] for d in range(3))
    spec = synth.PROGRAMS[program]
    sc = dict(zip([n for n, _ in spec.scalars], scalars)) if scalars is not None else synth.scalars(program)
    dt = host[spec.inputs[0].name].data.dtype
    if program == "hdiff":
        o = HostField(np.full((nk, nj, ni), np.nan, dtype=dt), tuple(dom_lb), tuple(dom_ub))
        capi.hdiff(host["in"], host["coeff"], o, dom_lb, dom_ub, capi.HDIFF_UNFUSED, nthreads)
        return {"out": o.data}
    if program == "vadv":
        o = HostField(np.full((nk, nj, ni), np.nan, dtype=dt), tuple(dom_lb), tuple(dom_ub))
        capi.vadv(host, o, sc["dtr_stage"], dom_lb, dom_ub, capi.VADV_UNFUSED, nthreads)
        return {"utens_stage_out": o.data}
    r = st.run_unfused(suite.PROGRAMS[program], host, sc, dom_lb, dom_ub)
    return {k: v.data for k, v in r.items()}


def domain_part(f: HostField, lo, hi):
    return f.data[lo[2] - f.lb[2]:hi[2] - f.lb[2], lo[1] - f.lb[1]:hi[1] - f.lb[1], lo[0] - f.lb[0]:hi[0] - f.lb[0]]


def outside_mask(f: HostField, lo, hi):
    m = np.ones(f.data.shape, bool)
    m[lo[2] - f.lb[2]:hi[2] - f.lb[2], lo[1] - f.lb[1]:hi[1] - f.lb[1], lo[0] - f.lb[0]:hi[0] - f.lb[0]] = False
    return m


def compare(gpu: np.ndarray, ref: np.ndarray):
    """Parity statistics: the gate is the per-element max relative error over
    r != 0 (<= 1e-12, north_star); we also report the normwise error and the bitwise count."""
    assert gpu.shape == ref.shape
    nz = ref != 0
    rel = np.max(np.abs(gpu[nz] - ref[nz]) / np.abs(ref[nz])) if nz.any() else 0.0
    zero_ok = np.all(gpu[~nz] == 0) if (~nz).any() else True
    norm = np.max(np.abs(gpu - ref)) / max(np.max(np.abs(ref)), 1e-300)
    assert gpu.dtype == ref.dtype, (gpu.dtype, ref.dtype)
    u = np.uint64 if gpu.dtype.itemsize == 8 else np.uint32
    nbits = int(np.sum(gpu.view(u) != ref.view(u)))
    return dict(max_rel=float(rel), zero_ok=bool(zero_ok), normwise=float(norm), n_bitdiff=nbits, n=gpu.size)
