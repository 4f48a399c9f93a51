"""GPU parity of liboec's stencil-language JIT (csrc/jit.cpp) through the C-ABI.

Every program text (tests/programs/*.oec: hdiff and the whole suite) and 40 seeded random programs
are compiled by liboec (parse, shape inference, inlining / unrolling / original level, NVRTC for
sm_100a) and run on the GPU; results must equal the oracle (oracle/dsl.py evaluated by
oracle/stencil.py, the "original" level of P:616) BIT FOR BIT in f64 and f32, and equal the
hand-written builtin kernels.  Output halos are sentinel-filled and must stay untouched.
"""
from __future__ import annotations

import glob
import os

import numpy as np
import pytest

import synth
from gpu_util import SENTINEL, compare, domain_part, outside_mask, run_gpu
from jit_programs import make_inputs as rnd_inputs, random_program, touched_boxes
from oracle import dsl, stencil
from synth import HostField

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "programs", "*.oec")))


def _oec():
    from paper_2005_13014_b200 import oec

    return oec


VARIANTS = [0, 1, 2, 3, 4, 5, 6, 7]  # AUTO (tuned), UNFUSED (original), NAIVE (inline), UNROLL2/4 (j), UNROLL2/4_K, TILED


def text_of(program):
    with open(os.path.join(HERE, "programs", program + ".oec")) as f:
        return f.read()


_registered = {}


def registered(text):
    oec = _oec()
    tp = dsl.parse(text)
    if tp.name not in _registered:
        _registered[tp.name] = oec.oec_program_create(text)
    return _registered[tp.name]


def run_jit(name, tp, host, domain, variant, dom_lb=(0, 0, 0), dom_ub=None, out_halo=(1, 1, 0), scalars=None):
    import torch

    oec = _oec()
    dom_ub = dom_ub or domain
    dt = host[tp.inputs[0]].data.dtype
    ins = [oec.field_from_host(host[n]) for n in tp.inputs]
    outs = [oec.oec_field_create(domain, out_halo, out_halo, dtype=dt).fill(SENTINEL) for _ in tp.outputs]
    sc = [v for _, v in tp.scalars] if scalars is None else scalars
    oec.oec_apply_program(name, ins, outs, sc, dom_lb, dom_ub, variant)
    n_launch = oec.oec_last_launch_count()
    torch.cuda.synchronize()
    return {o: HostField(f.download(), f.lb, f.ub) for o, f in zip(tp.outputs, outs)}, n_launch


def oracle(tp, host, dom_lb, dom_ub, scalars=None):
    sc = tp.scalar_values(scalars)
    r = stencil.run_unfused(tp.program, host, sc, dom_lb, dom_ub)
    return {o: r[o].data for o in tp.outputs}


def check(got, ref, dom_lb, dom_ub):
    for o, f in got.items():
        part = domain_part(f, dom_lb, dom_ub)
        st = compare(part, ref[o])
        assert st["n_bitdiff"] == 0 and st["max_rel"] <= 1e-12, (o, st)
        assert np.all(f.data[outside_mask(f, dom_lb, dom_ub)] == SENTINEL), f"{o}: write outside the domain"


@pytest.mark.parametrize("program", NAMES)
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_text_programs_bit_identical(program, variant, dtype):
    name = registered(text_of(program))
    tp = dsl.parse(text_of(program), dtype)
    domain = (33, 19, 5)
    host = synth.make_inputs(program, domain, seed=1, dtype=dtype)
    got, n_launch = run_jit(name, tp, host, domain, variant)
    check(got, oracle(tp, host, (0, 0, 0), domain), (0, 0, 0), domain)
    if variant >= 2:
        assert n_launch == 1
    elif variant == 1:
        assert n_launch == len(tp.program.applies)  # one kernel per (live) stencil.apply


@pytest.mark.parametrize("program", NAMES)
@pytest.mark.parametrize("domain", [(128, 128, 80), (200, 70, 9)])
def test_tiled_variant_large_and_ragged(program, domain):
    """OEC_VARIANT_TILED over many items per CTA (128x128x80) and ragged tiles (200 = 3x64 + 8,
    70 = 8x8 + 6), bit-identical to the oracle."""
    name = registered(text_of(program))
    tp = dsl.parse(text_of(program))
    host = synth.make_inputs(program, domain, seed=11)
    got, n = run_jit(name, tp, host, domain, 7)
    assert n == 1
    check(got, oracle(tp, host, (0, 0, 0), domain), (0, 0, 0), domain)


@pytest.mark.parametrize("program", NAMES)
def test_text_programs_equal_builtin_kernels(program):
    """JIT of the language version == the hand-written B200 kernel (AUTO) at 128x128x80 (configs[2])."""
    name = registered(text_of(program))
    tp = dsl.parse(text_of(program))
    domain = (128, 128, 80)
    host = synth.make_inputs(program, domain, seed=0)
    got, _ = run_jit(name, tp, host, domain, 0, out_halo=(0, 0, 0))
    ref = run_gpu(program, host, domain)
    for o in tp.outputs:
        assert np.array_equal(got[o].data, ref[o].data), o


@pytest.mark.parametrize("seed", range(40))
def test_random_programs_bit_identical(seed):
    text = random_program(seed)
    tp = dsl.parse(text)
    domain = (13, 11, 4)
    ext = touched_boxes(tp, domain)  # allocation from the ORACLE's brute-force trace
    host = rnd_inputs(tp, domain, ext, seed=seed)
    name = registered(text)
    ref = oracle(tp, host, (0, 0, 0), domain)
    for variant in (1, 2, 3, 4, 5, 6, 7, 0):
        try:
            got, _ = run_jit(name, tp, host, domain, variant)
        except Exception as e:  # TILED: boxes of very wide extents may not fit shared memory
            assert variant == 7 and getattr(e, "status", None) == 7, e
            continue
        check(got, ref, (0, 0, 0), domain)


def test_random_programs_f32():
    for seed in range(40, 50):
        text = random_program(seed)
        tp = dsl.parse(text, np.float32)
        domain = (9, 7, 3)
        ext = touched_boxes(tp, domain)
        host = rnd_inputs(tp, domain, ext, seed=seed, dtype=np.float32)
        name = registered(text)
        ref = oracle(tp, host, (0, 0, 0), domain)
        for variant in (1, 2, 4, 6, 7):
            try:
                got, _ = run_jit(name, tp, host, domain, variant)
            except Exception as e:
                assert variant == 7 and getattr(e, "status", None) == 7, e
                continue
            check(got, ref, (0, 0, 0), domain)


def test_sub_domain_and_scalars():
    program = "p_grad_c"
    name = registered(text_of(program))
    tp = dsl.parse(text_of(program))
    domain = (40, 30, 6)
    host = synth.make_inputs(program, domain, seed=5)
    lo, hi = (3, 2, 1), (37, 29, 5)
    got, _ = run_jit(name, tp, host, domain, 2, dom_lb=lo, dom_ub=hi, scalars=[0.37])
    check(got, oracle(tp, host, lo, hi, {"dt2": 0.37}), lo, hi)


def test_host_fields_end_to_end():
    """OEC_DEVICE_HOST fields: the library stages them (the e2e path) for JIT programs too."""
    oec = _oec()
    program = "fastwaves"
    name = registered(text_of(program))
    tp = dsl.parse(text_of(program))
    domain = (20, 12, 7)
    host = synth.make_inputs(program, domain, seed=2)
    ins = [oec.oec_field_wrap(host[n].data, host[n].lb, host[n].ub, k_invariant=host[n].k_invariant) for n in tp.inputs]
    outs_np = [np.full((domain[2], domain[1], domain[0]), np.nan) for _ in tp.outputs]
    outs = [oec.oec_field_wrap(a, (0, 0, 0), domain) for a in outs_np]
    oec.oec_apply_program(name, ins, outs, None, (0, 0, 0), domain, 0)
    ref = oracle(tp, host, (0, 0, 0), domain)
    for o, a in zip(tp.outputs, outs_np):
        assert np.array_equal(a, ref[o])


def test_graph_capture_after_first_compile():
    import torch

    oec = _oec()
    program = "uvbke"
    name = registered(text_of(program))
    tp = dsl.parse(text_of(program))
    domain = (64, 32, 8)
    host = synth.make_inputs(program, domain, seed=3)
    ins = [oec.field_from_host(host[n]) for n in tp.inputs]
    outs = [oec.oec_field_create(domain, (0, 0, 0), (0, 0, 0)).fill(SENTINEL) for _ in tp.outputs]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        oec.oec_apply_program(name, ins, outs, None, (0, 0, 0), domain, 0)  # compiles + caches
    torch.cuda.synchronize()
    for f in outs:
        f.fill(SENTINEL)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        oec.oec_apply_program(name, ins, outs, None, (0, 0, 0), domain, 0)
    g.replay()
    torch.cuda.synchronize()
    ref = oracle(tp, host, (0, 0, 0), domain)
    for o, f in zip(tp.outputs, outs):
        assert np.array_equal(f.download(), ref[o])


def test_auto_tuning_is_cached_and_bit_identical():
    """AUTO = empirical tuning: the first call times the inline / unrolled / tiled variants
    on R rotating copies of the fields (3 rounds of 2R launches each after one warm-up launch on the
    caller's fields) and then runs the choice on the caller's fields; later calls launch the cached
    choice once."""
    program = "nh_p_grad"
    name = registered(text_of(program))
    tp = dsl.parse(text_of(program))
    domain = (64, 48, 16)
    host = synth.make_inputs(program, domain, seed=7)
    ref = oracle(tp, host, (0, 0, 0), domain)
    got, n1 = run_jit(name, tp, host, domain, 0)
    check(got, ref, (0, 0, 0), domain)
    # 9 candidates (5 + 4 tiled configurations) x (1 warm-up + 3 x 2R timed) + the final launch,
    # 2 <= R <= 8 rotating copies (a small domain: R = 8)
    R = (n1 - 1 - 9) // (9 * 6)
    assert n1 == 9 * (1 + 6 * R) + 1 and 2 <= R <= 8, n1
    got, n2 = run_jit(name, tp, host, domain, 0)
    check(got, ref, (0, 0, 0), domain)
    assert n2 == 1


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
@pytest.mark.parametrize("program", ["hdiff", "nh_p_grad", "fvtp2d_qj", "fastwaves"])
def test_tiled_configurations(program, cfg, monkeypatch):
    """Every tiled configuration AUTO may pick (rows per thread x ring budget), ragged domain."""
    monkeypatch.setenv("OEC_JIT_TILE_CFG", str(cfg))
    name = registered(text_of(program))
    tp = dsl.parse(text_of(program))
    domain = (200, 70, 9)
    host = synth.make_inputs(program, domain, seed=cfg)
    got, _ = run_jit(name, tp, host, domain, 7)
    check(got, oracle(tp, host, (0, 0, 0), domain), (0, 0, 0), domain)


def test_first_auto_call_inside_capture():
    """No tuning or compilation inside a stream capture: a builtin suite program's first AUTO call
    on a new shape inside a capture runs its hand-written kernel (bit-identical); a text program
    raises OEC_ERR_UNSUPPORTED until it has been called once outside the capture."""
    import torch

    oec = _oec()
    program = "p_grad_c"
    domain = (72, 40, 6)  # a shape no other test tunes
    host = synth.make_inputs(program, domain, seed=9)
    ins = [oec.field_from_host(host[s.name]) for s in synth.PROGRAMS[program].inputs]
    outs = [oec.oec_field_create(domain, (0, 0, 0), (0, 0, 0)).fill(SENTINEL) for _ in synth.PROGRAMS[program].outputs]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        oec.oec_apply_program(program, ins, outs, [0.1125], (0, 0, 0), domain, 0)
    g.replay()
    torch.cuda.synchronize()
    ref = run_gpu(program, host, domain, variant=2)  # hand-written inline kernel, outside capture
    for o, f in zip(synth.PROGRAMS[program].outputs, outs):
        assert np.array_equal(f.download(), ref[o].data)
    # a text program's first AUTO call inside a capture
    name = registered(text_of("uvbke"))
    domain2 = (40, 24, 3)
    h2 = synth.make_inputs("uvbke", domain2, seed=1)
    ins2 = [oec.field_from_host(h2[s.name]) for s in synth.PROGRAMS["uvbke"].inputs]
    outs2 = [oec.oec_field_create(domain2, (0, 0, 0), (0, 0, 0)) for _ in range(2)]
    g2 = torch.cuda.CUDAGraph()
    with pytest.raises(oec.OecError) as ei:
        with torch.cuda.graph(g2, stream=s):
            oec.oec_apply_program(name, ins2, outs2, None, (0, 0, 0), domain2, 0)
    assert ei.value.status == 7


def test_odd_pitch_torch_fields_auto():
    """Torch-wrapped fields with an odd row pitch (not describable to TMA): AUTO tunes over the
    non-TMA kernels only, the explicit tiled variant reports OEC_ERR_LAYOUT; results bit-identical."""
    import torch

    oec = _oec()
    program = "nh_p_grad"
    name = registered(text_of(program))
    tp = dsl.parse(text_of(program))
    domain = (37, 21, 5)
    host = synth.make_inputs(program, domain, seed=13)
    ins = []
    for n in tp.inputs:
        h = host[n]
        shp = h.data.shape
        t = torch.full((shp[0], shp[1], shp[2] + 3), float("nan"), dtype=torch.float64, device="cuda")[:, :, 1:1 + shp[2]]
        t.copy_(torch.from_numpy(h.data))
        ins.append(oec.oec_field_wrap(t, h.lb, h.ub, k_invariant=h.k_invariant))
    outs = [oec.oec_field_create(domain, (0, 0, 0), (0, 0, 0)).fill(SENTINEL) for _ in tp.outputs]
    oec.oec_apply_program(name, ins, outs, None, (0, 0, 0), domain, 0)
    torch.cuda.synchronize()
    ref = oracle(tp, host, (0, 0, 0), domain)
    for o, f in zip(tp.outputs, outs):
        assert np.array_equal(f.download(), ref[o])
    with pytest.raises(oec.OecError) as ei:
        oec.oec_apply_program(name, ins, outs, None, (0, 0, 0), domain, 7)
    assert ei.value.status == 8
