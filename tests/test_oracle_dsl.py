"""Pins of the oracle's stencil-language reader (oracle/dsl.py) -- no GPU.

The reader is pinned against the hand-written oracle programs, which are themselves pinned
(test_oracle_hdiff.py, test_oracle_suite.py): the language versions of hdiff and of the whole
suite (tests/programs/*.oec) must give bit-identical results in f64 and f32 and the same Table II
census, and hdiff must also equal the plain-C oracle.  Precedence / associativity /
select / min / max semantics are pinned by closed forms; malformed programs are rejected.
"""
from __future__ import annotations

import glob
import os

import numpy as np
import pytest

import synth
from oracle import capi, dsl, stencil, suite
from synth import HostField

HERE = os.path.dirname(os.path.abspath(__file__))
PROGRAM_FILES = sorted(glob.glob(os.path.join(HERE, "programs", "*.oec")))
NAMES = [os.path.basename(p)[:-4] for p in PROGRAM_FILES]


def text_of(program):
    with open(os.path.join(HERE, "programs", program + ".oec")) as f:
        return f.read()


@pytest.mark.parametrize("program", NAMES)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_text_program_equals_handwritten_oracle(program, dtype):
    tp = dsl.parse(text_of(program), dtype)
    ref = suite.PROGRAMS[program]
    dom = (11, 9, 4)
    for seed in (0, 1):
        f = synth.make_inputs(program, dom, seed=seed, dtype=dtype)
        sc = synth.scalars(program)
        a = stencil.run_unfused(tp.program, f, sc, (0, 0, 0), dom)
        b = stencil.run_unfused(ref, f, sc, (0, 0, 0), dom)
        assert tp.outputs == [o for o, _ in ref.outputs]
        for o in tp.outputs:
            assert a[o].data.dtype == dtype
            assert np.array_equal(a[o].data, b[o].data), (program, o)


@pytest.mark.parametrize("program", NAMES)
def test_text_program_census_equals_handwritten(program):
    tp = dsl.parse(text_of(program))
    assert stencil.census(tp.program) == stencil.census(suite.PROGRAMS[program])


@pytest.mark.parametrize("program", sorted(suite.TABLE_II))
def test_text_program_table_ii(program):
    dims, applies, n_in, n_out, arith, access, cf = suite.TABLE_II[program]
    c = stencil.census(dsl.parse(text_of(program)).program)
    assert (c["applies"], c["inputs"], c["outputs"]) == (applies, n_in, n_out)
    assert (c["if"] > 0) == cf
    assert (c["arith"] + c["cmp"], c["access"]) == (arith, access)  # exact rows (R12, R15)


def test_text_hdiff_equals_c_oracle():
    tp = dsl.parse(text_of("hdiff"))
    dom = (17, 13, 3)
    f = synth.make_inputs("hdiff", dom, seed=4)
    a = stencil.run_unfused(tp.program, f, {}, (0, 0, 0), dom)
    o = HostField(np.full((dom[2], dom[1], dom[0]), np.nan), (0, 0, 0), dom)
    capi.hdiff(f["in"], f["coeff"], o, (0, 0, 0), dom)
    assert np.array_equal(a["out"].data, o.data)


def test_fused_equals_unfused_for_text_programs():
    for program in NAMES:
        tp = dsl.parse(text_of(program))
        dom = (5, 4, 3)
        f = synth.make_inputs(program, dom, seed=3)
        sc = synth.scalars(program)
        a = stencil.run_unfused(tp.program, f, sc, (0, 0, 0), dom)
        b, _ = stencil.run_fused(tp.program, f, sc, (0, 0, 0), dom)
        for o in tp.outputs:
            got = np.array([[[b[o][(i, j, k)] for i in range(dom[0])] for j in range(dom[1])] for k in range(dom[2])])
            assert np.array_equal(got, a[o].data), (program, o)


@pytest.mark.parametrize("seed", range(30))
def test_random_programs_fused_equals_unfused(seed):
    """The oracle's two evaluators (materialised temporaries vs per-point inlining) agree bit for
    bit on random language programs (f64 and f32), on inputs allocated from the brute-force trace."""
    from jit_programs import make_inputs, random_program, touched_boxes

    for dtype in (np.float64, np.float32):
        tp = dsl.parse(random_program(seed), dtype)
        dom = (6, 5, 3)
        host = make_inputs(tp, dom, touched_boxes(tp, dom), seed=seed, dtype=dtype)
        a = stencil.run_unfused(tp.program, host, tp.scalar_values(), (0, 0, 0), dom)
        b, _ = stencil.run_fused(tp.program, host, tp.scalar_values(), (0, 0, 0), dom)
        for o in tp.outputs:
            got = np.array([[[b[o][(i, j, k)] for i in range(dom[0])] for j in range(dom[1])] for k in range(dom[2])])
            assert got.dtype == dtype and np.array_equal(got, a[o].data), (seed, o)


def _point(text, values, scalars=None):
    """Evaluate a one-output program with 1x1x1 domain on constant inputs."""
    tp = dsl.parse(text)
    fields = {n: HostField(np.full((3, 3, 3), values[n]), (-1, -1, -1), (2, 2, 2)) for n in tp.inputs}
    r = stencil.run_unfused(tp.program, fields, tp.scalar_values(scalars), (0, 0, 0), (1, 1, 1))
    return float(r[tp.outputs[0]].data[0, 0, 0])


def test_left_associativity_and_precedence():
    # 1e16 + 1 - 1e16 = 0 left to right (1e16 + 1 rounds to 1e16); right-assoc would give 1
    assert _point("program p\ninput a\noutput o\napply r = a + 1.0 - a\nstore r -> o\n", {"a": 1e16}) == 0.0
    # * binds tighter than +, unary minus tighter than *
    assert _point("program p\ninput a\noutput o\napply r = 2.0 + 3.0 * -a\nstore r -> o\n", {"a": 4.0}) == -10.0
    assert _point("program p\ninput a\noutput o\napply r = (2.0 + 3.0) * a / 2.0\nstore r -> o\n", {"a": 4.0}) == 10.0
    # 8 / 4 / 2 = 1 (left) not 4
    assert _point("program p\ninput a\noutput o\napply r = 8.0 / a / 2.0\nstore r -> o\n", {"a": 4.0}) == 1.0


def test_select_min_max_abs_sqrt_semantics():
    prog = ("program p\ninput a\ninput b\noutput o\n"
            "apply r = select(a > b && !(a == 0.0) || b < -5.0, min(a, b) + max(a, b) * 10.0, abs(a) + sqrt(b))\n"
            "store r -> o\n")
    assert _point(prog, {"a": 3.0, "b": 2.0}) == 2.0 + 30.0
    assert _point(prog, {"a": -1.0, "b": 4.0}) == 1.0 + 2.0
    assert _point(prog, {"a": 0.0, "b": -9.0}) == -9.0 + 0.0
    # min(a, b) := b < a ? b : a  -> a NaN second operand is never chosen
    m = "program p\ninput a\ninput b\noutput o\napply r = min(a, b)\nstore r -> o\n"
    assert _point(m, {"a": 1.0, "b": np.nan}) == 1.0
    assert np.isnan(_point(m, {"a": np.nan, "b": 1.0}))


def test_locals_scalars_offsets():
    prog = ("program p\ninput a\nscalar s = 2.5\noutput o\n"
            "apply t { x = a[1,0,0] - a[-1,0,0]\n y = x * s\n return y + x }\n"
            "apply u = t[0,0,1] - t[0,0,-1]\nstore u -> o\n")
    tp = dsl.parse(prog)
    kk, jj, ii = np.meshgrid(np.arange(-2, 3), np.arange(-2, 3), np.arange(-2, 3), indexing="ij")
    a = HostField((ii * 3.0 + kk * 100.0).astype(np.float64), (-2, -2, -2), (3, 3, 3))
    r = stencil.run_unfused(tp.program, {"a": a}, tp.scalar_values(), (0, 0, 0), (1, 1, 1))
    # t = 3.5 * (a[i+1] - a[i-1]) = 3.5 * 6 = 21 at every level -> u = 0
    assert float(r["o"].data[0, 0, 0]) == 0.0
    r = stencil.run_unfused(tp.program, {"a": a}, tp.scalar_values({"s": -1.0}), (0, 0, 0), (1, 1, 1))
    assert float(r["o"].data[0, 0, 0]) == 0.0


def test_multi_result_operator():
    prog = ("program p\ninput a\noutput o1\noutput o2\n"
            "apply x, y { return a * 2.0, a - 1.0 }\nstore y -> o1\nstore x -> o2\n")
    tp = dsl.parse(prog)
    a = HostField(np.full((1, 1, 1), 5.0), (0, 0, 0), (1, 1, 1))
    r = stencil.run_unfused(tp.program, {"a": a}, {}, (0, 0, 0), (1, 1, 1))
    assert float(r["o1"].data[0, 0, 0]) == 4.0 and float(r["o2"].data[0, 0, 0]) == 10.0


BAD = [
    "input a\noutput o\napply r = a\nstore r -> o\n",                          # no program header
    "program p\ninput a\noutput o\napply r = b\nstore r -> o\n",               # undefined name
    "program p\ninput a\noutput o\napply r = a + o\nstore r -> o\n",           # output read
    "program p\ninput a\noutput o\napply r = r2\napply r2 = a\nstore r -> o\n",  # use before definition
    "program p\ninput a\noutput o\napply r = a\n",                             # output never stored
    "program p\ninput a\noutput o\napply r = a\nstore r -> o\nstore r -> o\n",  # stored twice
    "program p\ninput a\noutput o\napply r = a > 1.0\nstore r -> o\n",         # condition as value
    "program p\ninput a\noutput o\napply r = select(a, 1.0, 2.0)\nstore r -> o\n",  # value as condition
    "program p\ninput a\noutput o\napply r = a[1,0]\nstore r -> o\n",          # 2 offsets
    "program p\ninput a\noutput o\napply r, q = a\nstore r -> o\n",            # result count
    "program p\ninput a\ninput a\noutput o\napply r = a\nstore r -> o\n",      # duplicate
    "program p\ninput a\nscalar s\noutput o\napply r = s[1,0,0]\nstore r -> o\n",  # scalar offset
    "program p\ninput a\noutput o\napply r = foo(a)\nstore r -> o\n",          # unknown function
    "program p\ninput a\noutput o\napply r = a $ a\nstore r -> o\n",           # bad character
    "program p\ninput select\noutput o\napply r = 1.0\nstore r -> o\n",        # reserved word
]


@pytest.mark.parametrize("text", BAD)
def test_malformed_programs_rejected(text):
    with pytest.raises(dsl.DslError):
        dsl.parse(text)
