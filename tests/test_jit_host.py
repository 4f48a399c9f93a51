"""Host-side tests of liboec's stencil-language compiler (csrc/jit.cpp) -- no GPU.

* parse / verify: malformed programs rejected with line:col messages; builtin names and double
  registration rejected; destroy unregisters;
* shape inference: the extents liboec infers for the language versions of the suite
  equal the hand-derived builtin registry, and for 80 random programs equal the ORACLE's
  brute-force touched-index bounding boxes (oracle.stencil.run_fused);
* size-specialised code generation: every variant of every program generates CUDA that
  NVRTC compiles for sm_100a on this CPU-only host; sizes and strides are literals in the source.
"""
from __future__ import annotations

import glob
import os
import re

import numpy as np
import pytest

from jit_programs import random_program, touched_boxes
from oracle import dsl
from paper_2005_13014_b200 import oec

HERE = os.path.dirname(os.path.abspath(__file__))
NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "programs", "*.oec")))
VARIANTS = [oec.OEC_VARIANT_NAIVE, oec.OEC_VARIANT_UNROLL2, oec.OEC_VARIANT_UNROLL4, oec.OEC_VARIANT_UNFUSED,
            oec.OEC_VARIANT_UNROLL2_K, oec.OEC_VARIANT_UNROLL4_K]


def text_of(program):
    with open(os.path.join(HERE, "programs", program + ".oec")) as f:
        return f.read()


def _status(fn):
    try:
        fn()
    except oec.OecError as e:
        return e.status, str(e)
    return 0, ""


class Registered:
    """Register a program text for the duration of a test."""

    def __init__(self, text):
        self.name = oec.oec_program_create(text)

    def __enter__(self):
        return self.name

    def __exit__(self, *a):
        oec.oec_program_destroy(self.name)


def host_fields(name, domain, halo=3, dtype=np.float64):
    """Host descriptors (numpy arrays) with a generous halo for each input, outputs on the domain."""
    ins, outs = [], []
    sig_in, sig_out, _ = oec.program_signature(name)
    for (_, lo, hi, kinv) in sig_in:
        if kinv:
            a = np.zeros((1, domain[1] + 2 * halo, domain[0] + 2 * halo), dtype)
            ins.append(oec.oec_field_wrap(a, (-halo, -halo, 0), (domain[0] + halo, domain[1] + halo, 1), k_invariant=True))
        else:
            a = np.zeros(tuple(domain[d] + 2 * halo for d in (2, 1, 0)), dtype)
            ins.append(oec.oec_field_wrap(a, (-halo,) * 3, tuple(domain[d] + halo for d in range(3))))
    for _ in sig_out:
        outs.append(oec.oec_field_wrap(np.zeros((domain[2], domain[1], domain[0]), dtype), (0, 0, 0), domain))
    return ins, outs


@pytest.mark.parametrize("program", NAMES)
def test_inferred_extents_equal_builtin_registry(program):
    with Registered(text_of(program)) as name:
        assert name == program + "_text"
        a = oec.program_signature(name)
        b = oec.program_signature(program)
        assert a[0] == b[0]  # names, extents, k-invariance of every input
        assert a[1] == b[1]
        assert [n for n, _ in a[2]] == [n for n, _ in b[2]]


@pytest.mark.parametrize("seed", range(80))
def test_inferred_extents_equal_bruteforce_trace(seed):
    text = random_program(seed)
    tp = dsl.parse(text)
    ext = touched_boxes(tp, (5, 4, 3))
    with Registered(text) as name:
        sig_in, sig_out, sig_sc = oec.program_signature(name)
        assert [s[0] for s in sig_in] == tp.inputs
        assert sig_out == tp.outputs
        assert [s for s in sig_sc] == tp.scalars
        for (n, lo, hi, kinv) in sig_in:
            assert (lo, hi) == ext[n], (n, lo, hi, ext[n])
            assert kinv == tp.k_invariant[n]


def test_parse_errors_have_positions():
    st, msg = _status(lambda: oec.oec_program_create("program p\ninput a\noutput o\napply r = a +\nstore r -> o\n"))
    assert st == 1 and "line 5:" in msg
    st, msg = _status(lambda: oec.oec_program_create("program p\ninput a\noutput o\napply r = b\nstore r -> o\n"))
    assert st == 1 and "line 4:" in msg and "'b' is not defined" in msg


BAD = [
    "input a\noutput o\napply r = a\nstore r -> o\n",
    "program p\ninput a\noutput o\napply r = a + o\nstore r -> o\n",
    "program p\ninput a\noutput o\napply r = r2\napply r2 = a\nstore r -> o\n",
    "program p\ninput a\noutput o\napply r = a\n",
    "program p\ninput a\noutput o\napply r = a\nstore r -> o\nstore r -> o\n",
    "program p\ninput a\noutput o\napply r = a > 1.0\nstore r -> o\n",
    "program p\ninput a\noutput o\napply r = select(a, 1.0, 2.0)\nstore r -> o\n",
    "program p\ninput a\noutput o\napply r = a[1,0]\nstore r -> o\n",
    "program p\ninput a\noutput o\napply r, q = a\nstore r -> o\n",
    "program p\ninput a\ninput a\noutput o\napply r = a\nstore r -> o\n",
    "program p\ninput a\nscalar s\noutput o\napply r = s[1,0,0]\nstore r -> o\n",
    "program p\ninput a\noutput o\napply r = foo(a)\nstore r -> o\n",
    "program p\ninput a\noutput o\napply r = a $ a\nstore r -> o\n",
    "program p\ninput select\noutput o\napply r = 1.0\nstore r -> o\n",
]


@pytest.mark.parametrize("text", BAD)
def test_malformed_programs_rejected(text):
    st, msg = _status(lambda: oec.oec_program_create(text))
    assert st == 1, msg
    with pytest.raises(dsl.DslError):  # the oracle reader agrees
        dsl.parse(text)


def test_builtin_name_and_double_registration_rejected():
    st, msg = _status(lambda: oec.oec_program_create("program hdiff\ninput a\noutput o\napply r = a\nstore r -> o\n"))
    assert st == 1 and "builtin" in msg
    text = "program twice\ninput a\noutput o\napply r = a\nstore r -> o\n"
    with Registered(text):
        st, msg = _status(lambda: oec.oec_program_create(text))
        assert st == 1 and "already registered" in msg
    st, _ = _status(lambda: oec.oec_program_info("twice"))
    assert st == 1  # unregistered
    assert _status(lambda: oec.oec_program_destroy("hdiff"))[0] == 1
    assert _status(lambda: oec.oec_program_destroy("nope"))[0] == 1


def test_dead_operators_do_not_widen_extents():
    text = ("program dead\ninput a\ninput b\noutput o\n"
            "apply unused = b[5,5,1] + a[-7,0,0]\napply r = a[1,0,0]\nstore r -> o\n")
    with Registered(text) as name:
        (n0, lo0, hi0, _), (n1, lo1, hi1, _) = oec.program_signature(name)[0]
        assert (lo0, hi0) == ((0, 0, 0), (1, 0, 0))
        assert (lo1, hi1) == ((0, 0, 0), (0, 0, 0))


@pytest.mark.parametrize("program", NAMES)
@pytest.mark.parametrize("variant", VARIANTS)
def test_generated_source_compiles_for_sm100a(program, variant):
    domain = (33, 19, 5)  # ragged: 19 rows / 5 levels do not divide by 2 or 4
    with Registered(text_of(program)) as name:
        ins, outs = host_fields(name, domain)
        src, cubin = oec.oec_program_generate(name, ins, outs, (0, 0, 0), domain, variant, compile=True)
        assert cubin > 0
        assert "typedef double T;" in src
        # size specialisation: the domain bounds are literals, there are no size parameters
        assert re.search(r"\bi >= 33\b", src) and " 19" in src
        assert "int ni" not in src and "int nj" not in src
        if variant == oec.OEC_VARIANT_UNFUSED:
            n_live = len(re.findall(r"__global__", src))
            assert n_live >= 2
        else:
            assert src.count("__global__") == 1


def test_generated_source_f32_and_strides_are_constants():
    domain = (16, 8, 4)
    with Registered(text_of("hdiff")) as name:
        ins, outs = host_fields(name, domain, dtype=np.float32)
        src, cubin = oec.oec_program_generate(name, ins, outs, (0, 0, 0), domain, oec.OEC_VARIANT_NAIVE, compile=True)
        assert "typedef float T;" in src and cubin > 0
        # in: (16+6) x (8+6) allocation -> j stride 22, k stride 308: loads at immediate offsets
        assert "j0 * 22" in src and "k * 308" in src
        assert re.search(r"b0\[-22\]", src) and re.search(r"b0\[44\]", src)


def test_unroll_shares_loads_between_rows():
    """Stencil unrolling + CSE: with U rows per thread, the number of distinct
    (input, offset) loads per point drops (hdiff: 13 per point inlined, fewer per row unrolled)."""
    domain = (32, 32, 2)
    with Registered(text_of("hdiff")) as name:
        ins, outs = host_fields(name, domain)
        n = {}
        for v, u in ((oec.OEC_VARIANT_NAIVE, 1), (oec.OEC_VARIANT_UNROLL2, 2), (oec.OEC_VARIANT_UNROLL4, 4)):
            src, _ = oec.oec_program_generate(name, ins, outs, (0, 0, 0), domain, v)
            n[u] = len(re.findall(r"= b0\[", src)) / u
        assert n[1] == 13  # the 13-point diamond, each load once (CSE)
        assert n[2] < n[1] and n[4] < n[2]


def test_generate_argument_errors():
    with Registered(text_of("uvbke")) as name:
        ins, outs = host_fields(name, (8, 8, 2))
        assert _status(lambda: oec.oec_program_generate(name, ins[:2], outs, (0, 0, 0), (8, 8, 2)))[0] == 1
        assert _status(lambda: oec.oec_program_generate(name, ins, outs, (0, 0, 0), (8, 8, 2), variant=9))[0] == 1
    assert _status(lambda: oec.oec_program_generate("hdiff", [], [], (0, 0, 0), (8, 8, 2)))[0] == 1


def test_k_unroll_shares_levels():
    """Unrolling along k (P:451 'all unroll dimensions'): a thread evaluating 4 levels loads each
    k-offset plane once -- nh_p_grad's gz/pk3/pp k and k+1 accesses are shared between levels."""
    domain = (32, 16, 8)
    with Registered(text_of("nh_p_grad")) as name:
        ins, outs = host_fields(name, domain)
        src1, _ = oec.oec_program_generate(name, ins, outs, (0, 0, 0), domain, oec.OEC_VARIANT_NAIVE)
        src4, _ = oec.oec_program_generate(name, ins, outs, (0, 0, 0), domain, oec.OEC_VARIANT_UNROLL4_K)
        for f in ("b2", "b3", "b4"):  # pp, gz, pk3
            n1 = len(re.findall(rf"= {f}\[", src1))
            n4 = len(re.findall(rf"= {f}\[", src4)) / 4
            assert n4 < n1, (f, n1, n4)
        assert "k0 = blockIdx.z * 4" in src4


def test_k_unroll_rejected_for_builtins():
    st, msg = _status(lambda: oec.oec_apply_program("uvbke", [], [], None, (0, 0, 0), (8, 8, 2), oec.OEC_VARIANT_UNROLL2_K))
    assert st in (1, 7)


def test_embedded_suite_texts_equal_test_programs():
    """The library compiles its builtin suite programs' AUTO kernels from embedded stencil-language
    text (csrc/programs.cpp); it must be the very text the oracle reader is pinned on."""
    src = open(os.path.join(os.path.dirname(HERE), "paper_2005_13014_b200", "csrc", "programs.cpp")).read()
    for program in ("uvbke", "p_grad_c", "nh_p_grad", "fvtp2d_qi", "fvtp2d_qj", "fvtp2d_flux", "fastwaves"):
        assert 'R"OEC(' + text_of(program) + ')OEC"' in src, program
