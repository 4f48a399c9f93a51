"""Host-side tests of the C-ABI library (no GPU): it loads, exports every symbol include/oec.h
declares, its extent registry equals the oracle's brute-force touched-index trace, argument
validation returns the documented status codes, and the decomposition plan is consistent."""
import os
import re

import numpy as np
import pytest

import synth
from oracle import stencil as st
from oracle import suite
from paper_2005_13014_b200 import oec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "oec.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(oec_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = oec.lib()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    # and the binding declares a signature for every one of them
    assert set(names) == set(oec.SIGNATURES), set(names) ^ set(oec.SIGNATURES)


def test_no_oracle_symbols_in_product_library():
    import subprocess

    out = subprocess.run(["nm", "-D", oec.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle_" not in out
    assert "liboec_oracle" not in open(oec.LIB_PATH, "rb").read().decode("latin1")


def test_abi_version():
    assert oec.lib().oec_abi_version() == 1


@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
def test_registry_matches_recipe_and_trace(program):
    ins, outs, scs = oec.program_signature(program)
    spec = synth.PROGRAMS[program]
    assert [x[0] for x in ins] == [s.name for s in spec.inputs]
    assert outs == list(spec.outputs)
    assert [x[0] for x in scs] == [s[0] for s in spec.scalars]
    for (name, lo, hi, kinv), s in zip(ins, spec.inputs):
        assert lo == tuple(-h for h in s.halo_lo) and hi == tuple(s.halo_hi), name
        assert kinv == s.k_invariant
    for (name, dflt), (sname, sval) in zip(scs, spec.scalars):
        assert dflt == sval
    for q, (name, lo, hi, kinv) in enumerate(ins):  # oec_program_extent == oec_program_input
        assert oec.oec_program_extent(program, q) == (lo, hi)
    if program == "vadv":
        return  # vadv's extent is pinned by the oracle's range checks (test_oracle_vadv)
    # brute-force trace of the fused oracle evaluation on a small domain
    domain = (4, 5, 3)
    f = synth.make_inputs(program, domain, seed=0)
    _, touched = st.run_fused(suite.PROGRAMS[program], f, synth.scalars(program), (0, 0, 0), domain)
    for name, lo, hi, kinv in ins:
        blo, bhi = st.bbox(touched[name])
        for d in range(3):
            if d == 2 and kinv:
                assert (blo[2], bhi[2]) == (0, 1)
                continue
            assert blo[d] == lo[d] and bhi[d] == domain[d] + hi[d], (name, d)


def _host(shape_kji, lb, ub):
    arr = np.zeros(shape_kji)
    return oec.oec_field_wrap(arr, lb, ub)


def _hdiff_host_fields(domain=(8, 8, 2), halo=2):
    ni, nj, nk = domain
    inp = _host((nk, nj + 2 * halo, ni + 2 * halo), (-halo, -halo, 0), (ni + halo, nj + halo, nk))
    cf = _host((nk, nj, ni), (0, 0, 0), domain)
    out = _host((nk, nj, ni), (0, 0, 0), domain)
    return inp, cf, out


def _status(fn):
    try:
        fn()
    except oec.OecError as e:
        return e.status, str(e)
    return 0, ""


def test_error_halo_too_small():
    inp, cf, out = _hdiff_host_fields(halo=1)
    stt, msg = _status(lambda: oec.oec_hdiff(inp, cf, out, (0, 0, 0), (8, 8, 2)))
    assert stt == 2 and "does not cover" in msg


def test_error_alias():
    inp, cf, out = _hdiff_host_fields()
    stt, msg = _status(lambda: oec.oec_hdiff(inp, cf, cf, (0, 0, 0), (8, 8, 2)))
    assert stt == 3 and "overlaps" in msg


def test_error_arg_counts_and_program():
    inp, cf, out = _hdiff_host_fields()
    assert _status(lambda: oec.oec_apply_program("hdiff", [inp], [out], dom_ub=(8, 8, 2)))[0] == 1
    assert _status(lambda: oec.oec_apply_program("nope", [inp, cf], [out], dom_ub=(8, 8, 2)))[0] == 1
    assert _status(lambda: oec.oec_apply_program("hdiff", [inp, cf], [out], dom_ub=(8, 8, 2), variant=9))[0] == 1
    # unrolling along k exists for stencil-language programs only
    assert _status(lambda: oec.oec_apply_program("hdiff", [inp, cf], [out], dom_ub=(8, 8, 2), variant=5))[0] == 7


def test_unroll_variant_rejected_for_vadv():
    dom = (4, 4, 2)
    f = [_host((2, 4, 4), (0, 0, 0), dom) for _ in range(4)]
    w = _host((2, 4, 5), (0, 0, 0), (5, 4, 2))
    o = _host((2, 4, 4), (0, 0, 0), dom)
    for variant in (3, 4):
        stt, msg = _status(lambda: oec.oec_apply_program("vadv", [f[0], w, f[1], f[2], f[3]], [o], dom_ub=dom,
                                                         variant=variant))
        assert stt == 7 and "unroll" in msg


def test_error_layout_stride0():
    arr = np.zeros((2, 8, 8))
    stt, _ = _status(lambda: oec.oec_field_wrap(arr, (0, 0, 0), (8, 8, 2), stride=(2, 8, 64)))
    assert stt == 8


def test_error_vadv_k1():
    dom = (4, 4, 1)
    f = [_host((1, 4, 4), (0, 0, 0), dom) for _ in range(4)]
    w = _host((1, 4, 5), (0, 0, 0), (5, 4, 1))
    o = _host((1, 4, 4), (0, 0, 0), dom)
    stt, msg = _status(lambda: oec.oec_vadv(f[0], w, f[1], f[2], f[3], o, 0.15, (0, 0, 0), dom))
    assert stt == 2 and "K = 1" in msg


def test_error_mixed_dtypes():
    inp, cf, out = _hdiff_host_fields()
    o32 = oec.oec_field_wrap(np.zeros((2, 8, 8), np.float32), (0, 0, 0), (8, 8, 2))
    stt, msg = _status(lambda: oec.oec_hdiff(inp, cf, o32, (0, 0, 0), (8, 8, 2)))
    assert stt == 4 and "dtype" in msg
    bad = oec.oec_field_wrap(np.zeros((2, 8, 8), np.float32), (0, 0, 0), (8, 8, 2))
    bad.desc.dtype = 7
    assert _status(lambda: oec.oec_hdiff(inp, cf, bad, (0, 0, 0), (8, 8, 2)))[0] == 4


def test_error_mixed_devices():
    inp, cf, out = _hdiff_host_fields()
    out.desc.device = 0
    assert _status(lambda: oec.oec_hdiff(inp, cf, out, (0, 0, 0), (8, 8, 2)))[0] == 4


def test_empty_domain_is_a_noop():
    inp, cf, out = _hdiff_host_fields()
    oec.oec_hdiff(inp, cf, out, (0, 0, 0), (0, 8, 2))
    assert oec.oec_last_launch_count() == 0


def test_k_invariant_input_required():
    dom = (4, 4, 2)
    uc = _host((2, 5, 4), (0, -1, 0), (4, 4, 2))
    vc = _host((2, 4, 5), (-1, 0, 0), (4, 4, 2))
    cosa3d = _host((2, 4, 4), (0, 0, 0), dom)  # 3D where a 2D metric field is declared
    rs = oec.oec_field_wrap(np.zeros((1, 4, 4)), (0, 0, 0), (4, 4, 1), k_invariant=True)
    ub, vb = _host((2, 4, 4), (0, 0, 0), dom), _host((2, 4, 4), (0, 0, 0), dom)
    stt, msg = _status(lambda: oec.oec_apply_program("uvbke", [uc, vc, cosa3d, rs], [ub, vb], dom_ub=dom))
    assert stt == 2 and "k-invariant" in msg


# ---------------------------------------------------------------------------------------------
# decomposition plan (host logic)
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("g,px,py", [((16, 16, 3), 2, 2), ((17, 13, 2), 3, 2), ((32, 64, 4), 1, 8), ((9, 9, 1), 4, 1)])
@pytest.mark.parametrize("w", [((2, 2, 0), (2, 2, 0)), ((0, 1, 0), (1, 0, 0)), ((3, 3, 0), (2, 3, 0))])
def test_plan_consistency(g, px, py, w):
    wlo, whi = w
    R = px * py
    decs = [oec.oec_decomp_create(g, px, py, r) for r in range(R)]
    # sub-domains tile the global domain exactly
    cover = np.zeros((g[1], g[0]), int)
    for d in decs:
        cover[d.local_lb[1]:d.local_ub[1], d.local_lb[0]:d.local_ub[0]] += 1
        assert d.local_lb[2] == 0 and d.local_ub[2] == g[2]
    assert (cover == 1).all()
    plans = [oec.oec_decomp_plan(d, wlo, whi) for d in decs]
    # every recv of r from p equals a send of p to r with the same phase and box
    for r in range(R):
        for m in plans[r]:
            if not m["is_send"]:
                match = [x for x in plans[m["peer"]] if x["is_send"] and x["peer"] == r and x["phase"] == m["phase"]
                         and x["lo"] == m["lo"] and x["hi"] == m["hi"]]
                assert len(match) == 1, (r, m)
    # after both phases, every rank's halo box inside the global domain is received exactly once
    # (phase-1 boxes include the i-halo so corners arrive in two hops)
    for r, d in enumerate(decs):
        need = np.zeros((g[1] + 20, g[0] + 20), int)  # offset 10
        lo, hi = d.local_lb, d.local_ub
        for m in plans[r]:
            if not m["is_send"]:
                need[m["lo"][1] + 10:m["hi"][1] + 10, m["lo"][0] + 10:m["hi"][0] + 10] += 1
        for j in range(lo[1] - wlo[1], hi[1] + whi[1]):
            for i in range(lo[0] - wlo[0], hi[0] + whi[0]):
                inside_local = lo[0] <= i < hi[0] and lo[1] <= j < hi[1]
                inside_global = 0 <= j < g[1] and 0 <= i < g[0]
                in_i_halo_of_global = not (0 <= i < g[0]) and 0 <= j < g[1]
                got = need[j + 10, i + 10]
                if inside_local:
                    assert got == 0
                elif inside_global:
                    assert got == 1, (r, i, j)
                elif (lo[1] <= j < hi[1]) or not (0 <= j < g[1]):
                    assert got == 0 or in_i_halo_of_global


@pytest.mark.parametrize("g,px,py,per", [((16, 16, 3), 2, 2, (True, True)), ((17, 13, 2), 3, 2, (True, False)),
                                         ((12, 9, 2), 1, 1, (True, True)), ((12, 9, 2), 2, 1, (True, True)),
                                         ((32, 64, 4), 1, 8, (False, True))])
def test_periodic_plan_consistency(g, px, py, per):
    # periodic: every recv of r from p (phase, tag) pairs with exactly one send of p to r whose box
    # equals it modulo the period, and every halo cell of every rank is received exactly once
    # (in-domain cells and, across a periodic boundary, the wrapped ones)
    wlo, whi = (2, 1, 0), (1, 2, 0)
    R = px * py
    decs = [oec.oec_decomp_create(g, px, py, r) for r in range(R)]
    for d in decs:
        oec.oec_decomp_set_periodic(d, *per)
    plans = [oec.oec_decomp_plan(d, wlo, whi) for d in decs]

    def wrap(lo, hi):
        return tuple((lo[d] % g[d], hi[d] - lo[d]) if d < 2 and per[d] else (lo[d], hi[d] - lo[d]) for d in range(3))

    for r in range(R):
        for m in plans[r]:
            if m["is_send"]:
                continue
            match = [x for x in plans[m["peer"]] if x["is_send"] and x["peer"] == r and x["phase"] == m["phase"]
                     and x["tag"] == m["tag"]]
            assert len(match) == 1, (r, m)
            assert wrap(match[0]["lo"], match[0]["hi"]) == wrap(m["lo"], m["hi"]), (r, m, match[0])
    for r, d in enumerate(decs):
        lo, hi = d.local_lb, d.local_ub
        got = {}
        for m in plans[r]:
            if not m["is_send"]:
                for j in range(m["lo"][1], m["hi"][1]):
                    for i in range(m["lo"][0], m["hi"][0]):
                        got[(i, j)] = got.get((i, j), 0) + 1
        for j in range(lo[1] - wlo[1], hi[1] + whi[1]):
            for i in range(lo[0] - wlo[0], hi[0] + whi[0]):
                own = lo[0] <= i < hi[0] and lo[1] <= j < hi[1]
                reach = (per[0] or 0 <= i < g[0]) and (per[1] or 0 <= j < g[1])
                if own:
                    assert got.get((i, j), 0) == 0
                elif reach:
                    assert got.get((i, j), 0) == 1, (r, i, j)
