"""Pins of the binary32 oracle instance (§7.1: every benchmark is run in f32 and
f64; "results are within a relative error of 1e-5 for single-precision").  CPU-only.

The f32 oracle is the same definitions evaluated in IEEE binary32 (oec_oracle.c compiled with
-DORACLE_F32; numpy / oracle.stencil on float32 arrays).  Pinned to things other than itself:
  * the fp64 oracle on the same (exactly representable) inputs, within the paper's 1e-5;
  * evidence the arithmetic really is binary32 (results differ from the rounded fp64 result in
    many elements, while an fp64-evaluate-then-round oracle would agree everywhere);
  * the independent numpy writing of hdiff / vadv, bitwise;
  * closed forms that hold exactly in any binary format (constant / linear fields, the unit
    spike, the dense LU solve of the same rows within the binary32 error bound).
"""
import numpy as np
import pytest

import synth
from oracle import capi, numpy_oracle
from oracle import stencil as st
from oracle import suite
from synth import HostField

F32 = np.float32
TOL_PAPER = 1e-5


def _normwise(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b)) / max(np.max(np.abs(b)), 1e-300))


def _run_f32_f64(program, domain, seed):
    h32 = synth.make_inputs(program, domain, seed=seed, dtype=F32)
    h64 = synth.as_dtype(h32, np.float64)
    res = {}
    for tag, h in (("f32", h32), ("f64", h64)):
        if program == "hdiff":
            o = synth.empty_outputs("hdiff", domain, dtype=h["in"].data.dtype)["out"]
            res[tag] = {"out": capi.hdiff(h["in"], h["coeff"], o, (0, 0, 0), domain).data}
        elif program == "vadv":
            o = synth.empty_outputs("vadv", domain, dtype=h["u_pos"].data.dtype)["utens_stage_out"]
            res[tag] = {"utens_stage_out": capi.vadv(h, o, synth.scalars("vadv")["dtr_stage"], (0, 0, 0), domain).data}
        else:
            r = st.run_unfused(suite.PROGRAMS[program], h, synth.scalars(program), (0, 0, 0), domain)
            res[tag] = {k: v.data for k, v in r.items()}
    return res["f32"], res["f64"]


@pytest.mark.parametrize("program", synth.ALL_PROGRAMS)
def test_f32_within_paper_tolerance_of_f64_and_really_binary32(program):
    domain = (24, 20, 16)
    r32, r64 = _run_f32_f64(program, domain, seed=4)
    for name in r64:
        a, b = r32[name], r64[name]
        assert a.dtype == F32, (program, name)
        assert _normwise(a, b) <= TOL_PAPER, (program, name, _normwise(a, b))
        # evaluated in binary32, not fp64-then-rounded: many elements differ from round(fp64)
        ndiff = int(np.count_nonzero(a != b.astype(F32)))
        assert ndiff >= a.size // 50, (program, name, ndiff, a.size)


@pytest.mark.parametrize("domain", [(32, 32, 16), (33, 31, 5), (1, 1, 1)])
@pytest.mark.parametrize("seed", [0, 1])
def test_hdiff_f32_variants_and_numpy_agree_bitwise(domain, seed):
    h = synth.make_inputs("hdiff", domain, seed=seed, dtype=F32)
    ref = numpy_oracle.hdiff(h["in"], h["coeff"], (0, 0, 0), domain)
    assert ref.dtype == F32
    for v in (capi.HDIFF_UNFUSED, capi.HDIFF_FUSED, capi.HDIFF_FUSED_REVERSED):
        o = synth.empty_outputs("hdiff", domain, dtype=F32)["out"]
        assert np.array_equal(capi.hdiff(h["in"], h["coeff"], o, (0, 0, 0), domain, v).data, ref), v


@pytest.mark.parametrize("domain", [(32, 32, 16), (7, 3, 80), (1, 1, 2)])
@pytest.mark.parametrize("seed", [0, 1])
def test_vadv_f32_variants_and_numpy_agree_bitwise(domain, seed):
    f = synth.make_inputs("vadv", domain, seed=seed, dtype=F32)
    ref = numpy_oracle.vadv(f, 0.15, (0, 0, 0), domain)
    assert ref.dtype == F32
    for v in (capi.VADV_UNFUSED, capi.VADV_FUSED, capi.VADV_FUSED_REVERSED):
        o = synth.empty_outputs("vadv", domain, dtype=F32)["utens_stage_out"]
        assert np.array_equal(capi.vadv(f, o, 0.15, (0, 0, 0), domain, v).data, ref), v


@pytest.mark.parametrize("name", list(synth.SUITE) + ["hdiff"])
def test_suite_f32_unfused_equals_fused(name):
    domain = (5, 4, 3)
    f = synth.make_inputs(name, domain, seed=2, dtype=F32)
    r_unf = st.run_unfused(suite.PROGRAMS[name], f, synth.scalars(name), (0, 0, 0), domain)
    r_fus, _ = st.run_fused(suite.PROGRAMS[name], f, synth.scalars(name), (0, 0, 0), domain)
    for o in r_unf:
        a = r_unf[o].data
        b = np.array([[[r_fus[o][(i, j, k)] for i in range(domain[0])] for j in range(domain[1])]
                      for k in range(domain[2])], dtype=F32)
        assert a.dtype == F32 and np.array_equal(a, b), (name, o)


def test_hdiff_f32_closed_forms():
    # constant and linear fields: lap == 0 exactly in any binary format -> out == in
    domain = (9, 8, 3)
    k, j, i = np.meshgrid(np.arange(3), np.arange(-2, 10), np.arange(-2, 11), indexing="ij")
    for data in (np.full(i.shape, 1.75), i + 3.0 * j + 64.0 * k):
        inp = HostField(data.astype(F32), (-2, -2, 0), (11, 10, 3))
        cf = HostField(np.full((3, 8, 9), 0.0625, F32), (0, 0, 0), domain)
        out = HostField(np.full((3, 8, 9), np.nan, F32), (0, 0, 0), domain)
        res = capi.hdiff(inp, cf, out, (0, 0, 0), domain).data
        assert np.array_equal(res, inp.data[:, 2:10, 2:11])
    # unit spike, coeff 1/16: 16 out is the 13-point stencil (small integers, exact in binary32)
    data = ((i == 4) & (j == 4)).astype(F32)[:1]
    inp = HostField(np.ascontiguousarray(data), (-2, -2, 0), (11, 10, 1))
    cf = HostField(np.full((1, 8, 9), 0.0625, F32), (0, 0, 0), (9, 8, 1))
    out = HostField(np.full((1, 8, 9), np.nan, F32), (0, 0, 0), (9, 8, 1))
    res = capi.hdiff(inp, cf, out, (0, 0, 0), (9, 8, 1)).data[0] * 16
    assert res[4, 4] == -4.0 and res[4, 5] == 8.0 and res[4, 6] == -1.0 and res[5, 5] == -2.0 and res[0, 0] == 0.0


@pytest.mark.parametrize("K", [2, 5, 40])
def test_vadv_f32_within_binary32_bound_of_dense_lu(K):
    # Thomas in binary32 vs a float64 dense solve of the SAME binary32 rows: error O(K eps32)
    domain = (4, 2, K)
    f = synth.make_inputs("vadv", domain, seed=K, dtype=F32)
    o = synth.empty_outputs("vadv", domain, dtype=F32)["utens_stage_out"]
    res = capi.vadv(f, o, 0.15, (0, 0, 0), domain).data
    dtr = float(np.float32(0.15))
    for jj in range(2):
        for ii in range(4):
            a, b, c, d = capi.vadv_system(f, 0.15, ii, jj, 0, K)
            assert a.dtype == F32
            T = np.diag(b.astype(np.float64)) + np.diag(a[1:].astype(np.float64), -1) + np.diag(c[:-1].astype(np.float64), 1)
            x = np.linalg.solve(T, d.astype(np.float64))
            exp = dtr * (x - f["u_pos"].data[:, jj, ii].astype(np.float64))
            err = np.max(np.abs(res[:, jj, ii] - exp)) / max(1.0, np.max(np.abs(exp)))
            assert err <= 50 * K * np.finfo(F32).eps, (ii, jj, err)
