"""Pins of the hdiff oracle (oracle/oec_oracle.c) to things other than itself.

See DESIGN.md "Oracle pins".  Every test here is CPU-only.
"""
import os

import numpy as np
import pytest

import synth
from oracle import capi, numpy_oracle
from oracle import stencil as st
from oracle import suite
from synth import HostField

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _fields(data_in, domain, coeff_val=None, coeff=None, halo=2):
    ni, nj, nk = domain
    lb = (-halo, -halo, 0)
    ub = (ni + halo, nj + halo, nk)
    inp = HostField(np.ascontiguousarray(data_in, dtype=np.float64), lb, ub)
    if coeff is None:
        coeff = np.full((nk, nj, ni), coeff_val)
    cf = HostField(np.ascontiguousarray(coeff, dtype=np.float64), (0, 0, 0), domain)
    out = HostField(np.full((nk, nj, ni), np.nan), (0, 0, 0), domain)
    return inp, cf, out


def _grid(domain, halo=2):
    ni, nj, nk = domain
    k, j, i = np.meshgrid(np.arange(nk), np.arange(-halo, nj + halo), np.arange(-halo, ni + halo), indexing="ij")
    return i.astype(np.float64), j.astype(np.float64), k.astype(np.float64)


def _run(inp, cf, out, variant=capi.HDIFF_UNFUSED):
    domain = out.ub
    return capi.hdiff(inp, cf, out, (0, 0, 0), domain, variant).data


def _interior(inp, domain):
    ni, nj, nk = domain
    return inp.data[:, 2:2 + nj, 2:2 + ni]


@pytest.mark.parametrize("variant", [capi.HDIFF_UNFUSED, capi.HDIFF_FUSED])
@pytest.mark.parametrize("c", [0.0, 1.0, -3.75, 1e300, 7.123456789e-5])
def test_constant_field_is_identity(c, variant):
    # north_star: "a constant field gives a zero Laplacian and leaves hdiff unchanged"
    domain = (7, 6, 3)
    i, j, k = _grid(domain)
    rng = np.random.default_rng(1)
    inp, cf, out = _fields(np.full(i.shape, c), domain, coeff=rng.uniform(0, 0.1, (3, 6, 7)))
    res = _run(inp, cf, out, variant)
    assert np.array_equal(res, _interior(inp, domain))


@pytest.mark.parametrize("kind", ["linear", "quadratic"])
def test_linear_and_quadratic_fields_are_identity(kind):
    # closed form: lap of a linear field is 0, of i^2+j^2 is the constant 4 -> flx = fly = 0
    domain = (9, 8, 4)
    i, j, k = _grid(domain)
    data = i + 3 * j + 2.0**20 * k if kind == "linear" else i * i + j * j + 5 * k
    inp, cf, out = _fields(data, domain, coeff_val=0.0625)
    assert np.array_equal(_run(inp, cf, out), _interior(inp, domain))


def test_unit_spike_exact():
    # unit spike at (0,0) (shifted into the domain), coeff = 1/16: the limiter stays inactive and
    # 16*out is the 13-point stencil 1*16-20 at the centre, +8 axis +-1, -2 diagonals, -1 axis +-2
    domain = (9, 9, 1)
    i, j, k = _grid(domain)
    c0 = 4
    data = ((i == c0) & (j == c0)).astype(np.float64)
    inp, cf, out = _fields(data, domain, coeff_val=1.0 / 16.0)
    res = _run(inp, cf, out)[0] * 16.0
    exp = np.zeros((9, 9))
    exp[c0, c0] = 16.0 - 20.0
    for d in (-1, 1):
        exp[c0 + d, c0] = exp[c0, c0 + d] = 8.0
        exp[c0 + 2 * d, c0] = exp[c0, c0 + 2 * d] = -1.0
        exp[c0 + d, c0 + d] = exp[c0 + d, c0 - d] = -2.0
    assert np.array_equal(res, exp)


def test_quartic_limiter_everywhere():
    # in = i^4 (j-invariant): lap = 12 i^2 + 2, flx = 24 i + 12 has the sign of in(i+1)-in(i) for
    # every integer i, so the limiter zeroes every flux: out == in exactly; limiter off: in - 24 coeff
    domain = (12, 5, 2)
    i, j, k = _grid(domain)
    data = (i - 3.0) ** 4
    inp, cf, out = _fields(data, domain, coeff_val=0.125)
    assert np.array_equal(_run(inp, cf, out), _interior(inp, domain))
    inp, cf, out = _fields(data, domain, coeff_val=0.125)
    res = capi.hdiff(inp, cf, out, (0, 0, 0), domain, capi.HDIFF_NO_LIMITER).data
    assert np.array_equal(res, _interior(inp, domain) - 24 * 0.125)


def test_limiter_off_is_biharmonic():
    # textbook closed form: with the limiter off, hdiff is in - coeff * L(L(in)) with L the 5-point
    # Laplacian, i.e. the 13-point biharmonic 20u - 8 sum(axis 1) + 2 sum(diag) + sum(axis 2)
    domain = (10, 11, 3)
    rng = np.random.default_rng(7)
    inp, cf, out = _fields(rng.uniform(-1, 1, (3, 15, 14)), domain, coeff=rng.uniform(0, 0.1, (3, 11, 10)))
    res = capi.hdiff(inp, cf, out, (0, 0, 0), domain, capi.HDIFF_NO_LIMITER).data
    u = inp.data

    def U(di, dj):
        return u[:, 2 + dj:2 + dj + 11, 2 + di:2 + di + 10]

    bih = (20 * U(0, 0) - 8 * (U(1, 0) + U(-1, 0) + U(0, 1) + U(0, -1))
           + 2 * (U(1, 1) + U(1, -1) + U(-1, 1) + U(-1, -1)) + (U(2, 0) + U(-2, 0) + U(0, 2) + U(0, -2)))
    exp = U(0, 0) - cf.data * bih
    assert np.max(np.abs(res - exp)) / np.max(np.abs(exp)) < 4e-15


def _load_patches():
    lines = [ln for ln in open(os.path.join(GOLDEN, "hdiff_limiter_patches.txt")) if ln.strip() and not ln.startswith("#")]
    out = []
    for q in range(0, len(lines), 6):
        name, expect = lines[q].split()[:2]
        patch = np.array([[float(x) for x in lines[q + r].split()] for r in range(1, 6)])
        out.append((name, float(expect), patch))
    return out


@pytest.mark.parametrize("name,expect,patch", _load_patches(), ids=[p[0] for p in _load_patches()])
def test_hand_built_limiter_patches(name, expect, patch):
    # patch rows are i = -2..2, columns j = -2..2 -> array [k][j][i] = patch.T
    inp, cf, out = _fields(patch.T[None, :, :], (1, 1, 1), coeff_val=0.25)
    for variant in (capi.HDIFF_UNFUSED, capi.HDIFF_FUSED):
        res = capi.hdiff(inp, cf, out, (0, 0, 0), (1, 1, 1), variant).data
        assert res[0, 0, 0] == expect, (name, res[0, 0, 0])


def test_random_field_exercises_limiter():
    # guard that the parity workload is not vacuous: the limiter changes a large share of outputs
    domain = (32, 32, 4)
    f = synth.make_inputs("hdiff", domain, seed=0)
    o1 = HostField(np.zeros((4, 32, 32)), (0, 0, 0), domain)
    o2 = HostField(np.zeros((4, 32, 32)), (0, 0, 0), domain)
    capi.hdiff(f["in"], f["coeff"], o1, (0, 0, 0), domain, capi.HDIFF_UNFUSED)
    capi.hdiff(f["in"], f["coeff"], o2, (0, 0, 0), domain, capi.HDIFF_NO_LIMITER)
    frac = np.mean(o1.data != o2.data)
    assert 0.2 < frac < 0.6


@pytest.mark.parametrize("domain", [(32, 32, 16), (33, 31, 5), (1, 1, 1), (4, 3, 2)])
@pytest.mark.parametrize("seed", [0, 1])
def test_fused_unfused_reversed_numpy_stencil_agree_bitwise(domain, seed):
    f = synth.make_inputs("hdiff", domain, seed=seed)
    ni, nj, nk = domain
    outs = []
    for variant in (capi.HDIFF_UNFUSED, capi.HDIFF_FUSED, capi.HDIFF_FUSED_REVERSED):
        o = HostField(np.full((nk, nj, ni), np.nan), (0, 0, 0), domain)
        outs.append(capi.hdiff(f["in"], f["coeff"], o, (0, 0, 0), domain, variant, nthreads=2).data)
    outs.append(numpy_oracle.hdiff(f["in"], f["coeff"], (0, 0, 0), domain))
    outs.append(st.run_unfused(suite.HDIFF, f, {}, (0, 0, 0), domain)["out"].data)
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)
    assert not np.isnan(outs[0]).any()


def test_fused_per_point_stencil_matches_c():
    domain = (6, 5, 2)
    f = synth.make_inputs("hdiff", domain, seed=3)
    o = HostField(np.full((2, 5, 6), np.nan), (0, 0, 0), domain)
    ref = capi.hdiff(f["in"], f["coeff"], o, (0, 0, 0), domain).data
    vals, touched = st.run_fused(suite.HDIFF, f, {}, (0, 0, 0), domain)
    for (i, j, k), v in vals["out"].items():
        assert v == ref[k, j, i]


def test_thread_count_invariance():
    domain = (40, 24, 9)
    f = synth.make_inputs("hdiff", domain, seed=2)
    res = []
    for nt in (1, 3, 8):
        for variant in (capi.HDIFF_UNFUSED, capi.HDIFF_FUSED):
            o = HostField(np.zeros((9, 24, 40)), (0, 0, 0), domain)
            res.append(capi.hdiff(f["in"], f["coeff"], o, (0, 0, 0), domain, variant, nthreads=nt).data)
    for r in res[1:]:
        assert np.array_equal(res[0], r)


def test_subdomain_and_origin_offset():
    # the domain may be a sub-range of the allocation (P:336 ranges relative to the origin)
    domain = (16, 16, 3)
    f = synth.make_inputs("hdiff", domain, seed=4)
    full = HostField(np.zeros((3, 16, 16)), (0, 0, 0), domain)
    capi.hdiff(f["in"], f["coeff"], full, (0, 0, 0), domain)
    sub = HostField(np.full((3, 16, 16), -7.0), (0, 0, 0), domain)
    capi.hdiff(f["in"], f["coeff"], sub, (3, 5, 1), (11, 9, 3))
    assert np.array_equal(sub.data[1:3, 5:9, 3:11], full.data[1:3, 5:9, 3:11])
    mask = np.ones_like(sub.data, bool)
    mask[1:3, 5:9, 3:11] = False
    assert np.all(sub.data[mask] == -7.0)  # store range only


def test_halo_too_small_is_an_error():
    domain = (8, 8, 2)
    inp = HostField(np.zeros((2, 11, 11)), (-1, -1, 0), (10, 10, 2))  # halo 1 < 2
    cf = HostField(np.zeros((2, 8, 8)), (0, 0, 0), domain)
    out = HostField(np.zeros((2, 8, 8)), (0, 0, 0), domain)
    with pytest.raises(capi.OracleError):
        capi.hdiff(inp, cf, out, (0, 0, 0), domain)
