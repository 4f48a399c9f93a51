"""Pins of the suite oracle (oracle/suite.py) and of the extent recipe.  CPU-only.

* Table II census
* closed forms / special cases per program
* unfused (materialised) == fused (inlined, per point) bitwise
* brute-force touched-index bounding box == the synth allocation recipe (exact)
"""
import numpy as np
import pytest

import synth
from oracle import stencil as st
from oracle import suite
from synth import HostField

SUITE = synth.SUITE


@pytest.mark.parametrize("name", sorted(suite.TABLE_II))
def test_census_matches_table_ii_exactly(name):
    # every column of Table II for all six programs; the compare of the fvtp2d upwind
    # `if` counts as an arithmetic operation (reading R15)
    dims, applies, n_in, n_out, arith, access, cf = suite.TABLE_II[name]
    c = st.census(suite.PROGRAMS[name])
    assert (c["applies"], c["inputs"], c["outputs"], c["arith"] + c["cmp"], c["access"], c["if"] > 0) == (
        applies, n_in, n_out, arith, access, cf)


def _ppm_candidate(weights_as_quotients, c_reads):
    """One writing of the PPM flux program (R15 enumeration): the weights as literals or
    as the quotients 7/12, 1/12 of the text; c read once ('shared'), by the condition and each
    branch region ('regions'), or at every use ('uses')."""
    def prog(q, c, dim):
        def o(d):
            return (0, d) if dim == "j" else (d, 0)

        def f_al(a, s, sel):
            if weights_as_quotients:
                return st.kdiv(sel, 7.0, 12.0) * (a(q, *o(-1)) + a(q)) - st.kdiv(sel, 1.0, 12.0) * (a(q, *o(-2)) + a(q, *o(1)))
            return suite.P1 * (a(q, *o(-1)) + a(q)) + suite.P2 * (a(q, *o(-2)) + a(q, *o(1)))

        def f_blbr(a, s, sel):
            qq = a(q)
            return a("al", *o(0)) - qq, a("al", *o(1)) - qq

        def f_flux(a, s, sel):
            cc = a(c)
            if c_reads == "shared":
                c1 = c2 = c3 = c4 = cc
            elif c_reads == "regions":
                c1 = c2 = a(c)  # the c > 0 region's read
                c3 = c4 = a(c)  # the else region's read
            else:
                c1, c2, c3, c4 = a(c), a(c), a(c), a(c)
            blm, brm = a("bl", *o(-1)), a("br", *o(-1))
            bl0, br0 = a("bl"), a("br")
            return sel(cc > 0.0, a(q, *o(-1)) + (1.0 - c1) * (brm - c2 * (blm + brm)),
                       a(q) + (1.0 + c3) * (bl0 + c4 * (bl0 + br0)))

        return (st.Apply(("al",), f_al), st.Apply(("bl", "br"), f_blbr), st.Apply(("f",), f_flux))
    return prog


def test_fvtp2d_census_enumeration():
    # the enumeration behind reading R15: the extra arithmetic / access operations of each writing
    # of one PPM flux over the minimal one; only "quotient weights + c read per region" gives
    # Table II's +2 / +2 per PPM flux (27/23, 49/39, 28/22 in the three programs)
    def counts(wq, cr):
        p = st.Program("ppm", ("q", "c"), (("f", "f"),), _ppm_candidate(wq, cr)("q", "c", "j"))
        c = st.census(p)
        return c["arith"] + c["cmp"], c["access"]

    base = counts(False, "shared")
    assert base == (20, 14)
    table = {(wq, cr): tuple(x - y for x, y in zip(counts(wq, cr), base))
             for wq in (False, True) for cr in ("shared", "regions", "uses")}
    assert table == {(False, "shared"): (0, 0), (False, "regions"): (0, 2), (False, "uses"): (0, 4),
                     (True, "shared"): (2, 0), (True, "regions"): (2, 2), (True, "uses"): (2, 4)}
    # the suite's PPM is that writing
    qi = st.census(suite.PROGRAMS["fvtp2d_qi"])
    assert (qi["arith"] + qi["cmp"], qi["access"]) == (base[0] + 2 + 5, base[1] + 2 + 7)


def _dims_used(prog):
    offs = set()
    for ap in prog.applies:
        for _, di, dj, dk in st.accesses(ap, prog.scalars):
            offs.add((di != 0, dj != 0, dk != 0))
    return 3 if any(o[2] for o in offs) else 2


@pytest.mark.parametrize("name", list(suite.TABLE_II))
def test_census_dims(name):
    assert _dims_used(suite.PROGRAMS[name]) == suite.TABLE_II[name][0]


@pytest.mark.parametrize("name", list(SUITE) + ["hdiff"])
@pytest.mark.parametrize("domain", [(5, 4, 3), (3, 6, 2)])
def test_unfused_equals_fused_and_extents_equal_recipe(name, domain):
    prog = suite.PROGRAMS[name]
    f = synth.make_inputs(name, domain, seed=11)
    sc = synth.scalars(name)
    unf = st.run_unfused(prog, f, sc, (0, 0, 0), domain)
    fused, touched = st.run_fused(prog, f, sc, (0, 0, 0), domain)
    rev, _ = st.run_fused(prog, f, sc, (0, 0, 0), domain, reverse=True)
    for oname, _ in prog.outputs:
        for (i, j, k), v in fused[oname].items():
            u = unf[oname].data[k, j, i]
            assert v == u or (np.isnan(v) and np.isnan(u)), (oname, i, j, k)
            assert rev[oname][(i, j, k)] == v
    # the bounding box of what the fused evaluation touches is exactly the recipe's allocation
    for spec in synth.PROGRAMS[name].inputs:
        lb, ub = synth.alloc_range(spec, domain)
        blo, bhi = st.bbox(touched[spec.name])
        assert (blo, bhi) == (lb, ub), (spec.name, blo, bhi, lb, ub)


def test_hdiff_touched_set_is_diamond():
    # 13-point diamond: (N+4)^2 - 12 distinct `in` elements per level
    domain = (6, 6, 2)
    f = synth.make_inputs("hdiff", domain, seed=0)
    _, touched = st.run_fused(suite.HDIFF, f, {}, (0, 0, 0), domain)
    assert len(touched["in"]) == ((6 + 4) ** 2 - 12) * 2
    assert len(touched["coeff"]) == 6 * 6 * 2


def _const_inputs(name, domain, vals):
    f = synth.make_inputs(name, domain, seed=0)
    for n, v in vals.items():
        f[n].data[:] = v
    return f


def _unf(name, f, domain, sc=None):
    return st.run_unfused(suite.PROGRAMS[name], f, sc or synth.scalars(name), (0, 0, 0), domain)


def _grid(fld):
    k, j, i = np.meshgrid(np.arange(fld.lb[2], fld.ub[2]), np.arange(fld.lb[1], fld.ub[1]),
                          np.arange(fld.lb[0], fld.ub[0]), indexing="ij")
    return i.astype(float), j.astype(float), k.astype(float)


# ----------------------------------------------------------------------------------------------- uvbke
def test_uvbke_constant_closed_form():
    domain = (4, 5, 2)
    f = _const_inputs("uvbke", domain, {"uc": 0.75, "vc": -0.5, "cosa": 0.25, "rsina": 1.5})
    r = _unf("uvbke", f, domain, {"dt5": 0.125})
    assert np.all(r["ub"].data == 0.125 * (1.5 - (-1.0) * 0.25) * 1.5)
    assert np.all(r["vb"].data == 0.125 * (-1.0 - 1.5 * 0.25) * 1.5)


def _transpose(fld: HostField) -> HostField:
    return HostField(np.ascontiguousarray(fld.data.transpose(0, 2, 1)), (fld.lb[1], fld.lb[0], fld.lb[2]),
                     (fld.ub[1], fld.ub[0], fld.ub[2]), fld.k_invariant)


def test_uvbke_ij_symmetry():
    # vb(uc, vc) == transpose(ub(vc^T, uc^T)): pins which field is offset in which direction
    domain = (5, 5, 2)
    f = synth.make_inputs("uvbke", domain, seed=1)
    r = _unf("uvbke", f, domain)
    g = {"uc": _transpose(f["vc"]), "vc": _transpose(f["uc"]), "cosa": _transpose(f["cosa"]), "rsina": _transpose(f["rsina"])}
    r2 = _unf("uvbke", g, domain)
    assert np.array_equal(r["vb"].data, r2["ub"].data.transpose(0, 2, 1))


# -------------------------------------------------------------------------------------------- p_grad_c
def test_p_grad_c_flat_levels_no_force():
    # horizontally uniform gz and pkc: the two cross products cancel exactly -> uc, vc unchanged
    domain = (4, 4, 3)
    f = synth.make_inputs("p_grad_c", domain, seed=2)
    for n in ("gz", "pkc"):
        d = f[n].data
        d[:] = d[:, :1, :1]
    r = _unf("p_grad_c", f, domain)
    assert np.array_equal(r["uc_out"].data, f["uc"].data)
    assert np.array_equal(r["vc_out"].data, f["vc"].data)


def test_p_grad_c_tilted_surface_closed_form():
    # gz = al*i + be*k, pkc = ga*k, delpc = D: the bracket is (-al+be)ga + (-al-be)ga = -2 al ga
    # -> uc_out = uc + dt2*rdxc/(2D) * (-2 al ga); analogous in j with al -> 0 for vc
    domain = (4, 3, 2)
    f = synth.make_inputs("p_grad_c", domain, seed=3)
    al, be, ga, D = 0.25, -1.0, 0.5, 0.75
    i, j, k = _grid(f["gz"])
    f["gz"].data[:] = al * i + be * k
    i, j, k = _grid(f["pkc"])
    f["pkc"].data[:] = ga * k
    f["delpc"].data[:] = D
    r = _unf("p_grad_c", f, domain)
    dt2 = synth.scalars("p_grad_c")["dt2"]
    exp_u = f["uc"].data + dt2 * f["rdxc"].data / (2 * D) * (-2 * al * ga)
    assert np.allclose(r["uc_out"].data, exp_u, rtol=1e-15, atol=1e-16)
    assert np.array_equal(r["vc_out"].data, f["vc"].data)  # no j-tilt -> exact cancellation


# ------------------------------------------------------------------------------------------- nh_p_grad
def test_nh_p_grad_flat_levels():
    # horizontally uniform gz, pk3, pp: du = dv = 0 and the non-hydrostatic bracket cancels ->
    # u_out = u * rdx exactly
    domain = (4, 4, 3)
    f = synth.make_inputs("nh_p_grad", domain, seed=4)
    for n in ("gz", "pk3", "pp"):
        d = f[n].data
        d[:] = d[:, :1, :1]
    r = _unf("nh_p_grad", f, domain)
    assert np.array_equal(r["u_out"].data, f["u"].data * f["rdx"].data)
    assert np.array_equal(r["v_out"].data, f["v"].data * f["rdy"].data)


def test_nh_p_grad_tilted_closed_form():
    # gz = al*i - k, pk3 = k, pp = ga*k, delp = D: wk = 1;
    # du = dt/2 * ((1-... )) = dt/2 * ((-1-al)*1 + (1-al)*1) = -dt*al;
    # nonhydrostatic = dt/(2D) * ((-1-al)ga + (1-al)ga) = -dt*al*ga/D
    domain = (4, 3, 2)
    f = synth.make_inputs("nh_p_grad", domain, seed=5)
    al, ga, D = 0.5, 0.25, 2.0
    i, j, k = _grid(f["gz"])
    f["gz"].data[:] = al * i - k
    f["pk3"].data[:] = _grid(f["pk3"])[2]
    f["pp"].data[:] = ga * _grid(f["pp"])[2]
    f["delp"].data[:] = D
    dt = synth.scalars("nh_p_grad")["dt"]
    r = _unf("nh_p_grad", f, domain)
    exp = (f["u"].data + (-dt * al) + (-dt * al * ga / D)) * f["rdx"].data
    assert np.allclose(r["u_out"].data, exp, rtol=1e-15, atol=1e-16)
    assert np.array_equal(r["v_out"].data, f["v"].data * f["rdy"].data)


# ---------------------------------------------------------------------------------------------- fvtp2d
def test_ppm_exact_for_linear_q():
    # PPM textbook property: for linear q = j the 4th-order edge value is exact (al = j - 1/2),
    # bl = -1/2, br = +1/2, and the flux through face j-1/2 is the mean of q over the departure
    # interval, j - 1/2 - c/2, for either sign of c (both branches of the upwind `if`)
    domain = (3, 6, 2)
    f = synth.make_inputs("fvtp2d_qi", domain, seed=6)
    f["q"].data[:] = _grid(f["q"])[1]
    r = _unf("fvtp2d_qi", f, domain)
    j = np.arange(6).reshape(1, 6, 1)
    c = f["cry"].data[:, 0:6, :]
    assert (c > 0).any() and (c < 0).any()
    assert np.allclose(r["fy2"].data, j - 0.5 - c / 2, rtol=0, atol=2e-15)


def test_ppm_mirror_symmetry():
    # reflecting q in i and negating the Courant number mirrors the flux: flux(q, c)(face i) ==
    # flux(q_reflected, -c)(face mirrored) -- pins the two upwind branches against each other
    domain = (8, 2, 1)
    f = synth.make_inputs("fvtp2d_qj", domain, seed=7)
    r = _unf("fvtp2d_qj", f, domain)
    N = 8
    g = {n: v.copy() for n, v in f.items()}
    # q over i in [-3, N+3): reflection about the centre of the domain: q'(i) = q(N-1-i)
    g["q"].data[:] = f["q"].data[:, :, ::-1]
    # face i (between i-1 and i) maps to face N-i; c'(face N-i) = -c(face i)
    c = f["crx"].data  # faces 0..N
    g["crx"].data[:] = -c[:, :, ::-1]
    r2 = _unf("fvtp2d_qj", g, domain)
    # fx2(face i) for i in [1, N) compares with fx2'(face N-i)
    a = r["fx2"].data[:, :, 1:N]
    b = r2["fx2"].data[:, :, 1:N][:, :, ::-1]
    assert np.allclose(a, b, rtol=0, atol=1e-15)


def test_qi_uniform_state_closed_form():
    # q constant and yfx, cry uniform: the fluxes through both faces are identical, so
    # q_i = q * area / ra_y (mass conservation of a uniform state)
    domain = (3, 4, 2)
    f = synth.make_inputs("fvtp2d_qi", domain, seed=8)
    f["q"].data[:] = 0.625
    f["cry"].data[:] = 0.25
    f["yfx"].data[:] = -0.125
    r = _unf("fvtp2d_qi", f, domain)
    # (q*area + F) - F rounds once more than q*area: equal to ~1 ulp
    assert np.allclose(r["q_i"].data, 0.625 * f["area"].data / f["ra_y"].data, rtol=4e-16, atol=0)


def test_qi_flux_divergence_closed_form():
    # linear q = j, uniform cry = c and yfx = Y: the PPM flux is exact, fy2(j) = j - 1/2 - c/2, so
    # fyy(j) - fyy(j+1) = -Y and q_i = (j area - Y) / ra_y.  The sign of the divergence is pinned:
    # fyy(j+1) - fyy(j) would give (j area + Y) / ra_y.  Both branches of the upwind `if`.
    domain = (3, 6, 2)
    j = np.arange(6).reshape(1, 6, 1)
    for c, Y in ((0.25, 0.5), (-0.375, -0.75)):
        f = synth.make_inputs("fvtp2d_qi", domain, seed=21)
        f["q"].data[:] = _grid(f["q"])[1]
        f["cry"].data[:] = c
        f["yfx"].data[:] = Y
        r = _unf("fvtp2d_qi", f, domain)
        area = f["area"].data[:, 0:6, :]
        ra = f["ra_y"].data[:, 0:6, :]
        assert np.allclose(r["q_i"].data, (j * area - Y) / ra, rtol=1e-14, atol=1e-14)
        assert not np.allclose(r["q_i"].data, (j * area + Y) / ra, rtol=1e-3, atol=1e-3)


def test_qj_flux_divergence_closed_form():
    # the i analogue for q_j: q = i, uniform crx = c, xfx = X: fx2(i) = i - 1/2 - c/2,
    # q_j = (i area - X) / ra_x; fx (the flux of q_i) is independent of q
    domain = (6, 3, 2)
    i = np.arange(6).reshape(1, 1, 6)
    for c, X in ((0.375, 0.25), (-0.125, -0.5)):
        f = synth.make_inputs("fvtp2d_qj", domain, seed=22)
        f["q"].data[:] = _grid(f["q"])[0]
        f["crx"].data[:] = c
        f["xfx"].data[:] = X
        r = _unf("fvtp2d_qj", f, domain)
        area = f["area"].data[:, :, 0:6]
        ra = f["ra_x"].data[:, :, 0:6]
        assert np.allclose(r["fx2"].data, i - 0.5 - c / 2, rtol=0, atol=2e-15)
        assert np.allclose(r["q_j"].data, (i * area - X) / ra, rtol=1e-14, atol=1e-14)
        assert not np.allclose(r["q_j"].data, (i * area + X) / ra, rtol=1e-3, atol=1e-3)


def test_qj_uniform_state_closed_form():
    domain = (4, 3, 2)
    f = synth.make_inputs("fvtp2d_qj", domain, seed=9)
    f["q"].data[:] = -0.375
    f["q_i"].data[:] = 0.5
    f["crx"].data[:] = -0.25
    f["xfx"].data[:] = 0.75
    r = _unf("fvtp2d_qj", f, domain)
    assert np.allclose(r["q_j"].data, -0.375 * f["area"].data / f["ra_x"].data, rtol=4e-16, atol=0)
    assert np.allclose(r["fx"].data, 0.5, rtol=0, atol=1e-15)
    assert np.allclose(r["fx2"].data, -0.375, rtol=0, atol=1e-15)


def test_flux_average_closed_form():
    # fx_out = 0.5*(fx + fx2)*mfx exactly; fy of linear q_j = j is j - 1/2 - c/2
    domain = (3, 5, 2)
    f = synth.make_inputs("fvtp2d_flux", domain, seed=10)
    f["q_j"].data[:] = _grid(f["q_j"])[1]
    r = _unf("fvtp2d_flux", f, domain)
    assert np.array_equal(r["fx_out"].data, 0.5 * (f["fx"].data + f["fx2"].data) * f["mfx"].data)
    j = np.arange(5).reshape(1, 5, 1)
    fy = j - 0.5 - f["cry"].data / 2
    assert np.allclose(r["fy_out"].data, 0.5 * (fy + f["fy2"].data) * f["mfy"].data, rtol=0, atol=4e-15)


# ------------------------------------------------------------------------------------------- fastwaves
def test_fastwaves_constant_pressure():
    # ppuv constant, wgtfac = 1/2: ppgk == ppuv exactly, ppgc == 0, ppgu == ppgv == 0
    # -> u_out = u_pos + u_tens*dt exactly
    domain = (4, 4, 3)
    f = synth.make_inputs("fastwaves", domain, seed=11)
    f["ppuv"].data[:] = 0.375
    f["wgtfac"].data[:] = 0.5
    sc = synth.scalars("fastwaves")
    r = _unf("fastwaves", f, domain)
    assert np.array_equal(r["u_out"].data, f["u_pos"].data + f["u_tens"].data * sc["dt"])
    assert np.array_equal(r["v_out"].data, f["v_pos"].data + f["v_tens"].data * sc["dt"])


def test_fastwaves_flat_levels_horizontal_gradient():
    # horizontally uniform hhl: the terrain correction numerator is 0 -> ppgu = ppuv(i+1)-ppuv;
    # ppuv = al*i + be*j: u_out = u_pos + (u_tens - al*2*fx/(2 rho)) dt with rho constant
    domain = (4, 3, 2)
    f = synth.make_inputs("fastwaves", domain, seed=12)
    d = f["hhl"].data
    d[:] = d[:, :1, :1]
    al, be = 0.25, -0.5
    i, j, k = _grid(f["ppuv"])
    f["ppuv"].data[:] = al * i + be * j
    f["rho"].data[:] = 1.25
    sc = synth.scalars("fastwaves")
    r = _unf("fastwaves", f, domain)
    exp_u = f["u_pos"].data + (f["u_tens"].data - al * 2.0 * f["fx"].data / 2.5) * sc["dt"]
    exp_v = f["v_pos"].data + (f["v_tens"].data - be * 2.0 * sc["edadlat"] / 2.5) * sc["dt"]
    assert np.allclose(r["u_out"].data, exp_u, rtol=1e-15, atol=1e-16)
    assert np.allclose(r["v_out"].data, exp_v, rtol=1e-15, atol=1e-16)


def test_fastwaves_sloped_coordinate_closed_form():
    # ppuv = be*k (horizontally uniform), hhl = -k + tau*i: ppgc = be, and the terrain-following
    # correction gives ppgu = (2 be) 0.5 (-2 tau) / (-2) = be*tau (pressure gradient along the
    # sloped coordinate surface); ppgv = 0
    domain = (4, 3, 3)
    f = synth.make_inputs("fastwaves", domain, seed=13)
    be, tau = 0.5, 0.25
    f["ppuv"].data[:] = be * _grid(f["ppuv"])[2]
    i, j, k = _grid(f["hhl"])
    f["hhl"].data[:] = -k + tau * i
    f["wgtfac"].data[:] = 0.5
    f["rho"].data[:] = 1.0
    sc = synth.scalars("fastwaves")
    r = _unf("fastwaves", f, domain)
    exp_u = f["u_pos"].data + (f["u_tens"].data - (be * tau) * 2.0 * f["fx"].data / 2.0) * sc["dt"]
    assert np.allclose(r["u_out"].data, exp_u, rtol=1e-15, atol=1e-16)
    assert np.array_equal(r["v_out"].data, f["v_pos"].data + f["v_tens"].data * sc["dt"])
