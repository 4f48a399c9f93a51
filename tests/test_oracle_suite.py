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


@pytest.mark.parametrize("name", ["uvbke", "p_grad_c", "nh_p_grad"])
def test_census_matches_table_ii_exactly(name):
    dims, applies, n_in, n_out, arith, access, cf = suite.TABLE_II[name]
    c = st.census(suite.PROGRAMS[name])
    assert (c["applies"], c["inputs"], c["outputs"], c["arith"], c["access"], c["if"] > 0) == (
        applies, n_in, n_out, arith, access, cf)


@pytest.mark.parametrize("name", ["fvtp2d_qi", "fvtp2d_qj", "fvtp2d_flux"])
def test_census_fvtp2d_structure(name):
    # apply ops, inputs/outputs and control flow match Table II; the arith/access counts of the
    # reconstructed PPM differ by a fixed amount per PPM flux (reading R15)
    dims, applies, n_in, n_out, arith, access, cf = suite.TABLE_II[name]
    c = st.census(suite.PROGRAMS[name])
    assert (c["applies"], c["inputs"], c["outputs"], c["if"] > 0) == (applies, n_in, n_out, cf)
    n_ppm = 2 if name == "fvtp2d_qj" else 1
    assert c["arith"] + c["cmp"] == arith - 2 * n_ppm
    assert c["access"] == access - 2 * n_ppm


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
