"""The remaining benchmark stencil programs, written for oracle/stencil.py.  TEST INFRASTRUCTURE ONLY.

PAPER.md gives these programs only as a census (Table II: dims / apply ops /
inputs-outputs / arith ops / access ops / control flow) and one sentence each ("The
fvtp2d kernels implement a monotone two-dimensional finite volume advection operator, the
p_grad_c and nh_p_grad kernels compute the three-dimensional pressure gradient, and the uvbke
kernel is a preprocessing step for the kinetic energy computation").  The formulas are
reconstructions from the public FV3 sources [EXT] (readings R12-R17); fastwaves is
not in PAPER.md at all (north_star; COSMO fast-waves u/v [EXT], reading R17).

Pins (tests/test_oracle_suite.py):
  * census vs Table II -- all six programs match every column exactly (the fvtp2d PPM written
    as enumerated in DESIGN.md reading R15);
  * closed-form flux divergence of fvtp2d_qi / fvtp2d_qj (linear q, uniform Courant number);
  * closed forms / special cases for every program (constant, linear and flat fields);
  * unfused (materialised) == fused (inlined) bitwise, extents == brute-force touched set.
  The VALUES of these programs are "parity unpinned" against the paper: PAPER.md prints none.

Notation: a(name, di, dj, dk) = stencil.access; s[...] scalars; sel(c, x, y) = loop.if
with a yielded result.  Python evaluates `x * y / z` left to right, which fixes the
operation order the CUDA kernels reproduce.
"""
from __future__ import annotations

from oracle.stencil import Apply, Program, kdiv

# ---------------------------------------------------------------------------------------------
# uvbke (FV3 d_sw.F90 ub/vb)  -- Table II: 2 / 2 / 4/2 / 12 / 12 / -
# ---------------------------------------------------------------------------------------------
UVBKE = Program(
    "uvbke",
    inputs=("uc", "vc", "cosa", "rsina"),
    outputs=(("ub", "ub"), ("vb", "vb")),
    scalars=("dt5",),
    applies=(
        Apply(("ub",), lambda a, s, sel: s["dt5"] * ((a("uc", 0, -1) + a("uc")) - (a("vc", -1, 0) + a("vc")) * a("cosa")) * a("rsina")),
        Apply(("vb",), lambda a, s, sel: s["dt5"] * ((a("vc", -1, 0) + a("vc")) - (a("uc", 0, -1) + a("uc")) * a("cosa")) * a("rsina")),
    ),
)

# ---------------------------------------------------------------------------------------------
# p_grad_c (FV3 dyn_core.F90, non-hydrostatic: wk = delpc) -- Table II: 3 / 3 / 7/2 / 24 / 25 / -
# gz and pkc live on the K+1 interfaces (k+1 accesses).
# ---------------------------------------------------------------------------------------------
P_GRAD_C = Program(
    "p_grad_c",
    inputs=("uc", "vc", "delpc", "pkc", "gz", "rdxc", "rdyc"),
    outputs=(("uc_out", "uc_out"), ("vc_out", "vc_out")),
    scalars=("dt2",),
    applies=(
        Apply(("wk",), lambda a, s, sel: a("delpc")),
        Apply(
            ("uc_out",),
            lambda a, s, sel: a("uc")
            + s["dt2"] * a("rdxc") / (a("wk", -1, 0) + a("wk"))
            * ((a("gz", -1, 0, 1) - a("gz")) * (a("pkc", 0, 0, 1) - a("pkc", -1, 0))
               + (a("gz", -1, 0) - a("gz", 0, 0, 1)) * (a("pkc", -1, 0, 1) - a("pkc"))),
        ),
        Apply(
            ("vc_out",),
            lambda a, s, sel: a("vc")
            + s["dt2"] * a("rdyc") / (a("wk", 0, -1) + a("wk"))
            * ((a("gz", 0, -1, 1) - a("gz")) * (a("pkc", 0, 0, 1) - a("pkc", 0, -1))
               + (a("gz", 0, -1) - a("gz", 0, 0, 1)) * (a("pkc", 0, -1, 1) - a("pkc"))),
        ),
    ),
)

# ---------------------------------------------------------------------------------------------
# nh_p_grad (FV3 nh_utils.F90) -- Table II: 3 / 5 / 8/2 / 47 / 48 / -
# wk = pk3(k+1) - pk3(k); du/dv = hydrostatic gradient; u/v += du + non-hydrostatic part, * rdx/rdy
# ---------------------------------------------------------------------------------------------
NH_P_GRAD = Program(
    "nh_p_grad",
    inputs=("u", "v", "pp", "gz", "pk3", "delp", "rdx", "rdy"),
    outputs=(("u_out", "u_out"), ("v_out", "v_out")),
    scalars=("dt",),
    applies=(
        Apply(("wk",), lambda a, s, sel: a("pk3", 0, 0, 1) - a("pk3")),
        Apply(
            ("du",),
            lambda a, s, sel: s["dt"] / (a("wk") + a("wk", 1, 0))
            * ((a("gz", 0, 0, 1) - a("gz", 1, 0)) * (a("pk3", 1, 0, 1) - a("pk3"))
               + (a("gz") - a("gz", 1, 0, 1)) * (a("pk3", 0, 0, 1) - a("pk3", 1, 0))),
        ),
        Apply(
            ("dv",),
            lambda a, s, sel: s["dt"] / (a("wk") + a("wk", 0, 1))
            * ((a("gz", 0, 0, 1) - a("gz", 0, 1)) * (a("pk3", 0, 1, 1) - a("pk3"))
               + (a("gz") - a("gz", 0, 1, 1)) * (a("pk3", 0, 0, 1) - a("pk3", 0, 1))),
        ),
        Apply(
            ("u_out",),
            lambda a, s, sel: (a("u") + a("du") + s["dt"] / (a("delp") + a("delp", 1, 0))
                               * ((a("gz", 0, 0, 1) - a("gz", 1, 0)) * (a("pp", 1, 0, 1) - a("pp"))
                                  + (a("gz") - a("gz", 1, 0, 1)) * (a("pp", 0, 0, 1) - a("pp", 1, 0))))
            * a("rdx"),
        ),
        Apply(
            ("v_out",),
            lambda a, s, sel: (a("v") + a("dv") + s["dt"] / (a("delp") + a("delp", 0, 1))
                               * ((a("gz", 0, 0, 1) - a("gz", 0, 1)) * (a("pp", 0, 1, 1) - a("pp"))
                                  + (a("gz") - a("gz", 0, 1, 1)) * (a("pp", 0, 0, 1) - a("pp", 0, 1))))
            * a("rdy"),
        ),
    ),
)

# ---------------------------------------------------------------------------------------------
# fv_tp_2d (FV3 tp_core.F90) split into the paper's three programs.  The 1D PPM flux of q
# through the face at the lower side of cell (i,j) with Courant number c (reading R14):
#   al = (7/12) (q[-1] + q) - (1/12) (q[-2] + q[+1])                  (4th-order edge value)
#   bl = al - q,  br = al[+1] - q
#   flux = c > 0 ? q[-1] + (1 - c)(br[-1] - c (bl[-1] + br[-1]))       (upwind `if`)
#               : q    + (1 + c)(bl     + c (bl     + br    ))
# Written as the paper's programs are counted (reading R15): the weights are the quotients
# 7/12 and 1/12 of the text (two arithmetic operations), and the condition and each branch
# region of the `if` read c themselves (three accesses).  Numerically this is the same as
# literal weights p1 = 7/12, p2 = -1/12 and one read of c: a + (-p) x == a - p x exactly.
# ---------------------------------------------------------------------------------------------
P1 = 7.0 / 12.0
P2 = -1.0 / 12.0


def _ppm(q: str, c: str, al: str, bl: str, br: str, flux: str, dim: str):
    def o(d):
        return (0, d) if dim == "j" else (d, 0)

    def f_al(a, s, sel):
        return kdiv(sel, 7.0, 12.0) * (a(q, *o(-1)) + a(q)) - kdiv(sel, 1.0, 12.0) * (a(q, *o(-2)) + a(q, *o(1)))

    def f_blbr(a, s, sel):
        qq = a(q)
        return a(al) - qq, a(al, *o(1)) - qq

    def f_flux(a, s, sel):
        cc = a(c)  # the condition's read
        c1 = a(c)  # the c > 0 region's read
        c2 = a(c)  # the else region's read
        blm, brm = a(bl, *o(-1)), a(br, *o(-1))
        bl0, br0 = a(bl), a(br)
        return sel(cc > 0.0,
                   a(q, *o(-1)) + (1.0 - c1) * (brm - c1 * (blm + brm)),
                   a(q) + (1.0 + c2) * (bl0 + c2 * (bl0 + br0)))

    return (Apply((al,), f_al), Apply((bl, br), f_blbr), Apply((flux,), f_flux))


# Table II: 2 / 5 / 5/2 / 27 / 23 / if
FVTP2D_QI = Program(
    "fvtp2d_qi",
    inputs=("q", "cry", "yfx", "area", "ra_y"),
    outputs=(("q_i", "q_i"), ("fy2", "fy2")),
    applies=_ppm("q", "cry", "al", "bl", "br", "fy2", "j") + (
        Apply(("fyy",), lambda a, s, sel: a("yfx") * a("fy2")),
        Apply(("q_i",), lambda a, s, sel: (a("q") * a("area") + a("fyy") - a("fyy", 0, 1)) / a("ra_y")),
    ),
)

# Table II: 2 / 8 / 6/3 / 49 / 39 / if
FVTP2D_QJ = Program(
    "fvtp2d_qj",
    inputs=("q", "q_i", "crx", "xfx", "area", "ra_x"),
    outputs=(("q_j", "q_j"), ("fx", "fx"), ("fx2", "fx2")),
    applies=_ppm("q_i", "crx", "al", "bl", "br", "fx", "i")
    + _ppm("q", "crx", "al2", "bl2", "br2", "fx2", "i")
    + (
        Apply(("fx1",), lambda a, s, sel: a("xfx") * a("fx2")),
        Apply(("q_j",), lambda a, s, sel: (a("q") * a("area") + a("fx1") - a("fx1", 1, 0)) / a("ra_x")),
    ),
)

# Table II: 2 / 5 / 7/2 / 28 / 22 / if
FVTP2D_FLUX = Program(
    "fvtp2d_flux",
    inputs=("q_j", "cry", "fx", "fx2", "fy2", "mfx", "mfy"),
    outputs=(("fx_out", "fx_out"), ("fy_out", "fy_out")),
    applies=_ppm("q_j", "cry", "al", "bl", "br", "fy", "j") + (
        Apply(("fx_out",), lambda a, s, sel: 0.5 * (a("fx") + a("fx2")) * a("mfx")),
        Apply(("fy_out",), lambda a, s, sel: 0.5 * (a("fy") + a("fy2")) * a("mfy")),
    ),
)

# ---------------------------------------------------------------------------------------------
# fastwaves (COSMO fast_waves_sc u/v update) [EXT, reading R17].  Not in PAPER.md.
#   ppgk  = wgtfac ppuv + (1 - wgtfac) ppuv[k-1]          pressure at the half level k-1/2
#   ppgc  = ppgk[k+1] - ppgk                               vertical pressure difference
#   ppgu  = (ppuv[i+1] - ppuv) + (ppgc[i+1] + ppgc) 0.5 ((hhl[k+1] + hhl) - (hhl[i+1,k+1] + hhl[i+1]))
#                                                   / ((hhl[k+1] - hhl) + (hhl[i+1,k+1] - hhl[i+1]))
#   u_out = u_pos + (u_tens - ppgu 2 fx / (rho[i+1] + rho)) dt       (v: j, edadlat)
# The caller's k-halo of ppuv (k = -1, K) and of wgtfac/hhl (k = K) replaces the model's
# top/bottom special levels (reading R17).
# ---------------------------------------------------------------------------------------------
def _ppg(d):
    def o(x, dk=0):
        return (x, 0, dk) if d == "i" else (0, x, dk)

    return lambda a, s, sel: (a("ppuv", *o(1)) - a("ppuv")) + (a("ppgc", *o(1)) + a("ppgc")) * 0.5 * (
        (a("hhl", 0, 0, 1) + a("hhl")) - (a("hhl", *o(1, 1)) + a("hhl", *o(1)))
    ) / ((a("hhl", 0, 0, 1) - a("hhl")) + (a("hhl", *o(1, 1)) - a("hhl", *o(1))))


FASTWAVES = Program(
    "fastwaves",
    inputs=("u_pos", "v_pos", "u_tens", "v_tens", "rho", "ppuv", "fx", "wgtfac", "hhl"),
    outputs=(("u_out", "u_out"), ("v_out", "v_out")),
    scalars=("edadlat", "dt"),
    applies=(
        Apply(("ppgk",), lambda a, s, sel: a("wgtfac") * a("ppuv") + (1.0 - a("wgtfac")) * a("ppuv", 0, 0, -1)),
        Apply(("ppgc",), lambda a, s, sel: a("ppgk", 0, 0, 1) - a("ppgk")),
        Apply(("ppgu",), _ppg("i")),
        Apply(("ppgv",), _ppg("j")),
        Apply(("u_out",), lambda a, s, sel: a("u_pos") + (a("u_tens") - a("ppgu") * 2.0 * a("fx") / (a("rho", 1, 0) + a("rho"))) * s["dt"]),
        Apply(("v_out",), lambda a, s, sel: a("v_pos") + (a("v_tens") - a("ppgv") * 2.0 * s["edadlat"] / (a("rho", 0, 1) + a("rho"))) * s["dt"]),
    ),
)

# ---------------------------------------------------------------------------------------------
# hdiff in the same notation (a third, independent writing of the definition in
# oracle/oec_oracle.c; used for the extent / census checks and as a cross-check).
# ---------------------------------------------------------------------------------------------
HDIFF = Program(
    "hdiff",
    inputs=("in", "coeff"),
    outputs=(("out", "out"),),
    applies=(
        Apply(("lap",), lambda a, s, sel: ((a("in", -1, 0) + a("in", 1, 0)) + (a("in", 0, -1) + a("in", 0, 1))) - 4.0 * a("in")),
        Apply(("flx",), lambda a, s, sel: (lambda f: sel(f * (a("in", 1, 0) - a("in")) > 0.0, 0.0, f))(a("lap", 1, 0) - a("lap"))),
        Apply(("fly",), lambda a, s, sel: (lambda g: sel(g * (a("in", 0, 1) - a("in")) > 0.0, 0.0, g))(a("lap", 0, 1) - a("lap"))),
        Apply(("out",), lambda a, s, sel: a("in") - a("coeff") * ((a("flx") - a("flx", -1, 0)) + (a("fly") - a("fly", 0, -1)))),
    ),
)

PROGRAMS = {p.name: p for p in (UVBKE, P_GRAD_C, NH_P_GRAD, FVTP2D_QI, FVTP2D_QJ, FVTP2D_FLUX, FASTWAVES, HDIFF)}

# Table II: dims, apply ops, inputs, outputs, arith ops, access ops, control flow
TABLE_II = {
    "p_grad_c": (3, 3, 7, 2, 24, 25, False),
    "nh_p_grad": (3, 5, 8, 2, 47, 48, False),
    "uvbke": (2, 2, 4, 2, 12, 12, False),
    "fvtp2d_qi": (2, 5, 5, 2, 27, 23, True),
    "fvtp2d_qj": (2, 8, 6, 3, 49, 39, True),
    "fvtp2d_flux": (2, 5, 7, 2, 28, 22, True),
}
