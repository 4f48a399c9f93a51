"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no stencil, no solve): it only draws seeded
random numbers into host arrays of the right shape, following the input recipe of DESIGN.md
("Input recipe") / SURVEY.md §8(d).  Both the oracle (oracle/) and the CUDA path
(paper_2005_13014_b200/) receive exactly these arrays.

Data model (§4.2 "Shapes & Domains"): a field is a dense
host array over its allocated range [lb, ub) in absolute coordinates whose origin is the lower
bound of the computation domain.  Array index order is [k][j][i] (i fastest).  A k-invariant
("2D", metric) field has lb[2] = 0, ub[2] = 1 and is broadcast along k.

The allocation recipe (halo widths per input) below is configuration, not method arithmetic; the
oracle's brute-force touched-index tracer checks it covers what each program reads
(tests/test_oracle_extents.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field as dc_field
from typing import Dict, List, Tuple

import numpy as np

Int3 = Tuple[int, int, int]


@dataclass
class HostField:
    """Dense host array over [lb, ub) (absolute coords, origin = domain lower bound)."""

    data: np.ndarray  # float64 (or float32), shape (ub2-lb2, ub1-lb1, ub0-lb0) -> [k][j][i]
    lb: Int3
    ub: Int3
    k_invariant: bool = False

    def copy(self) -> "HostField":
        return HostField(self.data.copy(), self.lb, self.ub, self.k_invariant)

    @property
    def shape_ijk(self) -> Int3:
        return tuple(self.ub[d] - self.lb[d] for d in range(3))  # type: ignore[return-value]


@dataclass(frozen=True)
class InputSpec:
    name: str
    halo_lo: Int3  # cells below the domain lower bound, per dim (i, j, k)
    halo_hi: Int3  # cells above the domain upper bound, per dim (i, j, k)
    dist: str  # value distribution, see _draw
    k_invariant: bool = False  # 2D metric field broadcast along k


@dataclass(frozen=True)
class ProgramSpec:
    name: str
    inputs: Tuple[InputSpec, ...]
    outputs: Tuple[str, ...]
    scalars: Tuple[Tuple[str, float], ...] = ()


Z: Int3 = (0, 0, 0)


def _in(name, lo=Z, hi=Z, dist="u11", k_inv=False):
    return InputSpec(name, lo, hi, dist, k_inv)


# ---------------------------------------------------------------------------------------------
# Allocation recipe per program.  Inputs are listed in the C-ABI argument order (include/oec.h).
# ---------------------------------------------------------------------------------------------
PROGRAMS: Dict[str, ProgramSpec] = {
    # COSMO horizontal diffusion; BASELINE.json configs[0]: "single field + coeff, halo 2".
    "hdiff": ProgramSpec(
        "hdiff",
        (_in("in", (2, 2, 0), (2, 2, 0), "u11"), _in("coeff", dist="coeff")),
        ("out",),
    ),
    # Vertical advection (Thomas solve in k); wcon is staggered in i (+1 on the high side).
    "vadv": ProgramSpec(
        "vadv",
        (
            _in("u_stage"),
            _in("wcon", Z, (1, 0, 0), "wcon"),
            _in("u_pos"),
            _in("utens"),
            _in("utens_stage_in"),
        ),
        ("utens_stage_out",),
        (("dtr_stage", 3.0 / 20.0),),
    ),
    # FV3 d_sw ub/vb (Table II row uvbke).
    "uvbke": ProgramSpec(
        "uvbke",
        (
            _in("uc", (0, 1, 0), Z),
            _in("vc", (1, 0, 0), Z),
            _in("cosa", dist="cosa", k_inv=True),
            _in("rsina", dist="pos", k_inv=True),
        ),
        ("ub", "vb"),
        (("dt5", 0.5 * 225.0 / 1000.0),),
    ),
    # FV3 dyn_core p_grad_c, non-hydrostatic branch (Table II row p_grad_c).
    "p_grad_c": ProgramSpec(
        "p_grad_c",
        (
            _in("uc"),
            _in("vc"),
            _in("delpc", (1, 1, 0), Z, "pos"),
            _in("pkc", (1, 1, 0), (0, 0, 1), "levels_inc"),
            _in("gz", (1, 1, 0), (0, 0, 1), "levels_dec"),
            _in("rdxc", dist="pos", k_inv=True),
            _in("rdyc", dist="pos", k_inv=True),
        ),
        ("uc_out", "vc_out"),
        (("dt2", 0.5 * 225.0 / 1000.0),),
    ),
    # FV3 nh_utils nh_p_grad (Table II row nh_p_grad).
    "nh_p_grad": ProgramSpec(
        "nh_p_grad",
        (
            _in("u"),
            _in("v"),
            _in("pp", Z, (1, 1, 1), "u11"),
            _in("gz", Z, (1, 1, 1), "levels_dec"),
            _in("pk3", Z, (1, 1, 1), "levels_inc"),
            _in("delp", Z, (1, 1, 0), "pos"),
            _in("rdx", dist="pos", k_inv=True),
            _in("rdy", dist="pos", k_inv=True),
        ),
        ("u_out", "v_out"),
        (("dt", 225.0 / 1000.0),),
    ),
    # FV3 tp_core fv_tp_2d, inner y-update (Table II row fvtp2d_qi).
    "fvtp2d_qi": ProgramSpec(
        "fvtp2d_qi",
        (
            _in("q", (0, 3, 0), (0, 3, 0)),
            _in("cry", Z, (0, 1, 0), "courant"),
            _in("yfx", Z, (0, 1, 0), "courant"),
            _in("area", dist="pos", k_inv=True),
            _in("ra_y", dist="pos"),
        ),
        ("q_i", "fy2"),
    ),
    # x-direction inner update (Table II row fvtp2d_qj).
    "fvtp2d_qj": ProgramSpec(
        "fvtp2d_qj",
        (
            _in("q", (3, 0, 0), (3, 0, 0)),
            _in("q_i", (3, 0, 0), (2, 0, 0)),
            _in("crx", Z, (1, 0, 0), "courant"),
            _in("xfx", Z, (1, 0, 0), "courant"),
            _in("area", dist="pos", k_inv=True),
            _in("ra_x", dist="pos"),
        ),
        ("q_j", "fx", "fx2"),
    ),
    # final fluxes (Table II row fvtp2d_flux).
    "fvtp2d_flux": ProgramSpec(
        "fvtp2d_flux",
        (
            _in("q_j", (0, 3, 0), (0, 2, 0)),
            _in("cry", dist="courant"),
            _in("fx"),
            _in("fx2"),
            _in("fy2"),
            _in("mfx", dist="pos"),
            _in("mfy", dist="pos"),
        ),
        ("fx_out", "fy_out"),
    ),
    # COSMO fast-waves u/v update (north_star "fastwaves"; not in PAPER.md).
    "fastwaves": ProgramSpec(
        "fastwaves",
        (
            _in("u_pos"),
            _in("v_pos"),
            _in("u_tens"),
            _in("v_tens"),
            _in("rho", Z, (1, 1, 0), "pos"),
            _in("ppuv", (0, 0, 1), (1, 1, 1), "u11"),
            _in("fx", dist="pos", k_inv=True),
            _in("wgtfac", Z, (1, 1, 1), "wgt"),
            _in("hhl", Z, (1, 1, 1), "levels_dec"),
        ),
        ("u_out", "v_out"),
        (("edadlat", 0.25), ("dt", 10.0 / 1000.0)),
    ),
}

SUITE = ("uvbke", "p_grad_c", "nh_p_grad", "fvtp2d_qi", "fvtp2d_qj", "fvtp2d_flux", "fastwaves")
ALL_PROGRAMS = ("hdiff", "vadv") + SUITE


def alloc_range(spec: InputSpec, domain: Int3) -> Tuple[Int3, Int3]:
    if spec.k_invariant:
        lb = (-spec.halo_lo[0], -spec.halo_lo[1], 0)
        ub = (domain[0] + spec.halo_hi[0], domain[1] + spec.halo_hi[1], 1)
    else:
        lb = tuple(-spec.halo_lo[d] for d in range(3))
        ub = tuple(domain[d] + spec.halo_hi[d] for d in range(3))
    return lb, ub  # type: ignore[return-value]


def _draw(rng: np.random.Generator, dist: str, shape, lb_k: int) -> np.ndarray:
    """Value distributions of SURVEY §8(d) / DESIGN.md "Input recipe"."""
    if dist == "u11":  # prognostic fields
        return rng.uniform(-1.0, 1.0, shape)
    if dist == "coeff":  # hdiff diffusion coefficient
        return rng.uniform(0.0, 0.1, shape)
    if dist == "wcon":  # vadv contravariant vertical velocity: keeps the system diagonally dominant
        return rng.uniform(-0.1, 0.1, shape)
    if dist == "pos":  # strictly positive metric / thickness quantities
        return rng.uniform(0.5, 1.5, shape)
    if dist == "cosa":
        return rng.uniform(-0.1, 0.1, shape)
    if dist == "courant":  # mixed-sign Courant numbers / face fluxes exercise the upwind `if`
        return rng.uniform(-0.5, 0.5, shape)
    if dist == "wgt":  # interpolation weights
        return rng.uniform(0.4, 0.6, shape)
    if dist in ("levels_dec", "levels_inc"):
        # strictly monotone in k (heights decrease, pressures increase with k), level spacing 1 +- 0.2
        nk = shape[0]
        k = np.arange(lb_k, lb_k + nk, dtype=np.float64).reshape(nk, 1, 1)
        noise = rng.uniform(-0.1, 0.1, shape)
        return (-k if dist == "levels_dec" else k) + noise
    raise ValueError(f"unknown distribution {dist!r}")


def make_inputs(program: str, domain: Int3, seed: int = 0, smooth: bool = False,
                dtype=np.float64) -> Dict[str, HostField]:
    """Seeded inputs of `program` on `domain` = (Ni, Nj, Nk).

    Fields are drawn in the fixed order of PROGRAMS[program].inputs from one PCG64(seed)
    stream over their entire allocation.  `smooth` (hdiff only) replaces `in` by the smooth
    field of SURVEY §8(d): sin(2 pi i/Ni) cos(2 pi j/Nj) (1 + k/Nk) + 0.01 U[-1,1].
    dtype=np.float32 draws the same fp64 values and rounds them to binary32 (P:556 f32 runs).
    """
    spec = PROGRAMS[program]
    rng = np.random.Generator(np.random.PCG64(seed))
    out: Dict[str, HostField] = {}
    for s in spec.inputs:
        lb, ub = alloc_range(s, domain)
        shape = (ub[2] - lb[2], ub[1] - lb[1], ub[0] - lb[0])
        data = _draw(rng, s.dist, shape, lb[2])
        if smooth and program == "hdiff" and s.name == "in":
            kk, jj, ii = np.meshgrid(
                np.arange(lb[2], ub[2]), np.arange(lb[1], ub[1]), np.arange(lb[0], ub[0]), indexing="ij"
            )
            data = (
                np.sin(2 * np.pi * ii / domain[0]) * np.cos(2 * np.pi * jj / domain[1]) * (1.0 + kk / domain[2])
                + 0.01 * data
            )
        out[s.name] = HostField(np.ascontiguousarray(data, dtype=np.float64).astype(dtype), lb, ub, s.k_invariant)
    return out


def as_dtype(fields: Dict[str, HostField], dtype) -> Dict[str, HostField]:
    """The same fields converted to `dtype` (float32 -> float64 is exact)."""
    return {n: HostField(np.ascontiguousarray(f.data.astype(dtype)), f.lb, f.ub, f.k_invariant) for n, f in fields.items()}


def scalars(program: str) -> Dict[str, float]:
    return dict(PROGRAMS[program].scalars)


def empty_outputs(program: str, domain: Int3, fill: float = np.nan, dtype=np.float64) -> Dict[str, HostField]:
    """Output fields allocated exactly on the domain, pre-filled with `fill` (sentinel)."""
    res = {}
    for name in PROGRAMS[program].outputs:
        res[name] = HostField(np.full((domain[2], domain[1], domain[0]), fill, dtype=dtype), (0, 0, 0), tuple(domain))
    return res


def probe_field(lb: Int3, ub: Int3) -> HostField:
    """Integer-coded probe field, value = i + 2^10 j + 2^20 k (exact in fp64), SURVEY §4 halo tests."""
    kk, jj, ii = np.meshgrid(np.arange(lb[2], ub[2]), np.arange(lb[1], ub[1]), np.arange(lb[0], ub[0]), indexing="ij")
    return HostField((ii + 1024.0 * jj + 1048576.0 * kk).astype(np.float64), lb, ub)


__all__ = [
    "HostField",
    "InputSpec",
    "ProgramSpec",
    "PROGRAMS",
    "SUITE",
    "ALL_PROGRAMS",
    "alloc_range",
    "make_inputs",
    "as_dtype",
    "scalars",
    "empty_outputs",
    "probe_field",
]
