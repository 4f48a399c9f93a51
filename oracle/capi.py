"""ctypes loader for the C oracle (oracle/oec_oracle.c).  TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).  `build()` compiles it with gcc -O2 -fno-fast-math -ffp-contract=off
-fopenmp ("no fused multiply-add"), twice: the fp64 instance and the
binary32 instance (-DORACLE_F32, entry points *_f32; P:556 evaluates both precisions).  The
functions below pick the instance from the fields' numpy dtype (all fields of a call alike)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, Sequence

import numpy as np

from synth import HostField

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "oec_oracle.c")
LIB = os.path.join(_HERE, "liboec_oracle.so")

CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(__file__)):
        objs = []
        for tag, defs in (("f64", []), ("f32", ["-DORACLE_F32"])):
            obj = os.path.join(_HERE, f"oec_oracle_{tag}.o")
            subprocess.check_call(["gcc", *[f for f in CFLAGS if f != "-shared"], *defs, "-c", SRC, "-o", obj])
            objs.append(obj)
        subprocess.check_call(["gcc", "-shared", "-fopenmp", *objs, "-o", LIB, "-lm"])
        for o in objs:
            os.remove(o)
    return LIB


class OField(C.Structure):
    _fields_ = [
        ("d", C.c_void_p),
        ("lb", C.c_int64 * 3),
        ("ub", C.c_int64 * 3),
        ("k_invariant", C.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(LIB)
        P = C.POINTER(OField)
        I3 = C.POINTER(C.c_int64)
        for sfx in ("", "_f32"):
            getattr(_lib, "oracle_hdiff" + sfx).argtypes = [P, P, P, I3, I3, C.c_int, C.c_int]
            getattr(_lib, "oracle_vadv" + sfx).argtypes = [P, P, P, P, P, P, C.c_double, I3, I3, C.c_int, C.c_int]
            getattr(_lib, "oracle_vadv_system" + sfx).argtypes = [P, P, P, P, P, C.c_double, C.c_int64, C.c_int64,
                                                                  C.c_int64, C.c_int64] + [C.c_void_p] * 4
        _lib.oracle_max_threads.restype = C.c_int
    return _lib


def _sfx(*fields: HostField) -> str:
    dts = {f.data.dtype for f in fields}
    assert len(dts) == 1 and dts <= {np.dtype(np.float64), np.dtype(np.float32)}, dts
    return "_f32" if np.dtype(np.float32) in dts else ""


def _of(f: HostField) -> OField:
    assert f.data.dtype in (np.float64, np.float32) and f.data.flags.c_contiguous
    o = OField()
    o.d = f.data.ctypes.data
    o.lb = (C.c_int64 * 3)(*f.lb)
    o.ub = (C.c_int64 * 3)(*f.ub)
    o.k_invariant = int(f.k_invariant)
    return o


def _i3(v: Sequence[int]):
    return (C.c_int64 * 3)(*v)


class OracleError(RuntimeError):
    pass


HDIFF_UNFUSED, HDIFF_FUSED, HDIFF_FUSED_REVERSED, HDIFF_NO_LIMITER = 0, 1, 2, 3
VADV_UNFUSED, VADV_FUSED, VADV_FUSED_REVERSED = 0, 1, 2


def hdiff(inp: HostField, coeff: HostField, out: HostField, lo, hi, variant: int = HDIFF_UNFUSED, nthreads: int = 1):
    fn = getattr(lib(), "oracle_hdiff" + _sfx(inp, coeff, out))
    rc = fn(C.byref(_of(inp)), C.byref(_of(coeff)), C.byref(_of(out)), _i3(lo), _i3(hi), variant, nthreads)
    if rc:
        raise OracleError(f"oracle_hdiff returned {rc} (2 = out-of-range access)")
    return out


def vadv(f: Dict[str, HostField], out: HostField, dtr_stage: float, lo, hi, variant: int = VADV_UNFUSED, nthreads: int = 1):
    names = ("u_stage", "wcon", "u_pos", "utens", "utens_stage_in")
    fn = getattr(lib(), "oracle_vadv" + _sfx(out, *(f[n] for n in names)))
    rc = fn(
        C.byref(_of(f["u_stage"])),
        C.byref(_of(f["wcon"])),
        C.byref(_of(f["u_pos"])),
        C.byref(_of(f["utens"])),
        C.byref(_of(f["utens_stage_in"])),
        C.byref(_of(out)),
        dtr_stage,
        _i3(lo),
        _i3(hi),
        variant,
        nthreads,
    )
    if rc:
        raise OracleError(f"oracle_vadv returned {rc}")
    return out


def vadv_system(f: Dict[str, HostField], dtr_stage: float, i: int, j: int, k_lo: int, k_hi: int):
    n = k_hi - k_lo
    names = ("u_stage", "wcon", "u_pos", "utens", "utens_stage_in")
    sfx = _sfx(*(f[x] for x in names))
    a, b, c, d = (np.zeros(n, dtype=np.float32 if sfx else np.float64) for _ in range(4))
    ptr = lambda x: x.ctypes.data  # noqa: E731
    rc = getattr(lib(), "oracle_vadv_system" + sfx)(
        C.byref(_of(f["u_stage"])),
        C.byref(_of(f["wcon"])),
        C.byref(_of(f["u_pos"])),
        C.byref(_of(f["utens"])),
        C.byref(_of(f["utens_stage_in"])),
        dtr_stage,
        i,
        j,
        k_lo,
        k_hi,
        ptr(a),
        ptr(b),
        ptr(c),
        ptr(d),
    )
    if rc:
        raise OracleError(f"oracle_vadv_system returned {rc}")
    return a, b, c, d


def max_threads() -> int:
    return int(lib().oracle_max_threads())
