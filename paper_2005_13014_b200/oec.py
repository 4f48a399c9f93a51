"""Thin Python binding of liboec's C ABI (include/oec.h): argument marshalling only.

Every function keeps the C name.  Every step of the hot path runs in liboec's sm_100a kernels;
this module only builds `oec_field` descriptors from torch tensors / library allocations, passes
torch's current CUDA stream, and turns a non-OK status into an exception.  PyTorch provides device
memory, streams and process groups -- nothing else.

There is NO fallback: if liboec.so is missing, `lib()` raises.  (The CPU oracle lives in oracle/
and is never imported here.)
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OEC_LIB_PATH") or os.path.join(_HERE, "liboec.so")

OEC_OK = 0
OEC_DEVICE_HOST = -1
OEC_F64 = 0
OEC_F32 = 1
OEC_VARIANT_AUTO = 0
OEC_VARIANT_UNFUSED = 1
OEC_VARIANT_NAIVE = 2
OEC_VARIANT_UNROLL2 = 3
OEC_VARIANT_UNROLL4 = 4
OEC_VARIANT_UNROLL2_K = 5
OEC_VARIANT_UNROLL4_K = 6
OEC_VARIANT_TILED = 7
STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_SHAPE", 3: "ERR_ALIAS", 4: "ERR_DTYPE", 5: "ERR_CUDA", 6: "ERR_NCCL",
          7: "ERR_UNSUPPORTED", 8: "ERR_LAYOUT"}

I64x3 = C.c_int64 * 3
I32x3 = C.c_int32 * 3


class OecField(C.Structure):
    _fields_ = [
        ("data", C.c_void_p),
        ("lb", I64x3),
        ("ub", I64x3),
        ("stride", I64x3),
        ("dtype", C.c_int32),
        ("device", C.c_int32),
        ("owned", C.c_int32),
        ("reserved", C.c_int32),
    ]


class OecHaloMsg(C.Structure):
    _fields_ = [
        ("peer", C.c_int32),
        ("is_send", C.c_int32),
        ("phase", C.c_int32),
        ("tag", C.c_int32),
        ("lo", I64x3),
        ("hi", I64x3),
    ]


class OecError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


# ABI symbols (name, restype, argtypes) -- tests check liboec.so exports all of include/oec.h
_P = C.POINTER(OecField)
_PP = C.POINTER(_P)
SIGNATURES = {
    "oec_abi_version": (C.c_int32, []),
    "oec_build_info": (C.c_char_p, []),
    "oec_last_error": (C.c_char_p, []),
    "oec_last_launch_count": (C.c_int32, []),
    "oec_field_create": (C.c_int, [C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int32, C.c_int32,
                                   C.POINTER(C.c_int32), C.c_int32, _P]),
    "oec_field_wrap": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_int32,
                                 C.c_int32, _P]),
    "oec_field_destroy": (C.c_int, [_P]),
    "oec_program_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "oec_program_input": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(C.c_char_p), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "oec_program_extent": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "oec_program_output": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(C.c_char_p)]),
    "oec_program_scalar": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(C.c_char_p), C.POINTER(C.c_double)]),
    "oec_hdiff": (C.c_int, [_P, _P, _P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_void_p]),
    "oec_hdiff_variant": (C.c_int, [_P, _P, _P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_int32, C.c_void_p]),
    "oec_vadv": (C.c_int, [_P, _P, _P, _P, _P, _P, C.c_double, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_void_p]),
    "oec_apply_program": (C.c_int, [C.c_char_p, _PP, C.c_int32, _PP, C.c_int32, C.POINTER(C.c_double), C.c_int32,
                                    C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_int32, C.c_void_p]),
    "oec_decomp_create": (C.c_int, [C.POINTER(C.c_int64), C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                    C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "oec_decomp_plan": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(OecHaloMsg),
                                  C.c_int32, C.POINTER(C.c_int32)]),
    "oec_halo_exchange": (C.c_int, [C.c_void_p, _PP, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_void_p]),
    "oec_halo_exchange_local": (C.c_int, [C.POINTER(C.c_int64), C.c_int32, C.c_int32, _PP, C.c_int32,
                                          C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_void_p]),
    "oec_halo_exchange_local_periodic": (C.c_int, [C.POINTER(C.c_int64), C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                                   _PP, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                                   C.c_void_p]),
    "oec_decomp_set_periodic": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    "oec_decomp_destroy": (C.c_int, [C.c_void_p]),
    "oec_hdiff_pipeline_create": (C.c_int, [C.POINTER(C.c_int64), C.c_int32, C.c_int32, C.c_int32, _P, _P, _P,
                                            C.POINTER(C.c_void_p)]),
    "oec_hdiff_pipeline_signal_pad": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "oec_hdiff_pipeline_set_peer": (C.c_int, [C.c_void_p, C.c_int32, _P, _P, C.c_void_p]),
    "oec_hdiff_pipeline_run": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "oec_hdiff_pipeline_steps": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "oec_hdiff_pipeline_destroy": (C.c_int, [C.c_void_p]),
    "oec_ipc_export": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]),
    "oec_ipc_import": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_void_p)]),
    "oec_ipc_close": (C.c_int, [C.c_void_p]),
    "oec_program_create": (C.c_int, [C.c_char_p, C.POINTER(C.c_char_p)]),
    "oec_program_destroy": (C.c_int, [C.c_char_p]),
    "oec_program_generate": (C.c_int, [C.c_char_p, _PP, C.c_int32, _PP, C.c_int32, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int64), C.c_int32, C.c_int32, C.c_char_p, C.c_int64,
                                       C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "oec_selftest_rcp32": (C.c_int, [C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]),
    "oec_selftest_rcp": (C.c_int, [C.c_ulonglong, C.c_ulonglong, C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]),
}

_lib = None


def lib():
    """Load liboec.so (built in-tree by paper_2005_13014_b200.build).  Raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} is not built -- run `python -m paper_2005_13014_b200.build` "
                          "(there is no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def _check(status: int):
    if status != OEC_OK:
        raise OecError(status, lib().oec_last_error().decode())


def _i64(v: Sequence[int]):
    return I64x3(*[int(x) for x in v])


def _i32(v: Sequence[int]):
    return I32x3(*[int(x) for x in v])


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch

        if not torch.cuda.is_available():
            return None
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class _CudaArray:
    """__cuda_array_interface__ over a field's allocation, for zero-copy torch views."""

    def __init__(self, ptr: int, shape, strides_bytes, keep, typestr="<f8"):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape),
            "strides": tuple(strides_bytes),
            "typestr": typestr,
            "data": (ptr, False),
            "version": 3,
        }
        self._keep = keep


class Field:
    """An oec_field descriptor plus whatever keeps its memory alive (a torch tensor / numpy array)."""

    def __init__(self, desc: OecField, keep=None):
        self.desc = desc
        self._keep = keep

    @property
    def lb(self) -> Tuple[int, int, int]:
        return tuple(self.desc.lb)  # type: ignore[return-value]

    @property
    def ub(self) -> Tuple[int, int, int]:
        return tuple(self.desc.ub)  # type: ignore[return-value]

    @property
    def stride(self) -> Tuple[int, int, int]:
        return tuple(self.desc.stride)  # type: ignore[return-value]

    @property
    def device(self) -> int:
        return self.desc.device

    @property
    def dtype(self) -> int:
        return self.desc.dtype

    @property
    def itemsize(self) -> int:
        return 4 if self.desc.dtype == OEC_F32 else 8

    @property
    def ptr(self):
        return C.pointer(self.desc)

    def view(self):
        """torch view [k][j][i] of the allocated range [lb, ub) (device fields; zero copy)."""
        import torch

        if self.desc.device < 0:
            return torch.from_numpy(self._keep) if isinstance(self._keep, np.ndarray) else self._keep
        n = [self.desc.ub[d] - self.desc.lb[d] for d in range(3)]
        st = self.desc.stride
        es = self.itemsize
        arr = _CudaArray(self.desc.data, (n[2], n[1], n[0]), (st[2] * es, st[1] * es, st[0] * es), self,
                         "<f4" if es == 4 else "<f8")
        return torch.as_tensor(arr, device=f"cuda:{self.desc.device}")

    def upload(self, host) -> "Field":
        """Copy a dense host array [k][j][i] over [lb, ub) (numpy or synth.HostField) into the field."""
        import torch

        data = getattr(host, "data", host)
        self.view().copy_(torch.from_numpy(np.ascontiguousarray(data)))
        return self

    def fill(self, value: float) -> "Field":
        self.view().fill_(value)
        return self

    def download(self) -> np.ndarray:
        return self.view().cpu().numpy().copy()

    def destroy(self):
        if self.desc.owned:
            _check(lib().oec_field_destroy(C.byref(self.desc)))

    def __del__(self):
        try:
            if self.desc.owned and self.desc.data:
                lib().oec_field_destroy(C.byref(self.desc))
        except Exception:
            pass


# ---------------------------------------------------------------------------------------------
# fields
# ---------------------------------------------------------------------------------------------
def _dtype_code(dtype) -> int:
    """numpy / torch dtype (or an OEC_F* code) -> oec_dtype."""
    if isinstance(dtype, int):
        return dtype
    name = str(dtype).replace("torch.", "")
    if not name.startswith("float") and name not in ("double", "<f8", "<f4"):
        try:
            name = np.dtype(dtype).name  # numpy scalar types, np.dtype objects, strings like "f4"
        except TypeError:
            pass
    if name in ("float64", "double", "<f8"):
        return OEC_F64
    if name in ("float32", "float", "<f4"):
        return OEC_F32
    raise ValueError(f"unsupported dtype {dtype!r} (fp64 or f32)")


def oec_field_create(domain, halo_lo=(0, 0, 0), halo_hi=(0, 0, 0), device: int = 0, order=None,
                     k_invariant: bool = False, dtype=OEC_F64) -> Field:
    d = OecField()
    order_arg = _i32(order) if order is not None else None
    _check(lib().oec_field_create(_i64(domain), _i32(halo_lo), _i32(halo_hi), _dtype_code(dtype), device, order_arg,
                                  int(k_invariant), C.byref(d)))
    return Field(d)


def oec_field_wrap(array, lb, ub, stride=None, device: Optional[int] = None, k_invariant: bool = False) -> Field:
    """Describe caller memory as a field.  `array`: a torch tensor (CUDA -> device field, CPU ->
    OEC_DEVICE_HOST) or a numpy array (host), indexed [k][j][i] over [lb, ub) unless `stride`
    (elements, i/j/k) is given explicitly.  k_invariant: a 2D field broadcast along k."""
    import torch

    d = OecField()
    dt = _dtype_code(array.dtype)
    if isinstance(array, np.ndarray):
        es = array.itemsize
        ptr = array.ctypes.data
        st = stride or (array.strides[2] // es, array.strides[1] // es, array.strides[0] // es)
        dev = OEC_DEVICE_HOST
    else:
        ptr = array.data_ptr()
        st = stride or (array.stride(2), array.stride(1), array.stride(0))
        dev = array.device.index if array.is_cuda else OEC_DEVICE_HOST
        if array.is_cuda and dev is None:
            dev = torch.cuda.current_device()
    if device is not None:
        dev = device
    st = list(st)
    if k_invariant:
        st[2] = 0
    _check(lib().oec_field_wrap(C.c_void_p(ptr), _i64(lb), _i64(ub), _i64(st), dt, dev, C.byref(d)))
    return Field(d, keep=array)


def field_from_host(host, device: int = 0, order=None) -> Field:
    """Allocate a device field (oec_field_create) with the allocation [lb, ub) of a synth.HostField
    (lb <= 0) and upload its data.  The allocation [-halo_lo, domain + halo_hi) is requested as
    halo_lo = -lb, domain = ub, halo_hi = 0, which yields the same range and pitch."""
    lb, ub, kinv = host.lb, host.ub, getattr(host, "k_invariant", False)
    if any(lb[d] > 0 for d in range(3)) or any(ub[d] < 1 for d in range(3)):
        raise ValueError("field_from_host: allocation must contain the origin")
    data = getattr(host, "data", host)
    f = oec_field_create(ub, [-x for x in lb], (0, 0, 0), device=device, order=order, k_invariant=kinv,
                         dtype=data.dtype)
    return f.upload(host)


def empty_like_domain(domain, device: int = 0, order=None, fill: float = float("nan"), dtype=OEC_F64) -> Field:
    f = oec_field_create(domain, (0, 0, 0), (0, 0, 0), device=device, order=order, dtype=dtype)
    return f.fill(fill)


# ---------------------------------------------------------------------------------------------
# registry
# ---------------------------------------------------------------------------------------------
def oec_program_info(program: str) -> Tuple[int, int, int]:
    a, b, c = C.c_int32(), C.c_int32(), C.c_int32()
    _check(lib().oec_program_info(program.encode(), C.byref(a), C.byref(b), C.byref(c)))
    return a.value, b.value, c.value


def oec_program_input(program: str, idx: int):
    name = C.c_char_p()
    lo, hi = I64x3(), I64x3()
    kinv = C.c_int32()
    _check(lib().oec_program_input(program.encode(), idx, C.byref(name), lo, hi, C.byref(kinv)))
    return name.value.decode(), tuple(lo), tuple(hi), bool(kinv.value)


def oec_program_extent(program: str, idx: int):
    """(lo, hi): the access extent of input idx relative to the domain."""
    lo, hi = I64x3(), I64x3()
    _check(lib().oec_program_extent(program.encode(), idx, lo, hi))
    return tuple(lo), tuple(hi)


def oec_program_output(program: str, idx: int) -> str:
    name = C.c_char_p()
    _check(lib().oec_program_output(program.encode(), idx, C.byref(name)))
    return name.value.decode()


def oec_program_scalar(program: str, idx: int):
    name = C.c_char_p()
    v = C.c_double()
    _check(lib().oec_program_scalar(program.encode(), idx, C.byref(name), C.byref(v)))
    return name.value.decode(), v.value


def program_signature(program: str):
    n_in, n_out, n_sc = oec_program_info(program)
    return ([oec_program_input(program, q) for q in range(n_in)], [oec_program_output(program, q) for q in range(n_out)],
            [oec_program_scalar(program, q) for q in range(n_sc)])


# ---------------------------------------------------------------------------------------------
# the hot path
# ---------------------------------------------------------------------------------------------
def oec_hdiff(inp: Field, coeff: Field, out: Field, dom_lb, dom_ub, stream=None, variant: int = OEC_VARIANT_AUTO):
    _check(lib().oec_hdiff_variant(inp.ptr, coeff.ptr, out.ptr, _i64(dom_lb), _i64(dom_ub), variant,
                                   _stream(stream) if inp.device >= 0 else _stream(stream)))


def oec_vadv(u_stage: Field, wcon: Field, u_pos: Field, utens: Field, utens_stage_in: Field, utens_stage_out: Field,
             dtr_stage: float, dom_lb, dom_ub, stream=None):
    _check(lib().oec_vadv(u_stage.ptr, wcon.ptr, u_pos.ptr, utens.ptr, utens_stage_in.ptr, utens_stage_out.ptr,
                          float(dtr_stage), _i64(dom_lb), _i64(dom_ub), _stream(stream)))


def oec_apply_program(program: str, inputs: Sequence[Field], outputs: Sequence[Field], scalars=None,
                      dom_lb=(0, 0, 0), dom_ub=None, variant: int = OEC_VARIANT_AUTO, stream=None):
    ins = (_P * len(inputs))(*[f.ptr for f in inputs])
    outs = (_P * len(outputs))(*[f.ptr for f in outputs])
    if scalars is not None and len(scalars):
        sc = (C.c_double * len(scalars))(*[float(x) for x in scalars])
        nsc = len(scalars)
    else:
        sc, nsc = None, 0
    _check(lib().oec_apply_program(program.encode(), ins, len(inputs), outs, len(outputs), sc, nsc, _i64(dom_lb),
                                   _i64(dom_ub), variant, _stream(stream)))


def oec_program_create(source: str) -> str:
    """Compile a stencil-language program (include/oec.h) and register it; returns its name."""
    name = C.c_char_p()
    _check(lib().oec_program_create(source.encode(), C.byref(name)))
    return name.value.decode()


def oec_program_destroy(program: str):
    _check(lib().oec_program_destroy(program.encode()))


def oec_program_generate(program: str, inputs: Sequence[Field], outputs: Sequence[Field], dom_lb, dom_ub,
                         variant: int = OEC_VARIANT_AUTO, compile: bool = False) -> Tuple[str, int]:
    """The CUDA source liboec generates for this call (and, with compile=True, the NVRTC cubin size)."""
    ins = (_P * len(inputs))(*[f.ptr for f in inputs])
    outs = (_P * len(outputs))(*[f.ptr for f in outputs])
    n, cb = C.c_int64(), C.c_int64()
    _check(lib().oec_program_generate(program.encode(), ins, len(inputs), outs, len(outputs), _i64(dom_lb),
                                      _i64(dom_ub), variant, 0, None, 0, C.byref(n), None))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib().oec_program_generate(program.encode(), ins, len(inputs), outs, len(outputs), _i64(dom_lb),
                                      _i64(dom_ub), variant, int(compile), buf, n.value + 1, C.byref(n), C.byref(cb)))
    return buf.value.decode(), cb.value


def oec_last_launch_count() -> int:
    return int(lib().oec_last_launch_count())


# ---------------------------------------------------------------------------------------------
# decomposition
# ---------------------------------------------------------------------------------------------
class Decomp:
    def __init__(self, handle: C.c_void_p, local_lb, local_ub):
        self.handle = handle
        self.local_lb = tuple(local_lb)
        self.local_ub = tuple(local_ub)

    def __del__(self):
        try:
            if self.handle:
                lib().oec_decomp_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def oec_decomp_create(global_domain, px: int, py: int, rank: int, nccl_comm: Optional[int] = None) -> Decomp:
    h = C.c_void_p()
    lo, hi = I64x3(), I64x3()
    _check(lib().oec_decomp_create(_i64(global_domain), px, py, rank, C.c_void_p(nccl_comm or 0), C.byref(h), lo, hi))
    return Decomp(h, lo, hi)


def oec_decomp_set_periodic(d: Decomp, periodic_i: bool, periodic_j: bool):
    _check(lib().oec_decomp_set_periodic(d.handle, int(bool(periodic_i)), int(bool(periodic_j))))


def oec_decomp_plan(d: Decomp, width_lo, width_hi) -> List[dict]:
    n = C.c_int32()
    _check(lib().oec_decomp_plan(d.handle, _i32(width_lo), _i32(width_hi), None, 0, C.byref(n)))
    msgs = (OecHaloMsg * max(1, n.value))()
    _check(lib().oec_decomp_plan(d.handle, _i32(width_lo), _i32(width_hi), msgs, n.value, C.byref(n)))
    return [dict(peer=m.peer, is_send=bool(m.is_send), phase=m.phase, tag=m.tag, lo=tuple(m.lo), hi=tuple(m.hi))
            for m in msgs[: n.value]]


def oec_halo_exchange(d: Decomp, fields: Sequence[Field], width_lo, width_hi, stream=None):
    arr = (_P * len(fields))(*[f.ptr for f in fields])
    _check(lib().oec_halo_exchange(d.handle, arr, len(fields), _i32(width_lo), _i32(width_hi), _stream(stream)))


def oec_halo_exchange_local(global_domain, px: int, py: int, fields: Sequence[Field], n_per_rank: int, width_lo,
                            width_hi, stream=None, periodic=None):
    arr = (_P * len(fields))(*[f.ptr for f in fields])
    if periodic is None:
        _check(lib().oec_halo_exchange_local(_i64(global_domain), px, py, arr, n_per_rank, _i32(width_lo),
                                             _i32(width_hi), _stream(stream)))
    else:
        per = (C.c_int32 * 2)(int(bool(periodic[0])), int(bool(periodic[1])))
        _check(lib().oec_halo_exchange_local_periodic(_i64(global_domain), px, py, per, arr, n_per_rank,
                                                      _i32(width_lo), _i32(width_hi), _stream(stream)))


def oec_selftest_rcp32():
    """(mismatches, checked) of the exhaustive binary32 reciprocal self-test (include/oec.h)."""
    bad, used = C.c_ulonglong(), C.c_ulonglong()
    _check(lib().oec_selftest_rcp32(C.byref(bad), C.byref(used)))
    return bad.value, used.value


def oec_selftest_rcp(n: int, seed: int = 1):
    bad, used = C.c_ulonglong(), C.c_ulonglong()
    _check(lib().oec_selftest_rcp(n, seed, C.byref(bad), C.byref(used)))
    return bad.value, used.value


# ---------------------------------------------------------------------------------------------
# multi-step hdiff with the halo exchange fused into the kernel (oec_hdiff_pipeline)
# ---------------------------------------------------------------------------------------------
OEC_IPC_HANDLE_BYTES = 64


class HdiffPipeline:
    """oec_hdiff_pipeline: x_{t+1} = hdiff(x_t) on one rank's sub-domain, neighbours' cells read
    from their memory inside the kernel.  Keeps the Field objects alive."""

    def __init__(self, global_domain, px: int, py: int, rank: int, coeff: Field, x0: Field, x1: Field):
        h = C.c_void_p()
        _check(lib().oec_hdiff_pipeline_create(_i64(global_domain), px, py, rank, coeff.ptr, x0.ptr, x1.ptr, C.byref(h)))
        self.handle = h
        self._keep = [coeff, x0, x1]

    def signal_pad(self) -> Tuple[int, int]:
        p, n = C.c_void_p(), C.c_int64()
        _check(lib().oec_hdiff_pipeline_signal_pad(self.handle, C.byref(p), C.byref(n)))
        return p.value, n.value

    def set_peer(self, peer_rank: int, peer_x0: Field, peer_x1: Field, peer_pad: int):
        _check(lib().oec_hdiff_pipeline_set_peer(self.handle, peer_rank, peer_x0.ptr, peer_x1.ptr, C.c_void_p(peer_pad)))
        self._keep += [peer_x0, peer_x1]

    def run(self, nsteps: int, stream=None):
        _check(lib().oec_hdiff_pipeline_run(self.handle, nsteps, _stream(stream)))

    def steps(self) -> int:
        v = C.c_int64()
        _check(lib().oec_hdiff_pipeline_steps(self.handle, C.byref(v)))
        return v.value

    def __del__(self):
        try:
            if self.handle:
                lib().oec_hdiff_pipeline_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def oec_ipc_export(dev_ptr: int) -> Tuple[bytes, int]:
    h = (C.c_ubyte * OEC_IPC_HANDLE_BYTES)()
    off = C.c_int64()
    _check(lib().oec_ipc_export(C.c_void_p(dev_ptr), h, C.byref(off)))
    return bytes(h), off.value


def oec_ipc_import(handle: bytes, offset: int) -> int:
    h = (C.c_ubyte * OEC_IPC_HANDLE_BYTES).from_buffer_copy(handle)
    p = C.c_void_p()
    _check(lib().oec_ipc_import(h, int(offset), C.byref(p)))
    return p.value


def oec_ipc_close(dev_ptr: int):
    _check(lib().oec_ipc_close(C.c_void_p(dev_ptr)))


def field_descriptor(f: Field) -> dict:
    """Plain-data description of a field (to send to another process with its IPC handle)."""
    d = f.desc
    return dict(lb=tuple(d.lb), ub=tuple(d.ub), stride=tuple(d.stride), dtype=d.dtype, device=d.device)


def field_at(ptr: int, desc: dict, device: int) -> Field:
    """A borrowed field over `ptr` (e.g. an IPC-imported peer allocation) with a peer's layout."""
    d = OecField()
    _check(lib().oec_field_wrap(C.c_void_p(ptr), _i64(desc["lb"]), _i64(desc["ub"]), _i64(desc["stride"]),
                                desc["dtype"], device, C.byref(d)))
    return Field(d)
