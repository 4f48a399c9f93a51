"""A tiny stencil-program evaluator for the oracle.  TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

A stencil program (§4.4) loads input arrays, applies a sequence of dependent
stencil operators and stores results to output arrays.  Here a program is written as a list of
`Apply`s; each apply's function implements the operator for ONE point ("the scalar
operations are applied to all domain elements as in a loop nest") in terms of
`a(name, di, dj, dk)` -- stencil.access at a constant offset -- arithmetic, and
`sel(cond, x, y)` for control flow inside operators (loop.if / select).

Three evaluators share these definitions:

* `run_unfused` -- the paper's "original" level: each apply is materialised as a numpy
  temporary over the maximal box on which its accesses are in range, applies run in program
  order, outputs are stored on the domain (stencil.store range).  numpy elementwise fp64
  arithmetic is IEEE RNE without contraction.
* `run_fused` -- stencil inlining: every output point is evaluated by recursively
  evaluating producers at the accessed offsets (pure-Python scalars, small sizes only).  It also
  records every touched input index -- the brute-force extent oracle of SPEC S:382 / S:618.
* `census` -- counts apply ops, inputs/outputs, arithmetic ops and access ops of the definition
  (Table II) by running each apply once on symbolic tracers.

Because both evaluators perform the same scalar operations in the same order, they must agree
bitwise -- a test pins that.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Sequence, Set, Tuple

import numpy as np

from synth import HostField


@dataclass(frozen=True)
class Apply:
    results: Tuple[str, ...]
    fn: Callable  # fn(a, s, sel) -> value or tuple of values (one per result)


@dataclass(frozen=True)
class Program:
    name: str
    inputs: Tuple[str, ...]
    outputs: Tuple[Tuple[str, str], ...]  # (output array name, temp name stored to it)
    applies: Tuple[Apply, ...]
    scalars: Tuple[str, ...] = ()


def _as_tuple(v, n):
    if n == 1:
        return (v,)
    assert isinstance(v, tuple) and len(v) == n
    return v


# ------------------------------------------------------------------------------------------
# census (Table II)
# ------------------------------------------------------------------------------------------
class _T:
    """Symbolic value: every arithmetic op / comparison on it is counted."""

    def __init__(self, cnt):
        self.cnt = cnt

    def _op(self, kind="arith"):
        self.cnt[kind] += 1
        return _T(self.cnt)

    __add__ = __radd__ = __sub__ = __rsub__ = __mul__ = __rmul__ = __truediv__ = __rtruediv__ = lambda s, o: s._op()

    def __neg__(self):
        return self._op()

    def __gt__(self, o):
        return self._op("cmp")

    __lt__ = __ge__ = __le__ = __gt__


def census(prog: Program) -> Dict[str, int]:
    cnt = {"arith": 0, "cmp": 0, "access": 0, "if": 0}

    def a(name, di=0, dj=0, dk=0):
        cnt["access"] += 1
        return _T(cnt)

    def sel(c, x, y):
        cnt["if"] += 1
        return _T(cnt)

    sel.census_cnt = cnt  # kdiv / literal ops of the stencil language count as arithmetic ops
    s = {k: 1.0 for k in prog.scalars}
    for ap in prog.applies:
        ap.fn(a, s, sel)
    return {
        "applies": len(prog.applies),
        "inputs": len(prog.inputs),
        "outputs": len(prog.outputs),
        **cnt,
    }


def kdiv(sel, n: float, d: float) -> float:
    """A constant written in the definition as the quotient n / d (e.g. the PPM weight 7/12):
    numerically the IEEE double n / d, and for the census (Table II) one arithmetic operation,
    as the operation appears in the program text (reading R15)."""
    cnt = getattr(sel, "census_cnt", None)
    if cnt is not None:
        cnt["arith"] += 1
    return n / d


def accesses(ap: Apply, scalars: Sequence[str]) -> List[Tuple[str, int, int, int]]:
    acc = []
    cnt = {"arith": 0, "cmp": 0, "access": 0, "if": 0}

    def a(name, di=0, dj=0, dk=0):
        acc.append((name, di, dj, dk))
        return _T(cnt)

    ap.fn(a, {k: 1.0 for k in scalars}, lambda c, x, y: _T(cnt))
    return acc


# ------------------------------------------------------------------------------------------
# unfused evaluation (materialised temporaries)
# ------------------------------------------------------------------------------------------
def _where(c, x, y):
    return np.where(c, x, y)


def _dtype(fields, names):
    dts = {fields[n].data.dtype for n in names}
    assert len(dts) == 1 and dts <= {np.dtype(np.float64), np.dtype(np.float32)}, dts
    return dts.pop()


def run_unfused(prog: Program, fields: Dict[str, HostField], scalars: Dict[str, float], domain_lo, domain_hi,
                outputs: Optional[Dict[str, HostField]] = None) -> Dict[str, HostField]:
    # precision = the inputs' dtype (float64, or float32 for the paper's f32 runs): scalars
    # are rounded to it and numpy keeps float32 expressions in float32 (Python-float constants
    # are rounded to float32, NEP 50)
    dt = _dtype(fields, prog.inputs)
    scalars = {k: dt.type(v) for k, v in scalars.items()}
    env: Dict[str, HostField] = {n: fields[n] for n in prog.inputs}
    # universe: the bounding box of all input allocations (k-invariant fields: all k)
    # universe: the bounding box of the domain and all input allocations (k-invariant fields: no
    # k range), grown by the longest chain of access offsets -- a temporary may be needed (and be
    # computable) beyond the inputs' box when a consumer reads it at an offset.  It
    # only bounds applies whose accesses leave a dimension unconstrained (constants, k-invariant
    # inputs); every other box is the intersection of its accesses' in-range boxes.
    margin = [sum(max([abs(acc[1 + d]) for acc in accesses(ap, prog.scalars)] + [0]) for ap in prog.applies)
              for d in range(3)]
    ulo = [min([domain_lo[d]] + [f.lb[d] for f in env.values() if not (d == 2 and f.k_invariant)]) - margin[d]
           for d in range(3)]
    uhi = [max([domain_hi[d]] + [f.ub[d] for f in env.values() if not (d == 2 and f.k_invariant)]) + margin[d]
           for d in range(3)]
    for ap in prog.applies:
        lo, hi = list(ulo), list(uhi)
        for name, di, dj, dk in accesses(ap, prog.scalars):
            f = env[name]
            for d, off in enumerate((di, dj, dk)):
                if d == 2 and f.k_invariant:
                    continue
                lo[d] = max(lo[d], f.lb[d] - off)
                hi[d] = min(hi[d], f.ub[d] - off)
        shape = tuple(max(0, hi[d] - lo[d]) for d in (2, 1, 0))

        def a(name, di=0, dj=0, dk=0, lo=lo, hi=hi):
            f = env[name]
            i0, j0 = lo[0] + di - f.lb[0], lo[1] + dj - f.lb[1]
            i1, j1 = hi[0] + di - f.lb[0], hi[1] + dj - f.lb[1]
            if f.k_invariant:
                return f.data[0:1, j0:j1, i0:i1]
            k0, k1 = lo[2] + dk - f.lb[2], hi[2] + dk - f.lb[2]
            return f.data[k0:k1, j0:j1, i0:i1]

        with np.errstate(all="ignore"):
            vals = _as_tuple(ap.fn(a, scalars, _where), len(ap.results))
        for rname, v in zip(ap.results, vals):
            v = np.asarray(v)
            assert v.dtype == dt, (prog.name, rname, v.dtype)  # no silent promotion
            arr = np.ascontiguousarray(np.broadcast_to(v, shape))
            env[rname] = HostField(arr, tuple(lo), tuple(hi))
    res = outputs if outputs is not None else {}
    for oname, tname in prog.outputs:
        t = env[tname]
        for d in range(3):
            if t.lb[d] > domain_lo[d] or t.ub[d] < domain_hi[d]:
                raise ValueError(f"{prog.name}: temp {tname} range {t.lb}:{t.ub} does not cover the domain "
                                 f"{tuple(domain_lo)}:{tuple(domain_hi)} (input arrays too small, P:482)")
        sl = tuple(slice(domain_lo[d] - t.lb[d], domain_hi[d] - t.lb[d]) for d in (2, 1, 0))
        vals = t.data[sl]
        if oname in res:
            o = res[oname]
            osl = tuple(slice(domain_lo[d] - o.lb[d], domain_hi[d] - o.lb[d]) for d in (2, 1, 0))
            o.data[osl] = vals
        else:
            res[oname] = HostField(vals.copy(), tuple(domain_lo), tuple(domain_hi))
    return res


# ------------------------------------------------------------------------------------------
# fused per-point evaluation (inlining) with touched-index tracing
# ------------------------------------------------------------------------------------------
class RangeError(IndexError):
    pass


def run_fused(prog: Program, fields: Dict[str, HostField], scalars: Dict[str, float], domain_lo, domain_hi,
              points: Optional[Sequence[Tuple[int, int, int]]] = None, reverse: bool = False):
    """Returns (outputs as {name: {(i,j,k): value}}, touched {input: set of (i,j,k)})."""
    producer = {}
    for ap in prog.applies:
        for r_idx, r in enumerate(ap.results):
            producer[r] = (ap, r_idx)
    touched: Dict[str, Set[Tuple[int, int, int]]] = {n: set() for n in prog.inputs}
    dt = _dtype(fields, prog.inputs)
    memo: Dict[Tuple[str, int, int, int], np.floating] = {}
    sc = {k: dt.type(v) for k, v in scalars.items()}

    def value(name, i, j, k):
        if name in fields and name in touched:
            f = fields[name]
            kk = 0 if f.k_invariant else k
            if not (f.lb[0] <= i < f.ub[0] and f.lb[1] <= j < f.ub[1] and f.lb[2] <= kk < f.ub[2]):
                raise RangeError(f"{prog.name}: access {name}{(i, j, k)} outside {f.lb}:{f.ub}")
            touched[name].add((i, j, kk))
            return f.data[kk - f.lb[2], j - f.lb[1], i - f.lb[0]]
        key = (name, i, j, k)
        if key not in memo:
            ap, _ = producer[name]

            def a(n, di=0, dj=0, dk=0):
                return value(n, i + di, j + dj, k + dk)

            vals = _as_tuple(ap.fn(a, sc, lambda c, x, y: dt.type(x if c else y)), len(ap.results))
            for r, v in zip(ap.results, vals):
                assert np.asarray(v).dtype == dt, (prog.name, r)  # no silent promotion
                memo[(r, i, j, k)] = v
        return memo[key]

    if points is None:
        rng = [range(domain_lo[d], domain_hi[d]) for d in range(3)]
        points = [(i, j, k) for k in rng[2] for j in rng[1] for i in rng[0]]
    if reverse:
        points = list(reversed(points))
    out: Dict[str, Dict[Tuple[int, int, int], float]] = {o: {} for o, _ in prog.outputs}
    with np.errstate(all="ignore"):
        for p in points:
            for oname, tname in prog.outputs:
                out[oname][p] = value(tname, *p)
    return out, touched


def bbox(points: Set[Tuple[int, int, int]]):
    arr = np.array(sorted(points))
    return tuple(arr.min(0)), tuple(arr.max(0) + 1)
