"""Seeded random stencil-language programs (test input generator; no method arithmetic).

`random_program(seed)` writes the TEXT of a random acyclic stencil program in the language of
include/oec.h: a few 3D and k-invariant inputs, scalars, 3-7 operators (some multi-result, some
with locals) reading inputs and earlier results at offsets in [-2, 2] x [-2, 2] x [-1, 1], with
+ - * /, select on comparisons and && / || / !, min / max / abs / sqrt, and 1-3 stored outputs.
Divisions are by (abs(x) + 1) and roots of abs(x), so values stay finite.  Some operators are dead
(never read), which exercises dead-operator elimination.

Both sides receive the same text: the oracle (oracle/dsl.py + oracle/stencil.py) and liboec's JIT
(csrc/jit.cpp).  Inputs are allocated from the ORACLE's brute-force touched set (never from the
CUDA path's shape inference).
"""
from __future__ import annotations

import numpy as np

import synth
from synth import HostField


def _expr(rng, readable, scalars, depth):
    """A random numeric expression over `readable` [(name, is_k_invariant)] and `scalars`."""
    r = rng.random()
    if depth <= 0 or r < 0.25:
        if rng.random() < 0.12 and scalars:
            return str(rng.choice(scalars))
        if rng.random() < 0.1:
            return repr(float(np.round(rng.uniform(-2, 2), 3)))
        name, kinv = readable[rng.integers(len(readable))]
        di, dj = (int(x) for x in rng.integers(-2, 3, 2))
        dk = 0 if kinv else int(rng.integers(-1, 2))
        if di == dj == dk == 0 and rng.random() < 0.5:
            return name
        return f"{name}[{di},{dj},{dk}]"
    a = _expr(rng, readable, scalars, depth - 1)
    b = _expr(rng, readable, scalars, depth - 1)
    kind = rng.integers(10)
    if kind <= 2:
        return f"({a} {rng.choice(['+', '-', '*'])} {b})"
    if kind == 3:
        return f"{a} * {b} + {a}"
    if kind == 4:
        return f"({a}) / (abs({b}) + 1.0)"
    if kind == 5:
        c = f"{a} {rng.choice(['<', '>', '<=', '>=', '==', '!='])} {b}"
        if rng.random() < 0.3:
            c = f"({c}) {rng.choice(['&&', '||'])} !({b} > 0.25)"
        return f"select({c}, {a}, -{b})"
    if kind == 6:
        return f"{rng.choice(['min', 'max'])}({a}, {b})"
    if kind == 7:
        return f"sqrt(abs({a}))"
    if kind == 8:
        return f"-({a})"
    return f"({a} - {b}) * 0.5"


def random_program(seed: int, name: str = None) -> str:
    rng = np.random.Generator(np.random.PCG64(seed))
    name = name or f"rnd{seed}"
    n3 = int(rng.integers(1, 4))
    n2 = int(rng.integers(0, 3))
    inputs = [(f"a{q}", False) for q in range(n3)] + [(f"m{q}", True) for q in range(n2)]
    rng.shuffle(inputs)
    scalars = [f"s{q}" for q in range(int(rng.integers(0, 3)))]
    lines = [f"program {name}"]
    for n, kinv in inputs:
        lines.append(f"input {n}" + (" : ij" if kinv else ""))
    for q, s in enumerate(scalars):
        lines.append(f"scalar {s} = {0.5 + 0.25 * q}")
    readable = list(inputs)
    temps = []
    for t in range(int(rng.integers(3, 8))):
        nres = 2 if rng.random() < 0.2 else 1
        names = [f"t{t}" + ("" if nres == 1 else "abc"[r]) for r in range(nres)]
        depth = int(rng.integers(1, 4))
        if nres == 1 and rng.random() < 0.5:
            lines.append(f"apply {names[0]} = {_expr(rng, readable, scalars, depth)}")
        else:
            body = []
            locs = []
            for q in range(int(rng.integers(0, 3))):
                ln = f"l{t}_{q}"
                body.append(f"    {ln} = {_expr(rng, readable, scalars + locs, depth)}")
                locs.append(ln)
            # locals (operator-internal SSA values) are read by name only, like scalars
            rets = [_expr(rng, readable, scalars + locs, depth) for _ in names]
            lines.append(f"apply {', '.join(names)} {{")
            lines.extend(body)
            lines.append(f"    return {', '.join(rets)}")
            lines.append("}")
        temps.extend(names)
        readable.extend((n, False) for n in names)
    nout = int(rng.integers(1, min(3, len(temps)) + 1))
    stored = list(rng.choice(temps[len(temps) // 2:], size=min(nout, len(temps[len(temps) // 2:])), replace=False))
    for q, t in enumerate(stored):
        lines.append(f"output o{q}")
        lines.append(f"store {t} -> o{q}")
    return "\n".join(lines) + "\n"


def touched_boxes(tp, domain, halo=8):
    """Brute-force access extents of a parsed program (oracle.dsl.TextProgram): run the oracle's
    fused evaluator on generously allocated fields and take the bounding box of every input's
    touched set, relative to the domain (lo <= 0 <= hi like oec_program_input)."""
    from oracle import stencil

    fields = {}
    for n in tp.inputs:
        kinv = tp.k_invariant[n]
        lb = (-halo, -halo, 0 if kinv else -halo)
        ub = (domain[0] + halo, domain[1] + halo, 1 if kinv else domain[2] + halo)
        shape = (ub[2] - lb[2], ub[1] - lb[1], ub[0] - lb[0])
        fields[n] = HostField(np.full(shape, 0.5, dtype=tp.dtype), lb, ub, kinv)
    _, touched = stencil.run_fused(tp.program, fields, tp.scalar_values(), (0, 0, 0), domain)
    ext = {}
    for n in tp.inputs:
        pts = touched[n]
        if not pts:
            ext[n] = ((0, 0, 0), (0, 0, 0))
            continue
        arr = np.array(sorted(pts))
        lo = arr.min(0)
        hi = arr.max(0) + 1 - np.array(domain)
        if tp.k_invariant[n]:
            lo[2], hi[2] = 0, 0
        ext[n] = (tuple(int(min(x, 0)) for x in lo), tuple(int(max(x, 0)) for x in hi))
    return ext


def make_inputs(tp, domain, ext, seed=0, dtype=np.float64):
    """Seeded U[-1, 1] inputs over domain + extent (ext from touched_boxes, i.e. the oracle)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = {}
    for n in tp.inputs:
        lo, hi = ext[n]
        if tp.k_invariant[n]:
            lb, ub = (lo[0], lo[1], 0), (domain[0] + hi[0], domain[1] + hi[1], 1)
        else:
            lb, ub = tuple(lo), tuple(domain[d] + hi[d] for d in range(3))
        shape = (ub[2] - lb[2], ub[1] - lb[1], ub[0] - lb[0])
        out[n] = HostField(rng.uniform(-1.0, 1.0, shape).astype(dtype), lb, ub, tp.k_invariant[n])
    return out


__all__ = ["random_program", "touched_boxes", "make_inputs", "synth"]
