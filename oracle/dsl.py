"""Oracle reader of the stencil language (include/oec.h).  TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

A second, independent reading of a stencil-language program text: it turns the text into an
`oracle.stencil.Program` whose operators are plain Python closures, so the oracle's existing
evaluators apply unchanged --

  * stencil.run_unfused  -- the "original" level: every operator materialised as a numpy
    temporary, in program order;
  * stencil.run_fused    -- inlining: per-point recursive evaluation, with the brute-force
    touched-index trace that checks liboec's shape inference;
  * stencil.census       -- Table II counts.

It shares no code with liboec's C++ parser / code generator (csrc/jit.cpp): program texts are
inputs, like fields.  Grammar and semantics, restated from include/oec.h:

  program NAME | input NAME [: ij|ijk] | scalar NAME [= NUMBER] | output NAME
  apply R1[, R2...] { LOCAL = EXPR ... return EXPR[, EXPR...] } | apply R = EXPR | store R -> OUT
  EXPR: literals, scalars, locals, NAME / NAME[di,dj,dk] (stencil.access), unary -, + - * /
  (left-associative), select(c, x, y), min(a,b) := b < a ? b : a, max(a,b) := b > a ? b : a,
  abs, sqrt; conditions: < > <= >= == !=, &&, ||, !.  Precedence ||, &&, comparison, + -, * /, unary.
Literals and scalars are rounded once to the fields' precision (R21).

Pinned (tests/test_oracle_dsl.py) against the hand-written, independently pinned oracle programs
(oracle/suite.py, oracle/oec_oracle.c): the language versions of hdiff and the suite give
bit-identical results and the same Table II census; syntax/semantic errors are rejected.
"""
from __future__ import annotations

import re
from typing import Dict, List, Tuple

import numpy as np

from oracle.stencil import Apply, Program, _T

_TOKEN = re.compile(r"\s*(?:(#[^\n]*)|(\d+\.?\d*(?:[eE][+-]?\d+)?|\.\d+(?:[eE][+-]?\d+)?)|([A-Za-z_]\w*)|"
                    r"(->|<=|>=|==|!=|&&|\|\||[()\[\]{},=+\-*/<>!:;]))")
_RESERVED = {"program", "input", "scalar", "output", "apply", "return", "store", "end", "select", "min", "max",
             "abs", "sqrt", "ij", "ijk"}


class DslError(ValueError):
    pass


def _tokens(text: str) -> List[Tuple[str, str]]:
    out, pos = [], 0
    text = text.rstrip()
    while pos < len(text):
        m = _TOKEN.match(text, pos)
        if not m or m.end() == pos:
            raise DslError(f"unexpected character {text[pos:pos + 1]!r} at offset {pos}")
        pos = m.end()
        com, num, name, punct = m.groups()
        if com is not None or punct == ";":
            continue
        if num is not None:
            out.append(("num", num))
        elif name is not None:
            out.append(("name", name))
        elif punct is not None:
            out.append(("p", punct))
    out.append(("end", ""))
    return out


class _Reader:
    """Recursive descent over the token list; expressions become nested tuples."""

    def __init__(self, text: str):
        self.t = _tokens(text)
        self.i = 0
        self.inputs: List[Tuple[str, bool]] = []
        self.scalars: List[Tuple[str, float]] = []
        self.outputs: List[str] = []
        self.stores: Dict[str, str] = {}
        self.applies: List[Tuple[Tuple[str, ...], List[Tuple[str, tuple]], List[tuple]]] = []
        self.kind: Dict[str, str] = {}  # name -> input | scalar | output | temp
        self.local: Dict[str, tuple] = {}

    # -- token helpers
    def peek(self, k=0):
        return self.t[min(self.i + k, len(self.t) - 1)]

    def at(self, s):
        return self.peek()[0] == "p" and self.peek()[1] == s

    def kw(self, s):
        return self.peek() == ("name", s)

    def next(self):
        tok = self.t[self.i]
        self.i = min(self.i + 1, len(self.t) - 1)
        return tok

    def want(self, s):
        if not self.at(s):
            raise DslError(f"expected {s!r}, got {self.peek()[1]!r}")
        self.next()

    def ident(self):
        k, v = self.next()
        if k != "name":
            raise DslError(f"expected a name, got {v!r}")
        return v

    def define(self, name, kind):
        if name in _RESERVED:
            raise DslError(f"{name!r} is a reserved word")
        if name in self.kind:
            raise DslError(f"{name!r} is already defined")
        self.kind[name] = kind

    # -- expressions: ('lit', v) ('sc', name) ('acc', name, (di,dj,dk)) ('loc', node) ('neg', x)
    #    ('bin', op, x, y) ('cmp', op, x, y) ('and'|'or', x, y) ('not', x) ('sel', c, x, y)
    #    ('min'|'max', x, y) ('abs'|'sqrt', x)
    def expr(self):
        x = self.conj()
        while self.at("||"):
            self.next()
            x = ("or", self._cond(x), self._cond(self.conj()))
        return x

    def conj(self):
        x = self.comparison()
        while self.at("&&"):
            self.next()
            x = ("and", self._cond(x), self._cond(self.comparison()))
        return x

    def comparison(self):
        x = self.additive()
        for op in ("<", ">", "<=", ">=", "==", "!="):
            if self.at(op):
                self.next()
                return ("cmp", op, self._num(x), self._num(self.additive()))
        return x

    def additive(self):
        x = self.term()
        while self.at("+") or self.at("-"):
            op = self.next()[1]
            x = ("bin", op, self._num(x), self._num(self.term()))
        return x

    def term(self):
        x = self.unary()
        while self.at("*") or self.at("/"):
            op = self.next()[1]
            x = ("bin", op, self._num(x), self._num(self.unary()))
        return x

    def unary(self):
        if self.at("-"):
            self.next()
            return ("neg", self._num(self.unary()))
        if self.at("!"):
            self.next()
            return ("not", self._cond(self.unary()))
        return self.primary()

    @staticmethod
    def _is_cond(x):
        while x[0] == "loc":
            x = x[1]
        return x[0] in ("cmp", "and", "or", "not")

    def _num(self, x):
        if self._is_cond(x):
            raise DslError("a condition is used as a number")
        return x

    def _cond(self, x):
        if not self._is_cond(x):
            raise DslError("a number is used as a condition")
        return x

    def primary(self):
        k, v = self.peek()
        if k == "num":
            self.next()
            return ("lit", float(v))
        if self.at("("):
            self.next()
            x = self.expr()
            self.want(")")
            return x
        if k != "name":
            raise DslError(f"unexpected {v!r}")
        self.next()
        if self.at("("):
            self.next()
            args = [self.expr()]
            while self.at(","):
                self.next()
                args.append(self.expr())
            self.want(")")
            arity = {"select": 3, "min": 2, "max": 2, "abs": 1, "sqrt": 1}
            if v not in arity:
                raise DslError(f"unknown function {v!r}")
            if len(args) != arity[v]:
                raise DslError(f"{v}() takes {arity[v]} arguments")
            if v == "select":
                return ("sel", self._cond(args[0]), self._num(args[1]), self._num(args[2]))
            return (v,) + tuple(self._num(a) for a in args)
        off = None
        if self.at("["):
            self.next()
            off = []
            for d in range(3):
                sign = 1
                if self.at("-") or self.at("+"):
                    sign = -1 if self.next()[1] == "-" else 1
                kk, vv = self.next()
                if kk != "num" or not vv.isdigit():
                    raise DslError(f"expected an integer offset, got {vv!r}")
                off.append(sign * int(vv))
                if d < 2:
                    self.want(",")
            self.want("]")
            off = tuple(off)
        if off is None and v in self.local:
            return ("loc", self.local[v])
        kind = self.kind.get(v)
        if kind is None:
            raise DslError(f"{v!r} is not defined")
        if kind == "scalar":
            if off is not None:
                raise DslError(f"scalar {v!r} cannot be accessed at an offset")
            return ("sc", v)
        if kind == "output":
            raise DslError(f"output {v!r} cannot be read (P:381)")
        return ("acc", v, off or (0, 0, 0))

    # -- program
    def program(self):
        if not self.kw("program"):
            raise DslError("a program starts with 'program NAME'")
        self.next()
        self.name = self.ident()
        while self.peek()[0] != "end" and not self.kw("end"):
            word = self.ident()
            if word == "input":
                n = self.ident()
                kinv = False
                if self.at(":"):
                    self.next()
                    dims = self.ident()
                    if dims not in ("ij", "ijk"):
                        raise DslError("input dimensions are ij or ijk")
                    kinv = dims == "ij"
                self.define(n, "input")
                self.inputs.append((n, kinv))
            elif word == "scalar":
                n = self.ident()
                val = 0.0
                if self.at("="):
                    self.next()
                    neg = self.at("-")
                    if neg:
                        self.next()
                    k, v = self.next()
                    if k != "num":
                        raise DslError("expected a number")
                    val = -float(v) if neg else float(v)
                self.define(n, "scalar")
                self.scalars.append((n, val))
            elif word == "output":
                n = self.ident()
                self.define(n, "output")
                self.outputs.append(n)
            elif word == "apply":
                names = [self.ident()]
                while self.at(","):
                    self.next()
                    names.append(self.ident())
                self.local = {}
                stmts: List[Tuple[str, tuple]] = []
                if self.at("="):
                    self.next()
                    rets = [self.expr()]
                else:
                    self.want("{")
                    while not self.kw("return"):
                        ln = self.ident()
                        if ln in self.local or ln in self.kind or ln in _RESERVED:
                            raise DslError(f"{ln!r} is already defined")
                        self.want("=")
                        x = self.expr()
                        self.local[ln] = x
                        stmts.append((ln, x))
                    self.next()
                    rets = [self.expr()]
                    while self.at(","):
                        self.next()
                        rets.append(self.expr())
                    self.want("}")
                if len(rets) != len(names):
                    raise DslError(f"apply {names}: {len(names)} results but {len(rets)} return values")
                for r in rets:
                    self._num(r)
                for n in names:
                    self.define(n, "temp")
                self.applies.append((tuple(names), stmts, rets))
            elif word == "store":
                t = self.ident()
                self.want("->")
                o = self.ident()
                if self.kind.get(t) != "temp":
                    raise DslError(f"{t!r} is not an operator result")
                if self.kind.get(o) != "output":
                    raise DslError(f"{o!r} is not a declared output")
                if o in self.stores:
                    raise DslError(f"output {o!r} is stored twice")
                self.stores[o] = t
            else:
                raise DslError(f"unknown declaration {word!r}")
        if self.kw("end"):
            self.next()
        if self.peek()[0] != "end":
            raise DslError("text after 'end'")
        if not self.outputs:
            raise DslError("the program has no output")
        for o in self.outputs:
            if o not in self.stores:
                raise DslError(f"output {o!r} is never stored")


def _combine(op, x, kids, sel):
    """Apply node `x`'s operation to its evaluated children (`kids` = x[1:] with sub-expressions evaluated)."""
    tracer = next((k for k in kids if isinstance(k, _T)), None)
    if tracer is not None and op in ("and", "or", "not", "abs", "sqrt"):
        return tracer._op("cmp" if op in ("and", "or", "not") else "arith")  # census / access tracing
    if op == "neg":
        return -kids[0]
    if op == "bin":
        p, q = kids[1], kids[2]
        cnt = getattr(sel, "census_cnt", None)
        if cnt is not None and tracer is None and x[2][0] == "lit" and x[3][0] == "lit":
            cnt["arith"] += 1  # e.g. (7.0 / 12.0): an operation of the program text (census, R15)
        return {"+": lambda: p + q, "-": lambda: p - q, "*": lambda: p * q, "/": lambda: p / q}[x[1]]()
    if op == "cmp":
        p, q = kids[1], kids[2]
        return {"<": lambda: p < q, ">": lambda: p > q, "<=": lambda: p <= q, ">=": lambda: p >= q,
                "==": lambda: p == q, "!=": lambda: p != q}[x[1]]()
    if op == "and":
        return np.logical_and(kids[0], kids[1])
    if op == "or":
        return np.logical_or(kids[0], kids[1])
    if op == "not":
        return np.logical_not(kids[0])
    if op == "sel":
        return sel(kids[0], kids[1], kids[2])
    if op == "min":
        p, q = kids
        return sel(q < p, q, p)
    if op == "max":
        p, q = kids
        return sel(q > p, q, p)
    if op == "abs":
        return np.abs(kids[0])
    if op == "sqrt":
        return np.sqrt(kids[0])
    raise AssertionError(op)


class TextProgram:
    """A parsed stencil-language program: its oracle `Program` plus the declarations."""

    def __init__(self, text: str, dtype=np.float64):
        r = _Reader(text)
        r.program()
        self.name = r.name
        self.inputs = [n for n, _ in r.inputs]
        self.k_invariant = {n: k for n, k in r.inputs}
        self.scalars = list(r.scalars)
        self.outputs = list(r.outputs)
        self.dtype = np.dtype(dtype)
        typ = self.dtype.type
        applies = []
        for names, stmts, rets in r.applies:
            applies.append(Apply(names, _operator(stmts, rets, typ)))
        self.program = Program(self.name, inputs=tuple(self.inputs),
                               outputs=tuple((o, r.stores[o]) for o in self.outputs),
                               applies=tuple(applies), scalars=tuple(n for n, _ in self.scalars))

    def scalar_values(self, overrides=None) -> Dict[str, float]:
        vals = {n: v for n, v in self.scalars}
        vals.update(overrides or {})
        return vals


def _operator(stmts, rets, typ):
    """One stencil.apply as a closure fn(a, s, sel): locals evaluated once each, in order."""

    def fn(a, s, sel):
        env: Dict[int, object] = {}

        def ev(x):
            op = x[0]
            if op == "lit":
                return typ(x[1])
            if op == "sc":
                return s[x[1]]
            if op == "acc":
                return a(x[1], *x[2])
            if op == "loc":
                k = id(x[1])
                if k not in env:
                    env[k] = ev(x[1])
                return env[k]
            kids = [ev(c) if isinstance(c, tuple) else c for c in x[1:]]
            return _combine(op, x, kids, sel)

        for _, x in stmts:
            ev(("loc", x))
        out = tuple(ev(r) for r in rets)
        return out[0] if len(out) == 1 else out

    return fn


def parse(text: str, dtype=np.float64) -> TextProgram:
    return TextProgram(text, dtype)
