"""TDL — Tensor Description Language (oracle side).  TEST INFRASTRUCTURE ONLY.

Follows P:L380-409 §4.1: "we represent tensors as lambda functions that map
from coordinates (aka index variables) to values".  TDL expressions are index
variables, tensor elements, arithmetic, and a reduction (Sum/Max/Min/Prod,
P:L396-400).  Opaque functions have pass-through batch dims.

Concrete text syntax (the paper embeds TDL in Python; this text form is the
reading recorded in DESIGN.md §R1):

    def conv1d(data(3), filters(3)) -> lambda b, co, x:
        reduce(Sum; ci, dx; data[b, ci, x + dx] * filters[ci, co, dx])
    def batch_cholesky(M(3)) -> lambda b, i, j: opaque(Cholesky; M[b, :, :])[i, j]

Index expressions must be affine in index variables with integer
coefficients (Eq. 1 only admits affine intervals).  A single
index variable may not address two dimensions of one input tensor
(Assumption #1).  At most one reducer, at the top of the body.
"""
from __future__ import annotations

import re
from dataclasses import dataclass, field

REDUCERS = ("Sum", "Max", "Min", "Prod")
FUNCS = {"max": 2, "min": 2, "exp": 1, "tanh": 1, "sigmoid": 1, "select": 3, "sqrt": 1}


class TdlError(Exception):
    """Base error.  kind in {Syntax, UndeclaredTensor, RankMismatch,
    NonAffineIndex, NestedReduce, AssumptionViolation, UnknownVar}."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ----------------------------------------------------------------------------- AST
@dataclass(frozen=True)
class Affine:
    """sum(coef[v] * v) + const (+ quasi-affine terms); coefficients are ints.

    ``terms`` (reading R11): mult * floor(inner / d) ('div') or mult * (inner mod d) ('mod')
    with an affine ``inner`` — the ``I / k`` of Fig. int-arith taken as integer division
    of an index, plus its remainder; needed to describe the gradient of a strided convolution."""
    coef: tuple  # tuple of (var, int) sorted by var
    const: int
    terms: tuple = ()  # tuple of (kind 'div'|'mod', mult int, inner Affine, d int)

    def vars(self):
        vs = [v for v, c in self.coef if c != 0]
        for _, _, inner, _ in self.terms:
            vs += [v for v in inner.vars() if v not in vs]
        return vs

    def value(self, env):
        """Index value at a point (env: var -> int or numpy int array); floor division, non-negative mod."""
        acc = self.const
        for v, c in self.coef:
            acc = acc + c * env[v]
        for kind, mult, inner, d in self.terms:
            x = inner.value(env)
            acc = acc + mult * (x // d if kind == "div" else x % d)
        return acc

    def hull(self, box, off=0):
        """Closed integer range of the index over a var box (var -> (lo, hi)): linear part by interval
        arithmetic (exact for it), each div / mod term bounded separately (an over-approximation only
        when a term shares a variable with another part)."""
        lo = hi = self.const + off
        for v, c in self.coef:
            a, b = box[v]
            lo += min(c * a, c * b)
            hi += max(c * a, c * b)
        for kind, mult, inner, d in self.terms:
            ilo, ihi = inner.hull(box)
            if kind == "div":
                tl, th = ilo // d, ihi // d
            elif ihi - ilo + 1 >= d or ilo // d != ihi // d:
                tl, th = 0, d - 1
            else:
                tl, th = ilo % d, ihi % d
            lo += min(mult * tl, mult * th)
            hi += max(mult * tl, mult * th)
        return lo, hi

    def is_var(self, v=None):
        """Exactly one variable with coefficient 1 and nothing else."""
        return (len(self.coef) == 1 and self.coef[0][1] == 1 and self.const == 0 and not self.terms
                and (v is None or self.coef[0][0] == v))


@dataclass(frozen=True)
class Access:
    tensor: str
    index: tuple  # tuple of Affine or None (None = ':' slice inside opaque)


@dataclass
class Expr:
    kind: str  # 'num','var','access','bin','neg','call','opaque'
    val: object = None
    args: list = field(default_factory=list)


@dataclass
class OpDef:
    name: str
    params: list  # [(tensor, rank)]
    out_vars: list
    reducer: str | None
    red_vars: list
    body: Expr
    accesses: list  # [Access] in order of appearance (excluding opaque slices)
    opaque: bool = False
    opaque_free: list = field(default_factory=list)  # out vars usable for opaque split

    def param_rank(self, t):
        for n, r in self.params:
            if n == t:
                return r
        raise KeyError(t)

    def all_vars(self):
        return list(self.out_vars) + list(self.red_vars)


# ----------------------------------------------------------------------------- lexer
_TOK = re.compile(r"\s*(?:(\d+\.\d*|\d+)|([A-Za-z_][A-Za-z_0-9]*)|(->|>=|<=|==|[-+*/%()\[\],:;<>]))")


def _lex(src):
    toks = []
    pos = 0
    src = src.strip()
    while pos < len(src):
        m = _TOK.match(src, pos)
        if not m or m.end() == pos:
            if src[pos:].strip() == "":
                break
            raise TdlError("Syntax", f"bad character at {pos}: {src[pos:pos+10]!r}")
        num, ident, sym = m.groups()
        if num is not None:
            toks.append(("num", num, pos))
        elif ident is not None:
            toks.append(("id", ident, pos))
        else:
            toks.append(("sym", sym, pos))
        pos = m.end()
    toks.append(("eof", None, pos))
    return toks


class _P:
    def __init__(self, src):
        self.t = _lex(src)
        self.i = 0

    def peek(self):
        return self.t[self.i]

    def next(self):
        tok = self.t[self.i]
        self.i += 1
        return tok

    def expect(self, val):
        tok = self.next()
        if tok[1] != val:
            raise TdlError("Syntax", f"expected {val!r} at {tok[2]}, got {tok[1]!r}")
        return tok

    def ident(self):
        tok = self.next()
        if tok[0] != "id":
            raise TdlError("Syntax", f"expected identifier at {tok[2]}, got {tok[1]!r}")
        return tok[1]

    def accept(self, val):
        if self.peek()[1] == val:
            self.i += 1
            return True
        return False


# ----------------------------------------------------------------------------- parser
def _parse_affine(p, known_vars, stop=(",", "]")):
    """Parse an index: sum of [int *] var | int | [int *] '(' affine ')' ('/' | '%') int, with + / -
    (the parenthesised floor-division / remainder terms are reading R11)."""
    coef = {}
    const = 0
    terms = []
    sign = 1
    if p.accept("-"):
        sign = -1
    elif p.accept("+"):
        sign = 1
    while True:
        tok = p.next()
        mult = None
        if tok[0] == "num" and p.peek()[1] == "*" and p.t[p.i + 1][1] == "(":
            if "." in tok[1]:
                raise TdlError("NonAffineIndex", "non-integer constant in index")
            mult = int(tok[1])
            p.next()
            tok = p.next()
        if tok[1] == "(":
            inner = _parse_affine(p, known_vars, stop=(")",))
            p.expect(")")
            kind = p.next()
            if kind[1] not in ("/", "%"):
                raise TdlError("NonAffineIndex", f"parenthesised index term needs / or % at {kind[2]}")
            dtok = p.next()
            if dtok[0] != "num" or "." in dtok[1] or int(dtok[1]) <= 0:
                raise TdlError("NonAffineIndex", "index division by a positive integer constant only")
            terms.append(("div" if kind[1] == "/" else "mod", sign * (1 if mult is None else mult), inner,
                          int(dtok[1])))
        elif mult is not None:
            raise TdlError("Syntax", f"bad index term at {tok[2]}")
        elif tok[0] == "num":
            if "." in tok[1]:
                raise TdlError("NonAffineIndex", "non-integer constant in index")
            n = int(tok[1])
            if p.accept("*"):
                v = p.ident()
                if v not in known_vars:
                    raise TdlError("UnknownVar", v)
                coef[v] = coef.get(v, 0) + sign * n
            else:
                const += sign * n
        elif tok[0] == "id":
            v = tok[1]
            if v not in known_vars:
                raise TdlError("UnknownVar", v)
            if p.accept("*"):
                t2 = p.next()
                if t2[0] != "num":
                    raise TdlError("NonAffineIndex", f"product of index variables at {t2[2]}")
                coef[v] = coef.get(v, 0) + sign * int(t2[1])
            else:
                coef[v] = coef.get(v, 0) + sign
        else:
            raise TdlError("Syntax", f"bad index term at {tok[2]}")
        nxt = p.peek()[1]
        if nxt == "+":
            p.next()
            sign = 1
        elif nxt == "-":
            p.next()
            sign = -1
        elif nxt in stop:
            break
        elif nxt in ("*", "/", "%"):
            raise TdlError("NonAffineIndex", "non-affine index expression")
        else:
            raise TdlError("Syntax", f"unexpected {nxt!r} in index")
    return Affine(tuple(sorted((v, c) for v, c in coef.items() if c != 0)), const, tuple(terms))


class _BodyParser:
    def __init__(self, p, params, vars_):
        self.p = p
        self.params = dict(params)
        self.vars = set(vars_)
        self.accesses = []

    def access(self, name, allow_slice=False):
        p = self.p
        if name not in self.params:
            raise TdlError("UndeclaredTensor", name)
        p.expect("[")
        idx = []
        while True:
            if allow_slice and p.peek()[1] == ":":
                p.next()
                idx.append(None)
            else:
                idx.append(_parse_affine(p, self.vars))
            if p.accept("]"):
                break
            p.expect(",")
        if len(idx) != self.params[name]:
            raise TdlError("RankMismatch", f"{name} has rank {self.params[name]}, indexed with {len(idx)}")
        acc = Access(name, tuple(idx))
        return acc

    def primary(self):
        p = self.p
        tok = p.next()
        if tok[0] == "num":
            return Expr("num", float(tok[1]))
        if tok[1] == "(":
            e = self.expr()
            p.expect(")")
            return e
        if tok[1] == "-":
            return Expr("neg", None, [self.primary()])
        if tok[0] == "id":
            name = tok[1]
            if name in REDUCERS or name == "reduce":
                raise TdlError("NestedReduce", "reduce only allowed at top level")
            if p.peek()[1] == "[":
                acc = self.access(name)
                self.accesses.append(acc)
                return Expr("access", acc)
            if p.peek()[1] == "(":
                if name not in FUNCS:
                    raise TdlError("Syntax", f"unknown function {name}")
                p.next()
                args = [self.expr()]
                while p.accept(","):
                    args.append(self.expr())
                p.expect(")")
                if len(args) != FUNCS[name]:
                    raise TdlError("Syntax", f"{name} takes {FUNCS[name]} args")
                return Expr("call", name, args)
            if name in self.vars:
                return Expr("var", name)
            if name in self.params:
                raise TdlError("RankMismatch", f"tensor {name} used without index")
            raise TdlError("UnknownVar", name)
        raise TdlError("Syntax", f"unexpected {tok[1]!r} at {tok[2]}")

    def term(self):
        e = self.primary()
        while self.p.peek()[1] in ("*", "/"):
            op = self.p.next()[1]
            e = Expr("bin", op, [e, self.primary()])
        return e

    def arith(self):
        e = self.term()
        while self.p.peek()[1] in ("+", "-"):
            op = self.p.next()[1]
            e = Expr("bin", op, [e, self.term()])
        return e

    def expr(self):
        e = self.arith()
        if self.p.peek()[1] in (">", "<", ">=", "<=", "=="):
            op = self.p.next()[1]
            e = Expr("bin", op, [e, self.arith()])
        return e


def parse_def(src: str) -> OpDef:
    """parse_tdl for one ``def`` (grammar in module docstring)."""
    p = _P(src)
    if p.ident() != "def":
        raise TdlError("Syntax", "expected 'def'")
    name = p.ident()
    p.expect("(")
    params = []
    if not p.accept(")"):
        while True:
            t = p.ident()
            p.expect("(")
            r = p.next()
            if r[0] != "num":
                raise TdlError("Syntax", "expected rank")
            p.expect(")")
            params.append((t, int(r[1])))
            if p.accept(")"):
                break
            p.expect(",")
    names = [n for n, _ in params]
    if len(set(names)) != len(names):
        raise TdlError("Syntax", "duplicate parameter")
    p.expect("->")
    if p.ident() != "lambda":
        raise TdlError("Syntax", "expected lambda")
    out_vars = []
    if p.peek()[1] != ":":
        while True:
            out_vars.append(p.ident())
            if p.accept(":"):
                break
            p.expect(",")
    else:
        p.next()
    reducer = None
    red_vars = []
    opaque = False
    opaque_free = []
    tok = p.peek()
    if tok[1] == "reduce":
        p.next()
        p.expect("(")
        reducer = p.ident()
        if reducer not in REDUCERS:
            raise TdlError("Syntax", f"unknown reducer {reducer}")
        p.expect(";")
        while True:
            red_vars.append(p.ident())
            if p.accept(";"):
                break
            p.expect(",")
        if set(red_vars) & set(out_vars):
            raise TdlError("Syntax", "reduce vars overlap output vars")
        bp = _BodyParser(p, params, out_vars + red_vars)
        body = bp.expr()
        p.expect(")")
    elif tok[1] == "opaque":
        p.next()
        p.expect("(")
        fn = p.ident()
        p.expect(";")
        bp = _BodyParser(p, params, out_vars)
        tname = p.ident()
        acc = bp.access(tname, allow_slice=True)
        p.expect(")")
        p.expect("[")
        res = []
        while True:
            res.append(p.ident())
            if p.accept("]"):
                break
            p.expect(",")
        opaque = True
        # pass-through dims: output vars used directly as the index of a non-sliced dim
        for ix in acc.index:
            if ix is not None and ix.is_var():
                opaque_free.append(ix.coef[0][0])
        bp.accesses.append(acc)
        body = Expr("opaque", fn, [Expr("access", acc), res])
    else:
        bp = _BodyParser(p, params, out_vars)
        body = bp.expr()
    if p.peek()[0] != "eof":
        raise TdlError("Syntax", f"trailing input at {p.peek()[2]}")
    d = OpDef(name, params, out_vars, reducer, red_vars, body, bp.accesses, opaque, opaque_free)
    _validate(d)
    return d


def _validate(d: OpDef):
    used = set()
    for acc in d.accesses:
        seen = {}
        for dim, ix in enumerate(acc.index):
            if ix is None:
                continue
            for v in ix.vars():
                used.add(v)
                if v in seen and seen[v] != dim:
                    # Assumption #1: one output index accesses one dim per tensor
                    raise TdlError("AssumptionViolation", f"{v} indexes two dims of {acc.tensor}")
                seen[v] = dim
    for v in d.red_vars:
        if v not in used:
            raise TdlError("Syntax", f"reduce var {v} indexes no input")


def parse_program(src: str) -> dict:
    """Parse a file of defs separated by lines starting with 'def'.  '#' comments."""
    lines = [ln.split("#", 1)[0] for ln in src.splitlines()]
    chunks, cur = [], []
    for ln in lines:
        if ln.strip().startswith("def ") and cur:
            chunks.append("\n".join(cur))
            cur = []
        if ln.strip():
            cur.append(ln)
    if cur:
        chunks.append("\n".join(cur))
    out = {}
    for c in chunks:
        d = parse_def(c)
        if d.name in out:
            raise TdlError("Syntax", f"duplicate def {d.name}")
        out[d.name] = d
    return out


def classify(d: OpDef):
    """OpClass (§5.1: element-wise if inputs/outputs partitioned identically).

    ElementWise iff no reducer, not opaque, and every access is exactly the
    identity tuple of the output vars.  Returns ('ElementWise'|'Reduction'|
    'OpaqueBatched'|'General', payload)."""
    if d.opaque:
        return ("OpaqueBatched", list(d.opaque_free))
    if d.reducer:
        return ("Reduction", list(d.red_vars))
    ident = tuple(Affine(((v, 1),), 0) for v in d.out_vars)
    if d.accesses and all(a.index == ident for a in d.accesses):
        return ("ElementWise", None)
    return ("General", None)


def split_vars(d: OpDef):
    """Index variables a strategy may split: output vars (Case-1) and reduce
    vars (Case-2).  Opaque ops: only pass-through batch vars."""
    if d.opaque:
        return list(d.opaque_free)
    return list(d.out_vars) + list(d.red_vars)


def var_ranges(d: OpDef, in_shapes: dict, out_shape, given: dict | None = None) -> dict:
    """Concrete extent of every index variable.  Output vars from the output
    shape; reduce vars from the first input dim they index alone (coef 1,
    no other var) or, failing that, bounded by dim size."""
    R = {}
    for v, n in zip(d.out_vars, out_shape):
        R[v] = int(n)
    for v in d.red_vars:
        if given and v in given:
            R[v] = int(given[v])
            continue
        best = None
        for acc in d.accesses:
            for dim, ix in enumerate(acc.index):
                if ix is None:
                    continue
                if ix.is_var(v):
                    best = int(in_shapes[acc.tensor][dim])
                    break
            if best is not None:
                break
        if best is None:
            raise TdlError("UnknownVar", f"cannot infer range of reduce var {v}")
        R[v] = best
    return R
