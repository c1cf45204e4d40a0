"""Symbolic interval analysis (oracle side).  TEST INFRASTRUCTURE ONLY.

Eq. 1 (§4.2): an interval is an affine transformation of the
symbolic upper bounds 𝒳ᵢ,

    𝓘 ≜ [Σ lᵢ𝒳ᵢ + c, Σ uᵢ𝒳ᵢ + c],

with the arithmetic of Fig. int-arith: 𝓘 ± k, 𝓘 × k, 𝓘 / k,
𝓘 ± 𝓘'.  "Product or comparison between two intervals are not supported and
will raise an error".

Readings:
* 𝒳ᵢ is the largest index of variable i — "the range of index variable xi
  [is] [0, 𝒳ᵢ]" — so for an extent n, 𝒳ᵢ = n − 1 and the
  interval is closed.  Concretisation is [⌈lo⌉, ⌊hi⌋].  With this reading the
  paper's shift_two example is reproduced exactly and splits of
  a divisible extent into s parts are exact.
* Lower and upper bounds carry separate constants (c_lo, c_hi); the paper's
  single c cannot express the split initialiser ZV[l=½,u=1] shifted by a
  constant.  Multiplication by a negative constant swaps the bounds.
* Coefficients are exact rationals (fractions.Fraction).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction as F


class NonAffineError(Exception):
    pass


@dataclass(frozen=True)
class SymInterval:
    lo: tuple   # ((sym, Fraction), ...) sorted
    c_lo: F
    hi: tuple
    c_hi: F

    # -- construction ------------------------------------------------------
    @staticmethod
    def const(k) -> "SymInterval":
        k = F(k)
        return SymInterval((), k, (), k)

    @staticmethod
    def zv(sym, l=0, u=1) -> "SymInterval":
        """ZV[l_i=l, u_i=u]: all zeros except the coefficients of
        𝒳_sym.  Default ZV[u_i=1] = the full range [0, 𝒳ᵢ]."""
        lo = ((sym, F(l)),) if F(l) != 0 else ()
        hi = ((sym, F(u)),) if F(u) != 0 else ()
        return SymInterval(lo, F(0), hi, F(0))

    # -- Fig. int-arith ----------------------------------------------------
    def add_const(self, k):
        k = F(k)
        return SymInterval(self.lo, self.c_lo + k, self.hi, self.c_hi + k)

    def mul_const(self, k):
        k = F(k)
        lo = tuple((s, c * k) for s, c in self.lo if c * k != 0)
        hi = tuple((s, c * k) for s, c in self.hi if c * k != 0)
        if k >= 0:
            return SymInterval(lo, self.c_lo * k, hi, self.c_hi * k)
        return SymInterval(hi, self.c_hi * k, lo, self.c_lo * k)

    def div_const(self, k):
        return self.mul_const(F(1) / F(k))

    def add(self, other: "SymInterval"):
        return SymInterval(_addc(self.lo, other.lo), self.c_lo + other.c_lo,
                           _addc(self.hi, other.hi), self.c_hi + other.c_hi)

    def sub(self, other: "SymInterval"):
        return self.add(other.mul_const(-1))

    def mul(self, other):
        raise NonAffineError("product of two intervals (P:L526-529)")

    def compare(self, other):
        raise NonAffineError("comparison of two intervals (P:L526-529)")

    # -- concretisation ----------------------------------------------------
    def concretize(self, bounds: dict):
        """bounds: sym -> extent n (so 𝒳 = n − 1).  Returns closed integer
        range (lo, hi) with lo = ⌈lower⌉, hi = ⌊upper⌋ (empty if lo > hi)."""
        lo = self.c_lo + sum(c * (F(bounds[s]) - 1) for s, c in self.lo)
        hi = self.c_hi + sum(c * (F(bounds[s]) - 1) for s, c in self.hi)
        return (math.ceil(lo), math.floor(hi))

    def vector(self, syms):
        """⟨l₁..lₙ, u₁..uₙ, c_lo, c_hi⟩."""
        dl, dh = dict(self.lo), dict(self.hi)
        return [dl.get(s, F(0)) for s in syms] + [dh.get(s, F(0)) for s in syms] + [self.c_lo, self.c_hi]


def _addc(a, b):
    d = dict(a)
    for s, c in b:
        d[s] = d.get(s, F(0)) + c
    return tuple(sorted((s, c) for s, c in d.items() if c != 0))


def eval_affine(aff, env: dict) -> SymInterval:
    """Symbolically execute an affine index expression Σ aᵥ·v + c
    ("symbolically execute the lambda function")."""
    acc = SymInterval.const(aff.const)
    for v, a in aff.coef:
        acc = acc.add(env[v].mul_const(a))
    for kind, mult, inner, d in aff.terms:
        if kind == "div":   # 𝓘 / k (Fig. int-arith)
            acc = acc.add(eval_affine(inner, env).div_const(d).mul_const(mult))
        else:               # remainder: [0, d-1] (reading R11)
            acc = acc.add(SymInterval((), F(min(0, mult * (d - 1))), (), F(max(0, mult * (d - 1)))))
    return acc


def eval_access(opdef, init: dict):
    """AccessMap: for every input access, per dim, the SymInterval of accessed
    coordinates.  Uninitialised vars default to ZV[u=1] (full range)."""
    env = {v: init.get(v, SymInterval.zv(v)) for v in opdef.all_vars()}
    out = []
    for acc in opdef.accesses:
        dims = []
        for ix in acc.index:
            dims.append(None if ix is None else eval_affine(ix, env))
        out.append((acc.tensor, dims))
    return out
