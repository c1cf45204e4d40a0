"""Basic partition strategies (oracle side).  TEST INFRASTRUCTURE ONLY.

P:L532-561 §4.2 "Discover operator partition strategies":
* Case-1 — split an output variable: "We use two different initial intervals
  for lambda variable b, ZV[u_b=½] and ZV[l_b=½, u_b=1], in two separate
  analysis runs.  Each run calculates the input regions needed to compute half
  of the output tensor." Output = concatenation.
* Case-2 — split a reduction variable: "each partially reduced tensor will
  require half of the data tensor ... and half of the filter tensor";
  output = element-wise reduction of full-size partials.

For an s-way split the j-th worker's initialiser is ZV[l=j/s, u=(j+1)/s]
(P:L801-806 generalise the 2-way split to kᵢ-way steps).
"""
from __future__ import annotations

from fractions import Fraction as F

from .interval import SymInterval, eval_access
from .tdl import split_vars


def discover_strategies(opdef, s: int = 2):
    """One strategy per splittable variable, in declaration order (output
    vars then reduce vars).  Each strategy: dict(var, kind, ways, regions),
    regions[j] = [(tensor, [SymInterval|None per dim])] for worker j."""
    out = []
    for v in split_vars(opdef):
        kind = "Concat" if v in opdef.out_vars else "Reduce"
        regions = []
        for j in range(s):
            init = {v: SymInterval.zv(v, F(j, s), F(j + 1, s))}
            regions.append(eval_access(opdef, init))
        out.append(dict(var=v, kind=kind, ways=s, regions=regions,
                        reducer=opdef.reducer if kind == "Reduce" else None))
    return out


def classify_region(opdef, strategy, j, shapes: dict, var_extent: dict):
    """Concrete RegionSpec of worker j: per input, per dim one of
    ('Whole',), ('Slice', part, ways), ('Range', lo, hi) (halo/other)."""
    s = strategy["ways"]
    res = []
    for tensor, dims in strategy["regions"][j]:
        spec = []
        for d, iv in enumerate(dims):
            n = shapes[tensor][d]
            if iv is None:
                spec.append(("Whole",))
                continue
            lo, hi = iv.concretize(var_extent)
            lo, hi = max(lo, 0), min(hi, n - 1)
            if lo == 0 and hi == n - 1:
                spec.append(("Whole",))
            elif n % s == 0 and lo == j * n // s and hi == (j + 1) * n // s - 1:
                spec.append(("Slice", j, s))
            else:
                spec.append(("Range", lo, hi))
        res.append((tensor, spec))
    return res


def count_nd_partitions(n_dims: int, m_splits: int) -> int:
    """Ways to distribute m binary splits over n dims (multiset count
    C(n+m-1, m)); "20 different ways to partition [a 4-D tensor]
    evenly across 8 workers"."""
    from math import comb
    return comb(n_dims + m_splits - 1, m_splits)
