"""Communication cost of a partition plan (oracle side).  TEST INFRASTRUCTURE ONLY.

The paper minimises "the total communication cost" (§5).  The
Lemma's proof names the two sources of communication:

  * "The selected partition-n-reduce strategy requires input region that is
    not available locally."
  * "The selected partition-n-reduce strategy produces output region that is
    assigned to other devices."

Reading ("direct transfer" model): a k-way plan is a sequence
of basic plans ⟨p₁..p_m⟩ with step factors k₁..k_m.  Worker w
has mixed-radix digits (w₁..w_m), step 1 most significant.  Along a tensor
dim (or an op index variable) split by steps S = [i : dᵢ = dim] the part of
worker w is the nested even split by k_i, i ∈ S in step order.  Then

  cost(P) = Σ_ops Σ_w [ Σ_inputs |Req_w(in) \\ Own_w(in)| + |Prod_w(out) \\ Own_w(out)| ]

where Req_w is the (per-dim interval hull of the) region worker w's sub-op
reads, Prod_w its produced output box (a full-size partial when a reduction
variable is split; partials go to the owner, who sums them — the spread
reduction of P:L879-881).  This is exactly what a P2P executor moves, so the
executor's byte ledger must equal it.  A plan prefix of i steps is costed the
same way with Π_{j≤i} k_j worker groups; δᵢ = cost(prefix_i) − cost(prefix_{i−1})
(the per-step cost of P:L1646-1651).  Rank-0 tensors are not split and are
owned by worker 0.

Units: elements (the planner objective, uniform element weight — the Lemma's
"weighted sum of the size of each tensor").  Bytes use the
wire dtype: the tensor's dtype for fetches and complete outputs, fp32 (4 B)
for partial outputs.

Two independent evaluations: ``op_cost_box`` (interval arithmetic on boxes)
and ``op_cost_enum`` (enumerate iteration points and owned elements, tiny
shapes only).
"""
from __future__ import annotations

import itertools

from .graph import ITEMSIZE


def digits(w, factors):
    """Mixed-radix digits of worker w, step 1 most significant."""
    out = []
    for k in reversed(factors):
        out.append(w % k)
        w //= k
    return list(reversed(out))


def nested_range(n, splits):
    """Closed range [lo, hi] of the part selected by splits=[(k, digit)...]
    (step order) of an extent-n axis.  Requires divisibility at each level."""
    lo, size = 0, n
    for k, dgt in splits:
        assert size % k == 0, (n, splits)
        size //= k
        lo += dgt * size
    return lo, lo + size - 1


def _box(extents, seq, factors, dig, names=None):
    """Box of one worker: seq[i] = split axis (index into extents or a var
    name) at step i, or None (no split of this entity at step i)."""
    axes = names if names is not None else list(range(len(extents)))
    box = []
    for a, n in zip(axes, extents):
        sp = [(factors[i], dig[i]) for i in range(len(factors)) if seq[i] == a]
        box.append(nested_range(n, sp))
    return box


def owned_box(shape, dims_seq, factors, dig):
    if len(shape) == 0:
        return [] if all(d == 0 for d in dig) else None  # rank 0: worker 0 owns it
    return _box(shape, dims_seq, factors, dig)


def iter_box(ranges: dict, var_order, splits_seq, factors, dig):
    ext = [ranges[v] for v in var_order]
    return dict(zip(var_order, _box(ext, splits_seq, factors, dig, names=var_order)))


def access_hull(aff, ibox, off=0):
    return aff.hull(ibox, off)


def clip(box, shape):
    """Required region ∩ the tensor: elements outside a tensor read as zero (reading R11) and are never
    communicated."""
    return [(max(lo, 0), min(hi, n - 1)) for (lo, hi), n in zip(box, shape)]


def _vol(box):
    p = 1
    for lo, hi in box:
        p *= max(0, hi - lo + 1)
    return p


def _inter(a, b):
    return [(max(x[0], y[0]), min(x[1], y[1])) for x, y in zip(a, b)]


def op_cost_box(g, op, tdims, osplit, factors):
    """(elements, bytes, fetch_elems, out_elems) of one op under a plan
    prefix.  tdims[t] / osplit[op] are sequences of len(factors)."""
    sl = op_cost_slots(g, op, tdims, osplit, factors)
    fetch = sum(e for kind, _, e, _ in sl if kind == "in")
    out = sum(e for kind, _, e, _ in sl if kind == "out")
    return fetch + out, sum(b for _, _, _, b in sl), fetch, out


def op_cost_slots(g, op, tdims, osplit, factors):
    """The terms of op_cost_box, one per operand slot: [("in", param, elements, bytes) for each input
    param that is read, then ("out", output, elements, bytes)].  The cost above is the sum of these
    slots, and a slot's term reads only its own tensor's dim sequence (and the op's split sequence)."""
    d = g.opdef(op)
    R = g.ranges[op["name"]]
    var_order = d.all_vars()
    seq = osplit[op["name"]]
    nw = 1
    for k in factors:
        nw *= k
    partial = any(v in d.red_vars for v in seq)
    slots = {p_: [0, 0] for p_, _ in d.params}
    read = set()
    o_el = o_by = 0
    param_t = {p: t for (p, _), t in zip(d.params, op["inputs"])}
    param_off = {p: off for (p, _), off in zip(d.params, op["offsets"])}
    o_t = op["output"]
    for w in range(nw):
        dig = digits(w, factors)
        ib = iter_box(R, var_order, seq, factors, dig)
        for p_, _ in d.params:
            # one required region per param: the hull of all its accesses
            req = None
            t = param_t[p_]
            shape = g.shape(t)
            for acc in d.accesses:
                if acc.tensor != p_:
                    continue
                r = [(0, shape[dim] - 1) if ix is None else access_hull(ix, ib, param_off[p_][dim])
                     for dim, ix in enumerate(acc.index)]
                req = r if req is None else [(min(a[0], b[0]), max(a[1], b[1])) for a, b in zip(req, r)]
            if req is None:
                continue
            read.add(p_)
            req = clip(req, shape)
            own = owned_box(shape, tdims[t], factors, dig)
            n_req = _vol(req)
            n_loc = 0 if own is None else _vol(_inter(req, own))
            slots[p_][0] += n_req - n_loc
            slots[p_][1] += (n_req - n_loc) * ITEMSIZE[g.tensors[t]["dtype"]]
        prod = [(ib[v][0] + off, ib[v][1] + off) for v, off in zip(d.out_vars, op["out_offset"])]
        own = owned_box(g.shape(o_t), tdims[o_t], factors, dig)
        n_p = _vol(prod)
        n_loc = 0 if own is None else _vol(_inter(prod, own))
        o_el += n_p - n_loc
        o_by += (n_p - n_loc) * (4 if partial else ITEMSIZE[g.tensors[o_t]["dtype"]])
    return [("in", p_, slots[p_][0], slots[p_][1]) for p_, _ in d.params if p_ in read] + [("out", o_t, o_el, o_by)]


def _owner_of(idx, shape, dims_seq, factors):
    """Owner worker of element idx (independent of nested_range: successive
    integer division).  Rank-0 → worker 0."""
    m = len(factors)
    dig = [0] * m
    if len(shape) == 0:
        return 0
    for dim in range(len(shape)):
        steps = [i for i in range(m) if dims_seq[i] == dim]
        rem, size = idx[dim], shape[dim]
        for i in steps:
            size //= factors[i]
            dig[i] = rem // size
            rem = rem % size
    w = 0
    for i in range(m):
        w = w * factors[i] + dig[i]
    return w


def op_cost_enum(g, op, tdims, osplit, factors):
    """Element-enumeration evaluation of op_cost_box's element count (tiny
    shapes).  Iteration points are assigned to workers by successive division
    of each split variable; accessed elements are enumerated and hulled."""
    d = g.opdef(op)
    R = g.ranges[op["name"]]
    vars_ = d.all_vars()
    seq = osplit[op["name"]]
    m = len(factors)
    nw = 1
    for k in factors:
        nw *= k
    param_t = {p: t for (p, _), t in zip(d.params, op["inputs"])}
    param_off = {p: off for (p, _), off in zip(d.params, op["offsets"])}
    pts = {w: [] for w in range(nw)}
    for point in itertools.product(*[range(R[v]) for v in vars_]):
        env = dict(zip(vars_, point))
        dig = [0] * m
        for v in vars_:
            steps = [i for i in range(m) if seq[i] == v]
            rem, size = env[v], R[v]
            for i in steps:
                size //= factors[i]
                dig[i] = rem // size
                rem %= size
        w = 0
        for i in range(m):
            w = w * factors[i] + dig[i]
        pts[w].append(env)
    total = 0
    for w in range(nw):
        if not pts[w]:
            continue
        for p_, _ in d.params:
            t = param_t[p_]
            shape = g.shape(t)
            lo = [None] * len(shape)
            hi = [None] * len(shape)
            for acc in d.accesses:
                if acc.tensor != p_:
                    continue
                for env in pts[w]:
                    pt = [(0, shape[dim] - 1) if ix is None else (ix.value(env) + param_off[p_][dim],) * 2
                          for dim, ix in enumerate(acc.index)]
                    for dim, (a, b) in enumerate(pt):
                        lo[dim] = a if lo[dim] is None else min(lo[dim], a)
                        hi[dim] = b if hi[dim] is None else max(hi[dim], b)
            # the hull of the accessed indices ∩ the tensor (outside it: zeros, not data, R11)
            lo = [None if a is None else max(a, 0) for a in lo]
            hi = [None if b is None else min(b, n - 1) for b, n in zip(hi, shape)]
            if lo and lo[0] is None:
                continue
            for idx in itertools.product(*[range(a, b + 1) for a, b in zip(lo, hi)]):
                if _owner_of(idx, shape, tdims[t], factors) != w:
                    total += 1
        o_t = op["output"]
        oshape = g.shape(o_t)
        produced = {tuple(env[v] + off for v, off in zip(d.out_vars, op["out_offset"])) for env in pts[w]}
        for idx in produced:
            if _owner_of(idx, oshape, tdims[o_t], factors) != w:
                total += 1
    return total


def plan_cost(g, plan, upto=None):
    """Total (elements, bytes) of a plan (or of its first `upto` steps)."""
    factors = plan["factors"][:upto] if upto is not None else plan["factors"]
    m = len(factors)
    td = {t: list(s)[:m] for t, s in plan["tdims"].items()}
    osp = {o: list(s)[:m] for o, s in plan["osplit"].items()}
    el = by = 0
    for op in g.ops:
        e, b, _, _ = op_cost_box(g, op, td, osp, factors)
        el += e
        by += b
    return el, by


def step_costs(g, plan):
    """δᵢ = cost(prefix_i) − cost(prefix_{i−1}) in elements."""
    out = []
    prev = 0
    for i in range(1, len(plan["factors"]) + 1):
        c, _ = plan_cost(g, plan, upto=i)
        out.append(c - prev)
        prev = c
    return out


def stored_elements(g, plan, w):
    """Elements of all tensors owned by worker w (per-worker
    storage is 1/k of the total)."""
    f = plan["factors"]
    dig = digits(w, f)
    tot = 0
    for t, info in g.tensors.items():
        own = owned_box(info["shape"], plan["tdims"][t], f, dig)
        if own is not None:
            tot += _vol(own)
    return tot
