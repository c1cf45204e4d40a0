"""Partitioned execution on k simulated workers (oracle side).  TEST INFRASTRUCTURE ONLY.

Partition-n-reduce (§3.1): every worker runs the *same* operator
on its sub-box; "O is the concatenation of O₁ and O₂ along some dimension"
or "the element-wise reduction of O₁ and O₂".  Remote input regions are
assembled in place from their owners (MultiFetch) and partial
outputs are sent to the owner of each element, which sums them (reduction
spread over all GPUs).  Owners sum contributions in ascending
rank order, in fp64 unless ``partial_dtype`` says otherwise.

Ownership is computed element-wise by successive integer division (no box
arithmetic), and every transferred element is counted: the ledger must equal
``cost.plan_cost`` for the same plan.
"""
from __future__ import annotations

import itertools

import numpy as np

from .cost import digits, nested_range
from .exec_ref import fast_eval, store_round


def owner_map(shape, dims_seq, factors):
    """int array of shape `shape`: owner worker id of every element."""
    m = len(factors)
    if len(shape) == 0:
        return np.zeros((), dtype=np.int64)
    dig = [np.zeros(shape, dtype=np.int64) for _ in range(m)]
    for dim in range(len(shape)):
        steps = [i for i in range(m) if dims_seq[i] == dim]
        bshape = [1] * len(shape)
        bshape[dim] = shape[dim]
        rem = np.arange(shape[dim]).reshape(bshape)
        size = shape[dim]
        for i in steps:
            size //= factors[i]
            dig[i] = dig[i] + np.broadcast_to(rem // size, shape)
            rem = rem % size
    w = np.zeros(shape, dtype=np.int64)
    for i in range(m):
        w = w * factors[i] + dig[i]
    return w


def simulate(g, plan, values, emulate_storage=False):
    """Returns (result tensors assembled from owners, ledger dict).

    ledger: elements (total), bytes (wire dtypes, fp32 for partials),
    per-op element counts, per-worker sent/received elements."""
    factors = plan["factors"]
    nw = int(np.prod(factors)) if factors else 1
    owners = {t: owner_map(g.shape(t), plan["tdims"][t], factors) for t in g.tensors}
    # local storage: full-size arrays, NaN where not owned
    local = [dict() for _ in range(nw)]
    for t, v in values.items():
        v = np.asarray(v, dtype=np.float64)
        for w in range(nw):
            a = np.full(v.shape, np.nan)
            mask = owners[t] == w
            a[mask] = v[mask]
            local[w][t] = a
    ledger = {"elements": 0, "bytes": 0, "per_op": {}, "sent": [0] * nw, "recv": [0] * nw}
    isz = {"bf16": 2, "f32": 4, "f64": 8}
    for op in g.ops:
        d = g.opdef(op)
        R = g.ranges[op["name"]]
        vars_ = d.all_vars()
        seq = plan["osplit"][op["name"]]
        partial = any(v in d.red_vars for v in seq)
        o_t = op["output"]
        oshape = tuple(g.shape(o_t))
        contrib = []   # (worker, box, values)
        op_el = 0
        for w in range(nw):
            dig = digits(w, factors)
            box = {}
            for v in vars_:
                sp = [(factors[i], dig[i]) for i in range(len(factors)) if seq[i] == v]
                box[v] = nested_range(R[v], sp)
            ins = {}
            for (p, _), t, poff in zip(d.params, op["inputs"], op["offsets"]):
                shape = g.shape(t)
                # required hull of every access to this param
                lo = [None] * len(shape)
                hi = [None] * len(shape)
                for acc in d.accesses:
                    if acc.tensor != p:
                        continue
                    for dim, ix in enumerate(acc.index):
                        if ix is None:
                            a, b = 0, shape[dim] - 1
                        else:
                            a, b = ix.hull(box, poff[dim])
                            a, b = max(a, 0), min(b, shape[dim] - 1)   # outside the tensor: zeros (R11)
                        lo[dim] = a if lo[dim] is None else min(lo[dim], a)
                        hi[dim] = b if hi[dim] is None else max(hi[dim], b)
                sl = tuple(slice(a, b + 1) for a, b in zip(lo, hi))
                own = owners[t][sl]
                region = np.zeros(own.shape)
                for src in range(nw):
                    mask = own == src
                    if not mask.any():
                        continue
                    region[mask] = local[src][t][sl][mask]
                    if src != w:
                        n = int(mask.sum())
                        ledger["elements"] += n
                        op_el += n
                        ledger["bytes"] += n * isz[g.tensors[t]["dtype"]]
                        ledger["sent"][src] += n
                        ledger["recv"][w] += n
                assert not np.isnan(region).any(), (op["name"], t)
                ins[p] = (region, tuple(a - b for a, b in zip(lo, poff)))
            val = fast_eval(d, ins, box)
            obox = [(box[v][0] + off, box[v][1] + off) for v, off in zip(d.out_vars, op["out_offset"])]
            contrib.append((w, obox, np.asarray(val, dtype=np.float64).reshape(
                tuple(b - a + 1 for a, b in obox))))
        # route produced values to owners; owners sum in rank order.  Elements outside this op's output
        # view keep their current value (another op, or the initial value, owns them).
        cur = np.full(oshape, np.nan)
        if o_t in local[0]:
            for w in range(nw):
                mask = owners[o_t] == w
                cur[mask] = local[w][o_t][mask]
        cur = np.where(np.isnan(cur), 0.0, cur)
        lo_o = [min(c[1][dd][0] for c in contrib) for dd in range(len(oshape))]
        hi_o = [max(c[1][dd][1] for c in contrib) for dd in range(len(oshape))]
        view = tuple(slice(a, b + 1) for a, b in zip(lo_o, hi_o))
        acc = np.zeros(oshape)
        for w, obox, val in contrib:
            sl = tuple(slice(a, b + 1) for a, b in obox)
            own = owners[o_t][sl]
            acc[sl] += val
            n = int((own != w).sum())
            ledger["elements"] += n
            op_el += n
            ledger["bytes"] += n * (4 if partial else isz[g.tensors[o_t]["dtype"]])
            for dst in range(nw):
                c = int(((own == dst) & (own != w)).sum())
                if c:
                    ledger["sent"][w] += c
                    ledger["recv"][dst] += c
        if oshape:
            cur[view] = acc[view]
        else:
            cur = acc
        acc = cur
        if emulate_storage:
            acc = store_round(acc, g.tensors[o_t]["dtype"])
        for w in range(nw):
            a = np.full(oshape, np.nan)
            mask = owners[o_t] == w
            a[mask] = acc[mask]
            local[w][o_t] = a
        ledger["per_op"][op["name"]] = op_el
    result = {}
    for t in local[0]:
        full = np.full(g.shape(t), np.nan)
        for w in range(nw):
            mask = owners[t] == w
            full[mask] = local[w][t][mask]
        result[t] = full
    return result, ledger
