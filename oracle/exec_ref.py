"""Unpartitioned reference execution (oracle side).  TEST INFRASTRUCTURE ONLY.

* ``tdl_eval`` evaluates a TDL lambda literally ("the output
  tensor value at each index" is the lambda body; a reducer "aggregate[s]
  elements ... along one or more dimensions") over an iteration
  box, vectorised with numpy broadcasting, in fp64.
* ``fast_eval`` is the same for contraction defs (A[..] * B[..] summed) via
  one library einsum (allowed as a single step); pinned equal to ``tdl_eval``.
* ``run_graph`` executes a training graph op by op in list order and, when
  ``emulate_storage`` is set, rounds every stored tensor to its storage dtype
  (bf16 by round-to-nearest-even from fp64, fp32 by cast) — the points where
  the GPU path stores.  Reading §R5 in DESIGN.md.
"""
from __future__ import annotations

import numpy as np

from .tdl import Affine


def round_bf16(x):
    """Round fp64 values to the nearest bf16 (8 significant bits), ties to
    even.  Normal range only (finite, |x| < 3.4e38)."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)                   # x = m * 2**e, 0.5 <= |m| < 1
    r = np.rint(m * 256.0)               # 8 significant bits, half-to-even
    return np.ldexp(r, e - 8)


def store_round(x, dtype):
    if dtype == "bf16":
        return round_bf16(x)
    if dtype == "f32":
        return np.asarray(x, dtype=np.float32).astype(np.float64)
    return np.asarray(x, dtype=np.float64)


def _grid(vars_, box):
    n = len(vars_)
    out = {}
    for i, v in enumerate(vars_):
        lo, hi = box[v]
        shape = [1] * n
        shape[i] = hi - lo + 1
        out[v] = np.arange(lo, hi + 1).reshape(shape)
    return out


def _idx(aff: Affine, grid):
    return aff.value(grid)


def _slice_access(acc, arr, origin, grid, rank):
    """An access whose every index is a distinct plain variable, inside the array, is a slice of it: return
    that view laid out on the grid's axes (the same values _gather would produce, without index arrays)."""
    axes = []
    for ix in acc.index:
        if ix is None or not ix.is_var():
            return None
        axes.append(ix.coef[0][0])
    if len(set(axes)) != len(axes):
        return None
    order = list(grid)
    sl = []
    for d, v in enumerate(axes):
        g = grid[v]
        lo, hi = int(g.flat[0]) - origin[d], int(g.flat[-1]) - origin[d]
        if lo < 0 or hi >= arr.shape[d]:
            return None
        sl.append(slice(lo, hi + 1))
    sub = arr[tuple(sl)]
    pos = [order.index(v) for v in axes]
    sub = np.transpose(sub, np.argsort(pos))          # dims in grid-axis order
    shp = [1] * rank
    for p_, n in zip(sorted(pos), sub.shape):
        shp[p_] = n
    return sub.reshape(shp)


def _gather(arr, origin, index_arrays, shape):
    """arr[index] with zero for indices outside the array (reading R11: an access outside its tensor
    reads 0, i.e. zero padding).  Inside the tensor every access lies in the array by construction
    (the array is the tensor or a region covering the required hull)."""
    if any(n == 0 for n in arr.shape):
        return np.zeros(shape)
    local = [np.asarray(i - origin[d]) for d, i in enumerate(index_arrays)]
    if all(i.min() >= 0 and i.max() < arr.shape[d] for d, i in enumerate(local)):   # nothing outside
        return arr[tuple(np.broadcast_to(i, shape) for i in local)]
    ok = True
    idx = []
    for d, i in enumerate(local):
        i = np.broadcast_to(i, shape)
        inb = (i >= 0) & (i < arr.shape[d])
        ok = ok & inb
        idx.append(np.where(inb, i, 0))
    return np.where(ok, arr[tuple(idx)], 0.0)


def _ev(e, grid, inputs, shape):
    k = e.kind
    if k == "num":
        return np.float64(e.val)
    if k == "var":
        return grid[e.val].astype(np.float64)
    if k == "access":
        arr, origin = inputs[e.val.tensor]
        view = _slice_access(e.val, arr, origin, grid, len(shape))
        if view is not None:
            return view
        return _gather(arr, origin, [_idx(ix, grid) for ix in e.val.index], shape)
    if k == "neg":
        return -_ev(e.args[0], grid, inputs, shape)
    if k == "bin":
        a = _ev(e.args[0], grid, inputs, shape)
        b = _ev(e.args[1], grid, inputs, shape)
        op = e.val
        if op == "+":
            return a + b
        if op == "-":
            return a - b
        if op == "*":
            return a * b
        if op == "/":
            return a / b
        if op == ">":
            return (a > b).astype(np.float64)
        if op == "<":
            return (a < b).astype(np.float64)
        if op == ">=":
            return (a >= b).astype(np.float64)
        if op == "<=":
            return (a <= b).astype(np.float64)
        if op == "==":
            return (a == b).astype(np.float64)
    if k == "call":
        a = [_ev(x, grid, inputs, shape) for x in e.args]
        f = e.val
        if f == "max":
            return np.maximum(a[0], a[1])
        if f == "min":
            return np.minimum(a[0], a[1])
        if f == "exp":
            return np.exp(a[0])
        if f == "tanh":
            return np.tanh(a[0])
        if f == "sigmoid":
            return 1.0 / (1.0 + np.exp(-a[0]))
        if f == "sqrt":
            return np.sqrt(a[0])
        if f == "select":
            return np.where(np.broadcast_to(a[0], shape) != 0, a[1], a[2])
    raise ValueError(f"cannot evaluate {k}")


def tdl_eval(opdef, inputs: dict, box: dict):
    """inputs: param -> (array, origin) where origin is the global index of
    array[0,...,0].  box: var -> (lo, hi) closed, for all out and reduce vars.
    Returns the output over the out-var box (a partial if the reduce box is
    not the full range)."""
    if opdef.opaque:
        raise ValueError("opaque functions are not executable (P:L411-423)")
    vars_ = list(opdef.out_vars) + list(opdef.red_vars)
    grid = _grid(vars_, box)
    shape = tuple(box[v][1] - box[v][0] + 1 for v in vars_)
    val = np.broadcast_to(_ev(opdef.body, grid, inputs, shape), shape).astype(np.float64)
    nout = len(opdef.out_vars)
    if opdef.reducer:
        axes = tuple(range(nout, len(vars_)))
        r = opdef.reducer
        if r == "Sum":
            val = val.sum(axis=axes)
        elif r == "Max":
            val = val.max(axis=axes)
        elif r == "Min":
            val = val.min(axis=axes)
        elif r == "Prod":
            val = val.prod(axis=axes)
    return np.asarray(val, dtype=np.float64)


_MM = {
    # def name -> (A index fn, B index fn) as (rows-var-of-A...) realised with numpy
    "mm_nn": lambda A, B: A @ B,
    "mm_nt": lambda A, B: A @ B.T,
    "mm_tn": lambda A, B: A.T @ B,
}


def _contraction(opdef):
    """(A access, B access) when the body is exactly reduce(Sum; ..; A[..] * B[..]) with single-variable
    indices, else None."""
    b = opdef.body
    if opdef.reducer != "Sum" or b.kind != "bin" or b.val != "*":
        return None
    x, y = b.args
    if x.kind != "access" or y.kind != "access":
        return None
    for acc in (x.val, y.val):
        for ix in acc.index:
            if ix is None or not ix.is_var():
                return None
    return x.val, y.val


def _product(opdef):
    """(A access, B access) when the body is reduce(Sum; ..; A[..] * B[..]) with any index forms."""
    b = opdef.body
    if opdef.reducer != "Sum" or b.kind != "bin" or b.val != "*":
        return None
    x, y = b.args
    if x.kind != "access" or y.kind != "access" or any(ix is None for a in (x, y) for ix in a.val.index):
        return None
    return x.val, y.val


def tap_eval(opdef, inputs: dict, box: dict):
    """Sum-of-products defs whose indices mix variables (convolutions: ``X[b, y + ky - 1, ..]``) evaluated
    as the sum over "tap" values of one library einsum each: every index dimension that mixes several
    variables has all but one of them fixed (the smallest extents: the filter taps), the tap values are
    looped over, and for each the operands are gathered (zero outside the tensor, R11) into arrays with
    one axis per remaining variable and contracted by einsum.  The taps' partial sums are added in tap
    order.  Returns None when the def does not have this form (e.g. a variable left in two dims)."""
    con = _product(opdef)
    if con is None:
        return None
    ext = {v: box[v][1] - box[v][0] + 1 for v in opdef.all_vars()}
    fixed = []
    while True:
        cand = None
        for acc in con:
            for ix in acc.index:
                free = [v for v in ix.vars() if v not in fixed]
                if len(free) >= 2:
                    cand = min(free, key=lambda v: (ext[v], v))
                    break
            if cand:
                break
        if cand is None:
            break
        fixed.append(cand)
    plan = []   # per operand: [(dim, free var or None)]
    for acc in con:
        dims, seen = [], set()
        for d, ix in enumerate(acc.index):
            free = [v for v in ix.vars() if v not in fixed]
            if len(free) > 1 or (free and free[0] in seen):
                return None
            dims.append(free[0] if free else None)
            seen.update(free)
        plan.append(dims)
    letters = {v: chr(ord("a") + i) for i, v in enumerate(opdef.all_vars())}
    out_free = [v for v in opdef.out_vars if v not in fixed]
    out = np.zeros(tuple(ext[v] for v in opdef.out_vars))
    import itertools
    for tap in itertools.product(*[range(box[v][0], box[v][1] + 1) for v in fixed]):
        env = dict(zip(fixed, tap))
        ops, subs = [], []
        for acc, dims in zip(con, plan):
            arr, origin = inputs[acc.tensor]
            axes = [v for v in dims if v is not None]
            gshape = tuple(ext[v] for v in axes)
            grid = dict(env)
            for i, v in enumerate(axes):
                sh = [1] * len(axes)
                sh[i] = ext[v]
                grid[v] = np.arange(box[v][0], box[v][1] + 1).reshape(sh)
            idx = [np.asarray(ix.value(grid)) for ix in acc.index]
            ops.append(_gather(arr, origin, idx, gshape))
            subs.append("".join(letters[v] for v in axes))
        part = np.einsum(f"{subs[0]},{subs[1]}->{''.join(letters[v] for v in out_free)}", ops[0], ops[1], optimize=True)
        sl = tuple(env[v] - box[v][0] if v in env else slice(None) for v in opdef.out_vars)
        out[sl] += part
    return out


def fast_eval(opdef, inputs: dict, box: dict):
    """Library evaluation (numpy einsum -> BLAS) of contraction defs over a box — one library primitive
    for the whole sum, as the TDL text states it; anything else goes to tdl_eval."""
    con = _contraction(opdef)
    if con is None:
        r = tap_eval(opdef, inputs, box)
        return tdl_eval(opdef, inputs, box) if r is None else r
    letters = {v: chr(ord("a") + i) for i, v in enumerate(opdef.all_vars())}
    ops, subs = [], []
    for acc in con:
        arr, origin = inputs[acc.tensor]
        sl = []
        for d, ix in enumerate(acc.index):
            v = ix.coef[0][0]
            sl.append(slice(box[v][0] - origin[d], box[v][1] - origin[d] + 1))
        ops.append(np.asarray(arr[tuple(sl)], dtype=np.float64))
        subs.append("".join(letters[ix.coef[0][0]] for ix in acc.index))
    out = "".join(letters[v] for v in opdef.out_vars)
    return np.einsum(f"{subs[0]},{subs[1]}->{out}", ops[0], ops[1], optimize=True)


def full_box(g, op):
    R = g.ranges[op["name"]]
    return {v: (0, n - 1) for v, n in R.items()}


def run_graph(g, values: dict, emulate_storage=True, fast=True):
    """Execute every op of g in order on full tensors.  values: initial
    tensors (inputs / weights / state) as fp64 arrays.  Returns dict of all
    tensors (fp64 arrays holding storage-rounded values when emulating)."""
    env = {t: np.asarray(v, dtype=np.float64) for t, v in values.items()}
    for op in g.ops:
        d = g.opdef(op)
        # an input offset o means the def's index i reads tensor element i + o (output views, §R10)
        ins = {p: (env[t], tuple(-x for x in off)) for (p, _), t, off in zip(d.params, op["inputs"], op["offsets"])}
        box = full_box(g, op)
        out = (fast_eval if fast else tdl_eval)(d, ins, box)
        R = g.ranges[op["name"]]
        oshape = [R[v] for v in d.out_vars]
        out = np.asarray(out, dtype=np.float64).reshape(oshape)
        if emulate_storage:
            out = store_round(out, g.tensors[op["output"]]["dtype"])
        t = op["output"]
        if list(oshape) == list(g.shape(t)) and not any(op["out_offset"]):
            env[t] = out
        else:
            full = env.get(t)
            full = np.zeros(g.shape(t)) if full is None else full.copy()
            full[tuple(slice(o, o + n) for o, n in zip(op["out_offset"], oshape))] = out
            env[t] = full
    return env
