"""Partition search (oracle side).  TEST INFRASTRUCTURE ONLY.

* ``step_search`` — one basic-plan step: "run the DP algorithm with coarsening
  to partition G for two worker groups ... each tensor is only partitioned
  along one dimension" (§5.2).  The DP over the coarsened graph
  ([jia2018exploring], plus "brute-force combinatorial search
  among all member operators/tensors within the group") is
  realised as exact min-sum variable elimination over tensor-class and
  op-class variables; on a chain this is the chain DP.  All co-optimal step
  plans are enumerated (up to ``cap``).
* ``recursive_search`` — P:L755-764 §5.2 steps 1-3, for k = k₁·…·k_m with
  kᵢ ≥ kᵢ₊₁.  Each step minimises the exact cost of the
  prefix (cost.py); the set of co-optimal prefixes is carried forward
  (reading §R4: ties are kept because under the direct-transfer model the
  paper's commutativity argument, does not hold exactly).
* ``brute_force`` — exhaustive over all sequences of per-CLASS dims and
  per-op-class strategies (tiny graphs).
* ``brute_force_per_tensor`` — exhaustive over all per-TENSOR assignments
  (no coarsening): the optimum that pins both the coarsening
  and the searches.
* ``flat_search`` — the same variable elimination over *sequence-valued*
  variables (all m steps at once): exact global optimum for small graphs.
* ``auto_search`` — the recursion, plus the flat search when it is cheap,
  keeping the strictly cheaper plan (reading R4).
"""
from __future__ import annotations

import itertools

import numpy as np

from .cost import op_cost_box, op_cost_slots, plan_cost


def factorize(k: int):
    """k = k₁·k₂·…·k_m with kᵢ ≥ kᵢ₊₁: prime factors, sorted
    non-increasing."""
    out = []
    n = k
    p = 2
    while p * p <= n:
        while n % p == 0:
            out.append(p)
            n //= p
        p += 1
    if n > 1:
        out.append(n)
    return sorted(out, reverse=True)


# --------------------------------------------------------------------------- VE engine
class _VE:
    """Exact min-sum variable elimination with co-optimal enumeration."""

    def __init__(self, domains, factors):
        self.domains = domains                      # list of lists
        self.factors = [(tuple(s), np.asarray(t, dtype=np.int64)) for s, t in factors]

    def run(self, cap):
        active = list(self.factors)
        remaining = set(range(len(self.domains)))
        trace = []
        while remaining:
            best = None
            for x in sorted(remaining):
                nb = set()
                for s, _ in active:
                    if x in s:
                        nb |= set(s)
                w = 1
                for y in nb:
                    w *= len(self.domains[y])
                if best is None or w < best[0]:
                    best = (w, x)
            x = best[1]
            touching = [f for f in active if x in f[0]]
            active = [f for f in active if x not in f[0]]
            scope = sorted({y for s, _ in touching for y in s})
            shape = [len(self.domains[y]) for y in scope]
            comb = np.zeros(shape, dtype=np.int64)
            for s, t in touching:
                # broadcast t (axes s) into scope
                perm = [s.index(y) for y in scope if y in s]
                tt = np.transpose(t, perm) if t.ndim else t
                bshape = [len(self.domains[y]) if y in s else 1 for y in scope]
                comb = comb + tt.reshape(bshape)
            ax = scope.index(x)
            msg = comb.min(axis=ax)
            rest = [y for y in scope if y != x]
            trace.append((x, scope, comb))
            active.append((tuple(rest), msg))
            remaining.discard(x)
        total = int(sum(int(t) for _, t in active))
        sols = []

        def dfs(i, assign):
            if len(sols) >= cap:
                return
            if i < 0:
                sols.append(dict(assign))
                return
            x, scope, comb = trace[i]
            idx = tuple(slice(None) if y == x else assign[y] for y in scope)
            line = comb[idx]
            m = line.min()
            for v in np.nonzero(line == m)[0]:
                assign[x] = int(v)
                dfs(i - 1, assign)
                del assign[x]

        dfs(len(trace) - 1, {})
        return total, sols


# --------------------------------------------------------------------------- helpers
def _extent_after(n, seq, axis, factors):
    for i, a in enumerate(seq):
        if a == axis:
            n //= factors[i]
    return n


def _tensor_domain(g, members, prefix_tdims, factors_prev, k):
    t0 = members[0]
    rank = len(g.shape(t0))
    if rank == 0:
        return [None]
    dom = []
    for d in range(rank):
        ok = True
        for t in members:
            n = _extent_after(g.shape(t)[d], prefix_tdims[t], d, factors_prev)
            if n % k != 0:
                ok = False
        if ok:
            dom.append(d)
    return dom


def _op_domain(g, members, prefix_osplit, factors_prev, k):
    op0 = g.op(members[0])
    dom = []
    for v in g.split_vars(op0):
        ok = True
        for name in members:
            n = _extent_after(g.ranges[name][v], prefix_osplit[name], v, factors_prev)
            if n % k != 0:
                ok = False
        if ok:
            dom.append(v)
    return dom


class SearchError(Exception):
    pass


def _op_cost_cached(g, op, td, osp, factors):
    """op_cost_box memoised (per graph object) on exactly the arguments it reads: the op, its split
    sequence, its tensors' dim sequences and the factors — no change to the value."""
    memo = g.__dict__.setdefault("_cost_memo", {})
    key = (op["name"], tuple(factors), tuple(osp[op["name"]]),
           tuple(tuple(td[t]) for t in list(op["inputs"]) + [op["output"]]))
    v = memo.get(key)
    if v is None:
        v = op_cost_box(g, op, td, osp, factors)[0]
        memo[key] = v
    return v


def step_search(g, prefix, k, cap=256):
    """All co-optimal basic plans for the next step (size-k split) given a
    plan prefix.  Returns (cost_of_prefix_plus_step, [plans]) where plans are
    full prefix+step plans."""
    tclass, classes, oclass, op_classes = g.coarsen()
    fprev = list(prefix["factors"])
    factors = fprev + [k]
    tdom = [_tensor_domain(g, ms, prefix["tdims"], fprev, k) for ms in classes]
    odom = [_op_domain(g, ms, prefix["osplit"], fprev, k) for ms in op_classes]
    for c, dom in enumerate(tdom):
        if not dom:
            raise SearchError(f"no divisible dim for tensor class {classes[c]}")
    for c, dom in enumerate(odom):
        if not dom:
            raise SearchError(f"no divisible var for op class {op_classes[c]}")
    nT = len(classes)
    domains = tdom + odom
    factors_ve = []
    for oc, members in enumerate(op_classes):
        tcs = sorted({tclass[t] for name in members
                      for t in list(g.op(name)["inputs"]) + [g.op(name)["output"]]})
        scope = tcs + [nT + oc]
        shape = [len(domains[x]) for x in scope]
        table = np.zeros(shape, dtype=np.int64)
        for idx in itertools.product(*[range(s) for s in shape]):
            choice = {x: domains[x][i] for x, i in zip(scope, idx)}
            v = choice[nT + oc]
            val = 0
            for name in members:
                op = g.op(name)
                td = {}
                for t in list(op["inputs"]) + [op["output"]]:
                    td[t] = list(prefix["tdims"][t]) + [choice[tclass[t]]]
                osp = {name: list(prefix["osplit"][name]) + [v]}
                val += _op_cost_cached(g, op, td, osp, factors)
            table[idx] = val
        factors_ve.append((scope, table))
    total, sols = _VE(domains, factors_ve).run(cap)
    # untouched tensor classes (no op) are free: VE assigned them too.
    plans = []
    for s in sols:
        p = {"factors": factors,
             "tdims": {t: list(prefix["tdims"][t]) + [tdom[tclass[t]][s[tclass[t]]]] for t in g.tensors},
             "osplit": {o["name"]: list(prefix["osplit"][o["name"]]) + [odom[oclass[o["name"]]][s[nT + oclass[o["name"]]]]]
                        for o in g.ops}}
        plans.append(p)
    plans.sort(key=lambda p: canon_key(g, p))
    return total, plans


def canon_key(g, plan):
    _, classes, _, op_classes = g.coarsen()
    kt = tuple(tuple(-1 if d is None else d for d in plan["tdims"][ms[0]]) for ms in classes)
    ko = []
    for ms in op_classes:
        op = g.op(ms[0])
        sv = g.split_vars(op)
        ko.append(tuple(sv.index(v) for v in plan["osplit"][ms[0]]))
    return kt + tuple(ko)


def empty_plan(g):
    return {"factors": [], "tdims": {t: [] for t in g.tensors}, "osplit": {o["name"]: [] for o in g.ops}}


def recursive_search(g, k, cap=256, frontier_cap=64):
    """Recursive partitioning with the co-optimal frontier.
    Returns the plan with 'cost', 'bytes', 'deltas', 'frontier_truncated'."""
    plan0 = empty_plan(g)
    if k == 1:
        plan0.update(cost=0, bytes=0, deltas=[], frontier_truncated=False)
        return plan0
    frontier = [plan0]
    truncated = False
    for ki in factorize(k):
        cands = []
        best = None
        for pre in frontier:
            c, plans = step_search(g, pre, ki, cap)
            if len(plans) >= cap:
                truncated = True
            if best is None or c < best:
                best = c
                cands = list(plans)
            elif c == best:
                cands.extend(plans)
        uniq = {}
        for p in cands:
            uniq.setdefault(canon_key(g, p), p)
        cands = [uniq[key] for key in sorted(uniq)]
        if len(cands) > frontier_cap:
            truncated = True
            cands = cands[:frontier_cap]
        frontier = cands
    best = frontier[0]
    el, by = plan_cost(g, best)
    from .cost import step_costs
    best = dict(best, cost=el, bytes=by, deltas=step_costs(g, best), frontier_truncated=truncated)
    return best


def _seq_domain_tensor(g, members, factors):
    rank = len(g.shape(members[0]))
    if rank == 0:
        return [tuple([None] * len(factors))]
    out = []
    for seq in itertools.product(range(rank), repeat=len(factors)):
        ok = True
        for t in members:
            n = list(g.shape(t))
            for i, d in enumerate(seq):
                if n[d] % factors[i]:
                    ok = False
                    break
                n[d] //= factors[i]
            if not ok:
                break
        if ok:
            out.append(seq)
    return out


def _seq_domain_op(g, members, factors):
    sv = g.split_vars(g.op(members[0]))
    out = []
    for seq in itertools.product(sv, repeat=len(factors)):
        ok = True
        for name in members:
            n = dict(g.ranges[name])
            for i, v in enumerate(seq):
                if n[v] % factors[i]:
                    ok = False
                    break
                n[v] //= factors[i]
            if not ok:
                break
        if ok:
            out.append(seq)
    return out


def brute_force(g, k, limit=2_000_000):
    """Exhaustive minimum over all sequences of basic plans.  Tensor-class dim
    sequences are enumerated jointly; given them the op terms are separable,
    so each op class takes its best strategy sequence (still exhaustive)."""
    factors = factorize(k)
    tclass, classes, oclass, op_classes = g.coarsen()
    tseq = [_seq_domain_tensor(g, ms, factors) for ms in classes]
    oseq = [_seq_domain_op(g, ms, factors) for ms in op_classes]
    n = 1
    for d in tseq:
        n *= len(d)
    if n > limit:
        raise SearchError(f"brute force too large ({n})")
    best = None
    for combo in itertools.product(*tseq):
        tdims = {t: list(combo[tclass[t]]) for t in g.tensors}
        tot = 0
        osplit = {}
        for oc, members in enumerate(op_classes):
            bo = None
            for seq in oseq[oc]:
                val = 0
                for name in members:
                    val += op_cost_box(g, g.op(name), tdims, {name: list(seq)}, factors)[0]
                if bo is None or val < bo[0]:
                    bo = (val, seq)
            tot += bo[0]
            for name in members:
                osplit[name] = list(bo[1])
        if best is None or tot < best[0]:
            best = (tot, {"factors": factors, "tdims": tdims, "osplit": osplit})
    return best[0], best[1]


def flat_search(g, k, cap=1):
    """Exact optimum by variable elimination over sequence-valued variables
    (all steps jointly)."""
    factors = factorize(k)
    tclass, classes, oclass, op_classes = g.coarsen()
    tdom = [_seq_domain_tensor(g, ms, factors) for ms in classes]
    odom = [_seq_domain_op(g, ms, factors) for ms in op_classes]
    if any(not d for d in tdom + odom):
        raise SearchError("flat search: a class has no divisible split sequence")
    nT = len(classes)
    domains = tdom + odom
    fs = []
    for oc, members in enumerate(op_classes):
        tcs = sorted({tclass[t] for name in members
                      for t in list(g.op(name)["inputs"]) + [g.op(name)["output"]]})
        scope = tcs + [nT + oc]
        shape = [len(domains[x]) for x in scope]
        # the op cost is a sum of per-slot terms, each reading one tensor's sequence (cost.op_cost_slots):
        # table[tensor classes..., op] = Σ_members Σ_slots term(slot's class sequence, op sequence)
        table = np.zeros(shape, dtype=np.int64)
        for name in members:
            op = g.op(name)
            ts = list(op["inputs"]) + [op["output"]]
            base = {t: list(domains[tclass[t]][0]) for t in ts}
            slot_t = [t for (p_, _), t in zip(g.opdef(op).params, op["inputs"])] + [op["output"]]
            slot_p = [p_ for p_, _ in g.opdef(op).params] + [op["output"]]
            for si, (t, pname) in enumerate(zip(slot_t, slot_p)):
                c = tclass[t]
                ax = scope.index(c)
                term = np.zeros((len(domains[c]), len(odom[oc])), dtype=np.int64)
                for qi, q in enumerate(domains[c]):
                    td = dict(base)
                    td[t] = list(q)
                    for oi, oseq in enumerate(odom[oc]):
                        kind = "out" if si == len(slot_t) - 1 else "in"
                        term[qi, oi] = sum(e for k_, p2, e, _ in op_cost_slots(g, op, td, {name: list(oseq)}, factors)
                                           if k_ == kind and p2 == pname)
                bshape = [1] * len(scope)
                bshape[ax] = len(domains[c])
                bshape[-1] = len(odom[oc])
                table = table + term.reshape(bshape)
        fs.append((scope, table))
    total, sols = _VE(domains, fs).run(cap)
    s = sols[0]
    plan = {"factors": factors,
            "tdims": {t: list(tdom[tclass[t]][s[tclass[t]]]) for t in g.tensors},
            "osplit": {o["name"]: list(odom[oclass[o["name"]]][s[nT + oclass[o["name"]]]]) for o in g.ops}}
    return total, plan


# --------------------------------------------------------------------------- per-tensor brute force
def _seq_domain_single_tensor(shape, factors):
    """All split-dim sequences of ONE tensor (no class): dims whose extent stays divisible."""
    if len(shape) == 0:
        return [tuple([None] * len(factors))]
    out = []
    for seq in itertools.product(range(len(shape)), repeat=len(factors)):
        n = list(shape)
        ok = True
        for i, d in enumerate(seq):
            if n[d] % factors[i]:
                ok = False
                break
            n[d] //= factors[i]
        if ok:
            out.append(seq)
    return out


def _seq_domain_single_op(g, op, factors):
    out = []
    for seq in itertools.product(g.split_vars(op), repeat=len(factors)):
        n = dict(g.ranges[op["name"]])
        ok = True
        for i, v in enumerate(seq):
            if n[v] % factors[i]:
                ok = False
                break
            n[v] //= factors[i]
        if ok:
            out.append(seq)
    return out


def brute_force_per_tensor(g, k, limit=1 << 24):
    """Exhaustive minimum over ALL per-tensor partition assignments — every tensor and every op chooses
    its own split sequence, with no coarsening (no element-wise / timestep / alias classes) — the
    north star's "brute-force enumeration of all per-tensor partition assignments".

    Enumeration: a dense array over the joint assignment of every tensor (one axis per tensor, one entry
    per divisible sequence, so Π|domain| cells: every assignment is visited); each op adds, broadcast
    over its own tensors' axes, the cost of its best strategy sequence for that assignment of its tensors
    (given the tensors, the ops' terms are independent, so minimising each separately is exhaustive).
    No variable elimination: independent of ``flat_search``'s engine.  Returns (cost, plan)."""
    factors = factorize(k)
    names = sorted(g.tensors)
    tdom = [_seq_domain_single_tensor(g.shape(t), factors) for t in names]
    if any(not d for d in tdom):
        raise SearchError("a tensor has no divisible split sequence")
    axis = {t: i for i, t in enumerate(names)}
    cells = 1
    for d in tdom:
        cells *= len(d)
    if cells > limit:
        raise SearchError(f"brute force too large ({cells} assignments)")
    total = np.zeros([len(d) for d in tdom], dtype=np.int64)
    best_op = []
    for op in g.ops:
        odom = _seq_domain_single_op(g, op, factors)
        if not odom:
            raise SearchError(f"op {op['name']} has no divisible split sequence")
        ts = sorted({axis[t] for t in list(op["inputs"]) + [op["output"]]})
        shape = [len(tdom[a]) for a in ts]
        tab = np.zeros(shape, dtype=np.int64)
        arg = np.zeros(shape, dtype=np.int64)
        for idx in itertools.product(*[range(s) for s in shape]):
            td = {names[a]: list(tdom[a][i]) for a, i in zip(ts, idx)}
            vals = [op_cost_box(g, op, td, {op["name"]: list(s)}, factors)[0] for s in odom]
            j = int(np.argmin(vals))
            tab[idx] = vals[j]
            arg[idx] = j
        bshape = [len(tdom[a]) if a in ts else 1 for a in range(len(names))]
        total += tab.reshape(bshape)
        best_op.append((op, ts, arg, odom))
    flat_i = int(np.argmin(total))
    cost = int(total.reshape(-1)[flat_i])
    where = np.unravel_index(flat_i, total.shape)
    tdims = {t: list(tdom[axis[t]][where[axis[t]]]) for t in names}
    osplit = {}
    for op, ts, arg, odom in best_op:
        osplit[op["name"]] = list(odom[int(arg[tuple(where[a] for a in ts)])])
    return cost, {"factors": factors, "tdims": tdims, "osplit": osplit}


# --------------------------------------------------------------------------- auto (recursion + exact check)
FLAT_AUTO_CELLS = 1 << 20


def flat_cells(g, k):
    """Σ over op classes of the flat search's factor-table cells (Π of its scope's sequence-domain sizes):
    the size test of the ``auto`` search.  Domains are enumerated exactly as ``flat_search`` does."""
    factors = factorize(k)
    tclass, classes, oclass, op_classes = g.coarsen()
    tn = [len(_seq_domain_tensor(g, ms, factors)) for ms in classes]
    on = [len(_seq_domain_op(g, ms, factors)) for ms in op_classes]
    tot = 0
    for oc, members in enumerate(op_classes):
        tcs = sorted({tclass[t] for name in members for t in list(g.op(name)["inputs"]) + [g.op(name)["output"]]})
        n = on[oc]
        for c in tcs:
            n *= tn[c]
        tot += n
    return tot


def auto_search(g, k, cap=256, frontier_cap=64):
    """The paper's recursion, then — when the graph is small enough that the exact joint
    search is cheap (``flat_cells`` <= FLAT_AUTO_CELLS) — the flat exact search, keeping the flat plan
    only if it is strictly cheaper.  Reading R4: under the direct-transfer cost model the recursion is not
    always optimal (named cases in tests/test_oracle_optimality.py), so small graphs get the exact
    optimum.  Returns the plan dict of ``recursive_search`` plus 'search': 'recursive' | 'flat'."""
    rec = recursive_search(g, k, cap, frontier_cap)
    rec["search"] = "recursive"
    if k == 1 or flat_cells(g, k) > FLAT_AUTO_CELLS:
        return rec
    c, fp = flat_search(g, k)
    if c < rec["cost"]:
        from .cost import step_costs
        el, by = plan_cost(g, fp)
        return dict(fp, cost=el, bytes=by, deltas=step_costs(g, fp), frontier_truncated=rec["frontier_truncated"],
                    search="flat")
    return rec
