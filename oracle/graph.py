"""Dataflow graph and coarsening (oracle side).  TEST INFRASTRUCTURE ONLY.

Graph JSON (shared input format, produced by ``tofu_inputs.graphs``):

    {"defs":    {def_name: "def ... -> lambda ...: ..."},
     "tensors": {name: {"shape": [...], "dtype": "bf16"|"f32",
                        "role": "input"|"weight"|"state"|"act"|"grad"|"loss",
                        "grad_of": name|null, "merge": key|null}},
     "ops":     [{"name", "def", "inputs": [...], "output",
                  "backward_of": op|null, "merge": key|null}],
     "alias":   {new_tensor: old_tensor}}     # in-place update W2 -> W

Coarsening (§5.1):
* "Each forward operator ... and its auto-generated backward operators ...
  form a group"; "Each forward tensor ... and its gradient tensor form a
  group".  Group members may be partitioned differently
  (P:L656-661), so these groups only order the DP; they impose no equality.
* "Merging consecutive element-wise operators, because the input and output
  tensors of an element-wise operator should always be partitioned
  identically": inputs and output of every ElementWise op are
  unioned into one tensor class.
* "Merging unrolled timesteps ... they should be coalesced to share the same
  partition strategy": tensors / ops carrying the same "merge"
  key share one class.
* In-place aliases (W2 stored in W) are unioned (storage identity).
"""
from __future__ import annotations

import json

from .tdl import parse_def, classify, var_ranges, split_vars

ITEMSIZE = {"bf16": 2, "f32": 4, "f64": 8}


class GraphError(Exception):
    pass


class Graph:
    def __init__(self, spec: dict):
        self.spec = spec
        self.defs = {n: parse_def(src) for n, src in spec["defs"].items()}
        self.tensors = {n: dict(t) for n, t in spec["tensors"].items()}
        for t in self.tensors.values():
            t["shape"] = [int(x) for x in t["shape"]]
            t.setdefault("dtype", "f32")
            t.setdefault("merge", None)
        self.ops = [dict(o) for o in spec["ops"]]
        for o in self.ops:
            o.setdefault("merge", None)
            o.setdefault("backward_of", None)
            # output views (reading §R10): constant per-dim offsets added to an input's access indices
            # and to the output index, so one op reads / writes a slice (e.g. one timestep) of a tensor
            offs = o.get("offsets") or [None] * len(o["inputs"])
            o["offsets"] = [tuple(x) if x else (0,) * len(self.tensors[t]["shape"])
                            for x, t in zip(offs, o["inputs"])]
            oo = o.get("out_offset")
            o["out_offset"] = tuple(oo) if oo else (0,) * len(self.tensors[o["output"]]["shape"])
        self.alias = dict(spec.get("alias", {}))
        self._validate()
        self.ranges = {o["name"]: self._ranges(o) for o in self.ops}

    @staticmethod
    def from_json(text: str) -> "Graph":
        return Graph(json.loads(text))

    def shape(self, t):
        return self.tensors[t]["shape"]

    def opdef(self, op):
        return self.defs[op["def"]]

    def _ranges(self, op):
        """Extent of every index var: inferred from the output / input shapes
        (tdl.var_ranges), overridden by the op's explicit "ranges" (needed when
        the op reads or writes a view, §R10)."""
        d = self.opdef(op)
        shapes = {p: self.shape(t) for (p, _), t in zip(d.params, op["inputs"])}
        over = op.get("ranges") or {}
        oshape = [over.get(v, n) for v, n in zip(d.out_vars, self.shape(op["output"]))]
        R = var_ranges(d, shapes, oshape, over)
        R.update({v: int(n) for v, n in over.items()})
        return R

    def bound(self, op, tensor_param):
        return tensor_param

    def _validate(self):
        produced = {}
        for o in self.ops:
            if o["def"] not in self.defs:
                raise GraphError(f"UnknownOperator {o['def']}")
            d = self.defs[o["def"]]
            if len(d.params) != len(o["inputs"]):
                raise GraphError(f"ShapeMismatch {o['name']}: arity")
            for (p, r), t in zip(d.params, o["inputs"]):
                if t not in self.tensors:
                    raise GraphError(f"unknown tensor {t}")
                if len(self.shape(t)) != r:
                    raise GraphError(f"ShapeMismatch {o['name']}: {t} rank {len(self.shape(t))} != {r}")
            if len(self.shape(o["output"])) != len(d.out_vars):
                raise GraphError(f"ShapeMismatch {o['name']}: output rank")
            R = self._ranges(o)
            obox = [(off, off + R[v] - 1) for v, off in zip(d.out_vars, o["out_offset"])]
            for (lo, hi), n in zip(obox, self.shape(o["output"])):
                if lo < 0 or hi >= n:
                    raise GraphError(f"ShapeMismatch {o['name']}: output view out of range")
            for other in produced.get(o["output"], []):
                if all(a[0] <= b[1] and b[0] <= a[1] for a, b in zip(obox, other)):
                    raise GraphError(f"tensor {o['output']} produced twice (overlapping views)")
            produced.setdefault(o["output"], []).append(obox)
            # accesses may leave their tensor (zero padding, reading R11): nothing to check

    # ------------------------------------------------------------------ coarsening
    def coarsen(self):
        """Returns (tensor_class: name->class id, classes: [sorted names],
        op_class: op name->class id, op_classes: [[op names]])."""
        parent = {t: t for t in self.tensors}

        def find(x):
            while parent[x] != x:
                parent[x] = parent[parent[x]]
                x = parent[x]
            return x

        def union(a, b):
            ra, rb = find(a), find(b)
            if ra != rb:
                if ra < rb:
                    parent[rb] = ra
                else:
                    parent[ra] = rb

        for o in self.ops:
            d = self.opdef(o)
            if classify(d)[0] == "ElementWise" and not any(any(x) for x in o["offsets"]) \
                    and not any(o["out_offset"]):
                for t in o["inputs"]:
                    union(t, o["output"])
        for new, old in self.alias.items():
            union(new, old)
        bykey = {}
        for n, t in self.tensors.items():
            if t["merge"] is not None:
                bykey.setdefault(t["merge"], []).append(n)
        for ms in bykey.values():
            for m in ms[1:]:
                union(ms[0], m)
        # class ids in order of first appearance (inputs of ops in op order, then rest)
        order = []
        seen = set()
        for o in self.ops:
            for t in list(o["inputs"]) + [o["output"]]:
                r = find(t)
                if r not in seen:
                    seen.add(r)
                    order.append(r)
        for t in sorted(self.tensors):
            r = find(t)
            if r not in seen:
                seen.add(r)
                order.append(r)
        cid = {r: i for i, r in enumerate(order)}
        tclass = {t: cid[find(t)] for t in self.tensors}
        classes = [[] for _ in order]
        for t in sorted(self.tensors):
            classes[tclass[t]].append(t)
        for ms in classes:
            shapes = {tuple(self.shape(t)) for t in ms}
            ranks = {len(s) for s in shapes}
            if len(ranks) != 1:
                raise GraphError(f"tensor class {ms} mixes ranks")
        # op classes
        ok = {}
        op_classes = []
        oclass = {}
        for o in self.ops:
            key = o["merge"]
            if key is not None and key in ok:
                i = ok[key]
            else:
                i = len(op_classes)
                op_classes.append([])
                if key is not None:
                    ok[key] = i
            op_classes[i].append(o["name"])
            oclass[o["name"]] = i
        for members in op_classes:
            defs = {self.op(m)["def"] for m in members}
            if len(defs) != 1:
                raise GraphError(f"merged ops {members} have different defs")
        return tclass, classes, oclass, op_classes

    def op(self, name):
        for o in self.ops:
            if o["name"] == name:
                return o
        raise KeyError(name)

    def split_vars(self, op):
        return split_vars(self.opdef(op))
