"""Sampled per-op parity of a full-size training step (test helper; reads the oracle, never the product).

For workloads too large for the oracle to run whole (LSTM-6-4K, WResNet-152-4 at batch 32), every op of
the step is checked on sampled output boxes, on the GPU's own inputs:

* a box is a window of each output variable (a few rows, 32-64 channels, ...) with the FULL range of
  every reduce variable, so each sampled element is the complete result the op computes;
* the oracle evaluates the op's TDL over that box (``oracle.exec_ref.fast_eval``: the def's body as one
  library contraction or tap loop) from the required regions of its inputs — the interval hull of every
  access over the box (Eq. 1, ``Affine.hull``), clipped to the tensor (zero padding, reading R11);
* an input comes from the step's initial values when no op produces it (inputs, weights, state before
  the in-place update), else from the GPU's stored result;
* an input the GPU never stores (``tofu_exec_unmaterialized``: a weight gradient folded into the
  optimizer epilogue, a convolution output folded into its relu / residual add, DESIGN R8) is recomputed
  by the oracle from ITS producer's inputs over the needed region, without the intermediate bf16
  rounding the fused kernel also skips (reading R13); such tensors are checked through their consumers;
* the oracle result is rounded to the output's storage dtype and compared normwise over the sample with
  the north star's two classes: "bf16-input/fp32-accumulate outputs" <= 5e-3 — every output stored in
  bf16, and every fp32 output computed (directly, or through a fused intermediate) from bf16 operands,
  e.g. a weight gradient — and "fp32 paths" <= 1e-5: fp32 outputs of fp32 operands only (momentum from a
  stored fp32 gradient, the loss of fp32 values).  Measured: a 25k-term tensor-core weight gradient is
  ~4e-5 from fp64 (fp32 accumulation in TMEM), which is why the classes differ.

``source(name, box)`` returns a stored tensor's region as a float64 array (box: per-dim closed ranges).
"""
from __future__ import annotations

import numpy as np

from oracle.cost import clip
from oracle.exec_ref import fast_eval, store_round
from oracle.graph import Graph


def nrm(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    d = float(np.linalg.norm(b))
    return float(np.linalg.norm(a - b)) / d if d > 0 else float(np.linalg.norm(a - b))


class SampledChecker:
    def __init__(self, spec, initial, source, unmaterialized=(), seed=0, out_budget=256):
        self.g = Graph(spec)
        self.initial = initial                 # name -> numpy array, or callable (name, box) -> region
        self.source = source
        self.unmat = set(unmaterialized)
        self.rng = np.random.default_rng(seed)
        self.out_budget = out_budget
        self.producers = {}
        for op in self.g.ops:
            self.producers.setdefault(op["output"], []).append(op)

    # ------------------------------------------------------------------ regions of stored / initial tensors
    def _region(self, t, box):
        if any(lo > hi for lo, hi in box):
            return np.zeros([max(0, hi - lo + 1) for lo, hi in box])
        if t in self.unmat:
            return self._recompute(t, box)
        if t not in self.producers:
            if callable(self.initial):       # regenerated on demand (the largest configs)
                return np.asarray(self.initial(t, box), np.float64)
            v = np.asarray(self.initial[t], np.float64)
            return v[tuple(slice(lo, hi + 1) for lo, hi in box)] if v.ndim else v
        return self.source(t, box)

    def _recompute(self, t, box):
        """Region of an unmaterialised tensor from its (single) producer, unrounded (R13)."""
        prods = self.producers[t]
        assert len(prods) == 1, f"unmaterialised {t} has {len(prods)} producers"
        op = prods[0]
        d = self.g.opdef(op)
        obox = {v: (lo - off, hi - off) for v, (lo, hi), off in zip(d.out_vars, box, op["out_offset"])}
        return self.eval_op(op, obox, rounded=False)

    # ------------------------------------------------------------------ one op over an out-var box
    def eval_op(self, op, obox, rounded=True):
        g = self.g
        d = g.opdef(op)
        R = g.ranges[op["name"]]
        box = dict(obox)
        for v in d.red_vars:
            box[v] = (0, R[v] - 1)
        ins = {}
        for (p, _), t, off in zip(d.params, op["inputs"], op["offsets"]):
            shape = g.shape(t)
            req = None
            for acc in d.accesses:
                if acc.tensor != p:
                    continue
                r = [(0, shape[dim] - 1) if ix is None else ix.hull(box, off[dim]) for dim, ix in enumerate(acc.index)]
                req = r if req is None else [(min(a[0], b[0]), max(a[1], b[1])) for a, b in zip(req, r)]
            if req is None:
                continue
            req = clip(req, shape)
            arr = self._region(t, req)
            # fast_eval origin: the def's index i reads array element i + off - lo
            ins[p] = (arr, tuple(lo - o for (lo, _), o in zip(req, off)))
        out = np.asarray(fast_eval(d, ins, box), np.float64)
        out = out.reshape([obox[v][1] - obox[v][0] + 1 for v in d.out_vars])
        return store_round(out, g.tensors[op["output"]]["dtype"]) if rounded else out

    def sample_box(self, op):
        d = self.g.opdef(op)
        R = self.g.ranges[op["name"]]
        n = len(d.out_vars)
        win = []
        budget = self.out_budget
        for i, v in enumerate(reversed(d.out_vars)):       # last var (channels / columns) widest
            w = 64 if i == 0 else (4 if i == 1 else 2)
            w = max(1, min(R[v], w, budget))
            win.append(w)
            budget = max(1, budget // w)
        win = list(reversed(win))
        box = {}
        for v, w in zip(d.out_vars, win):
            lo = int(self.rng.integers(0, R[v] - w + 1))
            box[v] = (lo, lo + w - 1)
        return box

    def check_op(self, op, boxes=1):
        """Worst normwise error of op over `boxes` sampled boxes (None when its output is unmaterialised)."""
        g = self.g
        t = op["output"]
        if t in self.unmat:
            return None
        d = g.opdef(op)
        got, ref = [], []
        for _ in range(boxes if d.out_vars else 1):
            obox = self.sample_box(op)
            ref.append(self.eval_op(op, obox).reshape(-1))
            tbox = [(obox[v][0] + off, obox[v][1] + off) for v, off in zip(d.out_vars, op["out_offset"])]
            got.append(np.asarray(self.source(t, tbox), np.float64).reshape(-1))
        return nrm(np.concatenate(got), np.concatenate(ref))

    def reads_bf16(self, op):
        """True when the op's value depends on a bf16 operand: a bf16 input, or an unmaterialised input
        (recomputed through its producer) that does."""
        for t in op["inputs"]:
            if self.g.tensors[t]["dtype"] == "bf16":
                return True
            if t in self.unmat and any(self.reads_bf16(p) for p in self.producers[t]):
                return True
        return False

    def tolerance(self, op):
        if self.g.tensors[op["output"]]["dtype"] == "bf16" or self.reads_bf16(op):
            return 5e-3
        return 1e-5

    def check_all(self, boxes=1, ops=None):
        """{op name: (error, tolerance)} for every checked op; raises AssertionError listing failures."""
        res, bad = {}, []
        for op in self.g.ops:
            if ops is not None and op["name"] not in ops:
                continue
            e = self.check_op(op, boxes)
            if e is None:
                continue
            tol = self.tolerance(op)
            res[op["name"]] = (e, tol)
            if not e <= tol:
                bad.append((op["name"], e, tol))
        assert not bad, bad[:20]
        return res


def runner_source(R):
    """source(name, box) reading a TofuRunner's stored shards (any k, virtual or local ranks): the region
    is assembled from the intersections with the owners' shard boxes (each element owned once)."""
    import torch

    def src(name, box):
        out = np.zeros([hi - lo + 1 for lo, hi in box])
        if not box:
            for r in R.local:
                v = R.view(r, name)
                if v is not None:
                    return float(v.reshape(-1)[0].double().cpu())
            raise KeyError(name)
        for r in R.local:
            v = R.view(r, name)
            if v is None:
                continue
            _, sbox = R.shards[r][name]
            ib = [(max(a, c), min(b, d)) for (a, b), (c, d) in zip(box, sbox)]
            if any(lo > hi for lo, hi in ib):
                continue
            sv = v[tuple(slice(lo - c, hi - c + 1) for (lo, hi), (c, _) in zip(ib, sbox))]
            out[tuple(slice(lo - a, hi - a + 1) for (lo, hi), (a, _) in zip(ib, box))] = \
                sv.to(torch.float64).cpu().numpy()
        return out

    return src
