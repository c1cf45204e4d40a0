"""Oracle pins: symbolic interval analysis (Eq. 1, Fig. int-arith)
and strategy discovery (Case-1/Case-2)."""
import itertools
import json
import os
import random
from fractions import Fraction as F

import pytest

from oracle.interval import NonAffineError, SymInterval, eval_access
from oracle.strategy import classify_region, count_nd_partitions, discover_strategies
from oracle.tdl import parse_def, parse_program, var_ranges

HERE = os.path.dirname(__file__)
GOLD = json.load(open(os.path.join(HERE, "golden", "paper_examples.json")))
CORPUS = parse_program(open(os.path.join(HERE, "golden", "corpus.tdl")).read())


def test_shift_two_paper_regions():
    g = GOLD["shift_two"]
    d = parse_def(g["tdl"])
    for j, (b_range, a_range) in enumerate(g["halves"]):
        init = {"i": SymInterval.zv("i", F(j, 2), F(j + 1, 2))}
        (t, dims), = eval_access(d, init)
        assert t == "A"
        assert dims[0].concretize({"i": g["extent_i"]}) == tuple(a_range)
        assert init["i"].concretize({"i": g["extent_i"]}) == tuple(b_range)


def test_interval_product_is_error():
    a = SymInterval.zv("x", 0, F(1, 2))
    with pytest.raises(NonAffineError):
        a.mul(a)
    with pytest.raises(NonAffineError):
        a.compare(a)


def _random_shapes(d, rng):
    """Random concrete extents (even, <= 6) for every var of d."""
    return {v: rng.choice([2, 4, 6]) for v in d.all_vars()}


@pytest.mark.parametrize("name", ["matmul", "mm_nt", "mm_tn", "conv1d", "conv2d_s2", "shift_two",
                                  "reverse", "maxpool2", "bias_add", "lstm_gates", "lstm_cell", "transpose"])
def test_intervals_exact_vs_enumeration(name):
    """For every strategy and half: the concretised symbolic region equals the
    hull of the indices actually accessed, enumerated point by point."""
    d = CORPUS[name]
    rng = random.Random(hash(name) & 0xffff)
    for trial in range(3):
        ext = _random_shapes(d, rng)
        if name == "reverse":
            ext["i"] = 8
        for st in discover_strategies(d, 2):
            v = st["var"]
            for j in range(2):
                got = [(t, [iv.concretize(ext) if iv is not None else None for iv in dims])
                       for t, dims in st["regions"][j]]
                half = ext[v] // 2
                ranges = {u: range(ext[u]) for u in d.all_vars()}
                ranges[v] = range(j * half, (j + 1) * half)
                for (t, dims), acc in zip(got, d.accesses):
                    for dim, ix in enumerate(acc.index):
                        vals = [ix.const + sum(c * env[u] for u, c in ix.coef)
                                for env in (dict(zip(ranges, p)) for p in itertools.product(*ranges.values()))]
                        lo, hi = dims[dim]
                        # sound always; exact when every coefficient is +-1 (strided
                        # accesses over-approximate by the scaled fraction, Fig. int-arith)
                        assert lo <= min(vals) and hi >= max(vals), (name, v, j, t, dim)
                        if all(abs(c) == 1 for _, c in ix.coef):
                            assert (lo, hi) == (min(vals), max(vals)), (name, v, j, t, dim)


def test_conv1d_figure3_strategies():
    g = GOLD["conv1d"]
    d = parse_def(g["tdl"])
    st = {s["var"]: s for s in discover_strategies(d, 2)}
    assert list(st) == ["b", "co", "x", "ci", "dx"]
    shapes = {"data": [4, 6, 9], "filters": [6, 8, 2]}
    ext = {"b": 4, "co": 8, "x": 8, "ci": 6, "dx": 2}

    def spec(s, j):
        out = {}
        for t, sp in classify_region(d, s, j, shapes, ext):
            out[t] = ["Whole" if x[0] == "Whole" else ("Slice" if x[0] == "Slice" else "Range") for x in sp]
        return out
    for key, var in (("split_b", "b"), ("split_ci", "ci")):
        exp = g[key]
        assert st[var]["kind"] == exp["kind"]
        r0 = spec(st[var], 0)
        assert r0["data"] == exp["data"] and r0["filters"] == exp["filters"]
    # halo exchange on x: data dim 2 overlaps between the halves
    r0 = st["x"]["regions"][0][0][1][2].concretize(ext)
    r1 = st["x"]["regions"][1][0][1][2].concretize(ext)
    assert r0 == (0, 4) and r1 == (4, 8)


def test_matmul_three_strategies():
    st = discover_strategies(CORPUS["matmul"], 2)
    assert [(s["var"], s["kind"]) for s in st] == [("i", "Concat"), ("j", "Concat"), ("k", "Reduce")]


def test_partition_counts():
    c = GOLD["counts"]
    assert count_nd_partitions(4, 3) == c["ways_4d_8"]
    assert count_nd_partitions(4, 3) ** 6 == pytest.approx(c["conv_group_flat"], rel=0.01)
    assert count_nd_partitions(1, 3) == 1 and count_nd_partitions(2, 2) == 3


def test_strategy_partition_correctness():
    """Partition-n-reduce: concat (Case-1) or sum (Case-2) of the
    two workers' outputs equals the unpartitioned op, exactly on integers."""
    import numpy as np
    from oracle.exec_ref import tdl_eval
    rng = np.random.default_rng(0)
    for name in ["matmul", "conv1d", "bias_add", "lstm_gates", "maxpool2", "row_max", "sumsq", "mm_tn"]:
        d = CORPUS[name]
        ext = {v: 4 for v in d.all_vars()}
        if name == "conv1d":
            ext["dx"] = 2
        if name == "maxpool2":
            ext["dy"] = ext["dx"] = 2
        if name == "lstm_gates":
            ext["g"] = 4
        shapes = {}
        for acc in d.accesses:
            shapes[acc.tensor] = [ix.const + sum(max(0, c * (ext[u] - 1)) for u, c in ix.coef) + 1
                                  for ix in acc.index]
        ins = {t: (rng.integers(-3, 4, size=s).astype(float), (0,) * len(s)) for t, s in shapes.items()}
        full = {v: (0, ext[v] - 1) for v in d.all_vars()}
        ref = tdl_eval(d, ins, full)
        for s in discover_strategies(d, 2):
            v = s["var"]
            parts = []
            for j in range(2):
                box = dict(full)
                box[v] = (j * ext[v] // 2, (j + 1) * ext[v] // 2 - 1)
                parts.append(tdl_eval(d, ins, box))
            if s["kind"] == "Concat":
                ax = d.out_vars.index(v)
                got = np.concatenate(parts, axis=ax)
            else:
                red = {"Sum": np.add, "Max": np.maximum, "Min": np.minimum, "Prod": np.multiply}[d.reducer]
                got = red(parts[0], parts[1])
            assert np.array_equal(got, ref), (name, v)
