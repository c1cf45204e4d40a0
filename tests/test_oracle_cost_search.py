"""Oracle pins: cost model (Lemma P:L1604-1644) and search
(Appendix theorems)."""
import itertools
import json
import os
import random

import pytest

from fixtures import random_chain
from oracle.cost import op_cost_box, op_cost_enum, plan_cost, stored_elements
from oracle.graph import Graph
from oracle.search import (SearchError, _tensor_domain, brute_force, empty_plan, factorize,
                           flat_search, recursive_search, step_search)
from tofu_inputs.graphs import config, mlp

HERE = os.path.dirname(__file__)
GOLD = json.load(open(os.path.join(HERE, "golden", "paper_examples.json")))


def _mm_graph(n=8, dtype="f32"):
    return Graph({"defs": {"mm_nn": "def mm_nn(A(2), B(2)) -> lambda i, j: reduce(Sum; k; A[i, k] * B[k, j])"},
                  "tensors": {t: {"shape": [n, n], "dtype": dtype, "role": "act"} for t in "ABC"},
                  "ops": [{"name": "mm", "def": "mm_nn", "inputs": ["A", "B"], "output": "C"}]})


def test_matmul_row_split_256_bytes():
    """SPEC S:L298 worked example: C=A·B, 8x8 fp32, all split on dim0,
    Concat(i): B needed whole, half local -> 32 elements = 128 B per worker,
    256 B total."""
    g = _mm_graph()
    plan = {"factors": [2], "tdims": {"A": [0], "B": [0], "C": [0]}, "osplit": {"mm": ["i"]}}
    assert plan_cost(g, plan) == (64, 256)


def test_matmul_reduce_split_whole_partials():
    """Case-2 on k: each worker produces a full 8x8 partial and
    sends the half it does not own (32 elements, fp32)."""
    g = _mm_graph()
    plan = {"factors": [2], "tdims": {"A": [1], "B": [0], "C": [0]}, "osplit": {"mm": ["k"]}}
    assert plan_cost(g, plan) == (64, 256)


def _random_plan(g, factors, rng):
    td = {}
    for t, info in g.tensors.items():
        r = len(info["shape"])
        td[t] = [None if r == 0 else rng.randrange(r) for _ in factors]
    osp = {o["name"]: [rng.choice(g.split_vars(o)) for _ in factors] for o in g.ops}
    # keep only divisible plans
    for t, seq in td.items():
        n = list(g.shape(t))
        for i, d in enumerate(seq):
            if d is None:
                continue
            if n[d] % factors[i]:
                return None
            n[d] //= factors[i]
    for o in g.ops:
        n = dict(g.ranges[o["name"]])
        for i, v in enumerate(osp[o["name"]]):
            if n[v] % factors[i]:
                return None
            n[v] //= factors[i]
    return {"factors": factors, "tdims": td, "osplit": osp}


def test_box_cost_equals_element_enumeration():
    rng = random.Random(1)
    checked = 0
    for s in range(60):
        g = Graph(random_chain(s))
        for factors in ([2], [2, 2], [2, 2, 2]):
            p = _random_plan(g, factors, rng)
            if p is None:
                continue
            for op in g.ops:
                assert op_cost_box(g, op, p["tdims"], p["osplit"], factors)[0] == \
                    op_cost_enum(g, op, p["tdims"], p["osplit"], factors)
                checked += 1
    assert checked > 100


def test_aligned_elementwise_costs_nothing():
    g = Graph(random_chain(3))
    ew = Graph({"defs": {"add": "def add(A(2), B(2)) -> lambda i, j: A[i, j] + B[i, j]"},
                "tensors": {t: {"shape": [4, 8], "dtype": "f32", "role": "act"} for t in "ABC"},
                "ops": [{"name": "a", "def": "add", "inputs": ["A", "B"], "output": "C"}]})
    for d, v in ((0, "i"), (1, "j")):
        p = {"factors": [2, 2], "tdims": {t: [d, d] for t in "ABC"}, "osplit": {"a": [v, v]}}
        assert plan_cost(ew, p)[0] == 0


def test_lemma_linearity_under_scaling():
    """Lemma: a fixed plan's cost is a weighted sum of tensor
    sizes, so scaling every dim of a rank-2 graph by c scales cost by c^2."""
    rng = random.Random(7)
    for s in range(20):
        spec = random_chain(s)
        g1 = Graph(spec)
        p = _random_plan(g1, [2, 2], rng)
        if p is None:
            continue
        for c in (2, 3):
            spec2 = json.loads(json.dumps(spec))
            for t in spec2["tensors"].values():
                t["shape"] = [x * c for x in t["shape"]]
            g2 = Graph(spec2)
            assert plan_cost(g2, p)[0] == c * c * plan_cost(g1, p)[0]


def test_commutativity_when_steps_split_distinct_axes():
    """Theorem, under the direct-transfer model it holds when
    the two basic plans split different axes of every tensor and op (reading
    §R4 of DESIGN.md: repeated splits of one axis make the order matter)."""
    rng = random.Random(3)
    n = 0
    for s in range(40):
        g = Graph(random_chain(s))
        td = {}
        for t, info in g.tensors.items():
            d1 = rng.randrange(2)
            td[t] = [d1, 1 - d1]
        osp = {o["name"]: rng.sample(g.split_vars(o), 2) for o in g.ops}
        p = {"factors": [2, 2], "tdims": td, "osplit": osp}
        q = {"factors": [2, 2], "tdims": {t: s_[::-1] for t, s_ in td.items()},
             "osplit": {o: s_[::-1] for o, s_ in osp.items()}}
        assert plan_cost(g, p) == plan_cost(g, q)
        n += 1
    assert n >= 10


def test_per_worker_storage_is_one_kth():
    """storage per worker is 1/k of the total."""
    g = Graph(config(0))
    for k in (2, 4, 8):
        p = recursive_search(g, k)
        total = sum(max(1, __import__("math").prod(t["shape"])) for t in g.tensors.values())
        scal = sum(1 for t in g.tensors.values() if len(t["shape"]) == 0)
        for w in range(k):
            assert stored_elements(g, p, w) == (total - scal) // k + (scal if w == 0 else 0)


def test_factorize():
    assert factorize(8) == [2, 2, 2] and factorize(12) == [3, 2, 2] and factorize(7) == [7]


def test_step_dp_equals_exhaustive_single_step():
    """k = 2: one DP step is exact, so it must equal brute force."""
    for s in range(40):
        g = Graph(random_chain(s))
        try:
            p = recursive_search(g, 2)
        except SearchError:
            continue
        c, _ = brute_force(g, 2)
        assert p["cost"] == c


def test_conv_group_step_configurations():
    """one recursive step enumerates 4^6 = 4096 configurations of
    the six rank-4 tensors of a conv group; 3 steps -> 3*4096."""
    c = GOLD["counts"]
    conv = ("def conv(D(4), F(4)) -> lambda b, co, y, x: "
            "reduce(Sum; ci, ky, kx; D[b, ci, y + ky, x + kx] * F[co, ci, ky, kx])")
    shp = {"D": [8, 8, 9, 9], "F": [8, 8, 2, 2], "O": [8, 8, 8, 8],
           "dD": [8, 8, 8, 8], "dF": [8, 8, 8, 8], "dO": [8, 8, 8, 8]}
    g = Graph({"defs": {"conv": conv}, "tensors": {t: {"shape": s, "role": "act"} for t, s in shp.items()},
               "ops": [{"name": "c", "def": "conv", "inputs": ["D", "F"], "output": "O"}]})
    six = ["O", "dD", "dF", "dO"]
    # the four fully-even tensors: 4 choices each per step
    plan = empty_plan(g)
    total = 0
    for step in range(3):
        n = 1
        for t in six:
            n *= len(_tensor_domain(g, [t], plan["tdims"], plan["factors"], 2))
        n *= 4 * 4   # D and F with all 4 dims splittable (paper's idealisation)
        total += n
        plan["factors"].append(2)
        for t in g.tensors:
            plan["tdims"][t].append(0)
    assert n == c["conv_group_per_step"]
    assert total == c["conv_group_recursive_total"]


def test_recursion_vs_brute_force_random_fixtures():
    """SPEC S:L506 acceptance #4 idea: recursive search vs exhaustive optimum on
    random halo-free chains.  k = 2 must match exactly (single exact step).
    For k = 4 the paper's optimality proof relies on its
    halving cost model; under the direct-transfer model (reading §R4) the
    recursion is a heuristic — we pin that it is never below the optimum,
    matches it on >= 95% of fixtures (the exceptions are exactly the named cases of
    test_oracle_optimality.KNOWN_RECURSION_GAPS), and that delta_i is non-decreasing
    (Theorem P:L784-786) on every returned plan."""
    n = match = 0
    for s in range(60):
        g = Graph(random_chain(s))
        for k in (2, 4):
            try:
                p = recursive_search(g, k)
            except SearchError:
                continue
            c, _ = flat_search(g, k)
            if len(g.ops) <= 2:
                cb, _ = brute_force(g, k, limit=20000)
                assert cb == c
            assert p["cost"] >= c
            if k == 2:
                assert p["cost"] == c
            n += 1
            match += p["cost"] == c
            d = p["deltas"]
            assert all(d[i] <= d[i + 1] for i in range(len(d) - 1))
    assert n >= 60 and match >= 0.95 * n, (match, n)


@pytest.mark.parametrize("cfg,k", [(0, 2), (0, 4), (1, 2), (1, 4), (1, 8)])
def test_config_plans_are_optimal(cfg, k):
    """The recursive plan of the BASELINE configs equals the exact optimum (configs[0] at k = 8:
    test_oracle_optimality.test_mlp_plans_are_optimal)."""
    g = Graph(config(cfg))
    p = recursive_search(g, k)
    c, _ = flat_search(g, k)
    assert p["cost"] == c


def test_fc_plan_uses_partition_n_reduce():
    """configs[1]: the 8-way plan of the large FC layer includes the
    partition-n-reduce (reduction-split) case."""
    g = Graph(config(1))
    p = recursive_search(g, 8)
    assert "k" in p["osplit"]["fc1"]
