"""Oracle pins: reference execution and the partitioned simulator."""
import numpy as np
import pytest
import torch

from oracle.exec_ref import fast_eval, round_bf16, run_graph, tdl_eval
from oracle.graph import Graph
from oracle.search import recursive_search
from oracle.cost import plan_cost
from oracle.sim import simulate
from oracle.tdl import parse_def
from tofu_inputs.graphs import MM_DEFS, config, mlp
from tofu_inputs.tensors import make_values


def test_round_bf16_closed_forms():
    assert round_bf16(1.0 + 2 ** -9) == 1.0                 # tie -> even
    assert round_bf16(1.0 + 3 * 2 ** -9) == 1.0 + 2 ** -7   # above half -> up
    assert round_bf16(1.0 + 2 ** -8 + 2 ** -9) == 1.0 + 2 ** -7   # tie -> even (odd lsb)
    assert round_bf16(-3.0) == -3.0 and round_bf16(0.0) == 0.0


def test_round_bf16_matches_torch_on_fp32_values():
    x = np.random.default_rng(0).standard_normal(10000).astype(np.float32).astype(np.float64) * 37.0
    x = x.astype(np.float32).astype(np.float64)
    ref = torch.from_numpy(x).float().to(torch.bfloat16).double().numpy()
    assert np.array_equal(round_bf16(x), ref)


@pytest.mark.parametrize("name", list(MM_DEFS))
def test_fast_matmul_equals_tdl_interpreter(name):
    d = parse_def(MM_DEFS[name])
    rng = np.random.default_rng(1)
    shapes = {"mm_nn": ([5, 7], [7, 3]), "mm_nt": ([5, 7], [3, 7]), "mm_tn": ([7, 5], [7, 3])}[name]
    A, B = (rng.integers(-4, 5, s).astype(float) for s in shapes)
    ins = {"A": (A, (0, 0)), "B": (B, (0, 0))}
    box = {"i": (1, 4), "j": (0, 2), "k": (2, 6)}
    assert np.array_equal(fast_eval(d, ins, box), tdl_eval(d, ins, box))


@pytest.mark.parametrize("name,shapes,box", [
    ("gate", ([6, 5], [5, 4, 3]), {"b": (1, 4), "g": (0, 3), "h": (1, 2), "k": (0, 4)}),
    ("mm_rec", ([6, 4, 3], [5, 4, 3]), {"b": (0, 5), "k": (2, 4), "g": (1, 3), "h": (0, 2)}),
    ("gate_wgrad", ([6, 5], [6, 4, 3]), {"k": (0, 4), "g": (0, 3), "h": (0, 2), "b": (2, 5)}),
])
def test_fast_contractions_equal_tdl_interpreter(name, shapes, box):
    from tofu_inputs.graphs import LSTM_DEFS
    d = parse_def(LSTM_DEFS[name])
    rng = np.random.default_rng(3)
    A, B = (rng.integers(-4, 5, s).astype(float) for s in shapes)
    ins = {d.params[0][0]: (A, (0,) * A.ndim), d.params[1][0]: (B, (0,) * B.ndim)}
    assert np.array_equal(fast_eval(d, ins, box), tdl_eval(d, ins, box))


def test_lstm_graph_backward_is_the_gradient():
    """The LSTM cell backward defs (tofu_inputs.graphs.lstm) are the gradient
    of the loss: central finite differences on every weight tensor, fp64."""
    from tofu_inputs.graphs import lstm
    spec = lstm(2, 4, 3, 2)
    g = Graph(spec)
    vals = make_values(spec, seed=3)
    for n in vals:
        if n.endswith("Wx") or n.endswith("Wh"):
            vals[n] = vals[n] * 8
    env = run_graph(g, vals, emulate_storage=False, fast=False)
    h = 1e-6
    rng = np.random.default_rng(0)
    for w in ("L1.Wx", "L1.Wh", "L2.Wx", "L2.Wh"):
        for _ in range(4):
            idx = tuple(rng.integers(0, s) for s in vals[w].shape)
            vp = dict(vals); vp[w] = vals[w].copy(); vp[w][idx] += h
            vm = dict(vals); vm[w] = vals[w].copy(); vm[w][idx] -= h
            fd = (run_graph(g, vp, emulate_storage=False)["loss"] - run_graph(g, vm, emulate_storage=False)["loss"]) / (2 * h)
            gd = env[w.replace(".W", ".dW")][idx]
            assert abs(fd - gd) <= 1e-4 * max(abs(fd), 1e-9), (w, idx, fd, gd)


def test_lstm_partitioned_sim_equals_unpartitioned():
    from tofu_inputs.graphs import lstm
    spec = lstm(2, 8, 3, 4)
    g = Graph(spec)
    vals = make_values(spec, seed=4)
    ref = run_graph(g, vals, emulate_storage=False)
    plan = recursive_search(g, 2)
    res, ledger = simulate(g, plan, vals)
    for t in ref:
        assert np.allclose(res[t], ref[t], rtol=1e-12, atol=1e-14), t
    assert ledger["elements"] == plan["cost"]


def test_mlp_graph_backward_is_the_gradient():
    """The backward ops of tofu_inputs.mlp are the gradient of the loss op:
    compared with central finite differences in fp64."""
    spec = mlp(4, [6, 8, 4])
    g = Graph(spec)
    vals = make_values(spec, seed=3)
    env = run_graph(g, vals, emulate_storage=False, fast=False)
    h = 1e-6
    rng = np.random.default_rng(0)
    for w, dw in (("W1", "dW1"), ("W2", "dW2")):
        for _ in range(6):
            idx = tuple(rng.integers(0, s) for s in vals[w].shape)
            vp = dict(vals); vp[w] = vals[w].copy(); vp[w][idx] += h
            vm = dict(vals); vm[w] = vals[w].copy(); vm[w][idx] -= h
            lp = run_graph(g, vp, emulate_storage=False)["loss"]
            lm = run_graph(g, vm, emulate_storage=False)["loss"]
            fd = (lp - lm) / (2 * h)
            assert abs(fd - env[dw][idx]) <= 1e-6 * max(1.0, abs(fd)), (w, idx)
    # SGD with momentum: W_new = W - lr*(mu*M + dW)
    assert np.allclose(env["W1_new"], vals["W1"] - 0.0078125 * (0.875 * vals["M1"] + env["dW1"]))


@pytest.mark.parametrize("cfg,k", [(0, 2), (0, 4), (0, 8)])
def test_partitioned_equals_unpartitioned_and_ledger_equals_plan(cfg, k):
    """Semantic equivalence on integer data, and the
    simulated byte ledger equals the planned cost (north star: bytes vs plan)."""
    spec = config(cfg)
    g = Graph(spec)
    vals = make_values(spec, seed=5, mode="int")
    ref = run_graph(g, vals, emulate_storage=False)
    plan = recursive_search(g, k)
    res, ledger = simulate(g, plan, vals)
    for t in ref:
        assert np.array_equal(res[t], ref[t]), t
    el, by = plan_cost(g, plan)
    assert ledger["elements"] == el == plan["cost"]
    assert ledger["bytes"] == by


def test_fc_small_partitioned_k8():
    spec = mlp(16, [32, 32])
    g = Graph(spec)
    vals = make_values(spec, seed=2, mode="int")
    ref = run_graph(g, vals, emulate_storage=False)
    plan = recursive_search(g, 8)
    res, ledger = simulate(g, plan, vals)
    for t in ref:
        assert np.array_equal(res[t], ref[t]), t
    assert ledger["elements"] == plan_cost(g, plan)[0]
