"""The sampled per-op checker (tests/sampled_parity.py) validated on CPU against the oracle's own full
execution: with every tensor stored it reproduces run_graph exactly; tensors declared unmaterialised are
recomputed through their producers (R13); a corrupted stored tensor is caught."""
import numpy as np
import pytest

from oracle.exec_ref import run_graph
from oracle.graph import Graph
from sampled_parity import SampledChecker
from tofu_inputs.graphs import config, lstm, wresnet
from tofu_inputs.tensors import make_values


def _env_source(env):
    def src(name, box):
        v = env[name]
        return v[tuple(slice(lo, hi + 1) for lo, hi in box)] if box else v
    return src


@pytest.mark.parametrize("which", ["mlp", "lstm", "wresnet"])
def test_checker_reproduces_the_oracle(which):
    spec = {"mlp": lambda: config(0), "lstm": lambda: lstm(2, 16, 3, 4),
            "wresnet": lambda: wresnet([1, 1], 1, 2, 32, base=8, classes=8)}[which]()
    vals = make_values(spec, seed=3)
    env = run_graph(Graph(spec), vals, emulate_storage=True)
    res = SampledChecker(spec, vals, _env_source(env), seed=1).check_all(boxes=2)
    assert len(res) == len(spec["ops"])
    assert max(e for e, _ in res.values()) == 0.0


def test_checker_recomputes_unmaterialized_and_catches_corruption():
    spec = wresnet([1], 1, 2, 32, base=8, classes=8)
    vals = make_values(spec, seed=4)
    g = Graph(spec)
    env = run_graph(g, vals, emulate_storage=True)
    # pretend every convolution output read by exactly one relu is folded into it (never stored)
    readers = {}
    for op in g.ops:
        for t in op["inputs"]:
            readers.setdefault(t, []).append(op)
    unmat = [op["output"] for op in g.ops if op["def"].startswith("conv_")
             and len(readers.get(op["output"], [])) == 1 and readers[op["output"]][0]["def"].startswith("relu")]
    assert unmat
    hidden = {t: v for t, v in env.items() if t not in unmat}
    chk = SampledChecker(spec, vals, _env_source(hidden), unmaterialized=unmat, seed=2)
    res = chk.check_all(boxes=2)
    assert all(e <= tol for e, tol in res.values())
    # a 1% error in one stored fp32 weight gradient is caught (tolerance 1e-5)
    dw = "s0u0.dW2"
    bad = dict(hidden)
    bad[dw] = env[dw] * 1.01
    with pytest.raises(AssertionError):
        SampledChecker(spec, vals, _env_source(bad), unmaterialized=unmat, seed=2).check_all(boxes=2)
