"""GPU parity of the WResNet path (configs[3]): implicit-GEMM convolutions (forward, stride-1/2 data
gradients, weight gradients with split-K and the fused optimizer), max pool and its gradient, global
average pool, residual joins — through tofu_execute on one B200, per op on the GPU's own inputs against the
oracle (bf16 outputs normwise <= 5e-3, fp32 <= 1e-5), end to end, and partitioned (virtual ranks) with the
byte ledger equal to the plan."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.exec_ref import run_graph  # noqa: E402
from oracle.graph import Graph as OGraph  # noqa: E402
from test_gpu_exec import nrm, per_op_check, run_gpu  # noqa: E402
from tofu_inputs.graphs import wresnet  # noqa: E402
from tofu_inputs.tensors import make_values  # noqa: E402


def small(batch=2, image=64, base=8, units=(1, 1, 1, 1), classes=16):
    # stem 64 -> 32, pool 16, stages 16 / 8 / 4 / 2: every conv kind, stride-2 phases, ragged row tiles
    return wresnet(list(units), 1, batch, image, base=base, classes=classes)


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_wresnet_step_per_op_parity(k, monkeypatch):
    """k = 4, 8 plans split activations spatially (halo regions fetched from the neighbours)."""
    monkeypatch.setenv("TOFU_FUSE", "0")
    spec = small()
    vals = make_values(spec, seed=21)
    R, out = run_gpu(spec, k, vals)
    worst = per_op_check(spec, vals, out)
    assert len(worst) == len(spec["ops"])
    assert R.ledger() == R.plan.cost()


def test_wresnet_wide_channels_per_op_parity(monkeypatch):
    """Channel counts of the real model's scale (>= 64 per tap: one tap per k-block, BN = 256 tiles)."""
    monkeypatch.setenv("TOFU_FUSE", "0")
    spec = wresnet([2, 1], 1, 4, 32, base=64, classes=64)
    vals = make_values(spec, seed=22)
    _, out = run_gpu(spec, 1, vals)
    per_op_check(spec, vals, out)


@pytest.mark.parametrize("k", [1, 2])
def test_wresnet_fused_product_path(k, monkeypatch):
    """Product path: the optimizer folded into every weight-gradient epilogue (or its split-K reduction)."""
    monkeypatch.setenv("TOFU_FUSE", "1")
    spec = small()
    vals = make_values(spec, seed=23)
    R, out = run_gpu(spec, k, vals)
    ref = run_graph(OGraph(spec), vals, emulate_storage=True)
    checked = 0
    for t, info in spec["tensors"].items():
        if t.endswith((".M_new", "W_new")) or t in ("Y", "loss"):
            r = ref[t]
            e = nrm(out[t], r) if np.ndim(r) else abs(out[t] - r) / abs(r)
            assert e <= 3e-2, (t, e)
            checked += 1
    assert checked > 20
    assert R.ledger() == R.plan.cost()


def test_wresnet_partitioned_equals_unpartitioned():
    spec = small()
    vals = make_values(spec, seed=24)
    _, o1 = run_gpu(spec, 1, vals)
    for k in (2, 4):
        _, ok = run_gpu(spec, k, vals)
        for t in ("Y", "loss", "stem.W_new", "s3u0.W2_new", "fc.W_new"):
            e = nrm(ok[t], o1[t]) if np.ndim(o1[t]) else abs(ok[t] - o1[t]) / abs(o1[t])
            assert e <= 1e-2, (k, t, e)


@pytest.mark.parametrize("k", [1, 2, 8])
def test_wresnet_epilogue_fusion(k, monkeypatch):
    """Channel counts that enable the element-wise epilogue fusions (relu / residual add / relu-gradient mask
    folded into the convolution and GEMM producers): fused run vs the oracle end to end, and vs the unfused
    GPU run (identical up to the one skipped bf16 rounding of each fused intermediate, R13)."""
    spec = wresnet([2, 1], 1, 2, 64, base=32, classes=32)
    vals = make_values(spec, seed=25)
    monkeypatch.setenv("TOFU_FUSE", "1")
    R, fused = run_gpu(spec, k, vals)
    descs = [R.exec.launch_desc(i) for i in range(R.exec.num_launches())]
    assert sum("epilogue" in d.get("fused", "") for d in descs) >= 10
    ref = run_graph(OGraph(spec), vals, emulate_storage=True)
    for t in ("Y", "loss", "stem.W_new", "s0u1.W2_new", "s1u0.W3_new", "fc.W_new", "s0u0.W1.M_new"):
        r = ref[t]
        e = nrm(fused[t], r) if np.ndim(r) else abs(fused[t] - r) / abs(r)
        assert e <= 3e-2, (t, e)
    monkeypatch.setenv("TOFU_FUSE", "0")
    _, plain = run_gpu(spec, k, vals)
    for t in ("Y", "s0u1.W2_new", "s0u0.W1.M_new", "stem.W.M_new"):
        e = nrm(fused[t], plain[t])
        assert e <= 2e-2, (t, e)
    assert R.ledger() == R.plan.cost()
