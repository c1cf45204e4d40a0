"""Oracle pins for the WResNet path (configs[3]): convolution TDL (reading R11: zero padding, floor-division /
remainder index terms), the tap evaluation, and the WResNet training graph (reading R12).

Pins that do not reuse the oracle's own formulas:
* the literal TDL interpreter (tdl_eval, one lambda evaluation per point) on tiny inputs;
* torch.nn.functional.conv2d / max_pool2d / autograd in fp64 on CPU (the convolution, its data and weight
  gradients, and the max-pool gradient are textbook library routines);
* an independently written torch model of the whole network: loss and every weight gradient;
* Table 3: the total weight sizes of WResNet-50/101/152 at widening 4..10;
* the cost model's box arithmetic == element enumeration on conv graphs, and the partitioned simulator ==
  unpartitioned execution with the ledger equal to the plan.
"""
import random

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle.cost import op_cost_box, op_cost_enum, plan_cost
from oracle.exec_ref import fast_eval, run_graph, tap_eval, tdl_eval
from oracle.graph import Graph
from oracle.search import recursive_search
from oracle.sim import simulate
from oracle.tdl import TdlError, parse_def
from tofu_inputs.graphs import WRN_UNITS, conv_defs, wresnet
from tofu_inputs.tensors import make_values

CONVS = [(1, 1, 0), (3, 1, 1), (3, 2, 1), (1, 2, 0), (7, 2, 3)]


def _nhwc(t):
    return t.permute(0, 2, 3, 1)


def _w_torch(w):  # [co, ky, kx, ci] -> [co, ci, ky, kx]
    return torch.from_numpy(w).permute(0, 3, 1, 2)


def _rand(rng, shape):
    return rng.integers(-4, 5, shape).astype(np.float64)


def test_index_terms_parse_and_evaluate():
    d = parse_def("def f(A(1)) -> lambda y: reduce(Sum; t; A[(y - 2*t + 1) / 2] * A[2 * (y + 1) % 3])")
    acc = d.accesses[0].index[0]
    env = {"y": np.arange(-3, 6), "t": 1}
    assert list(acc.value(env)) == [(y - 2 + 1) // 2 for y in range(-3, 6)]
    assert list(d.accesses[1].index[0].value({"y": np.arange(5), "t": 0})) == [2 * ((y + 1) % 3) for y in range(5)]
    # hull: floor division is monotone (exact); remainder spans [0, d-1] once the range wraps
    assert acc.hull({"y": (0, 9), "t": (0, 1)}) == ((0 - 2 + 1) // 2, (9 + 1) // 2)
    assert d.accesses[1].index[0].hull({"y": (0, 0), "t": (0, 0)}) == (2, 2)
    assert d.accesses[1].index[0].hull({"y": (0, 5), "t": (0, 0)}) == (0, 4)
    for bad in ("def f(A(1)) -> lambda y: A[(y) / 0]", "def f(A(1)) -> lambda y: A[(y) * 2]",
                "def f(A(1)) -> lambda y: A[y / 2]"):
        with pytest.raises(TdlError):
            parse_def(bad)


@pytest.mark.parametrize("R,s,p", CONVS)
@pytest.mark.parametrize("kind", ["conv", "dconv", "wconv"])
def test_tap_eval_equals_literal_interpreter(R, s, p, kind):
    if kind == "dconv" and R == 7:
        pytest.skip("the stem has no data gradient")
    defs = conv_defs(R, s, p)
    d = parse_def(defs[f"{kind}_k{R}s{s}p{p}"])
    rng = np.random.default_rng(R * 10 + s)
    B, H, C, Co = 2, 6 if R < 7 else 8, 3, 2
    Ho = (H + 2 * p - R) // s + 1
    X, W, D = _rand(rng, (B, H, H, C)), _rand(rng, (Co, R, R, C)), _rand(rng, (B, Ho, Ho, Co))
    if kind == "conv":
        ins, box = {"X": X, "W": W}, {"b": B, "y": Ho, "x": Ho, "co": Co, "ky": R, "kx": R, "ci": C}
    elif kind == "dconv":
        T = (R + 1) // 2
        ins = {"D": D, "W": W}
        box = {"b": B, "y": H, "x": H, "ci": C, "co": Co}
        box.update({"ty": T, "tx": T} if s == 2 else {"ky": R, "kx": R})
    else:
        ins, box = {"D": D, "X": X}, {"co": Co, "ky": R, "kx": R, "ci": C, "b": B, "y": Ho, "x": Ho}
    ins = {k: (v, (0,) * v.ndim) for k, v in ins.items()}
    box = {k: (0, n - 1) for k, n in box.items()}
    got = tap_eval(d, ins, box)
    assert got is not None
    assert np.array_equal(got, tdl_eval(d, ins, box))
    # a sub-box (a worker's tile) of the same op
    sub = dict(box)
    first = d.out_vars[0]
    sub[first] = (box[first][1], box[first][1])
    assert np.array_equal(tap_eval(d, ins, sub), tdl_eval(d, ins, sub))


@pytest.mark.parametrize("R,s,p", CONVS)
def test_conv_and_gradients_equal_torch(R, s, p):
    """conv_, dconv_ and wconv_ defs are the convolution and its two gradients (torch fp64 autograd)."""
    defs = conv_defs(R, s, p)
    rng = np.random.default_rng(7)
    B, H, C, Co = 2, 9, 3, 4
    Ho = (H + 2 * p - R) // s + 1
    X, W, D = rng.standard_normal((B, H, H, C)), rng.standard_normal((Co, R, R, C)), rng.standard_normal((B, Ho, Ho, Co))
    xt = torch.from_numpy(X).permute(0, 3, 1, 2).requires_grad_(True)
    wt = _w_torch(W).requires_grad_(True)
    yt = F.conv2d(xt, wt, stride=s, padding=p)
    yt.backward(torch.from_numpy(D).permute(0, 3, 1, 2))
    n = f"k{R}s{s}p{p}"
    z = lambda a: (a, (0,) * a.ndim)
    full = lambda d, ext: {v: (0, ext[v] - 1) for v in d.all_vars()}
    d = parse_def(defs["conv_" + n])
    y = fast_eval(d, {"X": z(X), "W": z(W)}, full(d, {"b": B, "y": Ho, "x": Ho, "co": Co, "ky": R, "kx": R, "ci": C}))
    assert np.allclose(y, _nhwc(yt.detach()).numpy(), rtol=1e-12, atol=1e-12)
    d = parse_def(defs["wconv_" + n])
    dw = fast_eval(d, {"D": z(D), "X": z(X)}, full(d, {"co": Co, "ky": R, "kx": R, "ci": C, "b": B, "y": Ho, "x": Ho}))
    assert np.allclose(dw, wt.grad.permute(0, 2, 3, 1).numpy(), rtol=1e-12, atol=1e-12)
    if "dconv_" + n in defs:
        d = parse_def(defs["dconv_" + n])
        ext = {"b": B, "y": H, "x": H, "ci": C, "co": Co}
        ext.update({"ty": (R + 1) // 2, "tx": (R + 1) // 2} if s == 2 else {"ky": R, "kx": R})
        dx = fast_eval(d, {"D": z(D), "W": z(W)}, full(d, ext))
        assert np.allclose(dx, _nhwc(xt.grad).numpy(), rtol=1e-12, atol=1e-12)


def test_maxpool_and_gradient_equal_torch():
    g = wresnet([1], 1, 2, 16, base=4, classes=3)
    mp, mpg = parse_def(g["defs"]["maxpool"]), parse_def(g["defs"]["maxpool_grad"])
    rng = np.random.default_rng(2)
    B, H, C = 2, 8, 3
    X = np.abs(rng.standard_normal((B, H, H, C)))       # post-ReLU inputs, no ties
    X[0, 0, 0, 0] = 0.0
    xt = torch.from_numpy(X).permute(0, 3, 1, 2).requires_grad_(True)
    yt = F.max_pool2d(xt, 3, 2, 1)
    Ho = yt.shape[2]
    D = rng.standard_normal((B, Ho, Ho, C))
    yt.backward(torch.from_numpy(D).permute(0, 3, 1, 2))
    z = lambda a: (a, (0,) * a.ndim)
    Y = tdl_eval(mp, {"X": z(X)}, {"b": (0, B - 1), "y": (0, Ho - 1), "x": (0, Ho - 1), "c": (0, C - 1),
                                   "ky": (0, 2), "kx": (0, 2)})
    assert np.array_equal(Y, _nhwc(yt.detach()).numpy())
    dX = tdl_eval(mpg, {"X": z(X), "Y": z(Y), "D": z(D), "K": z(np.ones((3, 3, C)))},
                  {"b": (0, B - 1), "y": (0, H - 1), "x": (0, H - 1), "c": (0, C - 1), "ty": (0, 1), "tx": (0, 1)})
    assert np.allclose(dX, _nhwc(xt.grad).numpy(), rtol=1e-13, atol=1e-13)


def _torch_wresnet(units, width, base, vals, image):
    """The same network written directly with torch ops (NCHW), fp64: loss and weight gradients."""
    P = {k: torch.from_numpy(v).clone().requires_grad_(True) for k, v in vals.items()
         if k.endswith(("W", "W1", "W2", "W3", "Wp"))}
    cw = lambda w: w.permute(0, 3, 1, 2)
    x = torch.from_numpy(vals["X"]).permute(0, 3, 1, 2)
    h = F.relu(F.conv2d(x, cw(P["stem.W"]), stride=2, padding=3))
    x = F.max_pool2d(h, 3, 2, 1)
    for s, n in enumerate(units):
        for u in range(n):
            p = f"s{s}u{u}."
            st = 2 if (u == 0 and s > 0) else 1
            z = F.relu(F.conv2d(x, cw(P[p + "W1"])))
            z = F.relu(F.conv2d(z, cw(P[p + "W2"]), stride=st, padding=1))
            z = F.conv2d(z, cw(P[p + "W3"]))
            sc = F.conv2d(x, cw(P[p + "Wp"]), stride=st) if u == 0 else x
            x = F.relu(z + sc)
    y = x.mean(dim=(2, 3)) @ P["fc.W"]
    loss = ((y - torch.from_numpy(vals["T"])) ** 2).mean()
    loss.backward()
    return float(loss), {k: v.grad.numpy() for k, v in P.items()}


def test_wresnet_graph_equals_independent_torch_model():
    units, width, base, image = [2, 1], 1, 4, 16
    spec = wresnet(units, width, 2, image, base=base, classes=5)
    g = Graph(spec)
    vals = make_values(spec, seed=9)
    env = run_graph(g, vals, emulate_storage=False)
    loss, grads = _torch_wresnet(units, width, base, vals, image)
    assert abs(env["loss"] - loss) <= 1e-12 * abs(loss)
    for w, gw in grads.items():
        d = env[w.replace(".W", ".dW") if w in ("stem.W", "fc.W") else w[:-2] + "d" + w[-2:]]
        assert np.allclose(d, gw, rtol=1e-9, atol=1e-14 * np.abs(gw).max()), w
    # SGD with momentum applied to every weight
    for w in grads:
        m = vals[w + ".M"]
        assert np.allclose(env[w + "_new"], vals[w] - 0.0078125 * (0.875 * m + grads[w]), rtol=1e-12, atol=1e-15)


def test_table3_weight_sizes():
    """Table 3: weight + gradient + history in fp32 (3W), GiB.  The graph's
    weight tensors (RGB stem, i.e. without the 5 padding channels) reproduce every entry within 3%
    (the paper does not state its BN / bias parameters or rounding)."""
    table = {50: [4.2, 9.6, 17.1, 26.7], 101: [7.8, 17.1, 30.6, 47.7], 152: [10.5, 23.4, 41.7, 65.1]}
    for L, row in table.items():
        for w, gib in zip((4, 6, 8, 10), row):
            spec = wresnet(WRN_UNITS[L], w, 1, 32)
            n = 0
            for name, t in spec["tensors"].items():
                if t["role"] == "weight" and name not in spec["alias"]:
                    shp = list(t["shape"])
                    if name == "stem.W":
                        shp[-1] = 3
                    n += int(np.prod(shp))
            assert abs(n * 12 / 2 ** 30 - gib) <= 0.03 * gib, (L, w, n * 12 / 2 ** 30, gib)
    # the WResNet-152-4 model of configs[3]: 0.94 G parameters
    spec = wresnet(WRN_UNITS[152], 4, 32)
    assert len([o for o in spec["ops"] if o["def"].startswith("conv_")]) == 155


def _random_op_plan(g, op, factors, rng):
    """Random per-step split dims of the op's tensors and split vars of the op (divisible ones only)."""
    td = {}
    for t in list(op["inputs"]) + [op["output"]]:
        n = list(g.shape(t))
        seq = []
        for f in factors:
            ok = [d for d in range(len(n)) if n[d] % f == 0] if n else []
            d = rng.choice(ok) if ok else None
            if d is not None:
                n[d] //= f
            seq.append(d)
        td[t] = seq
    n = dict(g.ranges[op["name"]])
    seq = []
    for f in factors:
        ok = [v for v in g.split_vars(op) if n[v] % f == 0]
        if not ok:
            return None
        v = rng.choice(ok)
        n[v] //= f
        seq.append(v)
    if any(None in s for s in td.values()):
        return None
    return td, {op["name"]: seq}


def test_conv_box_cost_equals_element_enumeration():
    spec = wresnet([1, 1], 1, 2, 8, base=4, classes=4)
    g = Graph(spec)
    rng = random.Random(3)
    checked = 0
    conv_ops = [o for o in g.ops if "conv" in o["def"] or "pool" in o["def"] or o["def"] == "gap"]
    for op in conv_ops:
        for factors in ([2], [2, 2]):
            for _ in range(4):
                p = _random_op_plan(g, op, factors, rng)
                if p is None:
                    continue
                td, osp = p
                assert op_cost_box(g, op, td, osp, factors)[0] == op_cost_enum(g, op, td, osp, factors), \
                    (op["name"], td, osp)
                checked += 1
    assert checked > 100


@pytest.mark.parametrize("k,units", [(2, [1, 1]), (4, [1])])
def test_wresnet_partitioned_sim_equals_unpartitioned(k, units):
    spec = wresnet(units, 1, 4, 16 if k == 2 else 8, base=4, classes=4)
    g = Graph(spec)
    vals = make_values(spec, seed=4, mode="int")
    ref = run_graph(g, vals, emulate_storage=False)
    plan = recursive_search(g, k)
    res, ledger = simulate(g, plan, vals)
    for t in ref:
        assert np.array_equal(res[t], ref[t]), t
    el, by = plan_cost(g, plan)
    assert ledger["elements"] == el == plan["cost"]
    assert ledger["bytes"] == by
