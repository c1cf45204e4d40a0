"""Workload graph descriptions (the input of tofu_plan / tofu_execute).

Each builder returns the graph JSON dict documented in oracle/graph.py and
include/tofu.h: TDL defs (text), tensors with shapes/dtypes/roles, ops in
execution order (forward, loss, backward, optimizer) and in-place aliases.
Constants of the elementwise defs (loss scale, learning rate, momentum) are
powers of two or dyadic so every side represents them exactly.

Workloads follow BASELINE.json configs:
  configs[0]  mlp(64, [256, 512, 512])          2-layer MLP, k = 2
  configs[1]  mlp(512, [8192, 8192])            single large FC layer, k = 8
  configs[2]  lstm(6, 4096, 20, 128)             6-layer LSTM, hidden 4K, 20 steps, batch 128
"""
from __future__ import annotations

LR = 0.0078125      # 2^-7
MU = 0.875          # momentum

MM_DEFS = {
    "mm_nn": "def mm_nn(A(2), B(2)) -> lambda i, j: reduce(Sum; k; A[i, k] * B[k, j])",
    "mm_nt": "def mm_nt(A(2), B(2)) -> lambda i, j: reduce(Sum; k; A[i, k] * B[j, k])",
    "mm_tn": "def mm_tn(A(2), B(2)) -> lambda i, j: reduce(Sum; k; A[k, i] * B[k, j])",
}


def _num(c: float) -> str:
    s = ("%.40f" % c).rstrip("0")
    return s + "0" if s.endswith(".") else s


def mlp(batch: int, dims: list, lr: float = LR, mu: float = MU, relu_last: bool = False) -> dict:
    """MLP training step: H_l = relu(H_{l-1} · W_l) (no relu on the last
    layer), loss = mean((Y - T)^2), SGD with momentum.  No biases."""
    L = len(dims) - 1
    n_out = batch * dims[-1]
    defs = dict(MM_DEFS)
    defs["relu"] = "def relu(X(2)) -> lambda i, j: max(X[i, j], 0)"
    defs["relu_grad"] = "def relu_grad(X(2), D(2)) -> lambda i, j: select(X[i, j] > 0, D[i, j], 0)"
    defs["mse_grad"] = f"def mse_grad(Y(2), T(2)) -> lambda i, j: (Y[i, j] - T[i, j]) * {_num(2.0 / n_out)}"
    defs["sumsq"] = (f"def sumsq(Y(2), T(2)) -> lambda : reduce(Sum; i, j; "
                     f"(Y[i, j] - T[i, j]) * (Y[i, j] - T[i, j]) * {_num(1.0 / n_out)})")
    defs["mom"] = f"def mom(M(2), G(2)) -> lambda i, j: M[i, j] * {_num(mu)} + G[i, j]"
    defs["sgd"] = f"def sgd(W(2), M(2)) -> lambda i, j: W[i, j] - M[i, j] * {_num(lr)}"
    T = {}
    ops = []
    alias = {}

    def tensor(name, shape, dtype, role, grad_of=None):
        T[name] = {"shape": list(shape), "dtype": dtype, "role": role, "grad_of": grad_of, "merge": None}

    def op(name, d, ins, out, backward_of=None, attrs=None):
        ops.append({"name": name, "def": d, "inputs": list(ins), "output": out,
                    "backward_of": backward_of, "merge": None, "attrs": attrs or {}})

    tensor("X", (batch, dims[0]), "bf16", "input")
    tensor("T", (batch, dims[-1]), "bf16", "input")
    h = "X"
    for l in range(1, L + 1):
        tensor(f"W{l}", (dims[l - 1], dims[l]), "bf16", "weight")
        tensor(f"M{l}", (dims[l - 1], dims[l]), "f32", "state")
        z = f"Z{l}" if (l < L or relu_last) else "Y"
        tensor(z, (batch, dims[l]), "bf16", "act")
        op(f"fc{l}", "mm_nn", [h, f"W{l}"], z)
        if l < L or relu_last:
            tensor(f"H{l}", (batch, dims[l]), "bf16", "act")
            op(f"relu{l}", "relu", [z], f"H{l}")
            h = f"H{l}"
        else:
            h = z
    yname = h
    tensor("loss", (), "f32", "loss")
    tensor("dY", (batch, dims[-1]), "bf16", "grad", grad_of=yname)
    op("loss", "sumsq", [yname, "T"], "loss", attrs={"scale": 1.0 / n_out})
    op("loss_grad", "mse_grad", [yname, "T"], "dY", attrs={"scale": 2.0 / n_out})
    g = "dY"
    for l in range(L, 0, -1):
        if relu_last or l < L:
            zn = f"Z{l}"
            tensor(f"dZ{l}", (batch, dims[l]), "bf16", "grad", grad_of=zn)
            op(f"relu{l}_bwd", "relu_grad", [zn, g], f"dZ{l}", backward_of=f"relu{l}")
            g = f"dZ{l}"
        hin = "X" if l == 1 else f"H{l-1}"
        tensor(f"dW{l}", (dims[l - 1], dims[l]), "f32", "grad", grad_of=f"W{l}")
        op(f"fc{l}_wgrad", "mm_tn", [hin, g], f"dW{l}", backward_of=f"fc{l}")
        if l > 1:
            tensor(f"dH{l-1}", (batch, dims[l - 1]), "bf16", "grad", grad_of=f"H{l-1}")
            op(f"fc{l}_dgrad", "mm_nt", [g, f"W{l}"], f"dH{l-1}", backward_of=f"fc{l}")
            g = f"dH{l-1}"
    for l in range(1, L + 1):
        tensor(f"M{l}_new", (dims[l - 1], dims[l]), "f32", "state")
        tensor(f"W{l}_new", (dims[l - 1], dims[l]), "bf16", "weight")
        op(f"mom{l}", "mom", [f"M{l}", f"dW{l}"], f"M{l}_new", attrs={"mu": mu})
        op(f"sgd{l}", "sgd", [f"W{l}", f"M{l}_new"], f"W{l}_new", attrs={"lr": lr})
        alias[f"M{l}_new"] = f"M{l}"
        alias[f"W{l}_new"] = f"W{l}"
    used = {d for o in ops for d in [o["def"]]}
    defs = {k: v for k, v in defs.items() if k in used}
    return {"defs": defs, "tensors": T, "ops": ops, "alias": alias, "meta": {"samples_per_step": batch}}


def config(i: int) -> dict:
    if i == 0:
        return mlp(64, [256, 512, 512])
    if i == 1:
        return mlp(512, [8192, 8192])
    if i == 2:
        return lstm(6, 4096, 20, 128)
    raise ValueError(f"config {i} not built yet")


CONFIG_K = {0: 2, 1: 8}
CONFIG_NAME = {0: "mlp-2x512-b64", 1: "fc-8192x8192-b512"}


LSTM_DEFS = {
    "gate": "def gate(X(2), W(3)) -> lambda b, g, h: reduce(Sum; k; X[b, k] * W[k, g, h])",
    "mm_rec": "def mm_rec(A(3), W(3)) -> lambda b, k: reduce(Sum; g, h; A[b, g, h] * W[k, g, h])",
    "gate_wgrad": "def gate_wgrad(X(2), A(3)) -> lambda k, g, h: reduce(Sum; b; X[b, k] * A[b, g, h])",
}


def _lstm_cell_defs():
    a = lambda g: f"(GX[b, {g}, h] + GH[b, {g}, h])"
    I, F, G, O = f"sigmoid({a(0)})", f"sigmoid({a(1)})", f"tanh({a(2)})", f"sigmoid({a(3)})"
    TC = "tanh(C[b, h])"
    DH = "(DU[b, h] + DR[b, h])"
    DC = f"(DN[b, h] + {DH} * {O} * (1 - {TC} * {TC}))"
    d = {
        # c_t = f * c_{t-1} + i * g ;  h_t = o * tanh(c_t)   (LSTM cell, P:L1012-1013 [lstm])
        "cell_c": f"def cell_c(GX(3), GH(3), CP(2)) -> lambda b, h: {F} * CP[b, h] + {I} * {G}",
        "cell_h": f"def cell_h(GX(3), GH(3), C(2)) -> lambda b, h: {O} * {TC}",
        # gradients of the gate pre-activations (one output, gate index g selects the formula)
        "cell_bwd_a": (f"def cell_bwd_a(GX(3), GH(3), CP(2), C(2), DU(2), DR(2), DN(2)) -> lambda b, g, h: "
                       f"select(g == 0, {DC} * {G} * {I} * (1 - {I}), select(g == 1, {DC} * CP[b, h] * {F} * (1 - {F}), "
                       f"select(g == 2, {DC} * {I} * (1 - {G} * {G}), {DH} * {TC} * {O} * (1 - {O}))))"),
        # gradient wrt c_{t-1}
        "cell_bwd_c": f"def cell_bwd_c(GX(3), GH(3), C(2), DU(2), DR(2), DN(2)) -> lambda b, h: {DC} * {F}",
    }
    return d


def lstm(layers: int, hidden: int, steps: int, batch: int, lr: float = LR, mu: float = MU) -> dict:
    """Multi-layer LSTM RNN training step ("LSTM cell ... unrolled for 20 steps").

    Layout (reading §R10, output views): per layer the gate pre-activations of all timesteps from the
    layer input are one batched GEMM (Gx[T*B, 4, H]); the recurrent GEMM, the cell and its backward run
    per timestep and write their timestep's rows of stacked state tensors Cs / Hs [(T+1)*B, H] whose first
    B rows hold the zero initial state.  Weight gradients are single GEMMs over all T*B rows (in-place
    gradient aggregation over time).  Per-timestep ops/tensors of a layer share a merge key
    (timestep merging).  Loss: MSE of the top layer's outputs against a target sequence."""
    L, H, T, B = layers, hidden, steps, batch
    defs = dict(LSTM_DEFS)
    defs.update(_lstm_cell_defs())
    n_out = T * B * H
    defs["mse_grad"] = f"def mse_grad(Y(2), T(2)) -> lambda i, j: (Y[i, j] - T[i, j]) * {_num(2.0 / n_out)}"
    defs["sumsq"] = (f"def sumsq(Y(2), T(2)) -> lambda : reduce(Sum; i, j; "
                     f"(Y[i, j] - T[i, j]) * (Y[i, j] - T[i, j]) * {_num(1.0 / n_out)})")
    defs["mom3"] = f"def mom3(M(3), G(3)) -> lambda i, g, j: M[i, g, j] * {_num(mu)} + G[i, g, j]"
    defs["sgd3"] = f"def sgd3(W(3), M(3)) -> lambda i, g, j: W[i, g, j] - M[i, g, j] * {_num(lr)}"
    Tn, ops, alias = {}, [], {}

    def tensor(name, shape, dtype, role, merge=None, grad_of=None, init=None):
        Tn[name] = {"shape": list(shape), "dtype": dtype, "role": role, "grad_of": grad_of, "merge": merge}
        if init:
            Tn[name]["init"] = init

    def op(name, d, ins, out, offsets=None, out_offset=None, ranges=None, merge=None, backward_of=None, attrs=None):
        o = {"name": name, "def": d, "inputs": list(ins), "output": out, "backward_of": backward_of,
             "merge": merge, "attrs": attrs or {}}
        if offsets:
            o["offsets"] = offsets
        if out_offset:
            o["out_offset"] = out_offset
        if ranges:
            o["ranges"] = ranges
        ops.append(o)

    tensor("X", (T * B, H), "bf16", "input")
    tensor("T", (T * B, H), "bf16", "input")
    tensor("loss", (), "f32", "loss")
    for l in range(1, L + 1):
        p = f"L{l}."
        for w in ("Wx", "Wh"):
            tensor(p + w, (H, 4, H), "bf16", "weight")
            tensor(p + "M" + w[1], (H, 4, H), "f32", "state")
            tensor(p + "d" + w, (H, 4, H), "f32", "grad", grad_of=p + w)
        tensor(p + "Gx", (T * B, 4, H), "bf16", "act")
        tensor(p + "Cs", ((T + 1) * B, H), "f32", "state", init="zeros")   # rows 0..B-1: c_{-1} = 0
        tensor(p + "Hs", ((T + 1) * B, H), "bf16", "state", init="zeros")  # rows 0..B-1: h_{-1} = 0
        tensor(p + "dHs", (T * B, H), "bf16", "grad", grad_of=p + "Hs")
        tensor(p + "dA", (T * B, 4, H), "bf16", "grad")
        tensor(p + "Zr", (B, H), "f32", "state", init="zeros")     # zero recurrent gradients at t = T-1
        tensor(p + "Zc", (B, H), "f32", "state", init="zeros")
        for t in range(T):
            tensor(p + f"Gh{t}", (B, 4, H), "bf16", "act", merge=p + "Gh")
            if t > 0:
                tensor(p + f"R{t - 1}", (B, H), "f32", "grad", merge=p + "R")
                tensor(p + f"D{t - 1}", (B, H), "f32", "grad", merge=p + "D")
    # ---------------------------------------------------------------- forward
    for l in range(1, L + 1):
        p = f"L{l}."
        if l == 1:
            op(p + "gx", "gate", ["X", p + "Wx"], p + "Gx")
        else:
            op(p + "gx", "gate", [f"L{l - 1}.Hs", p + "Wx"], p + "Gx", offsets=[[B, 0], None],
               ranges={"b": T * B})
        for t in range(T):
            op(p + f"gh{t}", "gate", [p + "Hs", p + "Wh"], p + f"Gh{t}", offsets=[[t * B, 0], None],
               ranges={"b": B}, merge=p + "gh")
            op(p + f"c{t}", "cell_c", [p + "Gx", p + f"Gh{t}", p + "Cs"], p + "Cs",
               offsets=[[t * B, 0, 0], None, [t * B, 0]], out_offset=[(t + 1) * B, 0], ranges={"b": B},
               merge=p + "c")
            op(p + f"h{t}", "cell_h", [p + "Gx", p + f"Gh{t}", p + "Cs"], p + "Hs",
               offsets=[[t * B, 0, 0], None, [(t + 1) * B, 0]], out_offset=[(t + 1) * B, 0], ranges={"b": B},
               merge=p + "h")
    top = f"L{L}."
    op("loss", "sumsq", [top + "Hs", "T"], "loss", offsets=[[B, 0], None], ranges={"i": T * B},
       attrs={"scale": 1.0 / n_out})
    op("loss_grad", "mse_grad", [top + "Hs", "T"], top + "dHs", offsets=[[B, 0], None], attrs={"scale": 2.0 / n_out})
    # ---------------------------------------------------------------- backward through time
    for l in range(L, 0, -1):
        p = f"L{l}."
        for t in range(T - 1, -1, -1):
            R = p + ("Zr" if t == T - 1 else f"R{t}")
            D = p + ("Zc" if t == T - 1 else f"D{t}")
            op(p + f"da{t}", "cell_bwd_a", [p + "Gx", p + f"Gh{t}", p + "Cs", p + "Cs", p + "dHs", R, D], p + "dA",
               offsets=[[t * B, 0, 0], None, [t * B, 0], [(t + 1) * B, 0], [t * B, 0], None, None],
               out_offset=[t * B, 0, 0], ranges={"b": B}, merge=p + "da", backward_of=p + f"c{t}")
            if t > 0:
                op(p + f"dc{t}", "cell_bwd_c", [p + "Gx", p + f"Gh{t}", p + "Cs", p + "dHs", R, D], p + f"D{t - 1}",
                   offsets=[[t * B, 0, 0], None, [(t + 1) * B, 0], [t * B, 0], None, None], ranges={"b": B},
                   merge=p + "dc", backward_of=p + f"c{t}")
                op(p + f"rec{t}", "mm_rec", [p + "dA", p + "Wh"], p + f"R{t - 1}", offsets=[[t * B, 0, 0], None],
                   ranges={"b": B}, merge=p + "rec", backward_of=p + f"gh{t}")
        if l > 1:   # input gradient first: it reads Wx before the optimizer (fused into wgx) updates it
            op(p + "dx", "mm_rec", [p + "dA", p + "Wx"], f"L{l - 1}.dHs", backward_of=p + "gx")
        xin = "X" if l == 1 else f"L{l - 1}.Hs"
        xoff = None if l == 1 else [[B, 0], None]
        op(p + "wgx", "gate_wgrad", [xin, p + "dA"], p + "dWx", offsets=xoff, ranges={"b": T * B},
           backward_of=p + "gx")
        op(p + "wgh", "gate_wgrad", [p + "Hs", p + "dA"], p + "dWh", ranges={"b": T * B}, backward_of=p + "gh0")
    # ---------------------------------------------------------------- optimizer (SGD with momentum)
    for l in range(1, L + 1):
        p = f"L{l}."
        for w in ("Wx", "Wh"):
            m = p + "M" + w[1]
            tensor(m + "_new", (H, 4, H), "f32", "state")
            tensor(p + w + "_new", (H, 4, H), "bf16", "weight")
            op(p + "mom" + w[1], "mom3", [m, p + "d" + w], m + "_new", attrs={"mu": mu})
            op(p + "sgd" + w[1], "sgd3", [p + w, m + "_new"], p + w + "_new", attrs={"lr": lr})
            alias[m + "_new"] = m
            alias[p + w + "_new"] = p + w
    used = {o["def"] for o in ops}
    return {"defs": {k: v for k, v in defs.items() if k in used}, "tensors": Tn, "ops": ops, "alias": alias,
            "meta": {"samples_per_step": B, "tokens_per_step": T * B}}


CONFIG_K[2] = 8
CONFIG_NAME[2] = "lstm-6x4096-T20-b128"


def _config_lstm():
    return lstm(6, 4096, 20, 128)
