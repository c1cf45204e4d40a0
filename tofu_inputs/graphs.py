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
  configs[3]  wresnet_depth(152, 4, 32)          WResNet-152-4, batch 32, 224x224 images
  configs[4]  lstm(10, 8192, 20, 128) (bench config 4) and wresnet_depth(152, 10, 32) (bench config 5):
              the "models exceeding a single GPU's HBM" of the north star (both fit one B200's 180 GB at
              these batch sizes; reading R12 / SURVEY bite 4)
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
    if i == 3:
        return wresnet_depth(152, 4, 32)
    if i == 4:   # configs[4], first model: RNN-10-8K (batch 128 as the paper ran it)
        return lstm(10, 8192, 20, 128)
    if i == 5:   # configs[4], second model: WResNet-152-10, batch 32
        return wresnet_depth(152, 10, 32)
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


# ------------------------------------------------------------------------------------------------ WResNet
WRN_UNITS = {50: [3, 4, 6, 3], 101: [3, 4, 23, 3], 152: [3, 8, 36, 3]}


def conv_defs(R: int, s: int, p: int) -> dict:
    """TDL of a 2-D convolution (NHWC activations X[b, y, x, c], weights W[co, ky, kx, ci]) with an R x R
    filter, stride s, zero padding p (reading R11: an access outside its tensor reads 0), and its two
    gradients.  The data gradient of a stride-2 convolution is written with the floor-division /
    remainder index terms of reading R11: output pixel y receives from the input-gradient pixel
    (y + p - 2*ty) / 2 through filter tap (y + p) % 2 + 2*ty."""
    n = f"k{R}s{s}p{p}"
    sy = "y" if s == 1 else f"{s}*y"
    sx = "x" if s == 1 else f"{s}*x"
    d = {
        "conv_" + n: (f"def conv_{n}(X(4), W(4)) -> lambda b, y, x, co: reduce(Sum; ky, kx, ci; "
                      f"X[b, {sy} + ky - {p}, {sx} + kx - {p}, ci] * W[co, ky, kx, ci])"),
        "wconv_" + n: (f"def wconv_{n}(D(4), X(4)) -> lambda co, ky, kx, ci: reduce(Sum; b, y, x; "
                       f"D[b, y, x, co] * X[b, {sy} + ky - {p}, {sx} + kx - {p}, ci])"),
    }
    if s == 1:
        d["dconv_" + n] = (f"def dconv_{n}(D(4), W(4)) -> lambda b, y, x, ci: reduce(Sum; ky, kx, co; "
                           f"D[b, y - ky + {p}, x - kx + {p}, co] * W[co, ky, kx, ci])")
    elif s == 2:
        d["dconv_" + n] = (f"def dconv_{n}(D(4), W(4)) -> lambda b, y, x, ci: reduce(Sum; ty, tx, co; "
                           f"D[b, (y - 2*ty + {p}) / 2, (x - 2*tx + {p}) / 2, co] * "
                           f"W[co, (y + {p}) % 2 + 2*ty, (x + {p}) % 2 + 2*tx, ci])")
    return d


def wresnet(units: list, width: int, batch: int, image: int = 224, base: int = 64, classes: int = 1000,
            lr: float = LR, mu: float = MU) -> dict:
    """Wide ResNet training step (ResNet widened by a scalar on every convolution's channels,
    ImageNet 224x224 images).  Reading R12: bottleneck units (1x1, 3x3, 1x1; the stride of a
    stage's first unit on its 3x3 convolution and on its 1x1 projection shortcut), stem 7x7/2 convolution
    + ReLU + 3x3/2 max pool, global average pool, one FC layer, MSE loss, SGD with momentum; no batch
    normalisation; the RGB image is padded to 8 channels (3 live).  Channels: stem base*width, stage s
    bottleneck base*width*2^s, output 4*base*width*2^s."""
    defs = dict(MM_DEFS)
    T, ops, alias = {}, [], {}

    def tensor(name, shape, dtype, role, grad_of=None, **kw):
        T[name] = {"shape": list(shape), "dtype": dtype, "role": role, "grad_of": grad_of, "merge": None}
        T[name].update(kw)

    def op(name, d, ins, out, backward_of=None, ranges=None, attrs=None):
        o = {"name": name, "def": d, "inputs": list(ins), "output": out, "backward_of": backward_of,
             "merge": None, "attrs": attrs or {}}
        if ranges:
            o["ranges"] = ranges
        ops.append(o)

    def need_conv(R, s, p):
        defs.update(conv_defs(R, s, p))
        return f"k{R}s{s}p{p}"

    defs["relu4"] = "def relu4(X(4)) -> lambda b, y, x, c: max(X[b, y, x, c], 0)"
    defs["relu_grad4"] = "def relu_grad4(Y(4), D(4)) -> lambda b, y, x, c: select(Y[b, y, x, c] > 0, D[b, y, x, c], 0)"
    defs["addrelu"] = "def addrelu(A(4), B(4)) -> lambda b, y, x, c: max(A[b, y, x, c] + B[b, y, x, c], 0)"
    defs["add4"] = "def add4(A(4), B(4)) -> lambda b, y, x, c: A[b, y, x, c] + B[b, y, x, c]"
    # max pool 3x3 / 2, pad 1 (inputs are ReLU outputs >= 0, so zero padding equals -inf padding)
    defs["maxpool"] = ("def maxpool(X(4)) -> lambda b, y, x, c: reduce(Max; ky, kx; "
                       "X[b, 2*y + ky - 1, 2*x + kx - 1, c])")
    # its gradient: every input equal to its window's maximum receives the window's gradient; K[3, 3, c] = 1
    # masks the filter taps that exist (tap (y + 1) % 2 + 2*ty <= 2); it carries a channel dim so that it
    # can be split like the other operands (every tensor is split)
    defs["maxpool_grad"] = ("def maxpool_grad(X(4), Y(4), D(4), K(3)) -> lambda b, y, x, c: reduce(Sum; ty, tx; "
                            "select(X[b, y, x, c] == Y[b, (y - 2*ty + 1) / 2, (x - 2*tx + 1) / 2, c], "
                            "D[b, (y - 2*ty + 1) / 2, (x - 2*tx + 1) / 2, c] * K[(y + 1) % 2 + 2*ty, (x + 1) % 2 + 2*tx, c], 0))")
    cin = 8
    H = image
    X = "X"
    tensor(X, (batch, H, H, cin), "bf16", "input", live_channels=3)
    c0 = base * width
    # ------------------------------------------------------------------ forward
    fwd_units = []
    k = need_conv(7, 2, 3)
    H1 = (H + 2 * 3 - 7) // 2 + 1
    tensor("stem.W", (c0, 7, 7, cin), "bf16", "weight", fan_in=7 * 7 * 3)
    tensor("stem.Z", (batch, H1, H1, c0), "bf16", "act")
    tensor("stem.H", (batch, H1, H1, c0), "bf16", "act")
    op("stem.conv", "conv_" + k, [X, "stem.W"], "stem.Z")
    op("stem.relu", "relu4", ["stem.Z"], "stem.H")
    H2 = (H1 + 2 - 3) // 2 + 1
    tensor("pool.Y", (batch, H2, H2, c0), "bf16", "act")
    tensor("pool.K", (3, 3, c0), "bf16", "state", init="ones")
    op("pool", "maxpool", ["stem.H"], "pool.Y", ranges={"ky": 3, "kx": 3})
    x, c, Hc = "pool.Y", c0, H2
    for s, n in enumerate(units):
        mid, outc = base * width * 2 ** s, 4 * base * width * 2 ** s
        for u in range(n):
            p = f"s{s}u{u}."
            stride = 2 if (u == 0 and s > 0) else 1
            Ho = (Hc - 1) // stride + 1
            k1, k2, k3 = need_conv(1, 1, 0), need_conv(3, stride, 1), need_conv(1, 1, 0)
            tensor(p + "W1", (mid, 1, 1, c), "bf16", "weight", fan_in=c)
            tensor(p + "W2", (mid, 3, 3, mid), "bf16", "weight", fan_in=9 * mid)
            tensor(p + "W3", (outc, 1, 1, mid), "bf16", "weight", fan_in=mid)
            tensor(p + "Z1", (batch, Hc, Hc, mid), "bf16", "act")
            tensor(p + "H1", (batch, Hc, Hc, mid), "bf16", "act")
            tensor(p + "Z2", (batch, Ho, Ho, mid), "bf16", "act")
            tensor(p + "H2", (batch, Ho, Ho, mid), "bf16", "act")
            tensor(p + "Z3", (batch, Ho, Ho, outc), "bf16", "act")
            tensor(p + "O", (batch, Ho, Ho, outc), "bf16", "act")
            op(p + "conv1", "conv_" + k1, [x, p + "W1"], p + "Z1")
            op(p + "relu1", "relu4", [p + "Z1"], p + "H1")
            op(p + "conv2", "conv_" + k2, [p + "H1", p + "W2"], p + "Z2")
            op(p + "relu2", "relu4", [p + "Z2"], p + "H2")
            op(p + "conv3", "conv_" + k3, [p + "H2", p + "W3"], p + "Z3")
            proj = u == 0
            if proj:
                kp = need_conv(1, stride, 0)
                tensor(p + "Wp", (outc, 1, 1, c), "bf16", "weight", fan_in=c)
                tensor(p + "P", (batch, Ho, Ho, outc), "bf16", "act")
                op(p + "proj", "conv_" + kp, [x, p + "Wp"], p + "P")
                sc = p + "P"
            else:
                sc = x
            op(p + "add", "addrelu", [p + "Z3", sc], p + "O")
            fwd_units.append((p, x, c, Hc, mid, outc, stride, Ho, proj))
            x, c, Hc = p + "O", outc, Ho
    defs["gap"] = (f"def gap(X(4)) -> lambda b, c: reduce(Sum; y, x; X[b, y, x, c] * {_num(1.0 / (Hc * Hc))})")
    defs["gap_grad"] = f"def gap_grad(D(2)) -> lambda b, y, x, c: D[b, c] * {_num(1.0 / (Hc * Hc))}"
    tensor("gap.Y", (batch, c), "bf16", "act")
    op("gap", "gap", [x], "gap.Y", attrs={"scale": 1.0 / (Hc * Hc)})
    tensor("fc.W", (c, classes), "bf16", "weight")
    tensor("Y", (batch, classes), "bf16", "act")
    op("fc", "mm_nn", ["gap.Y", "fc.W"], "Y")
    n_out = batch * classes
    defs["mse_grad"] = f"def mse_grad(Y(2), T(2)) -> lambda i, j: (Y[i, j] - T[i, j]) * {_num(2.0 / n_out)}"
    defs["sumsq"] = (f"def sumsq(Y(2), T(2)) -> lambda : reduce(Sum; i, j; "
                     f"(Y[i, j] - T[i, j]) * (Y[i, j] - T[i, j]) * {_num(1.0 / n_out)})")
    tensor("T", (batch, classes), "bf16", "input")
    tensor("loss", (), "f32", "loss")
    tensor("dY", (batch, classes), "bf16", "grad", grad_of="Y")
    op("loss", "sumsq", ["Y", "T"], "loss", attrs={"scale": 1.0 / n_out})
    op("loss_grad", "mse_grad", ["Y", "T"], "dY", attrs={"scale": 2.0 / n_out})
    # ------------------------------------------------------------------ backward
    wgrads = []   # (weight, grad)
    tensor("gap.dY", (batch, c), "bf16", "grad", grad_of="gap.Y")
    op("fc_dgrad", "mm_nt", ["dY", "fc.W"], "gap.dY", backward_of="fc")
    tensor("fc.dW", (c, classes), "f32", "grad", grad_of="fc.W")
    op("fc_wgrad", "mm_tn", ["gap.Y", "dY"], "fc.dW", backward_of="fc")
    wgrads.append(("fc.W", "fc.dW"))
    dx = x + ".d"
    tensor(dx, (batch, Hc, Hc, c), "bf16", "grad", grad_of=x)
    op("gap_bwd", "gap_grad", ["gap.dY"], dx, backward_of="gap", attrs={"scale": 1.0 / (Hc * Hc)})
    for (p, xin, cin_u, Hin, mid, outc, stride, Ho, proj) in reversed(fwd_units):
        k1, k2, k3 = f"k1s1p0", f"k3s{stride}p1", "k1s1p0"
        dO = p + "O.d"
        tensor(p + "dS", (batch, Ho, Ho, outc), "bf16", "grad", grad_of=p + "Z3")
        op(p + "add_bwd", "relu_grad4", [p + "O", dO], p + "dS", backward_of=p + "add")
        tensor(p + "dH2", (batch, Ho, Ho, mid), "bf16", "grad", grad_of=p + "H2")
        op(p + "conv3_dgrad", "dconv_" + k3, [p + "dS", p + "W3"], p + "dH2", backward_of=p + "conv3")
        tensor(p + "dW3", (outc, 1, 1, mid), "f32", "grad", grad_of=p + "W3")
        op(p + "conv3_wgrad", "wconv_" + k3, [p + "dS", p + "H2"], p + "dW3", backward_of=p + "conv3")
        tensor(p + "dZ2", (batch, Ho, Ho, mid), "bf16", "grad", grad_of=p + "Z2")
        op(p + "relu2_bwd", "relu_grad4", [p + "H2", p + "dH2"], p + "dZ2", backward_of=p + "relu2")
        tensor(p + "dH1", (batch, Hin, Hin, mid), "bf16", "grad", grad_of=p + "H1")
        rng2 = {"ty": 2, "tx": 2} if stride == 2 else None
        op(p + "conv2_dgrad", "dconv_" + k2, [p + "dZ2", p + "W2"], p + "dH1", backward_of=p + "conv2",
           ranges=rng2)
        tensor(p + "dW2", (mid, 3, 3, mid), "f32", "grad", grad_of=p + "W2")
        op(p + "conv2_wgrad", "wconv_" + k2, [p + "dZ2", p + "H1"], p + "dW2", backward_of=p + "conv2")
        tensor(p + "dZ1", (batch, Hin, Hin, mid), "bf16", "grad", grad_of=p + "Z1")
        op(p + "relu1_bwd", "relu_grad4", [p + "H1", p + "dH1"], p + "dZ1", backward_of=p + "relu1")
        tensor(p + "dXm", (batch, Hin, Hin, cin_u), "bf16", "grad")
        op(p + "conv1_dgrad", "dconv_" + k1, [p + "dZ1", p + "W1"], p + "dXm", backward_of=p + "conv1")
        tensor(p + "dW1", (mid, 1, 1, cin_u), "f32", "grad", grad_of=p + "W1")
        op(p + "conv1_wgrad", "wconv_" + k1, [p + "dZ1", xin], p + "dW1", backward_of=p + "conv1")
        dxin = xin + ".d"
        tensor(dxin, (batch, Hin, Hin, cin_u), "bf16", "grad", grad_of=xin)
        if proj:
            kp = f"k1s{stride}p0"
            tensor(p + "dXp", (batch, Hin, Hin, cin_u), "bf16", "grad")
            op(p + "proj_dgrad", "dconv_" + kp, [p + "dS", p + "Wp"], p + "dXp", backward_of=p + "proj",
               ranges={"ty": 1, "tx": 1} if stride == 2 else None)
            tensor(p + "dWp", (outc, 1, 1, cin_u), "f32", "grad", grad_of=p + "Wp")
            op(p + "proj_wgrad", "wconv_" + kp, [p + "dS", xin], p + "dWp", backward_of=p + "proj")
            op(p + "dx_sum", "add4", [p + "dXm", p + "dXp"], dxin, backward_of=p + "add")
            wgrads.append((p + "Wp", p + "dWp"))
        else:
            op(p + "dx_sum", "add4", [p + "dXm", p + "dS"], dxin, backward_of=p + "add")
        wgrads += [(p + "W3", p + "dW3"), (p + "W2", p + "dW2"), (p + "W1", p + "dW1")]
    tensor("stem.dH", (batch, H1, H1, c0), "bf16", "grad", grad_of="stem.H")
    op("pool_bwd", "maxpool_grad", ["stem.H", "pool.Y", "pool.Y.d", "pool.K"], "stem.dH", backward_of="pool",
       ranges={"ty": 2, "tx": 2})
    tensor("stem.dZ", (batch, H1, H1, c0), "bf16", "grad", grad_of="stem.Z")
    op("stem.relu_bwd", "relu_grad4", ["stem.H", "stem.dH"], "stem.dZ", backward_of="stem.relu")
    tensor("stem.dW", (c0, 7, 7, cin), "f32", "grad", grad_of="stem.W")
    op("stem.wgrad", "wconv_k7s2p3", ["stem.dZ", X], "stem.dW", backward_of="stem.conv")
    wgrads.append(("stem.W", "stem.dW"))
    # ------------------------------------------------------------------ optimizer (SGD with momentum)
    defs["mom"] = f"def mom(M(2), G(2)) -> lambda i, j: M[i, j] * {_num(mu)} + G[i, j]"
    defs["sgd"] = f"def sgd(W(2), M(2)) -> lambda i, j: W[i, j] - M[i, j] * {_num(lr)}"
    defs["mom4"] = f"def mom4(M(4), G(4)) -> lambda a, b, c, d: M[a, b, c, d] * {_num(mu)} + G[a, b, c, d]"
    defs["sgd4"] = f"def sgd4(W(4), M(4)) -> lambda a, b, c, d: W[a, b, c, d] - M[a, b, c, d] * {_num(lr)}"
    for w, g in wgrads:
        shp = T[w]["shape"]
        r = "4" if len(shp) == 4 else ""
        m = w[:-1] + "M" + w[-1] if w.endswith(("1", "2", "3", "p")) else w + ".M"
        m = w + ".M"
        tensor(m, shp, "f32", "state")
        tensor(m + "_new", shp, "f32", "state")
        tensor(w + "_new", shp, "bf16", "weight")
        op(w + ".mom", "mom" + r, [m, g], m + "_new", attrs={"mu": mu})
        op(w + ".sgd", "sgd" + r, [w, m + "_new"], w + "_new", attrs={"lr": lr})
        alias[m + "_new"] = m
        alias[w + "_new"] = w
    used = {o["def"] for o in ops}
    return {"defs": {k_: v for k_, v in defs.items() if k_ in used}, "tensors": T, "ops": ops, "alias": alias,
            "meta": {"samples_per_step": batch}}


def wresnet_depth(L: int, width: int, batch: int, image: int = 224) -> dict:
    return wresnet(WRN_UNITS[L], width, batch, image)


CONFIG_K[3] = 8
CONFIG_NAME[3] = "wresnet-152-4-b32"

CONFIG_K[4] = 8
CONFIG_NAME[4] = "lstm-10x8192-T20-b128"
CONFIG_K[5] = 8
CONFIG_NAME[5] = "wresnet-152-10-b32"
