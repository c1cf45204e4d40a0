"""Workload graph descriptions (the input of tofu_plan / tofu_execute).

Each builder returns the graph JSON dict documented in oracle/graph.py and
include/tofu.h: TDL defs (text), tensors with shapes/dtypes/roles, ops in
execution order (forward, loss, backward, optimizer) and in-place aliases.
Constants of the elementwise defs (loss scale, learning rate, momentum) are
powers of two or dyadic so every side represents them exactly.

Workloads follow BASELINE.json configs:
  configs[0]  mlp(64, [256, 512, 512])          2-layer MLP, k = 2
  configs[1]  mlp(512, [8192, 8192])            single large FC layer, k = 8
  configs[2]  lstm(...)                          (next round)
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
    return {"defs": defs, "tensors": T, "ops": ops, "alias": alias}


def config(i: int) -> dict:
    if i == 0:
        return mlp(64, [256, 512, 512])
    if i == 1:
        return mlp(512, [8192, 8192])
    raise ValueError(f"config {i} not built yet")


CONFIG_K = {0: 2, 1: 8}
CONFIG_NAME = {0: "mlp-2x512-b64", 1: "fc-8192x8192-b512"}
