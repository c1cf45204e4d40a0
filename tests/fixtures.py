"""Random tiny graph fixtures for oracle property tests (test-only)."""
import random

from tofu_inputs.graphs import MM_DEFS

EW = {
    "add": "def add(A(2), B(2)) -> lambda i, j: A[i, j] + B[i, j]",
    "relu": "def relu(X(2)) -> lambda i, j: max(X[i, j], 0)",
}


def random_chain(seed, n_ops=None, dims=(2, 4, 8)):
    """A random fork-free chain of matmul / element-wise ops over 2-D
    tensors; every op output feeds the next op.  Halo-free (Assumption #2)."""
    rng = random.Random(seed)
    n_ops = n_ops or rng.randint(1, 4)
    defs = dict(MM_DEFS)
    defs.update(EW)
    T, ops = {}, []
    cnt = [0]

    def new(shape, role="act"):
        cnt[0] += 1
        name = f"t{cnt[0]}"
        T[name] = {"shape": list(shape), "dtype": "f32", "role": role, "grad_of": None, "merge": None}
        return name

    cur = new((rng.choice(dims), rng.choice(dims)), "input")
    for i in range(n_ops):
        m, n = T[cur]["shape"]
        kind = rng.choice(["mm_nn", "mm_nt", "mm_tn", "add", "relu"])
        p = rng.choice(dims)
        if kind == "mm_nn":
            w = new((n, p), "weight"); out = new((m, p)); ins = [cur, w]
        elif kind == "mm_nt":
            w = new((p, n), "weight"); out = new((m, p)); ins = [cur, w]
        elif kind == "mm_tn":
            w = new((m, p), "weight"); out = new((n, p)); ins = [cur, w]
        elif kind == "add":
            w = new((m, n), "weight"); out = new((m, n)); ins = [cur, w]
        else:
            out = new((m, n)); ins = [cur]
        ops.append({"name": f"op{i}", "def": kind, "inputs": ins, "output": out,
                    "backward_of": None, "merge": None})
        cur = out
    used = {o["def"] for o in ops}
    return {"defs": {k: v for k, v in defs.items() if k in used}, "tensors": T, "ops": ops, "alias": {}}
