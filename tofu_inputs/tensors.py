"""Seeded synthetic tensors for a graph's inputs, weights and state.

Every value drawn here is exactly representable in bf16 (a signed 8-bit
integer times a power of two), so both sides start from bit-identical
operands without any rounding code.  Recipes:

  input  X : q * 2^-7                    q ~ U{-128..128}
  input  T : q * 2^-8
  weight W : q * 2^-7 * 2^-round(log2(sqrt(fan_in)))   (He-like scale)
  state  M : q * 2^-17                    (non-zero so momentum is exercised)
  mode="int": all of the above replaced by q ~ U{-3..3} (exact fp64 sums,
              used for partitioned-vs-unpartitioned equality tests)
  mode="bf16": full-mantissa values — u ~ U(-1, 1) continuous, scaled as above (X: u, T: u/2,
              W: u * 2^-round(log2(sqrt(fan_in))), M: u * 2^-10), then rounded to the tensor's storage
              dtype (bf16: round-to-nearest-even on the fp32 bit pattern; f32: cast), so every mantissa
              bit is live and fp32 accumulation is not exact
  tensors with "init": "zeros" (initial recurrent state, zero gradients) are zero, "ones" are one
  a tensor's "fan_in" overrides shape[0] (convolution weights [co, ky, kx, ci]: ky*kx*ci)
  an input's "live_channels" n zeroes its last dim from n on (an RGB image padded to 8 channels)
"""
from __future__ import annotations

import math

import numpy as np


def _q(rng, shape, lo=-128, hi=128):
    return rng.integers(lo, hi + 1, size=shape).astype(np.float64)


def _to_storage(x, dtype):
    """fp64 -> the storage dtype's value set (an input generator step, not method arithmetic)."""
    f = np.asarray(x, np.float64).astype(np.float32)
    if dtype != "bf16":
        return f.astype(np.float64)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32).astype(np.float64)


def make_values(graph: dict, seed: int = 0, mode: str = "float") -> dict:
    rng = np.random.default_rng(seed)
    out = {}
    for name in sorted(graph["tensors"]):
        t = graph["tensors"][name]
        role = t["role"]
        shape = tuple(t["shape"])
        if role not in ("input", "weight", "state") or name in graph.get("alias", {}):
            continue
        if t.get("init") == "zeros":
            out[name] = np.zeros(shape)
            continue
        if t.get("init") == "ones":
            out[name] = np.ones(shape)
            continue
        if mode == "int":
            out[name] = _q(rng, shape, -3, 3)
            continue
        if mode == "bf16":
            u = rng.uniform(-1.0, 1.0, size=shape)
            if role == "input":
                u = u * (1.0 if name != "T" else 0.5)
                if t.get("live_channels") is not None:
                    u[..., int(t["live_channels"]):] = 0.0
            elif role == "weight":
                u = u * 2.0 ** -round(math.log2(math.sqrt(int(t.get("fan_in") or shape[0]))))
            else:
                u = u * 2.0 ** -10
            out[name] = _to_storage(u, t.get("dtype", "f32"))
            continue
        if role == "input":
            out[name] = _q(rng, shape) * (2.0 ** -7 if name != "T" else 2.0 ** -8)
            if t.get("live_channels") is not None:   # channel padding of an image (last dim) is zero
                out[name][..., int(t["live_channels"]):] = 0.0
        elif role == "weight":
            fan_in = int(t.get("fan_in") or shape[0])
            s = round(math.log2(math.sqrt(fan_in)))
            out[name] = _q(rng, shape) * 2.0 ** (-7 - s)
        else:
            out[name] = _q(rng, shape) * 2.0 ** -17
    return out


def make_values_device(graph: dict, seed: int = 0, device="cuda", names=None):
    """The same recipes drawn with torch's generator on the device (for models whose parameters would not
    fit in host memory as float64; used by bench.py for the largest configs).  Yields (name, tensor)."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    for name in sorted(graph["tensors"]):
        t = graph["tensors"][name]
        role = t["role"]
        shape = tuple(t["shape"])
        if role not in ("input", "weight", "state") or name in graph.get("alias", {}):
            continue
        if names is not None and name not in names:
            continue
        if t.get("init") == "zeros":
            yield name, torch.zeros(shape, device=device)
            continue
        if t.get("init") == "ones":
            yield name, torch.ones(shape, device=device)
            continue
        q = torch.randint(-128, 129, shape, generator=gen, device=device).float()
        if role == "input":
            q *= 2.0 ** -7 if name != "T" else 2.0 ** -8
            if t.get("live_channels") is not None:
                q[..., int(t["live_channels"]):] = 0.0
        elif role == "weight":
            fan_in = int(t.get("fan_in") or shape[0])
            q *= 2.0 ** (-7 - round(math.log2(math.sqrt(fan_in))))
        else:
            q *= 2.0 ** -17
        yield name, q


def make_value_device(graph: dict, name: str, seed: int = 0, device="cuda"):
    """One tensor of the recipes above (float32, on `device`) drawn from its OWN generator, seeded by (seed, the
    tensor's name) — so any single tensor can be regenerated on demand (the parity tests of the largest
    configs, whose parameters fit neither host memory as float64 nor a second device copy).  Returns None for
    tensors that are not inputs / weights / state."""
    import hashlib

    import torch
    t = graph["tensors"][name]
    role = t["role"]
    shape = tuple(t["shape"])
    if role not in ("input", "weight", "state") or name in graph.get("alias", {}):
        return None
    if t.get("init") == "zeros":
        return torch.zeros(shape, device=device)
    if t.get("init") == "ones":
        return torch.ones(shape, device=device)
    h = int.from_bytes(hashlib.sha256(f"{seed}:{name}".encode()).digest()[:8], "little") & ((1 << 63) - 1)
    gen = torch.Generator(device=device)
    gen.manual_seed(h)
    q = torch.randint(-128, 129, shape, generator=gen, device=device).float()
    if role == "input":
        q *= 2.0 ** -7 if name != "T" else 2.0 ** -8
        if t.get("live_channels") is not None:
            q[..., int(t["live_channels"]):] = 0.0
    elif role == "weight":
        fan_in = int(t.get("fan_in") or shape[0])
        q *= 2.0 ** (-7 - round(math.log2(math.sqrt(fan_in))))
    else:
        q *= 2.0 ** -17
    return q
