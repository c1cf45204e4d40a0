"""Partitioned training-step runner over libtofu (device memory plumbing only).

``TofuRunner(spec, k)`` plans the graph for k workers (tofu_plan), allocates
one arena per local rank (torch device memory), loads tensors into the ranks'
shards at the offsets libtofu reports, and runs steps through tofu_execute.

* virtual mode (default): all k ranks live on one GPU; peer pointers are
  local pointers and the same MultiFetch / reduce kernels run.
* multi-process mode (``rank``/``group`` given): one process per GPU; each
  rank's arena (+ barrier words) is exported with CUDA IPC and mapped by its
  peers; the mapped addresses are passed to libtofu, whose kernels then read
  peer HBM over NVLink directly.
"""
from __future__ import annotations

import os

import numpy as np

import torch

from . import tofu

_TD = {"bf16": torch.bfloat16, "f32": torch.float32}


class TofuRunner:
    def __init__(self, spec: dict, k: int, device="cuda", rank: int | None = None, group=None, plan_opts=None):
        self.spec = spec
        self.k = k
        self.device = torch.device(device)
        self.graph = tofu.Graph(spec)
        self.plan = tofu.Plan(self.graph, k, **(plan_opts or {}))
        self.plan_json = self.plan.json()
        self.multi = rank is not None
        self.local = [rank] if self.multi else list(range(k))
        self.arenas = {}
        self._symm = None
        if not self.multi:
            for r in self.local:
                n = max(256, self.plan.arena_bytes(r))
                self.arenas[r] = torch.zeros(n + 256, dtype=torch.uint8, device=self.device)
            ptrs = [self._aligned(self.arenas[r]) for r in range(k)]
            self.exec = tofu.Exec(self.graph, self.plan, self.local, ptrs)
        else:
            # one process per GPU: every rank allocates its own arena (+ 4 KiB of barrier words) and
            # exports it with CUDA IPC (tofu_ipc_export); each peer maps it on ITS OWN device with peer access
            # enabled explicitly (tofu_ipc_open), so libtofu's MultiFetch / reduce kernels load peer HBM
            # directly over NVLink.
            import torch.distributed as dist
            nbytes = (max(self.plan.arena_bytes(r) for r in range(k)) + 4095) // 4096 * 4096
            buf = torch.zeros(nbytes + 4096, dtype=torch.uint8, device=self.device)
            self.arenas[rank] = buf
            torch.cuda.synchronize()
            dev = self.device.index if self.device.index is not None else torch.cuda.current_device()
            handle, off = tofu.ipc_export(buf.data_ptr())
            handles = [None] * k
            dist.all_gather_object(handles, (rank, dev, handle, off), group=group)
            self._peer = {}
            ptrs = [0] * k
            for r, pdev, h, o in handles:
                if r == rank:
                    ptrs[r] = buf.data_ptr()
                else:
                    ptrs[r] = tofu.ipc_open(h, o, dev, pdev)
                    self._peer[r] = (ptrs[r], o)
            flags = [p + nbytes for p in ptrs]
            dist.barrier(group=group)
            self.exec = tofu.Exec(self.graph, self.plan, self.local, ptrs, flags)
        self.shards = {r: {t: self.plan.shard(r, t) for t in spec["tensors"]} for r in range(k)}

    def __del__(self):
        peers = getattr(self, "_peer", None)
        if not peers:
            return
        try:
            torch.cuda.synchronize()
            self.exec = None
            for ptr, off in peers.values():
                tofu.ipc_close(ptr, off)
        except Exception:
            pass
        self._peer = {}

    @staticmethod
    def _aligned(t):
        p = t.data_ptr()
        return (p + 255) // 256 * 256

    def _base(self, r):
        return self._aligned(self.arenas[r]) if not self.multi else self.arenas[r].data_ptr()

    def view(self, r: int, name: str) -> torch.Tensor | None:
        """The shard of tensor `name` held by rank r, as a torch view into the arena."""
        off, box = self.shards[r][name]
        if off < 0 or r not in self.arenas:
            return None
        info = self.spec["tensors"][name]
        dt = _TD[info["dtype"]]
        shape = [hi - lo + 1 for lo, hi in box]
        n = int(np.prod(shape)) if shape else 1
        arena = self.arenas[r]
        start = self._base(r) - arena.data_ptr() + off
        es = 2 if dt == torch.bfloat16 else 4
        return arena[start:start + n * es].view(dt).view(shape if shape else [])

    def load(self, values: dict):
        """Copy full tensors (numpy or torch, host or device) into every local rank's shards."""
        for name, v in values.items():
            src = torch.as_tensor(np.asarray(v)) if not torch.is_tensor(v) else v
            for r in self.local:
                dst = self.view(r, name)
                if dst is None:
                    continue
                _, box = self.shards[r][name]
                sl = tuple(slice(lo, hi + 1) for lo, hi in box)
                dst.copy_(src[sl].to(dst.dtype), non_blocking=True)

    def gather(self, name: str) -> torch.Tensor:
        """Assemble a full tensor from the local ranks' shards (virtual mode: all ranks)."""
        info = self.spec["tensors"][name]
        full = torch.empty(info["shape"], dtype=_TD[info["dtype"]], device=self.device)
        for r in self.local:
            v = self.view(r, name)
            if v is None:
                continue
            _, box = self.shards[r][name]
            sl = tuple(slice(lo, hi + 1) for lo, hi in box)
            full[sl] = v
        return full

    def step(self, stream=None):
        if getattr(self, "_graph", None) is not None:
            self._graph.replay()
        else:
            self.exec.run(stream)

    def capture(self):
        """Capture one step (all of its kernel launches) into a CUDA graph; later step() calls replay it.
        Run at least one eager step first (one-time kernel attribute setup happens outside capture)."""
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.exec.run()
        torch.cuda.synchronize()
        self._graph = g
        return g

    def uncapture(self):
        self._graph = None

    def ledger(self):
        return self.exec.ledger()

    def train(self, host_batches, steps: int, result: str = "loss", start_event=None):
        """End-to-end training loop through the public API: every step copies that step's inputs from
        pinned host memory into the ranks' shards and reads the step's `result` back to the host.
        The host->device copy of step s+1 runs on two copy streams while step s computes (double-buffered
        device staging); the result is read back asynchronously into pinned memory.

        host_batches: callable s -> {name: pinned host tensor (full shape)}.  Returns the pinned host
        tensor of per-step results (valid after the caller synchronises)."""
        comp = torch.cuda.current_stream()
        # two copy streams: one host->device stream reached ~27 GB/s on the B200 boxes, two ~51 GB/s
        # (tools/h2d_bench.py); every input is split in row halves across them
        copies = [torch.cuda.Stream() for _ in range(int(os.environ.get("TOFU_COPY_STREAMS", "2")))]
        names = list(host_batches(0).keys())
        slots = [(r, n) for r in self.local for n in names if self.view(r, n) is not None]
        bufs = [{s: torch.empty_like(self.view(*s)) for s in slots} for _ in range(2)]
        ready = [[torch.cuda.Event() for _ in copies] for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]
        used = [False, False]
        res_view = None
        for r in self.local:
            res_view = self.view(r, result) if res_view is None else res_view
        out = torch.empty([steps] + (list(res_view.shape) if res_view is not None else []),
                          dtype=res_view.dtype if res_view is not None else torch.float32).pin_memory()
        for c in copies:
            if start_event is not None:
                c.wait_event(start_event)
            else:
                c.wait_stream(comp)

        def issue(s):
            b = s % 2
            hb = host_batches(s)
            for ci, c in enumerate(copies):
                with torch.cuda.stream(c):
                    if used[b]:
                        c.wait_event(free[b])
                    for (r, n) in slots:
                        _, box = self.shards[r][n]
                        sl = tuple(slice(lo, hi + 1) for lo, hi in box)
                        src, dst = hb[n][sl], bufs[b][(r, n)]
                        if dst.dim() == 0:
                            if ci == 0:
                                dst.copy_(src, non_blocking=True)
                            continue
                        nc = len(copies)   # row blocks, one per copy stream
                        h = (dst.shape[0] + nc - 1) // nc
                        part = slice(min(ci * h, dst.shape[0]), min((ci + 1) * h, dst.shape[0]))
                        dst[part].copy_(src[part], non_blocking=True)
                    ready[b][ci].record(c)
            used[b] = True

        issue(0)
        for s in range(steps):
            b = s % 2
            if s + 1 < steps:
                issue(s + 1)
            for ev in ready[b]:
                comp.wait_event(ev)
            for sl in slots:
                self.view(*sl).copy_(bufs[b][sl], non_blocking=True)
            free[b].record(comp)
            self.step()
            if res_view is not None:
                out[s].copy_(res_view, non_blocking=True)
        return out
