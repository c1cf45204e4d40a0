"""Benchmark: Tofu-partitioned training step on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--impl reference]

One JSON line on rank 0.  N = 1 runs the workload unpartitioned on one GPU; N > 1 (torchrun, one
process per GPU) partitions every tensor k = N ways with tofu_plan and runs the partitioned step
through tofu_execute (MultiFetch / partition-n-reduce kernels reading peer HBM over NVLink).
The global batch is fixed as N grows (strong scaling, as in the paper: one model split over GPUs).
``--impl reference`` times the oracle (the CPU reference implementation) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from tofu_inputs.graphs import CONFIG_NAME, config  # noqa: E402
from tofu_inputs.tensors import make_values  # noqa: E402

METRIC = "samples/sec per training step"
NVLINK_GBS = 900.0   # NVLink 5 per direction per GPU (north star; B200_PROFILING.md)
CLOCK_Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
           "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
           "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={CLOCK_Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) > 8:
                for n, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def nvlink_counters(index):
    """(tx bytes, rx bytes) summed over the NVLink links of GPU `index` (nvidia-smi nvlink -gt d: cumulative data
    counters), or None when unavailable (no NVLink, no nvidia-smi)."""
    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(index)], capture_output=True, text=True,
                             timeout=20).stdout
    except Exception:
        return None
    unit = {"B": 1, "KiB": 1024, "MiB": 1024 ** 2, "GiB": 1024 ** 3}
    tx = rx = 0
    seen = False
    for line in out.splitlines():
        parts = line.replace(",", " ").split()
        for i, w in enumerate(parts):
            if w in ("Tx:", "Rx:") and i + 2 < len(parts) + 1 and i + 1 < len(parts):
                try:
                    v = float(parts[i + 1]) * unit.get(parts[i + 2] if i + 2 < len(parts) else "KiB", 1024)
                except ValueError:
                    continue
                seen = True
                if w == "Tx:":
                    tx += v
                else:
                    rx += v
    return (tx, rx) if seen else None


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


def oracle_step_time(spec, vals):
    from oracle.exec_ref import run_graph
    from oracle.graph import Graph
    g = Graph(spec)
    t = time.perf_counter()
    run_graph(g, vals, emulate_storage=True)
    return time.perf_counter() - t


def graph_work(spec):
    """Σ over ops of the iteration-space volume (multiply-adds of a contraction, elements otherwise): the
    oracle's work, used to extrapolate a bounded oracle sample to the full workload."""
    from oracle.graph import Graph
    g = Graph(spec)
    tot = 0
    for op in g.ops:
        v = 1
        for n in g.ranges[op["name"]].values():
            v *= n
        tot += v
    return tot


def oracle_sample(cfg):
    """(sample spec, full-workload samples represented per sample step, description) of the bounded CPU
    oracle run for workload cfg: about 10-30 s of fp64 work on the host cores."""
    full = config(cfg)
    batch = full.get("meta", {}).get("samples_per_step", full["tensors"]["X"]["shape"][0])
    if cfg == 2:
        from tofu_inputs.graphs import lstm
        spec = lstm(1, 4096, 20, 1)   # 1 of 6 layers, 1 sequence: 1/6 of a sequence's work
        return spec, 1.0 / 6.0, "1 LSTM layer (of 6), batch 1 sequence of 20 steps, fp64; samples/s = 1/(6 t)"
    if cfg in (3, 4, 5):
        from tofu_inputs.graphs import lstm, wresnet
        # cfg 3/5: stem + first bottleneck unit at full width, 1 image; cfg 4: one LSTM layer, 1 sequence
        spec = {3: lambda: wresnet([1], 4, 1, 224), 4: lambda: lstm(1, 8192, 2, 1),
                5: lambda: wresnet([1], 10, 1, 112)}[cfg]()
        frac = graph_work(spec) / (graph_work(full) / batch)
        what = {3: "WResNet-152-4 stem + first bottleneck unit, 1 image",
                4: "1 LSTM layer (of 10), 1 sequence of 2 steps (of 20)",
                5: "WResNet-152-10 stem + first bottleneck unit, 1 image at 112x112"}[cfg]
        return spec, frac, (f"{what}, fp64; extrapolated to the full network by iteration-space work (this sample "
                            f"= {frac:.4f} of a sample)")
    # MLP / FC: the whole training step of the workload itself (a few seconds of fp64 work)
    return full, float(batch), f"1 full training step of {CONFIG_NAME[cfg]} (batch {batch}), fp64"


def reference_arm(args, world, rank):
    """--impl reference: the oracle (fp64 CPU) on the host cores, rank 0 only."""
    if rank != 0:
        return
    spec, per_step, sample = oracle_sample(args.config)
    full = config(args.config)
    full_batch = full.get("meta", {}).get("samples_per_step", full["tensors"]["X"]["shape"][0])
    vals = make_values(spec, seed=0)
    for _ in range(args.warmup):
        oracle_step_time(spec, vals)
    ts = [oracle_step_time(spec, vals) for _ in range(args.steps)]
    t = sum(ts) / len(ts)
    v = per_step / t
    sb = per_step
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_NAME[args.config], "global_batch": full_batch, "parallelism": "cpu",
                       "oracle_samples_per_step": sb},
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cpu_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def virtual_partitioned(spec, vals, k, steps, k1_value=None):
    """The k-way partitioned step with all k ranks as virtual ranks on this one GPU: the same
    MultiFetch / reduce / sub-op kernels (peer pointers are local).  Not a scaling number — the k ranks
    run one after another on one device — but it exercises and times the partitioned path and its
    byte ledger on real hardware, and (total / k) is a proxy of one rank's step time, compared with the
    per-rank roofline: max(the busiest rank's flops at the tensor peak, its max(in, out) NVLink bytes at
    900 GB/s).  "ideal" = k x the k = 1 throughput (the paper's Ideal baseline)."""
    import torch
    from paper_1807_08887_b200.runner import TofuRunner
    R = TofuRunner(spec, k)
    if vals is None:   # the largest configs: each tensor regenerated on the device (tofu_inputs.make_value_device)
        from tofu_inputs.tensors import make_value_device
        for name in sorted(spec["tensors"]):
            v = make_value_device(spec, name, seed=0)
            if v is not None:
                R.load({name: v})
                del v
    else:
        R.load(vals)
    ex = R.exec
    for _ in range(3):
        ex.run()
    torch.cuda.synchronize()
    # timed as a CUDA-graph replay, as the k = 1 line (the ~6500 launches of an 8-way step issued one by one
    # from Python leave the host, not the GPU, on the critical path for stretches)
    graphed = True
    try:
        R.capture()
        for _ in range(3):
            R.step()
    except Exception:  # noqa: BLE001  (capture unavailable: eager launches)
        graphed = False
        R.uncapture()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        R.step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    R.uncapture()
    nl = ex.num_launches()
    descs = [ex.launch_desc(i) for i in range(nl)]
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)]
    evs[0].record()
    for i in range(nl):
        ex.run_range(i, i + 1)
        evs[i + 1].record()
    torch.cuda.synchronize()
    per = [evs[i].elapsed_time(evs[i + 1]) for i in range(nl)]
    comm_ms = sum(per[i] for i in range(nl) if descs[i]["kind"] in ("fetch", "reduce"))
    comm_bytes = sum(descs[i]["bytes"] for i in range(nl) if descs[i]["kind"] in ("fetch", "reduce"))
    by_kind, by_def, by_rank = {}, {}, {}
    flops_rank = {}
    for d, t in zip(descs, per):
        by_kind[d["kind"]] = by_kind.get(d["kind"], 0.0) + t
        key = d["def"] if d["kind"] == "compute" else d["kind"]
        by_def[key] = by_def.get(key, 0.0) + t
        r = d.get("rank", -1)
        by_rank[r] = by_rank.get(r, 0.0) + t
        if d["kind"] == "compute":
            flops_rank[r] = flops_rank.get(r, 0.0) + d["flops"]
    pk = peaks()
    io = [ex.rank_bytes(r) for r in range(k)]
    t_comp = max(flops_rank.values(), default=0.0) / (pk["bf16_tflops_sustained"] * 1e12)
    t_comm = max(max(x, y) for x, y in io) / NVLINK_GBS / 1e9
    roof_ms = max(t_comp, t_comm) * 1e3
    pe, pb = R.plan.cost()
    le, lb = R.ledger()
    out = {"k": k, "ranks": "virtual (all on one GPU)", "ms_per_step": ms, "cuda_graph": graphed, "plan_factors": R.plan_json["factors"],
           "plan_search": R.plan_json.get("search"),
           "plan_bytes": pb, "ledger_bytes": lb, "plan_elements": pe, "ledger_elements": le, "equal": pb == lb,
           "comm_kernels_ms": comm_ms, "comm_kernels_GBps": comm_bytes / (comm_ms / 1e3) / 1e9 if comm_ms else None,
           "launches_per_step": ex.launches(),
           "per_rank_ms_proxy": ms / k,
           "per_rank_roofline_ms": roof_ms,
           "per_rank_roofline": {"compute_ms": t_comp * 1e3, "nvlink_ms": t_comm * 1e3,
                                 "busiest_rank_in_out_bytes": max(max(x, y) for x, y in io)},
           "frac_per_rank": roof_ms / (ms / k) if ms else None,
           "breakdown_ms": {kk: round(v, 4) for kk, v in sorted(by_kind.items(), key=lambda kv: -kv[1])},
           "rank_ms": {str(r): round(v, 4) for r, v in sorted(by_rank.items())},
           "top_defs_ms": dict(sorted(((kk, round(v, 4)) for kk, v in by_def.items()), key=lambda kv: -kv[1])[:10])}
    if k1_value:
        out["ideal_samples_s"] = k * k1_value
    del R
    torch.cuda.empty_cache()
    return out


def run_workload(cfg, args, steps, world, rank, local_rank, group, shared, virtual_k, with_cpu):
    """One workload: instrumented pass, warmup, timed region (device events, max over ranks), end-to-end
    loop through TofuRunner.train, roofline objects.  Returns the JSON line (dict)."""
    import torch
    import torch.distributed as dist
    from paper_1807_08887_b200.runner import TofuRunner

    def all_reduce(t, op):
        if shared:
            c = t.cpu()
            dist.all_reduce(c, op=op)
            t.copy_(c)
        else:
            dist.all_reduce(t, op=op)

    spec = config(cfg)
    k = world
    big = cfg >= 4   # parameters drawn on the device (float64 host copies would not fit in RAM)
    vp_big = None
    if big and world == 1 and virtual_k > 1:   # the k-way plan first: both runners' arenas do not fit at once
        vp_big = virtual_partitioned(spec, None, virtual_k, max(steps, 5))
    vals = None if big else make_values(spec, seed=0)
    if world > 1:
        R = TofuRunner(spec, k, rank=rank, group=group)
    else:
        R = TofuRunner(spec, 1)
    if big:
        from tofu_inputs.tensors import make_values_device
        for name, v in make_values_device(spec, seed=0):
            R.load({name: v})
            del v
        vals = {n: v.cpu().numpy() for n, v in make_values_device(spec, seed=0, names=("X", "T"))}
    else:
        R.load(vals)
    ex = R.exec
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    # --- instrumented pass: per-launch device time (events between launches) -> dominant kernel
    nl = ex.num_launches()
    descs = [ex.launch_desc(i) for i in range(nl)]
    for _ in range(2):
        ex.run()
    per = [0.0] * nl
    reps = 3
    for _ in range(reps):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)]
        evs[0].record()
        for i in range(nl):
            ex.run_range(i, i + 1)
            evs[i + 1].record()
        torch.cuda.synchronize()
        for i in range(nl):
            per[i] += evs[i].elapsed_time(evs[i + 1]) / reps
    # dominant kernel: the kernel (def, or fetch / reduce) taking the largest share of the step; its longest
    # launch is the one timed live below
    cand = [i for i in range(nl) if descs[i]["kind"] in ("compute", "fetch", "reduce")]
    kkey = lambda i: descs[i]["def"] if descs[i]["kind"] == "compute" else descs[i]["kind"]
    share = {}
    for i in cand:
        share[kkey(i)] = share.get(kkey(i), 0.0) + per[i]
    top = max(share, key=share.get)
    dom = max((i for i in cand if kkey(i) == top), key=lambda i: per[i])
    dom_share = share[top] / max(sum(per), 1e-9)

    # --- warmup + timed region (inputs > L2: W 128 MiB + M 256 MiB + dW 256 MiB per step)
    for _ in range(args.warmup):
        ex.run()
    torch.cuda.synchronize()
    dom_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in dom_ev:   # torch creates the CUDA event lazily on first record; libtofu re-records them
        a.record(); b.record()
    torch.cuda.synchronize()
    # launch-bound steps (the RNN issues ~740 launches) are captured in a CUDA graph; libtofu records the
    # dominant kernel's events inside the graph, so every replay re-times it live
    use_graph = args.graph == "on" or (args.graph == "auto" and ex.launches() > 64)
    dom_a, dom_b = dom_ev[0]
    ex.time_launch(dom, dom_a, dom_b)
    if use_graph:
        R.capture()
    for _ in range(2):
        R.step()
    torch.cuda.synchronize()
    dom_samples = []
    soak_start = time.time()
    with ClockSampler(local_rank) as clk:
        barrier()
        torch.cuda.synchronize()
        nv0 = nvlink_counters(torch.cuda.current_device()) if world > 1 and not shared else None
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for s in range(steps):
            R.step()
        t1.record()
        torch.cuda.synchronize()
        nv1 = nvlink_counters(torch.cuda.current_device()) if nv0 is not None else None
        barrier()
        dom_samples.append(dom_a.elapsed_time(dom_b))   # last step of the timed region
        # keep the same step loop running (untimed) until nvidia-smi has >= 5 samples, so the clock
        # record covers this workload under load even when the timed region is only milliseconds
        # (every step holds device barriers across ranks: all ranks agree on each extra round, or they hang)
        deadline = time.time() + 3.0
        while True:
            more = (len(clk.rows) < 5 or time.time() < soak_start + 0.6) and time.time() < deadline
            if world > 1:
                flag = torch.tensor([1.0 if more else 0.0], device="cuda")
                all_reduce(flag, dist.ReduceOp.MAX)
                more = float(flag.item()) > 0
            if not more:
                break
            for _ in range(20):
                R.step()
            torch.cuda.synchronize()
            dom_samples.append(dom_a.elapsed_time(dom_b))
    R.uncapture()
    ex.time_launch(-1)
    ms = t0.elapsed_time(t1) / steps
    dom_ms = statistics.median(dom_samples)
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        all_reduce(tt, dist.ReduceOp.MAX)
        ms = float(tt.item())

    batch = spec.get("meta", {}).get("samples_per_step", spec["tensors"]["X"]["shape"][0])
    value = batch / (ms / 1e3)

    # --- end to end through the public API: H2D inputs (pinned) + step + D2H loss every step
    xs = {t: torch.from_numpy(np.asarray(vals[t], np.float32)).to(torch.bfloat16).pin_memory() for t in ("X", "T")}
    h2d = 0
    for t in ("X", "T"):
        for r in R.local:
            v = R.view(r, t)
            if v is not None:
                h2d += v.numel() * v.element_size()
    batches = lambda s: xs
    if use_graph:
        R.capture()
    R.train(batches, 2)
    torch.cuda.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    losses = R.train(batches, steps, start_event=e0)
    e1.record()
    torch.cuda.synchronize()
    barrier()
    R.uncapture()
    e2e_ms = e0.elapsed_time(e1) / steps
    if world > 1:
        tt = torch.tensor([e2e_ms, h2d], device="cuda", dtype=torch.float64)
        t0_ = tt[:1].clone()
        all_reduce(t0_, dist.ReduceOp.MAX)
        tt[:1] = t0_
        hh = tt[1:].clone()
        all_reduce(hh, dist.ReduceOp.SUM)
        e2e_ms, h2d = float(tt[0]), int(hh[0])

    pk = peaks()
    d = descs[dom]
    # bound = the resource whose peak time is larger for this kernel's algorithmic work
    t_flop = d["flops"] / (pk["bf16_tflops_sustained"] * 1e12)
    t_byte = d["bytes"] / (pk["hbm_gbs"] * 1e9)
    if t_flop >= t_byte:
        roof = {"bound": "tensor", "achieved": d["flops"] / (dom_ms / 1e3) / 1e12, "peak": pk["bf16_tflops_sustained"],
                "unit": "TFLOP/s"}
    else:
        roof = {"bound": "hbm", "achieved": d["bytes"] / (dom_ms / 1e3) / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["kernel"] = f"{d['kind']}:{d['op']}({d['def']})"
    roof["peak_src"] = pk["src"] + (" sustained bf16" if roof["bound"] == "tensor" else " hbm copy")
    roof["kernel_ms"] = dom_ms
    roof["kernel_step_share"] = dom_share   # share of the step taken by all launches of this kernel
    roof["algorithmic"] = {"flops": d["flops"], "bytes": d["bytes"], "fused": d.get("fused")}
    roof["traffic"] = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            pt = json.load(open(prof))
            key = f"{CONFIG_NAME[cfg]}|k{k}|{d['op']}"
            if key in pt:
                roof["traffic"] = pt[key]
        except Exception:
            pass

    ledger_el, ledger_b = R.ledger()
    plan_el, plan_b = R.plan.cost()
    # step roofline (north star): the slower of (a) the rank's sub-op flops at the tensor peak and (b) the
    # busiest rank's NVLink traffic at 900 GB/s per direction (max over ranks of max(bytes in, bytes out));
    # the HBM term (algorithmic bytes of the sub-ops at the measured copy bandwidth) is reported beside it
    flops_rank = sum(x["flops"] for x in descs if x["kind"] == "compute")
    t_comp = flops_rank / (pk["bf16_tflops_sustained"] * 1e12)
    io = [ex.rank_bytes(r) for r in range(k)]
    busiest = max((max(a, b) for a, b in io), default=0)
    t_comm = busiest / NVLINK_GBS / 1e9 if k > 1 else 0.0
    step_roof = max(t_comp, t_comm)
    hbm_rank = sum(x["bytes"] for x in descs if x["kind"] == "compute")
    t_hbm = hbm_rank / (pk["hbm_gbs"] * 1e9)

    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded, bf16-exact values)",
        "config": {"workload": CONFIG_NAME[cfg], "global_batch": batch, "parallelism": f"tofu-k{k}",
                   **({"shared_gpu": True} if world > 1 and shared else {}),
                   "plan_factors": R.plan_json["factors"], "l2": "inputs larger than L2 (W+M+dW 640 MiB)"},
        "roofline": roof,
        "step_roofline": {"compute_ms": t_comp * 1e3, "nvlink_ms": t_comm * 1e3, "hbm_ms": t_hbm * 1e3,
                          "frac": step_roof / (ms / 1e3),
                          "frac_incl_hbm": max(step_roof, t_hbm) / (ms / 1e3),
                          "busiest_rank_bytes": busiest,
                          "note": "frac = max(rank flops at the sustained bf16 peak, busiest rank's max(in, out) "
                                  "NVLink bytes at 900 GB/s per direction) / measured step (north star); "
                                  "frac_incl_hbm also takes the sub-ops' algorithmic HBM bytes at the copy peak"},
        "bytes_vs_plan": {"plan_bytes": plan_b, "ledger_bytes": ledger_b, "plan_elements": plan_el,
                          "ledger_elements": ledger_el, "equal": plan_b == ledger_b,
                          "rank_in_out_bytes": io,
                          # this rank's NVLink data counters over the timed steps (nvidia-smi nvlink -gt d), per
                          # step, beside the plan's bytes into / out of this rank (pull model: in = rx, out = tx)
                          "nvlink_measured": None if nv0 is None or nv1 is None else
                          {"rank": rank, "tx_per_step": (nv1[0] - nv0[0]) / steps,
                           "rx_per_step": (nv1[1] - nv0[1]) / steps,
                           "plan_out": io[rank][1], "plan_in": io[rank][0]}},
        "e2e": {"value": batch / (e2e_ms / 1e3), "unit": "samples/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 4, "api": "TofuRunner.train (H2D of step s+1 overlapped with step s)",
                "last_loss": float(losses[-1]) if losses.numel() else None},
        "gpu_launches": ex.launches() * steps,
        "cuda_graph": use_graph,
        "clocks": clk.summary(),
    }
    if world == 1 and virtual_k > 1:
        if big:
            vp_big["ideal_samples_s"] = virtual_k * value
            line["virtual_partitioned"] = vp_big
        else:
            line["virtual_partitioned"] = virtual_partitioned(spec, vals, virtual_k, max(steps, 5), k1_value=value)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sspec, per_step, sample = oracle_sample(cfg)
        t = oracle_step_time(sspec, make_values(sspec, seed=0))
        line["cpu_baseline"] = {"value": per_step / t, "unit": "samples/s", "cores": cpu_threads(), "kind": "oracle",
                                "sample": sample}
    del R, ex
    torch.cuda.empty_cache()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="tofu", choices=["tofu", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay the step as a CUDA graph (auto: when a step issues > 64 launches)")
    ap.add_argument("--virtual-k", type=int, default=8, help="N=1 only: also time the k-way plan on virtual ranks")
    ap.add_argument("--extra", default="1,2", help="N=1 only: other configs measured briefly, reported in the "
                    "same line under other_workloads (empty: none)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if os.environ.get("BENCH_TRACE_AFTER"):   # debugging aid: dump the Python stacks of a stuck run
        import faulthandler
        faulthandler.dump_traceback_later(int(os.environ["BENCH_TRACE_AFTER"]), exit=True)
    if args.impl == "reference":
        return reference_arm(args, world, rank)

    import torch
    import torch.distributed as dist
    from paper_1807_08887_b200.runner import TofuRunner

    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # one GPU per rank over NCCL; with fewer GPUs than ranks (a functional check of the multi-process path on
    # one GPU) the ranks share devices and the host collectives go over gloo (flagged in config.shared_gpu)
    shared = world > torch.cuda.device_count()
    dev = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    group = None
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        group = dist.group.WORLD

    line = run_workload(args.config, args, args.steps, world, rank, local_rank, group, shared, args.virtual_k,
                        rank == 0 and world == 1 and not args.no_cpu_baseline)
    # the other named workloads as compact sub-objects of the same line (N = 1 only; short runs)
    extra = [int(x) for x in args.extra.split(",") if x.strip() != ""] if world == 1 else []
    others = []
    for cfg in extra:
        if cfg == args.config:
            continue
        o = run_workload(cfg, args, max(5, args.steps // 2), world, rank, local_rank, group, shared, args.virtual_k,
                         False)
        others.append({key: o.get(key) for key in ("config", "value", "unit", "ms_per_step", "roofline", "step_roofline",
                                                   "e2e", "bytes_vs_plan", "virtual_partitioned", "gpu_launches",
                                                   "clocks")})
    if others:
        line["other_workloads"] = others
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
