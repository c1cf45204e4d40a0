"""Device time per kernel inside a CUDA-graph-replayed training step (torch.profiler / CUPTI: no per-launch
events, no host gaps): per kernel name count / total / mean, the step's busy time (union of kernel intervals)
and its idle time.  With K > 1 the step runs the k-way plan on K virtual ranks.

    K=8 python tools/kineto_step.py <config> [steps]
"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1807_08887_b200.runner import TofuRunner  # noqa: E402
from tofu_inputs.graphs import config  # noqa: E402
from tofu_inputs.tensors import make_values  # noqa: E402

cfg = int(sys.argv[1])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
k = int(os.environ.get("K", "1"))
spec = config(cfg)
R = TofuRunner(spec, k)
R.load(make_values(spec, seed=0))
for _ in range(2):
    R.step()
R.capture()
for _ in range(3):
    R.step()
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(steps):
    R.step()
e.record()
torch.cuda.synchronize()
step_ms = s.elapsed_time(e) / steps
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        R.step()
    torch.cuda.synchronize()
if os.environ.get("TRACE"):  # chrome trace of the profiled steps (streams as rows)
    prof.export_chrome_trace(os.environ["TRACE"])
evs = [ev for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA and ev.name != ""]
# comm kernels (MultiFetch / partition-n-reduce / barrier) running while a compute kernel runs: the overlap the
# executor's second stream buys (TOFU_STREAMS=2 on virtual ranks; always two in multi-process mode)
comm_names = ("pieces_kernel", "pieces_copy_kernel", "pieces_kernel_wide", "barrier_kernel")
ci = sorted((e.time_range.start, e.time_range.end) for e in evs if any(c in e.name for c in comm_names))
ki = sorted((e.time_range.start, e.time_range.end) for e in evs
            if not any(c in e.name for c in comm_names) and "Memcpy" not in e.name and "Memset" not in e.name)
ov, j = 0.0, 0
for a, b in ci:
    while j < len(ki) and ki[j][1] <= a:
        j += 1
    t = j
    while t < len(ki) and ki[t][0] < b:
        ov += max(0.0, min(b, ki[t][1]) - max(a, ki[t][0]))
        t += 1
ctot = sum(b - a for a, b in ci)
if ctot:
    print(f"comm kernels {ctot / steps / 1e3:.3f} ms/step, of which under compute kernels {ov / steps / 1e3:.3f} ms "
          f"({100 * ov / ctot:.0f}%)")
kern = [ev for ev in evs if "Memcpy" not in ev.name and "Memset" not in ev.name]
agg = collections.defaultdict(lambda: [0, 0.0])
iv = []
for ev in kern:
    name = ev.name.split("(")[0][:70]
    d = ev.time_range.elapsed_us()
    agg[name][0] += 1
    agg[name][1] += d
    iv.append((ev.time_range.start, ev.time_range.end))
iv.sort()
# per-step spans and the idle gaps between consecutive steps (kernels in launch order; a step = its share)
per = len(iv) // steps if steps else 0
if per:
    starts = [iv[i * per][0] for i in range(steps)]
    ends = [max(b for _, b in iv[i * per:(i + 1) * per]) for i in range(steps)]
    gaps = [(starts[i + 1] - ends[i]) for i in range(steps - 1)]
    print("per-step spans (ms):", [round((ends[i] - starts[i]) / 1e3, 3) for i in range(steps)],
          "gaps between steps (us):", [round(g, 1) for g in gaps])
s2, e2 = torch.cuda.Event(True), torch.cuda.Event(True)
s2.record()
for _ in range(steps):
    R.step()
e2.record()
torch.cuda.synchronize()
print(f"events after profiling: {s2.elapsed_time(e2) / steps:.3f} ms/step")
busy, cur_s, cur_e = 0.0, None, None
for a, b in iv:
    if cur_e is None or a > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = a, b
    else:
        cur_e = max(cur_e, b)
if cur_e is not None:
    busy += cur_e - cur_s
span = (iv[-1][1] - iv[0][0]) if iv else 0
tot = sum(a[1] for a in agg.values())
print(f"config {cfg} k={k}: step {step_ms:.3f} ms (events, graph replay); profiled {steps} steps: kernels "
      f"{len(kern) / steps:.0f}/step, sum of kernel time {tot / steps / 1e3:.3f} ms/step, busy (union) "
      f"{busy / steps / 1e3:.3f} ms/step, span {span / steps / 1e3:.3f} ms/step")
for name, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"  {us / steps / 1e3:8.3f} ms/step  n={n // steps:5d}  mean {us / n:8.2f} us  {name}")
