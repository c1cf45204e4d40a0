"""Per-launch device-time breakdown of one training step (CUDA events between launches).

    python tools/breakdown.py <config>            # e.g. 3 (WResNet-152-4, batch 32)
    python tools/breakdown.py wresnet L W B IMG   # another WResNet
    python tools/breakdown.py units 1,1 W B IMG   # a WResNet with the given units per stage
    python tools/breakdown.py lstm L H T B        # an LSTM (layers, hidden, steps, batch)
Prints per-def totals (count, ms, share, TFLOP/s, GB/s) and the slowest individual launches."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_08887_b200.runner import TofuRunner  # noqa: E402
from tofu_inputs.graphs import config, wresnet_depth  # noqa: E402
from tofu_inputs.tensors import make_values  # noqa: E402

if sys.argv[1] == "lstm":     # layers hidden steps batch
    from tofu_inputs.graphs import lstm
    spec = lstm(*map(int, sys.argv[2:6]))
elif sys.argv[1] == "wresnet":
    spec = wresnet_depth(*map(int, sys.argv[2:6]))
elif sys.argv[1] == "units":   # units "1,1" width batch image
    from tofu_inputs.graphs import wresnet
    spec = wresnet([int(u) for u in sys.argv[2].split(",")], *map(int, sys.argv[3:6]))
else:
    spec = config(int(sys.argv[1]))
k = int(os.environ.get("K", "1"))
R = TofuRunner(spec, k)
R.load(make_values(spec, seed=0))
ex = R.exec
for _ in range(2):
    ex.run()
torch.cuda.synchronize()
nl = ex.num_launches()
descs = [ex.launch_desc(i) for i in range(nl)]
evs = [torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)]
evs[0].record()
for i in range(nl):
    ex.run_range(i, i + 1)
    evs[i + 1].record()
torch.cuda.synchronize()
ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(nl)]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, d in enumerate(descs):
    key = d["def"] if d["kind"] == "compute" else d["kind"]
    a = agg[key]
    a[0] += 1
    a[1] += ms[i]
    a[2] += d["flops"]
    a[3] += d["bytes"]
tot = sum(ms)
for key, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{key:16s} n={a[0]:4d} ms={a[1]:8.3f} ({100 * a[1] / tot:4.1f}%) TF/s={a[2] / (a[1] / 1e3) / 1e12:7.1f} "
          f"GB/s={a[3] / (a[1] / 1e3) / 1e9:7.1f}")
print("total ms", tot, "flops", sum(d["flops"] for d in descs))
print("--- slowest launches")
for i in sorted(range(nl), key=lambda i: -ms[i])[:25]:
    d = descs[i]
    print(f"{ms[i]:7.3f} ms {d['kind']:8s} {d['op']:22s} {d['def']:14s} TF/s={d['flops'] / (ms[i] / 1e3) / 1e12:7.1f} "
          f"GB/s={d['bytes'] / (ms[i] / 1e3) / 1e9:7.1f} r{d.get('rank')} {d.get('mnk', '')} {d.get('fused', '')} "
          f"{d.get('weights', '')}")

if os.environ.get("UNIT"):
    print("--- launches of", os.environ["UNIT"])
    for i, d in enumerate(descs):
        if d["op"] and d["op"].startswith(os.environ["UNIT"] + "."):
            print(f"{ms[i]:7.3f} ms {d['kind']:8s} {d['op']:22s} {d['def']:14s} "
                  f"TF/s={d['flops'] / (ms[i] / 1e3) / 1e12:7.1f} GB/s={d['bytes'] / (ms[i] / 1e3) / 1e9:7.1f} "
                  f"{d.get('fused', '')}")

if os.environ.get("BY_SHAPE"):   # rank-0 launches aggregated by (def, shape, work split, fused)
    print("--- rank 0 by shape")
    agg2 = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, d in enumerate(descs):
        if d.get("rank") not in (0, -1):
            continue
        key = (d["kind"], d["def"], str(d.get("mnk", "")), d.get("splits", ""), d.get("bn", ""), d.get("fused", ""))
        a = agg2[key]
        a[0] += 1
        a[1] += ms[i]
        a[2] += d["flops"]
    for key, a in sorted(agg2.items(), key=lambda x: -x[1][1])[:40]:
        print(f"{a[1]:8.3f} ms n={a[0]:4d} TF/s={a[2] / (a[1] / 1e3) / 1e12:7.1f} {key}")
