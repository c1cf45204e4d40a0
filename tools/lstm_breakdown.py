import os, sys, json, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from tofu_inputs.graphs import config, lstm
from tofu_inputs.tensors import make_values
from paper_1807_08887_b200.runner import TofuRunner
spec = config(2) if len(sys.argv) < 2 else lstm(*map(int, sys.argv[1:5]))
R = TofuRunner(spec, 1); R.load(make_values(spec, seed=0))
ex = R.exec
for _ in range(2): ex.run()
torch.cuda.synchronize()
nl = ex.num_launches(); descs = [ex.launch_desc(i) for i in range(nl)]
evs = [torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)]
evs[0].record()
for i in range(nl):
    ex.run_range(i, i + 1); evs[i + 1].record()
torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, d in enumerate(descs):
    key = d["def"] if d["kind"] == "compute" else d["kind"]
    a = agg[key]; a[0] += 1; a[1] += evs[i].elapsed_time(evs[i + 1]); a[2] += d["flops"]; a[3] += d["bytes"]
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:12s} n={a[0]:4d} ms={a[1]:8.3f} ({100*a[1]/tot:4.1f}%) TF/s={a[2]/(a[1]/1e3)/1e12:7.1f} GB/s={a[3]/(a[1]/1e3)/1e9:7.1f}")
print("total ms", tot)
