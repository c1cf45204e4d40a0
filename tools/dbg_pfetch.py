import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1807_08887_b200.runner import TofuRunner
from tofu_inputs.graphs import config
from tofu_inputs.tensors import make_values
k = int(sys.argv[1]); cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = config(cfg)
vals = make_values(spec, seed=41)
outs = {}
for pf in sys.argv[3].split(","):
    os.environ["TOFU_PFETCH"] = pf
    R = TofuRunner(spec, k)
    R.load(vals)
    R.step()
    torch.cuda.synchronize()
    outs[pf] = {t: R.gather(t).float().cpu().numpy() for t in spec["tensors"]}
    print(pf, "ok", flush=True)
    del R
if len(outs) == 2:
    a, b = outs.values()
    for t in spec["tensors"]:
        d = np.abs(a[t] - b[t]).max() if np.ndim(a[t]) else abs(a[t] - b[t])
        print(t, d)
