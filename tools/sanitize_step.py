"""One small partitioned training step per workload family, for compute-sanitizer runs:

    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_step.py

(virtual ranks on cuda:0; MLP k = 2, a 2-unit WResNet k = 4, a 2-layer LSTM k = 4; fusion on)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_08887_b200.runner import TofuRunner  # noqa: E402
from tofu_inputs.graphs import config, lstm, wresnet  # noqa: E402
from tofu_inputs.tensors import make_values  # noqa: E402

for name, spec, k in [("mlp", config(0), 2), ("wresnet", wresnet([1, 1], 1, 4, 32, base=16, classes=16), 4),
                      ("lstm", lstm(2, 256, 3, 32), 4)]:
    R = TofuRunner(spec, k)
    R.load(make_values(spec, seed=1))
    R.step()
    torch.cuda.synchronize()
    print(name, "ok", R.exec.num_launches(), "launches", flush=True)
