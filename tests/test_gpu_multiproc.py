"""Multi-process executor (one process per rank, CUDA IPC peer mappings,
device barriers) vs the single-process virtual-rank executor: bitwise equal
results (same kernels, same rank-ordered sums).  Runs 2 processes; on a 1-GPU
box both share cuda:0 (IPC mapping of another process's memory on the same
device), on a multi-GPU box they use cuda:0 / cuda:1 over NVLink."""
import os
import pickle
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_two_process_step_equals_virtual(tmp_path):
    out = str(tmp_path / "res")
    port = str(29600 + os.getpid() % 1000)
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp_worker.py"), str(r), "2", out, port])
             for r in range(2)]
    try:
        rcs = [p.wait(timeout=240) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert rcs == [0, 0]
    res = [pickle.load(open(f"{out}.{r}", "rb")) for r in range(2)]
    from paper_1807_08887_b200.runner import TofuRunner
    from tofu_inputs.graphs import config
    from tofu_inputs.tensors import make_values
    spec = config(0)
    R = TofuRunner(spec, 2)
    R.load(make_values(spec, seed=31))
    for _ in range(2):
        R.step()
    torch.cuda.synchronize()
    for r in range(2):
        assert res[r]["ledger"] == res[r]["plan"]
        for t, (box, arr) in res[r]["shards"].items():
            ref = R.view(r, t).float().cpu().numpy()
            assert np.array_equal(arr, ref), (r, t)


def test_bench_two_ranks_shared_gpu(tmp_path):
    """bench.py at N = 2 under torchrun (one process per rank; on a 1-GPU box both ranks share the device
    and the host collectives go over gloo, config.shared_gpu): the whole multi-process bench path runs to
    its JSON line with the byte ledger equal to the plan.  Regression test for a hang: every step holds
    device barriers across ranks, so all ranks must run the same number of steps (the clock-soak loop)."""
    import json
    root = os.path.dirname(HERE)
    port = str(29700 + os.getpid() % 200)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", port, os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3"]
    p = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=400)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["bytes_vs_plan"]["equal"]
    assert line["config"]["parallelism"] == "tofu-k2"
    assert line["value"] > 0 and line["gpu_launches"] > 0
