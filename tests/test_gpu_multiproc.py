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


@pytest.mark.parametrize("world,which,jitter", [(2, "mlp", None), (2, "mlp", "7"), (4, "wres", None),
                                                (4, "wres", "11"), (4, "lstm", "5")])
def test_processes_step_equals_virtual(tmp_path, world, which, jitter):
    """world processes (one rank each, IPC-mapped peer arenas, device barriers) run two steps and match the
    virtual-rank executor bitwise.  With TOFU_JITTER every process injects pseudo-random 0-200 us delays
    before a quarter of its launches (different per rank), so a missing or misplaced barrier shows up as a
    read of stale / not-yet-produced peer data."""
    out = str(tmp_path / "res")
    port = str(29600 + (os.getpid() + world * 7 + (1 if jitter else 0)) % 1000)
    env = dict(os.environ)
    if jitter:
        env["TOFU_JITTER"] = jitter
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp_worker.py"), str(r), str(world), out, port,
                               which], env=env)
             for r in range(world)]
    try:
        rcs = [p.wait(timeout=300) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert rcs == [0] * world
    res = [pickle.load(open(f"{out}.{r}", "rb")) for r in range(world)]
    from mp_worker import worker_spec
    from paper_1807_08887_b200.runner import TofuRunner
    from tofu_inputs.tensors import make_values
    spec = worker_spec(which)
    R = TofuRunner(spec, world)
    R.load(make_values(spec, seed=31))
    for _ in range(2):
        R.step()
    torch.cuda.synchronize()
    for r in range(world):
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
