"""Worker for the multi-process executor test (2 processes, gloo, one GPU or two)."""
import os
import pickle
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker_spec(which):
    from tofu_inputs.graphs import config, wresnet
    if which == "wres":   # a small WResNet: halo / strided-gradient fetches, partition-n-reduce + fused consumers
        return wresnet([1, 1], 1, 8, 32, base=16, classes=16)
    if which == "lstm":   # a small LSTM: stacked-state views, fused cells, fused (in-place) GEMM operand fetches
        from tofu_inputs.graphs import lstm
        return lstm(2, 256, 4, 32)
    return config(0)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1807_08887_b200.runner import TofuRunner
    from tofu_inputs.graphs import config
    from tofu_inputs.tensors import make_values

    rank, world, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    which = sys.argv[5] if len(sys.argv) > 5 else "mlp"
    ngpu = torch.cuda.device_count()
    torch.cuda.set_device(rank % ngpu)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{sys.argv[4]}", rank=rank, world_size=world)
    spec = worker_spec(which)
    vals = make_values(spec, seed=31)
    dbg = os.environ.get("TOFU_MP_DEBUG")
    if dbg: print(f"[{rank}] init ok", file=sys.stderr, flush=True)
    R = TofuRunner(spec, world, device=f"cuda:{rank % ngpu}", rank=rank, group=dist.group.WORLD)
    if dbg: print(f"[{rank}] runner ok launches={R.exec.num_launches()}", file=sys.stderr, flush=True)
    R.load(vals)
    torch.cuda.synchronize()
    dist.barrier()
    for i in range(2):
        if dbg:
            for j in range(R.exec.num_launches()):
                R.exec.run_range(j, j + 1)
                torch.cuda.synchronize()
                print(f"[{rank}] step {i} launch {j} {R.exec.launch_desc(j)['kind']} ok", file=sys.stderr, flush=True)
        else:
            R.step()
    torch.cuda.synchronize()
    dist.barrier()
    shards = {}
    for t in spec["tensors"]:
        v = R.view(rank, t)
        if v is not None:
            shards[t] = (R.shards[rank][t][1], v.float().cpu().numpy())
    pickle.dump({"rank": rank, "shards": shards, "ledger": R.ledger(), "plan": R.plan.cost()},
                open(f"{out}.{rank}", "wb"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
