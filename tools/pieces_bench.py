"""Bandwidth of the piece kernel (tofu_pieces_run) on local HBM: bytes read + written per second.

    python tools/pieces_bench.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_08887_b200 import tofu  # noqa: E402


def run(name, shape, box, nsrc=1, sdt=0, ddt=0, reps=20):
    DT = {0: torch.bfloat16, 1: torch.float32}
    srcs = [torch.randn(shape, device="cuda").to(DT[sdt]) for _ in range(nsrc)]
    dst = torch.empty(shape, device="cuda", dtype=DT[ddt])
    sl = tuple(slice(a, b) for a, b in box)
    ps = (tofu.Piece * 1)()
    p = ps[0]
    sv = [s[sl] for s in srcs]
    dv = dst[sl]
    r = len(shape)
    ext = [1] * (4 - r) + list(dv.shape)
    dst_st = [0] * (4 - r) + list(dv.stride())
    src_st = [0] * (4 - r) + list(sv[0].stride())
    for d in range(4):
        p.extent[d], p.dst_stride[d], p.src_stride[d] = ext[d], dst_st[d], src_st[d]
    p.dst, p.nsrc, p.dst_dtype, p.src_dtype = dv.data_ptr(), nsrc, ddt, sdt
    for i, s in enumerate(sv):
        p.src[i] = s.data_ptr()
    tasks, nt = tofu.pieces_tasks(ps)
    pd = torch.frombuffer(bytearray(bytes(ps)), dtype=torch.uint8).cuda()
    td = torch.frombuffer(bytearray(bytes(tasks)), dtype=torch.uint8).cuda()
    raw = int(all(tasks[i].pad_ == 1 for i in range(nt)))  # (host work kept out of the timed loop)
    if not raw and nsrc >= 4:
        raw = 2  # the many-source kernel (as the executor picks it)
    for _ in range(3):
        tofu.pieces_run(pd.data_ptr(), td.data_ptr(), nt, raw)
    g = torch.cuda.CUDAGraph()  # graph replay: device time only, no per-call host cost
    with torch.cuda.graph(g):
        for _ in range(reps):
            tofu.pieces_run(pd.data_ptr(), td.data_ptr(), nt, raw, stream=torch.cuda.current_stream())
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    n = dv.numel()
    by = n * (srcs[0].element_size() * nsrc + dst.element_size())
    ref = sum(s.float() for s in sv).to(DT[ddt])
    ok = torch.equal(dv, ref)
    print(f"{name:38s} {ms * 1e3:8.1f} us {by / ms / 1e6:8.1f} GB/s  V={ps[0].pad_} tasks={nt} ok={ok}")


run("contiguous 256 MiB bf16", [128 * 1024 * 1024], [(0, 128 * 1024 * 1024)])
run("batch slice [4 of 32,56,56,256]", [32, 56, 56, 256], [(4, 8), (0, 56), (0, 56), (0, 256)])
run("channel slice [32,56,56,64 of 256]", [32, 56, 56, 256], [(0, 32), (0, 56), (0, 56), (64, 128)])
run("halo rows [32,28+2 of 56,56,256]", [32, 56, 56, 256], [(0, 32), (27, 57 - 1), (0, 56), (0, 256)])
run("reduce 8 x fp32 -> bf16 [1024,4096]", [1024, 4096], [(0, 1024), (0, 4096)], nsrc=8, sdt=1, ddt=0)
run("reduce 2 x fp32 -> fp32 [2048,2048]", [4096, 4096], [(0, 4096), (1024, 3072)], nsrc=2, sdt=1, ddt=1)
run("reduce 8 x fp32 -> bf16 [3136,512]", [3136, 512], [(0, 3136), (0, 512)], nsrc=8, sdt=1, ddt=0)
run("reduce 4 x fp32 -> bf16 [12544,1024]", [12544, 1024], [(0, 12544), (0, 1024)], nsrc=4, sdt=1, ddt=0)
