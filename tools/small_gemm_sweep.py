"""Work-split sweep for the per-rank recurrent GEMMs of the LSTM plans at k = 8 (M = 128 rows): device time of
tofu_gemm_bf16 per (bn, splits) for [128 x 2048 x 4096] (gate: K-major A, MN-major B) and [128 x 4096 x 2048]
(mm_rec: both K-major).  python tools/small_gemm_sweep.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_08887_b200 import tofu  # noqa: E402


def bench(fn, reps=50):
    """device time per call: a CUDA graph of reps calls (the per-call host work, tensor-map encoding and ctypes,
    outlasts these kernels and would otherwise be what is timed)"""
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


SHAPES = {"gate": (128, 2048, 4096, 0, 1), "mm_rec": (128, 4096, 2048, 0, 0)}
CMODE = 0
if len(sys.argv) > 1 and sys.argv[1] == "k1":  # configs[2] at k = 1: the full recurrent GEMMs (weights 134 MB)
    SHAPES = {"gate": (128, 16384, 4096, 0, 1), "mm_rec": (128, 4096, 16384, 0, 0)}
if len(sys.argv) > 1 and sys.argv[1] == "wres8":  # WResNet-152-4 1x1 sub-ops of a rank at k = 8, fp32 partials
    SHAPES = {"fwd": (1568, 1024, 2048, 0, 0), "dgrad": (1568, 2048, 1024, 0, 1), "wgrad": (1024, 2048, 1568, 1, 1)}
    CMODE = 1
for name, (M, N, K, am, bm) in SHAPES.items():
    a = torch.randn((K, M) if am else (M, K), device="cuda").bfloat16()
    b = torch.randn((K, N) if bm else (N, K), device="cuda").bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.float32 if CMODE == 1 else torch.bfloat16)
    for bn in (128, 256):
        for sp in ((1, 2, 3, 4) if CMODE == 1 else (1, 2, 4, 8, 16, 32)):
            try:
                t = bench(lambda: tofu.gemm(a, b, c, M, N, K, a.shape[1], am, b.shape[1], bm, N, CMODE, bn=bn,
                                            splits=sp, stream=torch.cuda.current_stream()))
            except Exception as ex:  # noqa: BLE001
                print(name, bn, sp, "error", ex)
                continue
            print(f"{name} [{M}x{N}x{K}] bn={bn} splits={sp}: {t:.1f} us {2 * M * N * K / t / 1e6:.0f} TF/s")
