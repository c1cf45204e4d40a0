"""GEMM micro-benchmark of the WResNet-152-4 (batch 32) 1x1-convolution shapes with and without the stream-K
workspace (and, via TOFU_LIB, across experimental builds): forward (A pixels x ci, B W[co][ci], both K-major)
with its fused epilogue, data gradient (B MN-major) with its fused epilogue."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_08887_b200 import tofu  # noqa: E402

SHAPES = [  # name, M pixels, N, K, b_mn, ep
    ("s0.conv1 fwd relu", 100352, 256, 1024, 0, 1),
    ("s0.conv3 fwd add+relu", 100352, 1024, 256, 0, 3),
    ("s0.conv1 dgrad add+mask", 100352, 1024, 256, 1, 6),
    ("s0.conv3 dgrad mask", 100352, 256, 1024, 1, 4),
    ("s2.conv1 fwd relu", 6272, 1024, 4096, 0, 1),
    ("s2.conv3 fwd add+relu", 6272, 4096, 1024, 0, 3),
    ("s2.conv1 dgrad add+mask", 6272, 4096, 1024, 1, 6),
    ("s2.conv3 dgrad mask", 6272, 1024, 4096, 1, 4),
    ("s3.conv1 fwd relu", 1568, 2048, 8192, 0, 1),
    ("s3.conv3 dgrad mask", 1568, 2048, 8192, 1, 4),
    ("fc fwd (mm_nn)", 512, 8192, 8192, 1, 0),
    ("s2.conv2 fwd-like", 6272, 1024, 9216, 0, 1),
]


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


ws = torch.zeros(tofu.sk_workspace_bytes(), dtype=torch.uint8, device="cuda")
for name, M, N, K, bmn, ep in SHAPES:
    A = (torch.randn(M, K, device="cuda") * 0.1).bfloat16()
    Bm = (torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).bfloat16()
    add = torch.randn(M, N, device="cuda").bfloat16()
    mask = torch.randn(M, N, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    res = []
    for sk in (None, ws):
        f = lambda: tofu.gemm(A, Bm, C, M, N, K, K, 0, N if bmn else K, bmn, N, 0, aux_add=add, aux_mask=mask,
                              ep=ep, sk_ws=sk, splits=-1 if sk is not None else 0)
        res.append(timeit(f))
    flops = 2 * M * N * K
    byts = 2 * (M * K + K * N + M * N) + 2 * M * N * (((ep >> 1) & 1) + ((ep >> 2) & 1))
    print(f"{name:26s} dp {res[0] * 1e3:7.1f} us ({flops / res[0] / 1e9:6.0f} TF/s {byts / res[0] / 1e6:5.0f} GB/s)"
          f"   sk {res[1] * 1e3:7.1f} us ({flops / res[1] / 1e9:6.0f} TF/s {byts / res[1] / 1e6:5.0f} GB/s)")
