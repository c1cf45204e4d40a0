"""Fused wgrad + momentum-SGD GEMM (c_mode 3) on the configs[1] shape: HBM GB/s vs the measured copy peak."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_08887_b200 import tofu  # noqa: E402

M = N = 8192
K = 512
a = torch.randn(K, M, device="cuda").bfloat16()
b = torch.randn(K, N, device="cuda").bfloat16()
m = torch.zeros(M, N, device="cuda")
w = torch.zeros(M, N, device="cuda").bfloat16()
for _ in range(3):
    tofu.gemm(a, b, m, M, N, K, M, 1, N, 1, N, 3, D=w, ldd=N, s0=0.875, s1=2 ** -7)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(20):
    tofu.gemm(a, b, m, M, N, K, M, 1, N, 1, N, 3, D=w, ldd=N, s0=0.875, s1=2 ** -7)
e.record()
torch.cuda.synchronize()
t = s.elapsed_time(e) / 20
byt = 2 * (M * K + K * N) + M * N * 12
print(os.environ.get("TOFU_LIB", "default"), f"{t * 1e3:.1f} us {byt / t / 1e6:.0f} GB/s")
