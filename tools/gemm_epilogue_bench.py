"""GEMM epilogue variants (bf16 store, fused relu / add / mask) on a stage-3 WResNet 1x1 shape, plus a
parity check of each fused epilogue against torch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_08887_b200 import tofu  # noqa: E402


def bench(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it


M, N, K = 6272, 1024, 4096
a = torch.randn(M, K, device="cuda").bfloat16()
b = torch.randn(N, K, device="cuda").bfloat16()
add = torch.randn(M, N, device="cuda").bfloat16()
mask = torch.randn(M, N, device="cuda").bfloat16()
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
ref = a.float() @ b.float().t()
for ep in (0, 1, 2, 3, 4, 6):
    t = bench(lambda: tofu.gemm(a, b, c, M, N, K, K, 0, K, 0, N, 0, bn=256, aux_add=add, aux_mask=mask, ep=ep))
    r = ref.clone()
    if ep & 2:
        r += add.float()
    if ep & 1:
        r = r.clamp_min(0)
    if ep & 4:
        r = torch.where(mask.float() > 0, r, torch.zeros_like(r))
    err = float((c.float() - r).norm() / r.norm())
    print(f"ep={ep} {t * 1e3:6.1f} us {2 * M * N * K / t / 1e9:6.0f} TF/s relerr {err:.2e}")
