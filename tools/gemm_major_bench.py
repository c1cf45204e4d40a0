import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1807_08887_b200 import tofu
def bench(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it
for (M, N, K) in [(6272, 1024, 4096), (6272, 4096, 1024), (8192, 8192, 8192)]:
    for am, bm in ((0, 0), (0, 1), (1, 0), (1, 1)):
        a = torch.randn((K, M) if am else (M, K), device="cuda").bfloat16()
        b = torch.randn((K, N) if bm else (N, K), device="cuda").bfloat16()
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t = bench(lambda: tofu.gemm(a, b, c, M, N, K, a.shape[1], am, b.shape[1], bm, N, 0, bn=256))
        print(M, N, K, "A_mn", am, "B_mn", bm, f"{t*1e3:.1f} us {2*M*N*K/t/1e9:.0f} TF/s")
