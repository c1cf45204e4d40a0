"""Microbench: libtofu tcgen05 GEMM vs torch.matmul (cuBLAS) at config shapes."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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

res = []
for (name, M, N, K, am, bm, cm) in [("fwd_nn", 512, 8192, 8192, 0, 1, 0), ("wgrad_tn", 8192, 8192, 512, 1, 1, 1),
                                    ("dgrad_nt", 512, 8192, 8192, 0, 0, 0), ("sq_nn", 8192, 8192, 8192, 0, 1, 1),
                                    ("k8_fwd", 512, 2048, 4096, 0, 1, 1), ("k8_wgrad", 4096, 2048, 512, 1, 1, 1)]:
    a = torch.randn((K, M) if am else (M, K), device="cuda").bfloat16()
    b = torch.randn((K, N) if bm else (N, K), device="cuda").bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16 if cm == 0 else torch.float32)
    for bn in (128, 256):
        t = bench(lambda: tofu.gemm(a, b, c, M, N, K, a.shape[1], am, b.shape[1], bm, N, cm, bn=bn))
        res.append(dict(name=name, bn=bn, ms=t, tflops=2 * M * N * K / t / 1e9))
    A = a.t() if am else a
    B = b if bm else b.t()
    tt = bench(lambda: torch.matmul(A, B))
    res.append(dict(name=name, bn="cublas", ms=tt, tflops=2 * M * N * K / tt / 1e9))
    # correctness vs cublas
    tofu.gemm(a, b, c, M, N, K, a.shape[1], am, b.shape[1], bm, N, cm)
    ref = torch.matmul(A.float(), B.float())
    res.append(dict(name=name, relerr=float((c.float() - ref).norm() / ref.norm())))
for r in res: print(json.dumps(r))
