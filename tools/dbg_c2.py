"""Debug helper: one 2-CTA GEMM (cl2=4) vs the single-CTA launch.  python tools/dbg_c2.py M N K [am bm]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1807_08887_b200 import tofu
M, N, K = map(int, sys.argv[1:4])
am, bm = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (0, 0)
A = torch.randn((K, M) if am else (M, K), device="cuda").bfloat16()
B = torch.randn((K, N) if bm else (N, K), device="cuda").bfloat16()
outs = []
for cl2 in (-1, 4):
    C = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    tofu.gemm(A, B, C, M, N, K, A.shape[1], am, B.shape[1], bm, N, 1, splits=1, cl2=cl2)
    torch.cuda.synchronize()
    outs.append(C)
print(M, N, K, am, bm, "maxdiff", float((outs[0] - outs[1]).abs().max()), flush=True)
