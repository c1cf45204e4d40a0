"""The LSTM-6-4K GEMM classes at k = 1 (configs[2]) in isolation: L.dx (dA . Wx^T: M 2560, N 4096, K 16384, both
K-major) and the gate weight gradient with the fused optimizer (X^T . dA: M 4096, N 16384, K 2560, both MN-major,
c_mode 3).  Prints device time and TF/s; run under ncu for DRAM bytes / L2 hit rate.
    python tools/lstm_gemm_probe.py [dx|wg|all] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_08887_b200 import tofu  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10


def bench(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


if which in ("dx", "all"):
    M, N, K = 2560, 4096, 16384
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t = bench(lambda: tofu.gemm(a, b, c, M, N, K, K, 0, K, 0, N, 0))
    print(f"L.dx {M}x{N}x{K}: {t * 1e3:.1f} us {2 * M * N * K / t / 1e9:.0f} TF/s")
if which in ("wg", "all"):
    M, N, K = 4096, 16384, 2560
    a = torch.randn(K, M, device="cuda").bfloat16()
    b = torch.randn(K, N, device="cuda").bfloat16()
    m = torch.zeros(M, N, device="cuda")
    w = torch.randn(M, N, device="cuda").bfloat16()
    t = bench(lambda: tofu.gemm(a, b, m, M, N, K, M, 1, N, 1, N, 3, D=w, ldd=N, s0=0.875, s1=2.0 ** -7))
    print(f"gate wgrad+opt {M}x{N}x{K}: {t * 1e3:.1f} us {2 * M * N * K / t / 1e9:.0f} TF/s")
