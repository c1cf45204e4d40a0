"""Driver of tools/epi_pattern.cu (experiment): GB/s of the fused add / mask epilogue's memory pattern alone,
beside torch's element-wise kernels on the same tensors (3 x 205 MB: add, mask read, out written)."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = C.CDLL(os.path.join(ROOT, "variants", "epi_pattern.so"))
M, N = 100352, 1024
add = torch.randn(M, N, device="cuda").bfloat16()
mask = torch.randn(M, N, device="cuda").bfloat16()
out = torch.empty_like(add)
nbytes = 3 * M * N * 2


def t(fn, it=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it


st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for cw, nb in ((32, 2), (32, 3), (32, 4), (32, 6), (64, 2), (64, 3)):
    f = lambda: L.epi_run(C.c_void_p(add.data_ptr()), C.c_void_p(mask.data_ptr()), C.c_void_p(out.data_ptr()), M, N, cw, nb, st)  # noqa
    assert f() == 0
    ms = t(f)
    ok = torch.equal(out, torch.where(mask.float() > 0, add, torch.zeros_like(add)))
    print(f"pattern cw={cw} nbuf={nb}: {ms * 1e3:7.1f} us {nbytes / ms / 1e6:7.0f} GB/s ok={ok}", flush=True)
z = torch.zeros_like(add)
ms = t(lambda: torch.where(mask > 0, add, z, out=out))
print(f"torch.where (4 tensors): {ms * 1e3:7.1f} us {4 * M * N * 2 / ms / 1e6:7.0f} GB/s")
ms = t(lambda: torch.add(add, mask, out=out))
print(f"torch.add (3 tensors): {ms * 1e3:7.1f} us {nbytes / ms / 1e6:7.0f} GB/s")
ms = t(lambda: out.copy_(add))
print(f"copy (2 tensors): {ms * 1e3:7.1f} us {2 * M * N * 2 / ms / 1e6:7.0f} GB/s")
