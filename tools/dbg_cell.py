import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1807_08887_b200 import tofu
L = tofu.lib()
f = L.tofu_lstm_cell
f.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
              C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p]
B, H = 16, 64
gx = torch.randn(B, 4, H, device="cuda").bfloat16(); gh = torch.randn(B, 4, H, device="cuda").bfloat16()
c = torch.randn(B, H, device="cuda")
out = torch.zeros(B, H, device="cuda").bfloat16()
ptrs = (C.c_void_p * 7)(gx.data_ptr(), gh.data_ptr(), 0, c.data_ptr(), 0, 0, 0)
lds = (C.c_int64 * 7)(4 * H, 4 * H, 0, H, 0, 0, 0)
gss = (C.c_int64 * 7)(H, H, 0, 0, 0, 0, 0)
dts = (C.c_int * 7)(0, 0, 1, 1, 1, 1, 1)
rc = f(1, B, H, 0, 0, ptrs, lds, gss, dts, out.data_ptr(), H, 0, 0, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
o = torch.sigmoid(gx[:, 3].float() + gh[:, 3].float())
ref = o * torch.tanh(c)
print("rc", rc, "err", float((out.float() - ref).norm() / ref.norm()))
