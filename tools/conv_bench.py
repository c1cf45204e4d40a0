"""Micro-benchmark of the implicit-GEMM convolution kernel on one stage-3 WResNet-152-4 shape
(batch 32, 14x14, 1024 -> 1024 channels, 3x3 pad 1): forward, data gradient with MN-major weights (as the
executor runs it), data gradient with K-major (transposed) weights, weight gradient."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_08887_b200 import tofu  # noqa: E402

B, H, C, R = int(os.environ.get("B", 32)), int(os.environ.get("H", 14)), int(os.environ.get("C", 1024)), 3
dev = "cuda"
X = (torch.randn(B, H, H, C, device=dev) * 0.1).bfloat16()
W = (torch.randn(C, R, R, C, device=dev) * 0.02).bfloat16()      # [co][ky][kx][ci]
WT = W.permute(3, 1, 2, 0).contiguous()                           # [ci][ky][kx][co]
Y = torch.empty(B, H, H, C, device=dev, dtype=torch.bfloat16)
dW = torch.zeros(C, R, R, C, device=dev, dtype=torch.float32)


def args(kind, S, out, Bmat=None, mn=0, flip=False):
    a = tofu.ConvArgs()
    a.kind = kind
    a.nb, a.ngy, a.ngx = B, H, H
    a.ay = a.ax = 1
    a.cy = a.cx = -1 if not flip else 1
    a.ntaps = 9
    for t in range(9):
        ky, kx = divmod(t, 3)
        a.tap_dy[t], a.tap_dx[t] = (-ky, -kx) if flip else (ky, kx)
        a.tap_w[t] = t
    a.nch = C
    a.S = S.data_ptr()
    a.s_sb, a.s_sy, a.s_sx = H * H * C, H * C, C
    a.sH = a.sW = H
    if kind == 0:
        a.n_out = C
        a.Bp = Bmat.data_ptr()
        a.ldb = 9 * C
        a.b_mn_major = mn
        a.b_tap = C
        a.b_rows, a.b_cols = C, 9 * C
        a.C = out.data_ptr()
        a.c_sb, a.c_sy, a.c_sx = H * H * C, H * C, C
        a.c_ys = a.c_xs = 1
    else:
        a.m_out = C
        a.Ap = Y.data_ptr()
        a.lda = C
        a.C = out.data_ptr()
        a.ldc = 9 * C
        a.c_mode = 1
    return a


SKWS = torch.zeros(tofu.sk_workspace_bytes(), dtype=torch.uint8, device=dev) if os.environ.get("SK") == "1" else None
# WS=1: a caller split-K workspace (as the executor passes; the one-shot path otherwise allocates one per call)
WS = torch.empty(16 * 9 * C * C, dtype=torch.float32, device=dev) if os.environ.get("WS") == "1" else None


def timeit(a, n=20):
    if SKWS is not None:  # stream-K workspace (as the executor passes): few-tile launches may spread their K loop
        a.sk_ws = SKWS.data_ptr()
    if WS is not None:
        a.ws = WS.data_ptr()
    if a.kind == 1 and os.environ.get("SPLITS"):  # weight gradient: force the split count (A/B)
        a.splits = int(os.environ["SPLITS"])
    for _ in range(3):
        tofu.conv(a)
    torch.cuda.synchronize()
    if os.environ.get("GRAPH") == "1":  # device time without the per-call host planning (tensor maps)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(n):
                tofu.conv(a, stream=torch.cuda.current_stream())
        g.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / n
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        tofu.conv(a)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


flops = 2 * B * H * H * C * C * 9
mask = (torch.randn(B, H, H, C, device=dev)).bfloat16()
dm = args(0, X, Y, WT, 0, flip=True)
dm.ep, dm.aux_mask = 4, mask.data_ptr()
fr = args(0, X, Y, W, 0)
fr.ep = 1
for name, a in [("fwd  (B K-major)", args(0, X, Y, W, 0)),
                ("fwd + relu epilogue", fr),
                ("dgrad(B MN-major)", args(0, X, Y, W, 1, flip=True)),
                ("dgrad(B K-major, W^T)", args(0, X, Y, WT, 0, flip=True)),
                ("dgrad(W^T) + mask epilogue", dm),
                ] + ([] if os.environ.get("GRAPH") == "1" and SKWS is None and WS is None else [("wgrad", args(1, X, dW))]):
    ms = timeit(a)
    print(f"{name:24s} {ms * 1e3:8.1f} us  {flops / ms / 1e9:7.1f} TF/s")
