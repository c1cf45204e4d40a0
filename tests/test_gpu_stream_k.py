"""GPU parity of the stream-K work split (common.cuh WorkList) in the implicit-GEMM convolution kernel: a
WResNet-like 3x3 convolution (16 x 14 x 14 pixels, 768 channels) whose output tiles cannot fill 148 SMs
evenly (75 tiles for the forward / data gradient, 162 for the weight gradient; all compute-bound), so tiles' k-loops are cut across CTAs
and finished from the fp32 partials of the others.  Forward (with the fused add+relu+mask
epilogue), data gradient (MN-major weights, flipped taps) and weight gradient (store and fused momentum-SGD)
against the oracle's fp64 evaluation of the convolution TDL defs (cross-checked with torch's fp64 convolution)
on the same bf16-exact inputs, and against the same launch without a stream-K workspace.  Tolerances as the north star: bf16 outputs normwise <= 5e-3,
fp32 <= 1e-5."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

B, H, C = 16, 14, 768


def _tofu():
    from paper_1807_08887_b200 import tofu
    tofu.lib()
    return tofu


def nrm(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def q(rng, shape, scale):
    return rng.integers(-128, 129, size=shape).astype(np.float64) * scale


def conv_args(t, kind, S, out, Bmat=None, mn=0, flip=False, Y=None):
    a = t.ConvArgs()
    a.kind = kind
    a.nb, a.ngy, a.ngx = B, H, H
    a.ay = a.ax = 1
    a.cy = a.cx = 1 if flip else -1
    a.ntaps = 9
    for k in range(9):
        ky, kx = divmod(k, 3)
        a.tap_dy[k], a.tap_dx[k] = (-ky, -kx) if flip else (ky, kx)
        a.tap_w[k] = k
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


@pytest.fixture(scope="module")
def data():
    rng = np.random.default_rng(31)
    X = q(rng, (B, H, H, C), 2 ** -7)
    W = q(rng, (C, 3, 3, C), 2 ** -11)        # [co][ky][kx][ci]
    D = q(rng, (B, H, H, C), 2 ** -7)         # an output gradient
    Xt = torch.from_numpy(X).permute(0, 3, 1, 2)
    Wt = torch.from_numpy(W).permute(0, 3, 1, 2)
    Dt = torch.from_numpy(D).permute(0, 3, 1, 2)
    # references: the oracle's evaluation of the convolution TDL defs (oracle.exec_ref.fast_eval, fp64), checked
    # against torch's fp64 convolution as a second, independent computation
    from oracle.exec_ref import fast_eval
    from oracle.tdl import parse_def
    from tofu_inputs.graphs import conv_defs
    defs = {n: parse_def(src) for n, src in conv_defs(3, 1, 1).items()}
    z4 = (0, 0, 0, 0)
    full = lambda **kw: {v: (0, n - 1) for v, n in kw.items()}
    ref = {
        "fwd": fast_eval(defs["conv_k3s1p1"], {"X": (X, z4), "W": (W, z4)},
                         full(b=B, y=H, x=H, co=C, ky=3, kx=3, ci=C)),
        "dgrad": fast_eval(defs["dconv_k3s1p1"], {"D": (D, z4), "W": (W, z4)},
                           full(b=B, y=H, x=H, ci=C, ky=3, kx=3, co=C)),
        "wgrad": fast_eval(defs["wconv_k3s1p1"], {"D": (D, z4), "X": (X, z4)},
                           full(co=C, ky=3, kx=3, ci=C, b=B, y=H, x=H)),
    }
    F = torch.nn.functional
    tref = {
        "fwd": F.conv2d(Xt, Wt, padding=1).permute(0, 2, 3, 1).numpy(),
        "dgrad": F.conv_transpose2d(Dt, Wt, padding=1).permute(0, 2, 3, 1).numpy(),
        "wgrad": torch.nn.grad.conv2d_weight(Xt, Wt.shape, Dt, padding=1).permute(0, 2, 3, 1).numpy(),
    }
    for k in ref:
        assert nrm(np.asarray(ref[k]), tref[k]) < 1e-12, k
    return rng, X, W, D, ref


def cuda_bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).cuda()


@pytest.mark.parametrize("which", ["fwd", "fwd_ep", "dgrad", "wgrad", "wgrad_opt"])
def test_conv_stream_k(data, which):
    t = _tofu()
    rng, X, W, D, ref = data
    ws = torch.zeros(t.sk_workspace_bytes(), dtype=torch.uint8, device="cuda")
    Xd, Wd, Dd = cuda_bf16(X), cuda_bf16(W), cuda_bf16(D)
    add, mask = q(rng, (B, H, H, C), 2 ** -6), q(rng, (B, H, H, C), 2 ** -6)
    M0, W0 = q(rng, (C, 3, 3, C), 2 ** -12), q(rng, (C, 3, 3, C), 2 ** -7)
    mu, lr = 0.875, 0.0078125
    outs = []
    for sk in (ws, None, ws):
        keep = []
        if which.startswith("fwd") or which == "dgrad":
            out = torch.zeros((B, H, H, C), dtype=torch.bfloat16, device="cuda")
            a = (conv_args(t, 0, Xd, out, Wd, 0) if which != "dgrad"
                 else conv_args(t, 0, Dd, out, Wd, 1, flip=True))
            if which == "fwd_ep":
                keep = [cuda_bf16(add), cuda_bf16(mask)]
                a.ep, a.aux_add, a.aux_mask = 7, keep[0].data_ptr(), keep[1].data_ptr()
        else:
            out = (torch.from_numpy(M0).float().cuda() if which == "wgrad_opt"
                   else torch.zeros((C, 3, 3, C), dtype=torch.float32, device="cuda"))
            a = conv_args(t, 1, Xd, out, Y=Dd)
            if which == "wgrad_opt":
                keep = [cuda_bf16(W0)]
                a.c_mode, a.D, a.ldd, a.s0, a.s1 = 3, keep[0].data_ptr(), 9 * C, mu, lr
            a.splits = 1   # stream-K (with ws) vs one data-parallel pass (without)
        a.sk_ws = sk.data_ptr() if sk is not None else None
        t.conv(a)
        torch.cuda.synchronize()
        outs.append((out.double().cpu().numpy(), keep[0].double().cpu().numpy() if which == "wgrad_opt" else None))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    assert int(ws[-sms * 32:].count_nonzero()) == 0          # flags lowered by the finishers
    assert np.array_equal(outs[0][0], outs[2][0])            # deterministic
    got, plain = outs[0][0], outs[1][0]
    if which in ("fwd", "dgrad"):
        assert nrm(got, ref[which]) <= 5e-3
        assert nrm(got, plain) <= 5e-3
    elif which == "fwd_ep":
        r = np.where(mask > 0, np.maximum(ref["fwd"] + add, 0.0), 0.0)
        assert nrm(got, r) <= 5e-3
    elif which == "wgrad":
        assert nrm(got, ref["wgrad"]) <= 1e-5
        assert nrm(got, plain) <= 1e-5
    else:
        mref = M0 * mu + ref["wgrad"]
        assert nrm(got, mref) <= 1e-5
        assert nrm(outs[0][1], np.asarray(torch.from_numpy(W0 - got * lr).to(torch.bfloat16).double())) <= 5e-3


@pytest.mark.parametrize("which", ["fwd", "fwd_ep", "dgrad", "wgrad", "wgrad_opt"])
def test_conv_im2col_equals_gather(data, which):
    """The activation operand loaded by TMA in im2col mode (tofu_conv_args.im2col; the A operand of the forward
    / data gradient, the B operand of the weight gradient) vs the cp.async gather warps: the same operand tiles
    reach the tensor cores, so the outputs are bitwise equal; both within tolerance of the fp64 convolution."""
    t = _tofu()
    rng, X, W, D, ref = data
    Xd, Wd, Dd = cuda_bf16(X), cuda_bf16(W), cuda_bf16(D)
    add, mask = q(rng, (B, H, H, C), 2 ** -6), q(rng, (B, H, H, C), 2 ** -6)
    keep = [cuda_bf16(add), cuda_bf16(mask)]
    outs, modes = [], []
    M0, W0 = q(rng, (C, 3, 3, C), 2 ** -12), q(rng, (C, 3, 3, C), 2 ** -7)
    for i2c in (-1, 0):
        if which.startswith("wgrad"):   # kind 1: the gathered activations are the B operand
            out = (torch.from_numpy(M0).float().cuda() if which == "wgrad_opt"
                   else torch.zeros((C, 3, 3, C), dtype=torch.float32, device="cuda"))
            a = conv_args(t, 1, Xd, out, Y=Dd)
            if which == "wgrad_opt":
                keep = [cuda_bf16(W0)]
                a.c_mode, a.D, a.ldd, a.s0, a.s1 = 3, keep[0].data_ptr(), 9 * C, 0.875, 0.0078125
        else:
            out = torch.zeros((B, H, H, C), dtype=torch.bfloat16, device="cuda")
            a = (conv_args(t, 0, Xd, out, Wd, 0) if which != "dgrad" else conv_args(t, 0, Dd, out, Wd, 1, flip=True))
            if which == "fwd_ep":
                a.ep, a.aux_add, a.aux_mask = 7, keep[0].data_ptr(), keep[1].data_ptr()
        a.im2col = i2c
        modes.append(t.conv_plan(a).im2col)
        t.conv(a)
        torch.cuda.synchronize()
        outs.append(out.double().cpu().numpy())
    assert modes == [0, 1]
    assert np.array_equal(outs[0], outs[1])
    if which.startswith("wgrad"):
        r = ref["wgrad"] + (M0 * 0.875 if which == "wgrad_opt" else 0.0)
        assert nrm(outs[1], r) <= 1e-5
        return
    r = ref["dgrad" if which == "dgrad" else "fwd"]
    if which == "fwd_ep":
        r = np.where(mask > 0, np.maximum(r + add, 0.0), 0.0)
    assert nrm(outs[1], r) <= 5e-3


@pytest.mark.parametrize("kind", [0, 1])
def test_conv_im2col_stride2(kind):
    """Stride-2 3x3 convolution (pad 1, the stage transitions of WResNet): the im2col map walks the input with
    traversal stride 2 (elementStrides) — forward (kind 0) and weight gradient (kind 1), bitwise equal to the
    gather path and within tolerance of the fp64 convolution."""
    t = _tofu()
    Bs, Hs, Cs = 8, 28, 256
    Ho = Hs // 2
    rng = np.random.default_rng(57)
    X = q(rng, (Bs, Hs, Hs, Cs), 2 ** -7)
    W = q(rng, (Cs, 3, 3, Cs), 2 ** -10)
    D = q(rng, (Bs, Ho, Ho, Cs), 2 ** -7)
    F = torch.nn.functional
    Xt, Wt, Dt = (torch.from_numpy(v) for v in (X, W, D))
    Xd, Wd, Dd = cuda_bf16(X), cuda_bf16(W), cuda_bf16(D)

    def args(out):
        a = t.ConvArgs()
        a.kind = kind
        a.nb, a.ngy, a.ngx = Bs, Ho, Ho
        a.ay = a.ax = 2
        a.cy = a.cx = -1
        a.ntaps = 9
        for k in range(9):
            a.tap_dy[k], a.tap_dx[k] = divmod(k, 3)
            a.tap_w[k] = k
        a.nch = Cs
        a.S = Xd.data_ptr()
        a.s_sb, a.s_sy, a.s_sx = Hs * Hs * Cs, Hs * Cs, Cs
        a.sH = a.sW = Hs
        if kind == 0:
            a.n_out = Cs
            a.Bp = Wd.data_ptr()
            a.ldb = 9 * Cs
            a.b_tap = Cs
            a.b_rows, a.b_cols = Cs, 9 * Cs
            a.C = out.data_ptr()
            a.c_sb, a.c_sy, a.c_sx = Ho * Ho * Cs, Ho * Cs, Cs
            a.c_ys = a.c_xs = 1
        else:
            a.m_out = Cs
            a.Ap = Dd.data_ptr()
            a.lda = Cs
            a.C = out.data_ptr()
            a.ldc = 9 * Cs
            a.c_mode = 1
            a.splits = 1
        return a

    outs, modes = [], []
    for i2c in (-1, 0):
        out = (torch.zeros((Bs, Ho, Ho, Cs), dtype=torch.bfloat16, device="cuda") if kind == 0
               else torch.zeros((Cs, 3, 3, Cs), dtype=torch.float32, device="cuda"))
        a = args(out)
        a.im2col = i2c
        modes.append(t.conv_plan(a).im2col)
        t.conv(a)
        torch.cuda.synchronize()
        outs.append(out.double().cpu().numpy())
    assert modes == [0, 1]
    assert np.array_equal(outs[0], outs[1])
    # reference: the oracle's evaluation of the stride-2 convolution TDL (R11), cross-checked with torch fp64
    from oracle.exec_ref import fast_eval
    from oracle.tdl import parse_def
    from tofu_inputs.graphs import conv_defs
    defs = {n: parse_def(src) for n, src in conv_defs(3, 2, 1).items()}
    z4 = (0, 0, 0, 0)
    if kind == 0:
        ref = fast_eval(defs["conv_k3s2p1"], {"X": (X, z4), "W": (W, z4)},
                        {"b": (0, Bs - 1), "y": (0, Ho - 1), "x": (0, Ho - 1), "co": (0, Cs - 1), "ky": (0, 2),
                         "kx": (0, 2), "ci": (0, Cs - 1)})
        tref = F.conv2d(Xt.permute(0, 3, 1, 2), Wt.permute(0, 3, 1, 2), stride=2, padding=1).permute(0, 2, 3, 1).numpy()
        assert nrm(np.asarray(ref), tref) < 1e-12
        assert nrm(outs[1], ref) <= 5e-3
    else:
        ref = fast_eval(defs["wconv_k3s2p1"], {"D": (D, z4), "X": (X, z4)},
                        {"co": (0, Cs - 1), "ky": (0, 2), "kx": (0, 2), "ci": (0, Cs - 1), "b": (0, Bs - 1),
                         "y": (0, Ho - 1), "x": (0, Ho - 1)})
        tref = torch.nn.grad.conv2d_weight(Xt.permute(0, 3, 1, 2), (Cs, Cs, 3, 3), Dt.permute(0, 3, 1, 2), stride=2,
                                           padding=1).permute(0, 2, 3, 1).numpy()
        assert nrm(np.asarray(ref), tref) < 1e-12
        assert nrm(outs[1], ref) <= 1e-5


@pytest.mark.parametrize("which", ["wgrad", "wgrad_opt"])
def test_conv_wgrad_cluster_pairs(data, which):
    """Weight gradient as clusters of 2 CTAs on adjacent output-channel tiles sharing the im2col-loaded
    activations (tofu_conv_args.cl2): multicast halves (bitwise equal to the single-CTA launch) and 2-CTA MMA
    pairs (cta_group::2, each CTA staging half of the activation tile; equal within fp32 rounding)."""
    t = _tofu()
    rng, X, W, D, ref = data
    Xd, Dd = cuda_bf16(X), cuda_bf16(D)
    M0, W0 = q(rng, (C, 3, 3, C), 2 ** -12), q(rng, (C, 3, 3, C), 2 ** -7)
    outs, modes = [], []
    for cl2 in (-1, 2, 4):
        out = (torch.from_numpy(M0).float().cuda() if which == "wgrad_opt"
               else torch.zeros((C, 3, 3, C), dtype=torch.float32, device="cuda"))
        a = conv_args(t, 1, Xd, out, Y=Dd)
        keep = []
        if which == "wgrad_opt":
            keep = [cuda_bf16(W0)]
            a.c_mode, a.D, a.ldd, a.s0, a.s1 = 3, keep[0].data_ptr(), 9 * C, 0.875, 0.0078125
        a.splits = 1
        a.cl2 = cl2
        modes.append(t.conv_plan(a).cl2)
        t.conv(a)
        torch.cuda.synchronize()
        outs.append((out.double().cpu().numpy(), keep[0].double().cpu().numpy() if keep else None))
    assert modes == [0, 1, 3]   # single CTA, multicast pairs, 2-CTA MMA pairs
    assert np.array_equal(outs[0][0], outs[1][0])
    assert nrm(outs[2][0], outs[0][0]) <= 1e-6
    if which == "wgrad_opt":
        assert np.array_equal(outs[0][1], outs[1][1])
        assert nrm(outs[2][1], outs[0][1]) <= 2e-3
        assert nrm(outs[1][0], M0 * 0.875 + ref["wgrad"]) <= 1e-5
    else:
        assert nrm(outs[1][0], ref["wgrad"]) <= 1e-5


@pytest.mark.parametrize("which", ["fwd", "fwd_ep", "dgrad_kmajor"])
def test_conv_fwd_2cta_mma(data, which):
    """Forward / data gradient (K-major weights) with 2-CTA MMA pairs over adjacent pixel tiles
    (tofu_conv_args.cl2 = 3: each CTA im2col-loads its 128 pixels and half of the weight tile, the leader
    issues M = 256 MMAs): equal to the single-CTA launch and within tolerance of the fp64 convolution."""
    t = _tofu()
    rng, X, W, D, ref = data
    Xd, Dd = cuda_bf16(X), cuda_bf16(D)
    Wd = cuda_bf16(W)
    WT = cuda_bf16(np.ascontiguousarray(W.transpose(3, 1, 2, 0)))   # [ci][ky][kx][co]: K-major for the dgrad
    add, mask = q(rng, (B, H, H, C), 2 ** -6), q(rng, (B, H, H, C), 2 ** -6)
    keep = [cuda_bf16(add), cuda_bf16(mask)]
    outs, modes = [], []
    for cl2 in (-1, 4):
        out = torch.zeros((B, H, H, C), dtype=torch.bfloat16, device="cuda")
        if which == "dgrad_kmajor":
            # tap k = (ky, kx) reads D at (y + 1 - ky, x + 1 - kx) and the weight column block (ky, kx) of
            # WT[ci][ky][kx][co] (K-major: rows = ci)
            a = conv_args(t, 0, Dd, out, WT, 0, flip=True)
        else:
            a = conv_args(t, 0, Xd, out, Wd, 0)
        if which == "fwd_ep":
            a.ep, a.aux_add, a.aux_mask = 7, keep[0].data_ptr(), keep[1].data_ptr()
        a.cl2 = cl2
        modes.append(t.conv_plan(a).cl2)
        t.conv(a)
        torch.cuda.synchronize()
        outs.append(out.double().cpu().numpy())
    assert modes == [0, 3]
    assert nrm(outs[1], outs[0]) <= 2e-3
    r = ref["dgrad" if which == "dgrad_kmajor" else "fwd"]
    if which == "fwd_ep":
        r = np.where(mask > 0, np.maximum(r + add, 0.0), 0.0)
    assert nrm(outs[1], r) <= 5e-3


@pytest.mark.parametrize("which", ["fwd", "fwd_ep", "fwd_f32", "dgrad"])
def test_conv_fwd_dgrad_split_k(data, which):
    """Split-K for a few-tile forward / data-gradient launch (a rank's sub-op under a k-way plan; chosen when the
    caller passes a workspace): the fp32 partial planes summed in split order by splitk_reduce_rows, which also
    applies the fused add / relu / mask epilogue or stores fp32 (c_mode 1).  4 of the 16 images (21 tiles): checked
    against the oracle's fp64 evaluation of the TDL defs and the one-pass launch; deterministic."""
    t = _tofu()
    rng, X, W, D, ref = data
    nb = 4
    Xd, Wd, Dd = cuda_bf16(X[:nb]), cuda_bf16(W), cuda_bf16(D[:nb])
    add, mask = q(rng, (nb, H, H, C), 2 ** -6), q(rng, (nb, H, H, C), 2 ** -6)
    keep = [cuda_bf16(add), cuda_bf16(mask)]
    ws = torch.zeros(16 * nb * H * H * C, dtype=torch.float32, device="cuda")
    outs = []
    for use_ws in (True, False, True):
        f32 = which == "fwd_f32"
        out = torch.zeros((nb, H, H, C), dtype=torch.float32 if f32 else torch.bfloat16, device="cuda")
        a = (conv_args(t, 0, Dd, out, Wd, 1, flip=True) if which == "dgrad" else conv_args(t, 0, Xd, out, Wd, 0))
        a.nb = nb
        if f32:
            a.c_mode = 1
        if which == "fwd_ep":
            a.ep, a.aux_add, a.aux_mask = 7, keep[0].data_ptr(), keep[1].data_ptr()
        a.ws = ws.data_ptr() if use_ws else None
        planned = t.conv_plan(a)
        assert (planned.splits > 1) == use_ws, planned.splits
        t.conv(a)
        torch.cuda.synchronize()
        outs.append(out.double().cpu().numpy())
    assert np.array_equal(outs[0], outs[2])  # deterministic (split order)
    got, plain = outs[0], outs[1]
    r = ref["dgrad" if which == "dgrad" else "fwd"][:nb]
    if which == "fwd_ep":
        r = np.where(mask > 0, np.maximum(r + add, 0.0), 0.0)
    tol = 1e-5 if which == "fwd_f32" else 5e-3
    assert nrm(got, r) <= tol
    assert nrm(got, plain) <= tol
