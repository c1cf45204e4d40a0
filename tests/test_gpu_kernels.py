"""GPU parity: kernels of libtofu vs the oracle (fp64) on the same seeded
bf16-exact inputs.  Tolerances (north star): normwise relative error <= 5e-3
for bf16 outputs, <= 1e-5 for fp32 outputs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.exec_ref import fast_eval, round_bf16  # noqa: E402
from oracle.tdl import parse_def  # noqa: E402
from tofu_inputs.graphs import MM_DEFS  # noqa: E402


def _tofu():
    from paper_1807_08887_b200 import tofu
    tofu.lib()
    return tofu


def nrm(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def q(rng, shape, scale):
    return rng.integers(-128, 129, size=shape).astype(np.float64) * scale


def cuda_bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).cuda()


DEF_MAJOR = {"mm_nn": (0, 1), "mm_nt": (0, 0), "mm_tn": (1, 1)}


@pytest.mark.parametrize("defname", ["mm_nn", "mm_nt", "mm_tn"])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (200, 300, 104), (64, 520, 1000), (512, 1024, 2048),
                                   (1, 8, 8), (384, 128, 4096)])
@pytest.mark.parametrize("c_mode", [0, 1, 2])
def test_gemm_parity(defname, M, N, K, c_mode):
    t = _tofu()
    am, bm = DEF_MAJOR[defname]
    if (am and M % 8) or (bm and N % 8) or (not am and K % 8) or (not bm and K % 8):
        pytest.skip("pitch must be a multiple of 8 elements")
    if (N * (2 if c_mode == 0 else 4)) % 16:
        pytest.skip("output pitch must be a multiple of 16 bytes (TMA store)")
    rng = np.random.default_rng(M * 7 + N * 13 + K)
    a_shape = (K, M) if am else (M, K)
    b_shape = (K, N) if bm else (N, K)
    A = q(rng, a_shape, 2 ** -7)
    B = q(rng, b_shape, 2 ** -9)
    d = parse_def(MM_DEFS[defname])
    ref = fast_eval(d, {"A": (A, (0, 0)), "B": (B, (0, 0))},
                    {"i": (0, M - 1), "j": (0, N - 1), "k": (0, K - 1)})
    Ad, Bd = cuda_bf16(A), cuda_bf16(B)
    if c_mode == 0:
        Cd = torch.full((M, N), 7.0, dtype=torch.bfloat16, device="cuda")
    else:
        C0 = q(rng, (M, N), 2 ** -5) if c_mode == 2 else np.zeros((M, N))
        Cd = torch.from_numpy(C0).float().cuda()
        if c_mode == 2:
            ref = ref + C0
    t.gemm(Ad, Bd, Cd, M, N, K, lda=a_shape[1], a_mn=am, ldb=b_shape[1], b_mn=bm, ldc=N, c_mode=c_mode)
    torch.cuda.synchronize()
    got = Cd.double().cpu().numpy()
    if c_mode == 0:
        assert nrm(got, ref) <= 5e-3
        # most elements equal the correctly rounded fp64 result
        assert np.mean(got == round_bf16(ref)) > 0.97
    else:
        assert nrm(got, ref) <= 1e-5


@pytest.mark.parametrize("defname", ["mm_tn", "mm_nn"])
@pytest.mark.parametrize("M,N,K,splits", [(256, 512, 128, 0), (200, 328, 72, 0), (1024, 2048, 512, 0),
                                          (256, 512, 2048, 4), (200, 328, 1000, 3)])
def test_gemm_fused_momentum_sgd(defname, M, N, K, splits):
    """c_mode 3: M = M*mu + A.B (fp32, 1e-5), W = bf16(W - lr*M) (5e-3); with split-K the optimizer is
    applied by the ordered reduction (vectorised when N is a multiple of 4, scalar otherwise)."""
    t = _tofu()
    am, bm = DEF_MAJOR[defname]
    rng = np.random.default_rng(M + N + K)
    a_shape = (K, M) if am else (M, K)
    b_shape = (K, N) if bm else (N, K)
    A, B = q(rng, a_shape, 2 ** -7), q(rng, b_shape, 2 ** -9)
    d = parse_def(MM_DEFS[defname])
    acc = fast_eval(d, {"A": (A, (0, 0)), "B": (B, (0, 0))}, {"i": (0, M - 1), "j": (0, N - 1), "k": (0, K - 1)})
    M0 = q(rng, (M, N), 2 ** -12)
    W0 = q(rng, (M, N), 2 ** -7)
    Md = torch.from_numpy(M0).float().cuda()
    Wd = cuda_bf16(W0)
    mu, lr = 0.875, 0.0078125
    t.gemm(cuda_bf16(A), cuda_bf16(B), Md, M, N, K, a_shape[1], am, b_shape[1], bm, N, 3, D=Wd, ldd=N, s0=mu, s1=lr,
           splits=splits)
    torch.cuda.synchronize()
    mref = M0 * mu + acc
    got_m = Md.double().cpu().numpy()
    assert nrm(got_m, mref) <= 1e-5
    wref = round_bf16(W0 - got_m * lr)
    assert nrm(Wd.double().cpu().numpy(), wref) <= 5e-3


@pytest.mark.parametrize("defname", ["mm_nn", "mm_nt", "mm_tn"])
@pytest.mark.parametrize("M,N,K,splits", [(128, 4096, 16384, 0), (128, 512, 4096, 5), (200, 264, 3000, 3),
                                          (64, 256, 1024, 16)])
@pytest.mark.parametrize("c_mode", [0, 1, 2])
def test_gemm_split_k(defname, M, N, K, splits, c_mode):
    """Split-K (auto for few output tiles, or forced) reduces fp32 partials in
    fixed split order: same tolerances as the unsplit GEMM, and deterministic."""
    t = _tofu()
    am, bm = DEF_MAJOR[defname]
    if (am and M % 8) or (not am and K % 8) or (N * (2 if c_mode == 0 else 4)) % 16:
        pytest.skip("pitch")
    rng = np.random.default_rng(M + 3 * N + K)
    a_shape = (K, M) if am else (M, K)
    b_shape = (K, N) if bm else (N, K)
    A, B = q(rng, a_shape, 2 ** -7), q(rng, b_shape, 2 ** -9)
    d = parse_def(MM_DEFS[defname])
    ref = fast_eval(d, {"A": (A, (0, 0)), "B": (B, (0, 0))}, {"i": (0, M - 1), "j": (0, N - 1), "k": (0, K - 1)})
    C0 = q(rng, (M, N), 2 ** -5) if c_mode == 2 else np.zeros((M, N))
    if c_mode == 2:
        ref = ref + C0
    outs = []
    for rep in range(2):
        Cd = (torch.from_numpy(C0).float().cuda() if c_mode else torch.zeros((M, N), dtype=torch.bfloat16, device="cuda"))
        t.gemm(cuda_bf16(A), cuda_bf16(B), Cd, M, N, K, a_shape[1], am, b_shape[1], bm, N, c_mode, splits=splits)
        torch.cuda.synchronize()
        outs.append(Cd.double().cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    assert nrm(outs[0], ref) <= (5e-3 if c_mode == 0 else 1e-5)


@pytest.mark.parametrize("M,N,K", [(1000, 2048, 1024),      # 64 tiles < 148 SMs: every tile stream-K (splits=-1)
                                   (6272, 1024, 4096),      # 196 tiles (WResNet stage-2 1x1): all stream-K
                                   (2600, 2304, 520),       # 189 tiles, ragged M/N/K tails
                                   (3840, 3072, 512)])      # 360 tiles: 148 data-parallel + 212 stream-K
@pytest.mark.parametrize("mode", [0, 1, 2, 3, 5])
def test_gemm_stream_k(M, N, K, mode):
    """Stream-K (common.cuh WorkList): tiles whose k-loop is cut across CTAs are finished by adding the other
    CTAs' fp32 partials in CTA order.  Same tolerances as the data-parallel GEMM, bitwise deterministic, the
    workspace flags left zeroed; mode 5 = bf16 output with the fused add+relu+mask epilogue (ep = 7)."""
    t = _tofu()
    rng = np.random.default_rng(M + N + K + mode)
    A, B = q(rng, (M, K), 2 ** -7), q(rng, (N, K), 2 ** -9)   # mm_nt: both K-major
    acc = A @ B.T
    c_mode = 0 if mode == 5 else mode
    ws = torch.zeros(t.sk_workspace_bytes(), dtype=torch.uint8, device="cuda")
    C0 = q(rng, (M, N), 2 ** -5) if mode in (2, 3) else np.zeros((M, N))
    W0 = q(rng, (M, N), 2 ** -7)
    X0, K0 = q(rng, (M, N), 2 ** -6), q(rng, (M, N), 2 ** -6)
    outs = []
    for rep in range(2):
        kw = {}
        if mode in (1, 2, 3):
            Cd = torch.from_numpy(C0).float().cuda()
        else:
            Cd = torch.zeros((M, N), dtype=torch.bfloat16, device="cuda")
        if mode == 3:
            kw = dict(D=cuda_bf16(W0), ldd=N, s0=0.875, s1=0.0078125)
        if mode == 5:
            kw = dict(aux_add=cuda_bf16(X0), aux_mask=cuda_bf16(K0), ep=7)
        t.gemm(cuda_bf16(A), cuda_bf16(B), Cd, M, N, K, K, 0, K, 0, N, c_mode, sk_ws=ws, splits=-1, **kw)
        torch.cuda.synchronize()
        outs.append((Cd.double().cpu().numpy(), kw["D"].double().cpu().numpy() if mode == 3 else None))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    assert int(ws[-sms * 32:].count_nonzero()) == 0   # flags lowered again by the finishers
    assert np.array_equal(outs[0][0], outs[1][0])
    got = outs[0][0]
    if mode == 0:
        assert nrm(got, acc) <= 5e-3
        assert np.mean(got == round_bf16(acc)) > 0.97
    elif mode == 1:
        assert nrm(got, acc) <= 1e-5
    elif mode == 2:
        assert nrm(got, C0 + acc) <= 1e-5
    elif mode == 3:
        mref = C0 * 0.875 + acc
        assert nrm(got, mref) <= 1e-5
        assert nrm(outs[0][1], round_bf16(W0 - got * 0.0078125)) <= 5e-3
    else:
        ref = np.where(K0 > 0, np.maximum(acc + X0, 0.0), 0.0)
        assert nrm(got, ref) <= 5e-3


def test_gemm_strided_output_and_bn():
    t = _tofu()
    rng = np.random.default_rng(9)
    M, N, K = 256, 512, 256
    A, B = q(rng, (M, K), 2 ** -7), q(rng, (K, N), 2 ** -7)
    for bn in (128, 256):
        Cd = torch.zeros((M, N + 64), dtype=torch.float32, device="cuda")
        t.gemm(cuda_bf16(A), cuda_bf16(B), Cd, M, N, K, K, 0, N, 1, N + 64, 1, bn=bn, max_ctas=3)
        torch.cuda.synchronize()
        got = Cd.double().cpu().numpy()
        assert nrm(got[:, :N], A @ B) <= 1e-5
        assert np.all(got[:, N:] == 0)


@pytest.mark.parametrize("kind", ["relu", "relu_grad", "mse_grad", "mom", "sgd", "sgd_mom", "sumsq"])
@pytest.mark.parametrize("n", [8, 1000, 1 << 20, 3 * 1024 + 5])
def test_elementwise(kind, n):
    t = _tofu()
    rng = np.random.default_rng(n)
    a = q(rng, n, 2 ** -7)
    b = q(rng, n, 2 ** -7)
    s0, s1 = 0.875, 0.0078125
    if kind in ("relu", "relu_grad", "mse_grad", "sumsq"):
        x0, x1 = cuda_bf16(a), cuda_bf16(b)
        y = torch.zeros(n, dtype=torch.float32 if kind == "sumsq" else torch.bfloat16, device="cuda")
        if kind == "sumsq":
            y = torch.zeros(4, dtype=torch.float32, device="cuda")
        t.elementwise(kind, n, y, x0, x1 if kind != "relu" else None, None, s0, s1)
        torch.cuda.synchronize()
        got = y.double().cpu().numpy()
        if kind == "relu":
            ref = round_bf16(np.maximum(a, 0))
        elif kind == "relu_grad":
            ref = round_bf16(np.where(a > 0, b, 0))
        elif kind == "mse_grad":
            ref = round_bf16((a - b) * s0)
        else:
            assert abs(got[0] - np.sum((a - b) ** 2) * s0) <= 1e-5 * np.sum((a - b) ** 2) * s0
            return
        assert np.array_equal(got, ref)
    elif kind == "mom":
        x0 = torch.from_numpy(a).float().cuda(); x1 = torch.from_numpy(b).float().cuda()
        y = torch.empty(n, dtype=torch.float32, device="cuda")
        t.elementwise(kind, n, y, x0, x1, None, s0, s1)
        torch.cuda.synchronize()
        assert nrm(y.double().cpu().numpy(), a * s0 + b) <= 1e-6
    elif kind == "sgd":
        x0 = cuda_bf16(a); x1 = torch.from_numpy(b).float().cuda()
        y = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        t.elementwise(kind, n, y, x0, x1, None, s0, s1)
        torch.cuda.synchronize()
        assert nrm(y.double().cpu().numpy(), round_bf16(a - b * s0)) <= 5e-3
    else:
        m = torch.from_numpy(a * 2 ** -6).float().cuda(); g = torch.from_numpy(b).float().cuda()
        w = cuda_bf16(q(rng, n, 2 ** -7)); w0 = w.double().cpu().numpy()
        t.elementwise(kind, n, None, m, g, w, s0, s1)
        torch.cuda.synchronize()
        mref = a * 2 ** -6 * s0 + b
        assert nrm(m.double().cpu().numpy(), mref) <= 1e-6
        assert nrm(w.double().cpu().numpy(), round_bf16(w0 - mref * s1)) <= 5e-3


@pytest.mark.parametrize("co,taps,ci", [(1024, 9, 1024), (256, 49, 8), (72, 9, 200), (13, 9, 7)])
def test_transpose_taps(co, taps, ci):
    """The data gradients' K-major weight copy WT[ci][t][co] = W[co][t][ci]: a pure permutation, bit-exact
    (16-byte vector path when co and ci are multiples of 8, scalar path otherwise, ragged 64-tiles)."""
    t = _tofu()
    W = torch.randn(co, taps, ci, device="cuda").bfloat16()
    WT = torch.zeros(ci, taps, co, device="cuda", dtype=torch.bfloat16)
    t.transpose_taps(W, WT, co, taps, ci)
    torch.cuda.synchronize()
    assert torch.equal(WT.cpu(), W.permute(2, 1, 0).contiguous().cpu())


@pytest.mark.parametrize("M,N,K", [(1000, 2048, 1024), (6272, 1024, 640), (384, 512, 200)])
@pytest.mark.parametrize("am,bm", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("mode", [0, 1, 3, 5])
def test_gemm_cluster_pairs(M, N, K, am, bm, mode):
    """Cluster pairs sharing B (tofu_gemm_args.cl2: two CTAs on vertically adjacent tiles, each TMA-loading half
    of the B tile and multicasting it to both, a stage freed by both CTAs' MMA commits): bitwise equal to the
    single-CTA launch (same per-tile arithmetic), including an odd number of m tiles (the last pair's second
    tile lies past M) and a ragged K tail; within tolerance of fp64."""
    t = _tofu()
    rng = np.random.default_rng(M + N + K + mode + 3 * am + 5 * bm)
    A = q(rng, (K, M) if am else (M, K), 2 ** -7)
    B = q(rng, (K, N) if bm else (N, K), 2 ** -9)
    acc = (A.T if am else A) @ (B if bm else B.T)
    c_mode = 0 if mode == 5 else mode
    C0, W0 = q(rng, (M, N), 2 ** -5), q(rng, (M, N), 2 ** -7)
    X0, K0 = q(rng, (M, N), 2 ** -6), q(rng, (M, N), 2 ** -6)
    outs = []
    for cl2 in (-1, 2):
        kw = {}
        if mode in (1, 3):
            Cd = torch.from_numpy(C0 if mode == 3 else np.zeros((M, N))).float().cuda()
        else:
            Cd = torch.zeros((M, N), dtype=torch.bfloat16, device="cuda")
        if mode == 3:
            kw = dict(D=cuda_bf16(W0), ldd=N, s0=0.875, s1=0.0078125)
        if mode == 5:
            kw = dict(aux_add=cuda_bf16(X0), aux_mask=cuda_bf16(K0), ep=7)
        t.gemm(cuda_bf16(A), cuda_bf16(B), Cd, M, N, K, M if am else K, am, N if bm else K, bm, N, c_mode, splits=1,
               cl2=cl2, **kw)
        torch.cuda.synchronize()
        outs.append((Cd.double().cpu().numpy(), kw["D"].double().cpu().numpy() if mode == 3 else None))
    assert np.array_equal(outs[0][0], outs[1][0])
    if mode == 3:
        assert np.array_equal(outs[0][1], outs[1][1])
        assert nrm(outs[1][0], C0 * 0.875 + acc) <= 1e-5
    elif mode == 1:
        assert nrm(outs[1][0], acc) <= 1e-5
    elif mode == 0:
        assert nrm(outs[1][0], acc) <= 5e-3
    else:
        assert nrm(outs[1][0], np.where(K0 > 0, np.maximum(acc + X0, 0.0), 0.0)) <= 5e-3


@pytest.mark.parametrize("M,N,K", [(1000, 2048, 1024), (6272, 1024, 640), (384, 512, 200)])
@pytest.mark.parametrize("am,bm", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("mode", [0, 1, 3, 5])
def test_gemm_2cta_mma(M, N, K, am, bm, mode):
    """2-CTA MMA pairs (tcgen05.mma.cta_group::2, M = 256 over a cluster of 2: each CTA stages its own 128 rows
    of A and half of the B tile, the leader issues the MMAs, loads complete on the leader's barriers, both
    CTAs' epilogues read their TMEM halves): same results as the single-CTA launch, within tolerance of fp64."""
    t = _tofu()
    rng = np.random.default_rng(M + N + K + mode + 3 * am + 5 * bm + 1)
    A = q(rng, (K, M) if am else (M, K), 2 ** -7)
    B = q(rng, (K, N) if bm else (N, K), 2 ** -9)
    acc = (A.T if am else A) @ (B if bm else B.T)
    c_mode = 0 if mode == 5 else mode
    C0, W0 = q(rng, (M, N), 2 ** -5), q(rng, (M, N), 2 ** -7)
    X0, K0 = q(rng, (M, N), 2 ** -6), q(rng, (M, N), 2 ** -6)
    outs = []
    for cl2 in (-1, 4):
        kw = {}
        if mode in (1, 3):
            Cd = torch.from_numpy(C0 if mode == 3 else np.zeros((M, N))).float().cuda()
        else:
            Cd = torch.zeros((M, N), dtype=torch.bfloat16, device="cuda")
        if mode == 3:
            kw = dict(D=cuda_bf16(W0), ldd=N, s0=0.875, s1=0.0078125)
        if mode == 5:
            kw = dict(aux_add=cuda_bf16(X0), aux_mask=cuda_bf16(K0), ep=7)
        t.gemm(cuda_bf16(A), cuda_bf16(B), Cd, M, N, K, M if am else K, am, N if bm else K, bm, N, c_mode, splits=1,
               cl2=cl2, **kw)
        torch.cuda.synchronize()
        outs.append(Cd.double().cpu().numpy())
    if mode in (1, 3):
        assert nrm(outs[1], outs[0]) <= 1e-6
    else:
        assert nrm(outs[1], outs[0]) <= 2e-3
    ref = {0: acc, 1: acc, 3: C0 * 0.875 + acc, 5: np.where(K0 > 0, np.maximum(acc + X0, 0.0), 0.0)}[mode]
    assert nrm(outs[1], ref) <= (1e-5 if mode in (1, 3) else 5e-3)
