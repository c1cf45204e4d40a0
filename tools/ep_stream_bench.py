"""The headline's HBM-bound GEMM class: WResNet-152-4 b32 stage-0 1x1 convolutions as GEMMs with fused
element-wise epilogues (the dominant launch is s0 conv1's data gradient, [100352 x 1024] = dY[100352 x 256] W,
+ residual gradient, relu-gradient mask).  Prints per shape: us, algorithmic GB/s (operands once + output side
bytes) and the fraction of the measured HBM copy peak.  Inputs are larger than L2 (no flush needed).

  python tools/ep_stream_bench.py            # env switches (TOFU_EW8, TOFU_CL2, TOFU_C2W8, TOFU_EP_BN, ...) apply
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_08887_b200 import tofu  # noqa: E402

PEAK = 6448.1
try:
    PEAK = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass


def bench(fn, it=30):
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


# (name, M, N, K, b_mn, ep): ep bit 0 relu, bit 1 add, bit 2 mask
SHAPES = [
    ("s0.conv1_dgrad+add+mask", 100352, 1024, 256, 1, 6),
    ("s0.conv3_fwd+add+relu", 100352, 1024, 256, 0, 3),
    ("s0.conv3_dgrad+mask", 100352, 256, 1024, 1, 4),
    ("s0.conv1_fwd+relu", 100352, 256, 1024, 0, 1),
    ("s1.conv1_dgrad+add+mask", 25088, 2048, 512, 1, 6),
]


def main():
    torch.manual_seed(0)
    only = [a for a in sys.argv[1:] if "," not in a] or None
    shapes = [("custom",) + tuple(int(x) for x in a.split(",")) for a in sys.argv[1:] if "," in a]
    if shapes and not only:
        only = ["custom"]
    for name, M, N, K, b_mn, ep in SHAPES + shapes:
        if only and not any(o in name for o in only):
            continue
        a = (torch.randn(M, K, device="cuda") * 0.1).bfloat16()
        b = (torch.randn(K, N, device="cuda") * 0.1).bfloat16() if b_mn else (torch.randn(N, K, device="cuda") * 0.1).bfloat16()
        add = torch.randn(M, N, device="cuda").bfloat16() if ep & 2 else None
        mask = torch.randn(M, N, device="cuda").bfloat16() if ep & 4 else None
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ldb = N if b_mn else K
        fn = lambda: tofu.gemm(a, b, c, M, N, K, K, 0, ldb, b_mn, N, 0, aux_add=add, aux_mask=mask, ep=ep)  # noqa
        t = bench(fn)
        nbytes = 2 * M * K + 2 * N * K + M * N * (2 + 2 * ((ep >> 1) & 1) + 2 * ((ep >> 2) & 1))
        gbs = nbytes / t / 1e6
        # parity spot check (fp32 reference of a few rows)
        rows = torch.arange(0, M, max(1, M // 64), device="cuda")
        ref = a[rows].float() @ (b.float() if b_mn else b.float().t())
        if ep & 2:
            ref += add[rows].float()
        if ep & 1:
            ref = ref.clamp_min(0)
        if ep & 4:
            ref = torch.where(mask[rows].float() > 0, ref, torch.zeros_like(ref))
        err = float((c[rows].float() - ref).abs().max() / ref.abs().max().clamp_min(1e-6))
        print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "ep": ep, "us": round(t * 1e3, 2),
                          "GBps": round(gbs, 1), "frac": round(gbs / PEAK, 3), "maxrel": float(f"{err:.2e}")}),
              flush=True)
        del a, b, add, mask, c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
