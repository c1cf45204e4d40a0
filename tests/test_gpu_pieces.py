"""MultiFetch / partition-n-reduce piece kernel (a5/a6, include/tofu.h tofu_pieces_tasks / tofu_pieces_run)
vs a torch reference: boxes of rank 1-4 cut from larger buffers (strided rows, odd offsets that force every
vector width), bf16 / fp32 sources and destinations, 1-8 sources summed in rank order in fp32.  Copies and
sums are bitwise equal to the same fp32 operations in torch."""
import ctypes as C
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1807_08887_b200 import tofu  # noqa: E402

DT = {0: torch.bfloat16, 1: torch.float32}   # TOFU_BF16 = 0, TOFU_F32 = 1 (include/tofu.h)


def _case(rng, n_pieces):
    pieces = (tofu.Piece * n_pieces)()
    refs = []
    keep = []
    for i in range(n_pieces):
        rank = rng.randint(1, 4)
        ext = [rng.choice([1, 2, 3, 5, 8, 16, 37, 64, 128, 200]) for _ in range(rank)]
        ext[-1] = rng.choice([1, 3, 8, 24, 64, 256, 1000, 4096])
        sdt, ddt = rng.choice([(0, 0), (1, 1), (1, 0), (0, 1)])
        nsrc = rng.choice([1, 1, 2, 3, 8])
        pad = [rng.choice([0, 0, 1, 3, 8]) for _ in range(rank)]
        srcs = []
        for s in range(nsrc):
            big = torch.randn([e + p + 2 for e, p in zip(ext, pad)], device="cuda").to(DT[sdt])
            sl = tuple(slice(p, p + e) for p, e in zip(pad, ext))
            srcs.append((big, big[sl]))
        dpad = pad[::-1]
        dbig = torch.zeros([e + p + 1 for e, p in zip(ext, dpad)], device="cuda", dtype=DT[ddt])
        dsl = tuple(slice(p, p + e) for p, e in zip(dpad, ext))
        dview = dbig[dsl]
        pc = pieces[i]
        e4 = [1] * (4 - rank) + ext
        for d in range(4):
            pc.extent[d] = e4[d]
        st = [0] * (4 - rank) + list(dview.stride())
        for d in range(4):
            pc.dst_stride[d] = st[d]
        pc.dst = dview.data_ptr()
        pc.dst_dtype, pc.src_dtype, pc.nsrc = ddt, sdt, nsrc
        sst = [0] * (4 - rank) + list(srcs[0][1].stride())
        for s, (_, v) in enumerate(srcs):
            assert list(v.stride()) == list(srcs[0][1].stride())
            pc.src[s] = v.data_ptr()
        for d in range(4):
            pc.src_stride[d] = sst[d]
        acc = srcs[0][1].float().clone()
        for _, v in srcs[1:]:
            acc += v.float()
        refs.append((dbig, dsl, acc.to(DT[ddt])))
        keep.append(srcs)
    return pieces, refs, keep


@pytest.mark.parametrize("wide", [False, True])
@pytest.mark.parametrize("seed", range(6))
def test_pieces_copy_and_ordered_sum(seed, wide):
    """wide: the many-source kernel (tofu_pieces_run all_raw = 2: every source's vector in flight at once) on
    the same pieces, bitwise equal to the ordered sum as the general kernel."""
    rng = random.Random(seed)
    pieces, refs, keep = _case(rng, rng.randint(1, 12))
    tasks, nt = tofu.pieces_tasks(pieces)
    pd = torch.empty(C.sizeof(pieces), dtype=torch.uint8, device="cuda")
    td = torch.empty(max(C.sizeof(tasks), 1), dtype=torch.uint8, device="cuda")
    pd.copy_(torch.frombuffer(bytearray(bytes(pieces)), dtype=torch.uint8))
    td.copy_(torch.frombuffer(bytearray(bytes(tasks)), dtype=torch.uint8)[:td.numel()])
    raw = int(all(tasks[i].pad_ == 1 for i in range(nt)))
    tofu.pieces_run(pd.data_ptr(), td.data_ptr(), nt, 2 if wide and not raw else raw)
    torch.cuda.synchronize()
    for dbig, dsl, ref in refs:
        exp = torch.zeros_like(dbig)
        exp[dsl] = ref                      # the box holds the ordered sum; nothing outside it was written
        assert torch.equal(dbig, exp)
