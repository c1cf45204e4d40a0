"""CPU tests of libtofu's host side (C ABI): the library loads and exports
every symbol include/tofu.h declares; describe_op and tofu_plan equal the
oracle bit-exactly; the executor's lowered byte ledger equals the plan cost
(no GPU needed: device allocations are deferred to the first tofu_execute)."""
import ctypes as C
import json
import os
import re
from fractions import Fraction

import pytest

from fixtures import random_chain
from oracle.cost import owned_box, digits, plan_cost
from oracle.graph import Graph as OGraph
from oracle.search import SearchError, auto_search, flat_search, recursive_search
from oracle.strategy import discover_strategies
from oracle.tdl import parse_def, parse_program
from tofu_inputs.graphs import config, mlp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tofu():
    from paper_1807_08887_b200 import build, tofu as t
    build.build(verbose=False)
    t.lib()
    return t


def test_library_exports_every_declared_symbol(tofu):
    hdr = open(os.path.join(ROOT, "include", "tofu.h")).read()
    names = set(re.findall(r"\b(tofu_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 20
    L = tofu.lib()
    missing = [n for n in sorted(names) if not hasattr(L, n)]
    assert not missing, missing


def test_describe_op_matches_oracle(tofu):
    corpus = parse_program(open(os.path.join(ROOT, "tests", "golden", "corpus.tdl")).read())
    for name, d in corpus.items():
        src = [l for l in open(os.path.join(ROOT, "tests", "golden", "corpus.tdl")).read().splitlines()
               if l.startswith(f"def {name}(")][0]
        for ways in (2, 3):
            got = tofu.describe_op(src, ways)
            assert got["out_vars"] == d.out_vars and got["red_vars"] == d.red_vars
            assert got["class"] == {"ElementWise": "ElementWise"}.get(got["class"], got["class"])
            from oracle.tdl import classify
            assert got["class"] == classify(d)[0]
            ost = discover_strategies(d, ways)
            assert [s["var"] for s in got["strategies"]] == [s["var"] for s in ost]
            for gs, os_ in zip(got["strategies"], ost):
                assert gs["kind"] == os_["kind"]
                for j in range(ways):
                    for greg, (t, dims) in zip(gs["regions"][j], os_["regions"][j]):
                        assert greg["tensor"] == t
                        for gd, od in zip(greg["dims"], dims):
                            if od is None:
                                assert gd is None
                                continue
                            lo = {k: Fraction(*v) for k, v in gd["lo"].items()}
                            hi = {k: Fraction(*v) for k, v in gd["hi"].items()}
                            assert lo == dict(od.lo) and hi == dict(od.hi)
                            q = lambda x: Fraction(*x) if isinstance(x, list) else Fraction(x)
                            assert q(gd["c_lo"]) == od.c_lo and q(gd["c_hi"]) == od.c_hi


@pytest.mark.parametrize("src", ["def bad(A(2)) -> lambda i: A[i, i]", "def bad(A(1)) -> lambda i, j: A[i * j]",
                                 "def bad(A(1)) -> lambda i: B[i]", "def bad(A(1)) -> lambda i: A[i"])
def test_describe_op_errors(tofu, src):
    with pytest.raises(tofu.TofuError):
        tofu.describe_op(src)


def _canon(plan):
    return {"tdims": {t: [None if d is None else d for d in s] for t, s in plan["tdims"].items()},
            "osplit": plan["osplit"]}


@pytest.mark.parametrize("cfg,k", [(0, 2), (0, 4), (0, 8), (1, 2), (1, 4), (1, 8)])
def test_plan_bit_exact_vs_oracle_configs(tofu, cfg, k):
    spec = config(cfg)
    g = tofu.Graph(spec)
    p = tofu.Plan(g, k).json()
    o = recursive_search(OGraph(spec), k)
    assert p["cost"] == o["cost"] and p["bytes"] == o["bytes"] and p["deltas"] == o["deltas"]
    assert p["tdims"] == o["tdims"] and p["osplit"] == o["osplit"]
    assert p["factors"] == o["factors"]


def test_plan_bit_exact_vs_oracle_random(tofu):
    n = 0
    for s in range(40):
        spec = random_chain(s)
        og = OGraph(spec)
        for k in (2, 4, 8):
            try:
                o = auto_search(og, k)
            except SearchError:
                with pytest.raises(tofu.TofuError):
                    tofu.Plan(tofu.Graph(spec), k)
                continue
            p = tofu.Plan(tofu.Graph(spec), k).json()
            assert (p["cost"], p["bytes"], p["deltas"], p["search"]) == \
                (o["cost"], o["bytes"], o["deltas"], o["search"]), (s, k)
            if not o["frontier_truncated"]:
                assert p["tdims"] == o["tdims"] and p["osplit"] == o["osplit"], (s, k)
            n += 1
    assert n > 60


@pytest.mark.parametrize("args,k", [((1, 8, 3, 4), 2), ((1, 8, 3, 4), 4), ((1, 8, 3, 4), 8), ((2, 8, 2, 4), 4)])
def test_plan_bit_exact_vs_oracle_lstm(tofu, args, k):
    """LSTM graphs (timestep merging, views, 3-D gate tensors): the C++ plan equals the oracle's bit for bit
    (auto search: the recursion here, the flat search at k = 2 confirms it is optimal)."""
    from tofu_inputs.graphs import lstm
    spec = lstm(*args)
    o = auto_search(OGraph(spec), k)
    p = tofu.Plan(tofu.Graph(spec), k).json()
    assert (p["cost"], p["bytes"], p["deltas"], p["search"]) == (o["cost"], o["bytes"], o["deltas"], o["search"])
    assert p["tdims"] == o["tdims"] and p["osplit"] == o["osplit"]


def test_auto_plan_reaches_the_optimum_on_known_gaps(tofu):
    """The named recursion gaps (tests/test_oracle_optimality.py): the library's default (auto) search
    returns the exact optimum, equal to the oracle's auto search; search = 0 keeps the paper's recursion."""
    from test_oracle_optimality import KNOWN_RECURSION_GAPS
    for (s, k), (rec, opt) in sorted(KNOWN_RECURSION_GAPS.items()):
        spec = random_chain(s)
        p = tofu.Plan(tofu.Graph(spec), k).json()
        o = auto_search(OGraph(spec), k)
        assert p["cost"] == o["cost"] == opt and p["search"] == o["search"] == "flat", (s, k)
        assert p["deltas"] == o["deltas"] and p["bytes"] == o["bytes"]
        assert tofu.Plan(tofu.Graph(spec), k, search=0).json()["cost"] == rec


def test_flat_search_equals_oracle(tofu):
    for s in range(15):
        spec = random_chain(s)
        try:
            c, _ = flat_search(OGraph(spec), 4)
        except SearchError:
            continue
        p = tofu.Plan(tofu.Graph(spec), 4, search=1).json()
        assert p["cost"] == c


def test_shards_match_oracle_owned_boxes(tofu):
    spec = config(0)
    g = tofu.Graph(spec)
    plan = tofu.Plan(g, 8)
    pj = plan.json()
    og = OGraph(spec)
    for r in range(8):
        dig = digits(r, pj["factors"])
        offs = set()
        for t in spec["tensors"]:
            off, box = plan.shard(r, t)
            ob = owned_box(og.shape(t), pj["tdims"][t], pj["factors"], dig)
            if ob is None:
                assert off == -1
            else:
                assert [tuple(b) for b in box] == [tuple(b) for b in ob]
                assert off % 256 == 0
        assert plan.arena_bytes(r) > 0


@pytest.mark.parametrize("cfg,k", [(0, 2), (0, 4), (0, 8), (1, 8)])
def test_lowered_ledger_equals_plan(tofu, cfg, k):
    """Bytes the executor will move (counted from its lowered MultiFetch and
    reduce pieces) == planned cost (north star: bytes moved equal the plan)."""
    spec = config(cfg)
    g = tofu.Graph(spec)
    plan = tofu.Plan(g, k)
    fake = [0x100000000 * (r + 1) for r in range(k)]  # never dereferenced before tofu_execute
    ex = tofu.Exec(g, plan, list(range(k)), fake)
    assert ex.ledger() == plan.cost()
    assert ex.launches() > 0


def test_plan_time_table2_scale(tofu):
    """Search time (Table 2 reports 8.3 s for WResNet-152 on 8
    workers): a 1500-op-scale chain plans for 8 workers in seconds."""
    import time
    spec = mlp(64, [256] * 41)   # 40 layers: 40 fwd + 80 bwd + 80 optimizer + 40 relu pairs ~ 280 ops
    g = tofu.Graph(spec)
    t = time.time()
    p = tofu.Plan(g, 8).json()
    assert time.time() - t < 60
    assert p["cost"] >= 0


@pytest.mark.parametrize("k,units", [(2, [1, 1]), (4, [1])])
def test_wresnet_plan_bit_exact_and_ledger(tofu, k, units):
    """Convolution graphs (configs[3] family): the C++ plan equals the oracle's, and the lowered
    executor moves exactly the planned bytes (halo and strided-gradient regions included)."""
    from tofu_inputs.graphs import wresnet
    spec = wresnet(units, 1, 8, 16 if k == 2 else 8, base=4, classes=8)
    o = auto_search(OGraph(spec), k)   # k = 4: the flat search beats the recursion (5871 vs 5999 elements)
    g = tofu.Graph(spec)
    plan = tofu.Plan(g, k)
    p = plan.json()
    assert (p["cost"], p["bytes"], p["deltas"], p["search"]) == (o["cost"], o["bytes"], o["deltas"], o["search"])
    if not o["frontier_truncated"]:
        assert p["tdims"] == o["tdims"] and p["osplit"] == o["osplit"]
    fake = [0x100000000 * (r + 1) for r in range(k)]
    ex = tofu.Exec(g, plan, list(range(k)), fake)
    assert ex.ledger() == plan.cost()


@pytest.mark.parametrize("k", [2, 4, 8])
def test_wresnet_ledger_equals_plan_larger(tofu, k):
    """A 2-stage WResNet at k = 2/4/8 (C++ planner only; the oracle's search is too slow here)."""
    from tofu_inputs.graphs import wresnet
    spec = wresnet([2, 1], 1, 8, 32, base=8, classes=16)
    g = tofu.Graph(spec)
    plan = tofu.Plan(g, k)
    ex = tofu.Exec(g, plan, list(range(k)), [0x100000000 * (r + 1) for r in range(k)])
    assert ex.ledger() == plan.cost()


@pytest.mark.parametrize("cfg,k", [(1, 8), (0, 4)])
def test_rank_bytes_partition_the_ledger(tofu, cfg, k):
    """tofu_exec_rank_bytes: every ledger byte is read by one rank and served by another, so Σ in = Σ out
    = the ledger = the plan's bytes; FC k = 8 moves 9437184 B into every rank (3/8 of X twice, quarters of
    dY / partials: the per-step pieces of tests/golden/fc_k8_deltas.json spread evenly) plus rank 0's 7
    loss partials (28 B)."""
    spec = config(cfg)
    g = tofu.Graph(spec)
    plan = tofu.Plan(g, k)
    ex = tofu.Exec(g, plan, list(range(k)), [0x100000000 * (r + 1) for r in range(k)])
    io = [ex.rank_bytes(r) for r in range(k)]
    assert sum(a for a, _ in io) == sum(b for _, b in io) == ex.ledger()[1] == plan.cost()[1]
    if cfg == 1:
        assert [a for a, _ in io] == [9437184 + 28] + [9437184] * 7


def _mlp_with_defs(**edits):
    spec = config(0)
    spec = json.loads(json.dumps(spec))
    for old, (new_name, new_src) in edits.items():
        src = spec["defs"].pop(old)
        spec["defs"][new_name] = new_src if new_src else src.replace(f"def {old}(", f"def {new_name}(")
        for o in spec["ops"]:
            if o["def"] == old:
                o["def"] = new_name
    return spec


def _exec(tofu, spec, k=1):
    g = tofu.Graph(spec)
    plan = tofu.Plan(g, k)
    return tofu.Exec(g, plan, list(range(k)), [0x100000000 * (r + 1) for r in range(k)])


def test_kernels_are_bound_by_tdl_body_not_name(tofu, monkeypatch):
    """an operator is its TDL description.  Renamed defs keep their kernels; the constants the
    kernels use are the TDL literals (not the op attrs)."""
    monkeypatch.setenv("TOFU_FUSE", "0")      # every op its own launch
    spec = _mlp_with_defs(relu=("rectify", None), sgd=("update", None))
    for o in spec["ops"]:
        o["attrs"] = {"lr": 123.0, "mu": 7.0, "scale": 9.0}    # ignored: the TDL text decides
    ex = _exec(tofu, spec)
    descs = [ex.launch_desc(i) for i in range(ex.num_launches())]
    kern = {d["op"]: (d.get("kernel"), d.get("kconst")) for d in descs if d["kind"] == "compute"}
    assert kern["relu1"] == ("relu", [])
    assert kern["loss"][0] == "sumsq" and kern["loss"][1] == [1.0 / (64 * 512)]
    assert kern["mom1"] == ("mom", [0.875])     # (sgd1 runs inside mom1's launch: "mom+sgd")


@pytest.mark.parametrize("name,src", [
    ("relu", "def relu(X(2)) -> lambda i, j: max(X[i, j], 1)"),                   # another function, same name
    ("sgd", "def sgd(W(2), M(2)) -> lambda i, j: W[i, j] + M[i, j] * 0.0078125"),  # sign flipped
    ("mom", "def mom(M(2), G(2)) -> lambda i, j: M[i, j] * 0.875 * G[i, j]"),     # product, not sum
])
def test_edited_bodies_are_rejected(tofu, name, src):
    """A def whose body matches no kernel is refused at tofu_exec_create (TOFU_ERR_ARG), whatever its name."""
    spec = _mlp_with_defs(**{name: (name, src)})
    with pytest.raises(tofu.TofuError):
        _exec(tofu, spec)


def test_conv_body_must_be_a_contraction(tofu):
    from tofu_inputs.graphs import wresnet
    spec = wresnet([1], 1, 2, 32, base=8, classes=8)
    n = [d for d in spec["defs"] if d.startswith("conv_k3")][0]
    spec["defs"][n] = spec["defs"][n].replace("] * W[", "] + W[")
    with pytest.raises(tofu.TofuError):
        _exec(tofu, spec)


def test_piece_tasks_normalise_and_cover(tofu):
    """tofu_pieces_tasks (host): contiguous dims merge (a whole-row box becomes one long row), the vector
    width follows the alignment, and the tasks cover every segment (<= 256 vectors of a row) of every piece exactly once."""
    ps = (tofu.Piece * 3)()
    # [4, 6, 64] bf16 box that is whole rows in dst and src: merges to one row of 1536 elements, V = 8
    p = ps[0]
    for d, (e, s) in enumerate(zip([1, 4, 6, 64], [0, 384, 64, 1])):
        p.extent[d], p.dst_stride[d], p.src_stride[d] = e, s, s
    p.dst, p.src[0], p.nsrc, p.dst_dtype, p.src_dtype = 4096, 8192, 1, 0, 0
    # [10, 3] fp32 rows inside a wider buffer, odd base offset: V = 1
    p = ps[1]
    for d, (e, ds_, ss_) in enumerate(zip([1, 1, 10, 3], [0, 0, 7, 1], [0, 0, 5, 1])):
        p.extent[d], p.dst_stride[d], p.src_stride[d] = e, ds_, ss_
    p.dst, p.src[0], p.src[1], p.nsrc, p.dst_dtype, p.src_dtype = 4100, 8192, 16384, 2, 1, 1
    # big 2-D piece: 3 x 10000 bf16 in a pitch-10240 buffer: rows stay, V = 8, several tasks
    p = ps[2]
    for d, (e, s) in enumerate(zip([1, 1, 3, 10000], [0, 0, 10240, 1])):
        p.extent[d], p.dst_stride[d], p.src_stride[d] = e, s, s
    p.dst, p.src[0], p.nsrc, p.dst_dtype, p.src_dtype = 1 << 20, 1 << 24, 1, 0, 0
    tasks, nt = tofu.pieces_tasks(ps)
    assert [list(ps[0].extent), ps[0].pad_] == [[1, 1, 1, 1536], 8]
    assert ps[1].pad_ == 1 and list(ps[1].extent) == [1, 1, 10, 3]
    assert ps[2].pad_ == 8 and list(ps[2].extent) == [1, 1, 3, 10000]
    cover = {}
    for i in range(nt):
        t = tasks[i]
        cover.setdefault(t.piece, []).append((t.q0, t.nq))
    for i, p in enumerate(ps):
        rv = p.extent[3] // p.pad_
        nv = p.extent[0] * p.extent[1] * p.extent[2] * ((rv + 255) // 256)
        segs = sorted(cover[i])
        assert segs[0][0] == 0 and all(a + n == b for (a, n), (b, _) in zip(segs, segs[1:]))
        assert segs[-1][0] + segs[-1][1] == nv


def test_fig10_wresnet_152_10_partition_shape(tofu):
    """§7.4 / Fig. 10, the partition Tofu finds for WResNet-152-10 at k = 8, reproduced by the
    library's planner: (1) both the batch and the channel dimensions are partitioned; (2) the repeated residual
    blocks of a group are partitioned identically, the first block of a group differently; (3) the lower
    layers (large feature maps, small weights) split the batch — their weights are fetched — and the higher
    layers split channels — their activations are fetched."""
    import re
    spec = config(5)
    p = tofu.Plan(tofu.Graph(spec), 8).json()
    os_ = p["osplit"]
    by = {}
    for o in spec["ops"]:
        m = re.match(r"s(\d)u(\d+)\.(conv\d(?:_dgrad|_wgrad)?)$", o["name"])
        if m:
            by.setdefault((int(m.group(1)), m.group(3)), []).append((int(m.group(2)), tuple(os_[o["name"]])))
    used = {v for seq in os_.values() for v in seq}
    assert "b" in used and ({"ci", "co"} & used)                                   # (1)
    for (stage, kind), lst in by.items():                                          # (2)
        lst.sort()
        assert len({s for u, s in lst[1:]}) <= 1, (stage, kind, lst)
    assert any(lst[0][1] != lst[1][1] for lst in by.values() if len(lst) > 1)
    for (stage, kind), lst in by.items():                                          # (3)
        for u, seq in lst:
            if stage == 0:
                assert set(seq) == {"b"}, (stage, kind, u, seq)
            if stage == 3:
                assert "b" not in seq and set(seq) & {"ci", "co"}, (stage, kind, u, seq)


def _lifetimes_py(spec):
    """Tensor lifetimes re-derived here (op indices): [earliest op that may write it — its producer or, by
    fusion, a producer of the producer's inputs two levels up, or the op before — , last reader]."""
    ops = spec["ops"]
    prod = {}
    for i, o in enumerate(ops):
        prod.setdefault(o["output"], []).append(i)
    life = {}
    for i, o in enumerate(ops):
        start = i
        for x in o["inputs"]:
            for p in prod.get(x, []):
                start = min(start, p)
                for y in ops[p]["inputs"]:
                    for q in prod.get(y, []):
                        start = min(start, q)
        if i > 0:
            start = min(start, i - 1)
        lo, hi = life.get(o["output"], (10 ** 9, -1))
        life[o["output"]] = (min(lo, start), max(hi, i))
        for x in o["inputs"]:
            lo, hi = life.get(x, (10 ** 9, -1))
            life[x] = (lo, max(hi, i))
    return life


@pytest.mark.parametrize("which", ["mlp", "lstm", "wresnet"])
def test_memory_planner_layout(tofu, which, monkeypatch):
    """TOFU_MEMPLAN=1: transient tensors (activations, gradients) share arena bytes only when their
    lifetimes are disjoint; persistent tensors (inputs, weights, state, loss) keep their own; the arena shrinks;
    the ledger still equals the plan."""
    from tofu_inputs.graphs import lstm, wresnet
    spec = {"mlp": lambda: config(0), "lstm": lambda: lstm(2, 64, 4, 8),
            "wresnet": lambda: wresnet([1, 2], 2, 4, 64, base=16, classes=16)}[which]()
    g = tofu.Graph(spec)
    plan = tofu.Plan(g, 4)
    monkeypatch.setenv("TOFU_MEMPLAN", "0")
    before = [plan.arena_bytes(r) for r in range(4)]
    monkeypatch.setenv("TOFU_MEMPLAN", "1")
    after = [plan.arena_bytes(r) for r in range(4)]
    assert all(a <= b for a, b in zip(after, before)), (before, after)
    if which == "wresnet":
        assert all(a < b for a, b in zip(after, before)), (before, after)
    life = _lifetimes_py(spec)
    isz = {"bf16": 2, "f32": 4}
    alias = set(spec.get("alias", {})) | set(spec.get("alias", {}).values())
    for r in range(4):
        iv = []
        for t, info in spec["tensors"].items():
            off, box = plan.shard(r, t)
            if off < 0 or t in spec.get("alias", {}):
                continue
            n = 1
            for lo, hi in box:
                n *= hi - lo + 1
            iv.append((off, off + n * isz[info["dtype"]], t))
        for i, (a0, a1, ta) in enumerate(iv):
            for b0, b1, tb in iv[i + 1:]:
                if a0 < b1 and b0 < a1:   # shared bytes: both transient, lifetimes disjoint
                    for t in (ta, tb):
                        assert spec["tensors"][t]["role"] in ("act", "grad") and t not in alias, t
                    la, lb = life[ta], life[tb]
                    assert la[1] < lb[0] or lb[1] < la[0], (ta, la, tb, lb)
    ex = tofu.Exec(g, plan, list(range(4)), [0x100000000 * (r + 1) for r in range(4)])
    assert ex.ledger() == plan.cost()


def test_many_source_reduce_kernel_is_chosen_from_four_sources(tofu):
    """Partition-n-reduce launches with >= 4 sources run the many-source piece kernel (every source's vector in
    flight at once, tofu_pieces_run all_raw = 2), fewer sources the general one, plain copies the copy kernel."""
    ex = _exec(tofu, config(1), k=8)
    seen = set()
    for i in range(ex.num_launches()):
        d = ex.launch_desc(i)
        if d["kind"] not in ("fetch", "reduce"):
            continue
        want = "many_source" if d["max_src"] >= 4 else None
        if want:
            assert d["piece_kernel"] == want, d
        else:
            assert d["piece_kernel"] in ("copy", "general"), d
        seen.add(d["piece_kernel"])
    assert "many_source" in seen


def test_staged_conv_weights_are_transposed_for_the_data_gradient(tofu, monkeypatch):
    """Every 3x3 convolution data gradient reads its weight K-major: owned weights from a per-op transposed
    copy, weights fetched into staging (batch-split layers under a k-way plan) from one per-rank scratch the
    launch transposes into (exec.cpp; the arena grows by the scratch only).  TOFU_WT=0: none transposed."""
    from tofu_inputs.graphs import wresnet
    spec = wresnet([2, 1], 2, 8, 64, base=32, classes=24)
    counts = {}
    for wt in ("1", "0"):
        monkeypatch.setenv("TOFU_WT", wt)
        ex = _exec(tofu, spec, k=8)
        descs = [ex.launch_desc(i) for i in range(ex.num_launches())]
        dg = [d for d in descs if d["kind"] == "compute" and d["def"].startswith("dconv_k3")]
        counts[wt] = (len(dg), sum(d.get("weights") == "transposed" for d in dg),
                      sum(d.get("weights_from") == "staging" for d in dg))
        assert ex.ledger() == tuple(tofu.Plan(tofu.Graph(spec), 8).cost())
    assert counts["1"][0] > 0 and counts["1"][1] == counts["1"][0]
    assert counts["1"][2] > 0                                # some of them from staging
    assert counts["0"][1] == 0


def test_gate_gemm_cell_fusion_lowering(tofu, monkeypatch):
    """TOFU_FUSE_GATE_CELL=1: every forward gate GEMM whose output GH_t feeds the fused cell pair of step t
    carries the pair in its launch (desc "gemm+lstm-cell"; the cell ops launch nothing), the ledger still equals
    the plan; off by default."""
    from tofu_inputs.graphs import lstm
    spec = lstm(2, 512, 3, 64)
    got = {}
    for v in ("0", "1"):
        monkeypatch.setenv("TOFU_FUSE_GATE_CELL", v)
        for k in (1, 2):
            ex = _exec(tofu, spec, k=k)
            descs = [ex.launch_desc(i) for i in range(ex.num_launches())]
            got[(v, k)] = (sum(d.get("fused") == "gemm+lstm-cell" for d in descs),
                           sum(d["kind"] == "compute" and d["def"] == "cell_c" for d in descs))
            assert ex.ledger() == tuple(tofu.Plan(tofu.Graph(spec), k).cost())
    for k in (1, 2):
        assert got[("0", k)][0] == 0
        assert got[("1", k)][0] == 2 * 3 * k                 # layers x steps x ranks
        assert got[("1", k)][1] == got[("0", k)][1] - 2 * 3 * k  # those cell launches are gone
