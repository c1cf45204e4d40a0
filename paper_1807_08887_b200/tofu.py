"""Thin ctypes binding of libtofu (include/tofu.h).  Argument marshalling only:
every step of the hot path runs in libtofu's kernels / host code.  Raises
loudly when the library is missing — there is no fallback path.
"""
from __future__ import annotations

import ctypes as C
import json
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TOFU_LIB") or os.path.join(_PKG, "libtofu.so")  # TOFU_LIB: an experimental build

TOFU_BF16, TOFU_F32 = 0, 1
EW = {"relu": 0, "relu_grad": 1, "mse_grad": 2, "mom": 3, "sgd": 4, "sgd_mom": 5, "sumsq": 6}
MAX_SRC = 8


class TofuError(RuntimeError):
    pass


class GemmArgs(C.Structure):
    _fields_ = [("M", C.c_int), ("N", C.c_int), ("K", C.c_int),
                ("A", C.c_void_p), ("lda", C.c_int), ("a_mn_major", C.c_int),
                ("B", C.c_void_p), ("ldb", C.c_int), ("b_mn_major", C.c_int),
                ("C", C.c_void_p), ("ldc", C.c_int), ("c_mode", C.c_int),
                ("bn", C.c_int), ("max_ctas", C.c_int), ("D", C.c_void_p), ("ldd", C.c_int),
                ("s0", C.c_float), ("s1", C.c_float), ("splits", C.c_int), ("ws", C.c_void_p),
                ("aux_add", C.c_void_p), ("aux_mask", C.c_void_p), ("ep", C.c_int), ("sk_ws", C.c_void_p),
                ("a_pieces", C.c_void_p), ("b_pieces", C.c_void_p), ("cl2", C.c_int), ("defer_reduce", C.c_int),
                ("k_reverse", C.c_int)]


MAX_PIECES = 8


class OperandPieces(C.Structure):
    _fields_ = [("n", C.c_int), ("dim", C.c_int), ("start", C.c_int * MAX_PIECES),
                ("ptr", C.c_void_p * MAX_PIECES), ("ld", C.c_int64 * MAX_PIECES)]


MAX_TAPS = 64


class ConvArgs(C.Structure):
    _fields_ = [("kind", C.c_int), ("nb", C.c_int), ("ngy", C.c_int), ("ngx", C.c_int),
                ("ay", C.c_int), ("ax", C.c_int), ("cy", C.c_int), ("cx", C.c_int), ("sb0", C.c_int),
                ("ntaps", C.c_int), ("nch", C.c_int),
                ("tap_dy", C.c_short * MAX_TAPS), ("tap_dx", C.c_short * MAX_TAPS), ("tap_w", C.c_short * MAX_TAPS),
                ("S", C.c_void_p), ("s_sb", C.c_int64), ("s_sy", C.c_int64), ("s_sx", C.c_int64),
                ("sH", C.c_int), ("sW", C.c_int), ("sc0", C.c_int),
                ("n_out", C.c_int), ("m_out", C.c_int),
                ("Bp", C.c_void_p), ("ldb", C.c_int64), ("b_mn_major", C.c_int), ("b_tap", C.c_int),
                ("b_rows", C.c_int), ("b_cols", C.c_int),
                ("Ap", C.c_void_p), ("lda", C.c_int64),
                ("C", C.c_void_p), ("c_sb", C.c_int64), ("c_sy", C.c_int64), ("c_sx", C.c_int64),
                ("c_ys", C.c_int), ("c_y0", C.c_int), ("c_xs", C.c_int), ("c_x0", C.c_int),
                ("ldc", C.c_int64), ("c_mode", C.c_int), ("D", C.c_void_p), ("ldd", C.c_int64),
                ("s0", C.c_float), ("s1", C.c_float), ("splits", C.c_int), ("ws", C.c_void_p),
                ("aux_add", C.c_void_p), ("aux_mask", C.c_void_p), ("ep", C.c_int), ("sk_ws", C.c_void_p),
                ("direct", C.c_int), ("im2col", C.c_int), ("i2c_dy0", C.c_int), ("i2c_dx0", C.c_int),
                ("cl2", C.c_int)]


class Piece(C.Structure):
    _fields_ = [("extent", C.c_int64 * 4), ("dst", C.c_void_p), ("dst_stride", C.c_int64 * 4),
                ("dst_dtype", C.c_int), ("nsrc", C.c_int), ("src", C.c_void_p * MAX_SRC),
                ("src_stride", C.c_int64 * 4), ("src_dtype", C.c_int), ("pad_", C.c_int)]


class PlanOptions(C.Structure):
    _fields_ = [("frontier_cap", C.c_int), ("solution_cap", C.c_int), ("search", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise TofuError(f"libtofu.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.tofu_last_error.restype = C.c_char_p
        L.tofu_version.restype = C.c_char_p
        vp, i64p = C.c_void_p, C.POINTER(C.c_int64)
        sig = {
            "tofu_gemm_bf16": [C.POINTER(GemmArgs), vp],
            "tofu_gemm_plan_tmaps": [C.POINTER(GemmArgs), vp, C.POINTER(C.c_int)],
            "tofu_gemm_launch_planned": [C.POINTER(GemmArgs), vp, C.c_int, vp],
            "tofu_pieces_run": [vp, vp, C.c_int64, C.c_int, vp],
            "tofu_pieces_tasks": [vp, C.c_int, vp, C.c_int64, i64p],
            "tofu_conv_bf16": [C.POINTER(ConvArgs), vp],
            "tofu_elementwise": [C.c_int, C.c_int64, vp, vp, vp, vp, C.c_float, C.c_float, vp],
            "tofu_elementwise_ws": [C.c_int, C.c_int64, vp, vp, vp, vp, C.c_float, C.c_float, vp, vp],
            "tofu_describe_op": [C.c_char_p, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
            "tofu_graph_create": [C.c_char_p, C.POINTER(vp)],
            "tofu_graph_destroy": [vp],
            "tofu_plan_create": [vp, C.c_int, C.POINTER(PlanOptions), C.POINTER(vp)],
            "tofu_plan_destroy": [vp],
            "tofu_plan_json": [vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
            "tofu_plan_cost": [vp, i64p, i64p],
            "tofu_exec_arena_bytes": [vp, vp, C.c_int, i64p],
            "tofu_exec_shard": [vp, vp, C.c_int, C.c_char_p, i64p, i64p, C.POINTER(C.c_int)],
            "tofu_exec_create": [vp, vp, C.c_int, C.POINTER(C.c_int), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)],
            "tofu_exec_destroy": [vp],
            "tofu_execute": [vp, vp],
            "tofu_exec_ledger": [vp, i64p, i64p],
            "tofu_exec_launch_count": [vp, i64p],
            "tofu_exec_set_skip_comm": [vp, C.c_int],
            "tofu_exec_num_launches": [vp, C.POINTER(C.c_int)],
            "tofu_exec_launch_desc": [vp, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
            "tofu_exec_unmaterialized": [vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
            "tofu_exec_rank_bytes": [vp, C.c_int, i64p, i64p],
            "tofu_ipc_export": [vp, vp, i64p],
            "tofu_ipc_open": [vp, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_void_p)],
            "tofu_ipc_close": [vp, C.c_int64],
            "tofu_execute_range": [vp, C.c_int, C.c_int, vp],
            "tofu_exec_time_launch": [vp, C.c_int, vp, vp],
            "tofu_transpose_taps": [vp, vp, C.c_int, C.c_int, C.c_int, vp],
            "tofu_conv_plan": [C.POINTER(ConvArgs), vp],
        }
        for name, args in sig.items():
            f = getattr(L, name, None)
            if f is None:
                continue
            f.argtypes = args
            f.restype = None if name.endswith("_destroy") else C.c_int
        if hasattr(L, "tofu_sk_workspace_bytes"):   # (absent from experimental builds of older sources)
            L.tofu_sk_workspace_bytes.argtypes = []
            L.tofu_sk_workspace_bytes.restype = C.c_int64
        if hasattr(L, "tofu_sumsq_workspace_bytes"):
            L.tofu_sumsq_workspace_bytes.argtypes = []
            L.tofu_sumsq_workspace_bytes.restype = C.c_int64
        _lib = L
    return _lib


def check(rc, what=""):
    if rc != 0:
        raise TofuError(f"{what} failed ({rc}): {lib().tofu_last_error().decode()}")


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


# ----------------------------------------------------------------------------- kernels
def gemm(A, B, Cout, M, N, K, lda, a_mn, ldb, b_mn, ldc, c_mode, bn=0, max_ctas=0, stream=None, D=None, ldd=0,
         s0=0.0, s1=0.0, splits=0, aux_add=None, aux_mask=None, ep=0, sk_ws=None, a_pieces=None, b_pieces=None,
         cl2=0):
    """tofu_gemm_bf16 (include/tofu.h).  sk_ws: a zero-filled uint8 device tensor of tofu_sk_workspace_bytes()
    bytes enables stream-K (left zeroed by the launch).  a_pieces / b_pieces: (dim, [(start, tensor, ld), ...])
    piecewise operands (tofu_operand_pieces; A / B are then only shape references)."""
    def pieces(p):
        if p is None:
            return None
        dim, lst = p
        op = OperandPieces()
        op.n, op.dim = len(lst), dim
        for i, (st, t, ld) in enumerate(lst):
            op.start[i], op.ptr[i], op.ld[i] = st, t.data_ptr(), ld
        return op
    pa, pb = pieces(a_pieces), pieces(b_pieces)
    a = GemmArgs(M, N, K, A.data_ptr(), lda, a_mn, B.data_ptr(), ldb, b_mn, Cout.data_ptr(), ldc, c_mode, bn, max_ctas,
                 D.data_ptr() if D is not None else None, ldd, s0, s1, splits, None,
                 aux_add.data_ptr() if aux_add is not None else None,
                 aux_mask.data_ptr() if aux_mask is not None else None, ep,
                 sk_ws.data_ptr() if sk_ws is not None else None,
                 C.addressof(pa) if pa is not None else None, C.addressof(pb) if pb is not None else None, cl2)
    check(lib().tofu_gemm_bf16(C.byref(a), _stream(stream)), "tofu_gemm_bf16")


def transpose_taps(W, WT, co, taps, ci, stream=None):
    """tofu_transpose_taps: WT[ci][taps][co] = W[co][taps][ci] (bf16 device tensors)."""
    check(lib().tofu_transpose_taps(C.c_void_p(W.data_ptr()), C.c_void_p(WT.data_ptr()), co, taps, ci,
                                    _stream(stream)), "tofu_transpose_taps")


def sk_workspace_bytes() -> int:
    return int(lib().tofu_sk_workspace_bytes())


def conv_plan(args: ConvArgs) -> ConvArgs:
    """tofu_conv_plan on a copy of args (the descriptors are discarded): reports splits / direct / im2col."""
    c = ConvArgs.from_buffer_copy(args)
    buf = C.create_string_buffer(5 * 128 + 64)
    ptr = (C.addressof(buf) + 63) // 64 * 64
    check(lib().tofu_conv_plan(C.byref(c), C.c_void_p(ptr)), "tofu_conv_plan")
    return c


def conv(args: ConvArgs, stream=None):
    """tofu_conv_bf16 (include/tofu.h): one implicit-GEMM convolution sub-op."""
    check(lib().tofu_conv_bf16(C.byref(args), _stream(stream)), "tofu_conv_bf16")


def elementwise(kind, n, y=None, x0=None, x1=None, x2=None, s0=0.0, s1=0.0, stream=None):
    p = lambda t: None if t is None else C.c_void_p(t.data_ptr())
    check(lib().tofu_elementwise(EW[kind] if isinstance(kind, str) else kind, n, p(y), p(x0), p(x1), p(x2),
                                 s0, s1, _stream(stream)), "tofu_elementwise")


class Piece(C.Structure):
    """tofu_piece (include/tofu.h)."""
    _fields_ = [("extent", C.c_int64 * 4), ("dst", C.c_void_p), ("dst_stride", C.c_int64 * 4), ("dst_dtype", C.c_int),
                ("nsrc", C.c_int), ("src", C.c_void_p * 8), ("src_stride", C.c_int64 * 4), ("src_dtype", C.c_int),
                ("pad_", C.c_int), ("ep", C.c_int), ("s0", C.c_float), ("s1", C.c_float), ("pad2_", C.c_int),
                ("aux0", C.c_void_p)]


class PieceTask(C.Structure):
    _fields_ = [("piece", C.c_int), ("pad_", C.c_int), ("q0", C.c_int64), ("nq", C.c_int64)]


def pieces_tasks(pieces):
    """tofu_pieces_tasks on a ctypes array of Piece (normalised in place): returns a PieceTask array."""
    n = C.c_int64(0)
    check(lib().tofu_pieces_tasks(C.addressof(pieces), len(pieces), None, 0, C.byref(n)), "tofu_pieces_tasks")
    tasks = (PieceTask * max(n.value, 1))()
    check(lib().tofu_pieces_tasks(C.addressof(pieces), len(pieces), C.addressof(tasks), n.value, C.byref(n)),
          "tofu_pieces_tasks")
    return tasks, n.value


def pieces_run(pieces_dev_ptr, tasks_dev_ptr, ntasks, all_raw=0, stream=None):
    """tofu_pieces_run over device copies of the pieces and tasks (all_raw: every task's pad_ == 1)."""
    check(lib().tofu_pieces_run(C.c_void_p(pieces_dev_ptr), C.c_void_p(tasks_dev_ptr), ntasks, all_raw,
                                _stream(stream)), "tofu_pieces_run")


def ipc_export(ptr: int):
    """tofu_ipc_export: (64-byte handle, offset of ptr in its allocation)."""
    h = (C.c_char * 64)()
    off = C.c_int64()
    check(lib().tofu_ipc_export(C.c_void_p(ptr), h, C.byref(off)), "tofu_ipc_export")
    return bytes(h), off.value


def ipc_open(handle: bytes, offset: int, local_device: int, peer_device: int) -> int:
    """tofu_ipc_open: map a peer's exported allocation on local_device; returns the mapped address."""
    h = (C.c_char * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    check(lib().tofu_ipc_open(h, offset, local_device, peer_device, C.byref(p)), "tofu_ipc_open")
    return p.value


def ipc_close(ptr: int, offset: int):
    check(lib().tofu_ipc_close(C.c_void_p(ptr), offset), "tofu_ipc_close")


# ----------------------------------------------------------------------------- host API
def describe_op(tdl: str, ways: int = 2) -> dict:
    n = C.c_size_t(0)
    check(lib().tofu_describe_op(tdl.encode(), ways, None, 0, C.byref(n)), "tofu_describe_op")
    buf = C.create_string_buffer(n.value + 1)
    check(lib().tofu_describe_op(tdl.encode(), ways, buf, n.value + 1, C.byref(n)), "tofu_describe_op")
    return json.loads(buf.value.decode())


class Graph:
    def __init__(self, spec: dict):
        self.spec = spec
        h = C.c_void_p()
        check(lib().tofu_graph_create(json.dumps(spec).encode(), C.byref(h)), "tofu_graph_create")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.tofu_graph_destroy(self.h)
            self.h = None


class Plan:
    def __init__(self, graph: Graph, k: int, frontier_cap=64, solution_cap=256, search=2):
        self.graph = graph
        self.k = k
        h = C.c_void_p()
        opts = PlanOptions(frontier_cap, solution_cap, search)
        check(lib().tofu_plan_create(graph.h, k, C.byref(opts), C.byref(h)), "tofu_plan_create")
        self.h = h

    def json(self) -> dict:
        n = C.c_size_t(0)
        check(lib().tofu_plan_json(self.h, None, 0, C.byref(n)), "tofu_plan_json")
        buf = C.create_string_buffer(n.value + 1)
        check(lib().tofu_plan_json(self.h, buf, n.value + 1, C.byref(n)), "tofu_plan_json")
        return json.loads(buf.value.decode())

    def cost(self):
        e, b = C.c_int64(), C.c_int64()
        check(lib().tofu_plan_cost(self.h, C.byref(e), C.byref(b)), "tofu_plan_cost")
        return e.value, b.value

    def arena_bytes(self, rank: int) -> int:
        n = C.c_int64()
        check(lib().tofu_exec_arena_bytes(self.graph.h, self.h, rank, C.byref(n)), "tofu_exec_arena_bytes")
        return n.value

    def shard(self, rank: int, tensor: str):
        off = C.c_int64()
        box = (C.c_int64 * 8)()
        r = C.c_int()
        check(lib().tofu_exec_shard(self.graph.h, self.h, rank, tensor.encode(), C.byref(off), box, C.byref(r)),
              "tofu_exec_shard")
        return off.value, [(box[2 * d], box[2 * d + 1]) for d in range(r.value)]

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.tofu_plan_destroy(self.h)
            self.h = None


class Exec:
    """Executor over local ranks.  arenas: list of k device pointers (ints)."""

    def __init__(self, graph: Graph, plan: Plan, local_ranks, arenas, flags=None):
        self.graph, self.plan = graph, plan
        n = len(local_ranks)
        lr = (C.c_int * n)(*local_ranks)
        ar = (C.c_void_p * len(arenas))(*arenas)
        fl = (C.c_void_p * len(arenas))(*(flags or [0] * len(arenas)))
        h = C.c_void_p()
        check(lib().tofu_exec_create(graph.h, plan.h, n, lr, ar, fl if flags else None, C.byref(h)),
              "tofu_exec_create")
        self.h = h

    def run(self, stream=None):
        check(lib().tofu_execute(self.h, _stream(stream)), "tofu_execute")

    def ledger(self):
        e, b = C.c_int64(), C.c_int64()
        check(lib().tofu_exec_ledger(self.h, C.byref(e), C.byref(b)), "tofu_exec_ledger")
        return e.value, b.value

    def launches(self):
        n = C.c_int64()
        check(lib().tofu_exec_launch_count(self.h, C.byref(n)), "tofu_exec_launch_count")
        return n.value

    def num_launches(self) -> int:
        n = C.c_int()
        check(lib().tofu_exec_num_launches(self.h, C.byref(n)), "tofu_exec_num_launches")
        return n.value

    def launch_desc(self, i: int) -> dict:
        buf = C.create_string_buffer(1024)
        n = C.c_size_t()
        check(lib().tofu_exec_launch_desc(self.h, i, buf, 1024, C.byref(n)), "tofu_exec_launch_desc")
        return json.loads(buf.value.decode())

    def rank_bytes(self, rank: int):
        """(bytes rank reads from peers, bytes peers read from rank) per step."""
        a, b = C.c_int64(), C.c_int64()
        check(lib().tofu_exec_rank_bytes(self.h, rank, C.byref(a), C.byref(b)), "tofu_exec_rank_bytes")
        return a.value, b.value

    def unmaterialized(self) -> list:
        """Tensors the step never writes to HBM (fused intermediates, include/tofu.h)."""
        cap = 1 << 20
        buf = C.create_string_buffer(cap)
        n = C.c_size_t()
        check(lib().tofu_exec_unmaterialized(self.h, buf, cap, C.byref(n)), "tofu_exec_unmaterialized")
        return json.loads(buf.value.decode())

    def run_range(self, first: int, last: int, stream=None):
        check(lib().tofu_execute_range(self.h, first, last, _stream(stream)), "tofu_execute_range")

    def time_launch(self, index: int, ev_start=None, ev_stop=None):
        a = C.c_void_p(ev_start.cuda_event) if ev_start is not None else None
        b = C.c_void_p(ev_stop.cuda_event) if ev_stop is not None else None
        check(lib().tofu_exec_time_launch(self.h, index, a, b), "tofu_exec_time_launch")

    def skip_comm(self, on: bool):
        check(lib().tofu_exec_set_skip_comm(self.h, 1 if on else 0), "tofu_exec_set_skip_comm")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.tofu_exec_destroy(self.h)
            self.h = None
