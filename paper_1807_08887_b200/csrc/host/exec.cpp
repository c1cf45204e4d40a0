// Lowering of a plan to per-rank programs and their execution (a3, a8).
//
// "For each operator in the original graph, Tofu generates a copy for each GPU worker in the partitioned
// graph" (§6).  Per (op, rank) the lowering computes the sub-op's iteration box, the required
// region of every input (MultiFetch pieces from each owner into a staging buffer unless the region is
// already local), and the produced output box: written straight into the owner's shard when
// it is exactly the rank's own shard, otherwise staged and pulled by the owners (fp32 partials summed in
// rank order when a reduction variable is split — partition-n-reduce P:L255-256, spread over all GPUs
// P:L879-881).  The ledger counts every element moved between distinct ranks; it equals the plan cost.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <tuple>
#include <cstring>
#include <map>
#include <set>

#include "common.h"
#include "graph.h"
#include "json.h"
#include "plan.h"

extern "C" int tofu_barrier_run(void* flags_ptrs_dev, int rank, int n, void* stream);
extern "C" int tofu_spin(int64_t ns, void* stream);
extern "C" int tofu_lstm_cell(int kind, int64_t nb, int64_t nh, int g0, int ng, const void* const* ptrs,
                              const int64_t* lds, const int64_t* gss, const int* dts, void* out, int64_t out_ld,
                              int64_t out_gs, int out_dt, void* out2, int64_t out2_ld, int out2_dt, void* stream);
extern "C" int tofu_lstm_cell_splitk(int kind, int64_t nb, int64_t nh, int g0, int ng, const void* const* ptrs,
                                     const int64_t* lds, const int64_t* gss, const int* dts, void* out, int64_t out_ld,
                                     int64_t out_gs, int out_dt, void* out2, int64_t out2_ld, int out2_dt,
                                     const float* ghws, int gh_splits, int64_t gh_plane, int64_t gh_wld,
                                     int64_t gh_wgs, void* stream);

namespace tofu {

namespace {

constexpr int64_t kAlign = 256;
int64_t align_up(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

int64_t vol(const std::vector<Rng>& b) {
  int64_t p = 1;
  for (auto& r : b) p *= r.len();
  return p;
}
bool inter(const std::vector<Rng>& a, const std::vector<Rng>& b, std::vector<Rng>& out) {
  out.resize(a.size());
  for (size_t i = 0; i < a.size(); ++i) {
    out[i] = {std::max(a[i].lo, b[i].lo), std::min(a[i].hi, b[i].hi)};
    if (out[i].len() <= 0) return false;
  }
  return true;
}
bool same(const std::vector<Rng>& a, const std::vector<Rng>& b) {
  for (size_t i = 0; i < a.size(); ++i)
    if (a[i].lo != b[i].lo || a[i].hi != b[i].hi) return false;
  return true;
}
bool contains(const std::vector<Rng>& outer, const std::vector<Rng>& in) {
  for (size_t i = 0; i < outer.size(); ++i)
    if (in[i].lo < outer[i].lo || in[i].hi > outer[i].hi) return false;
  return true;
}
// row-major strides (elements) of a dense box
std::vector<int64_t> strides_of(const std::vector<Rng>& box) {
  std::vector<int64_t> s(box.size());
  int64_t acc = 1;
  for (int i = (int)box.size() - 1; i >= 0; --i) {
    s[i] = acc;
    acc *= box[i].len();
  }
  return s;
}
int64_t offset_in(const std::vector<Rng>& buf, const std::vector<Rng>& at) {
  auto s = strides_of(buf);
  int64_t o = 0;
  for (size_t i = 0; i < buf.size(); ++i) o += (at[i].lo - buf[i].lo) * s[i];
  return o;
}

struct Layout {  // one rank's arena
  std::vector<int64_t> shard_off;             // per tensor (bytes), -1 = not owned
  std::vector<std::vector<Rng>> shard_box;    // per tensor
  int64_t staging_off = 0, staging_bytes = 0, total = 0;
};

struct Buf {  // an operand buffer of one (op, rank)
  struct RPiece {
    int src;        // owner rank
    int64_t off;    // bytes into the owner's arena of the piece's element (0, 0)
    int64_t ld;     // row pitch (elements) of the piece's 2-D view
    int start;      // first index along the cut GEMM dimension
  };
  std::vector<RPiece> rp;  // fused fetch: a GEMM operand read in place from its owners' shards (else empty)
  int rp_dim = 0;          // 0: M / N, 1: K (tofu_operand_pieces.dim)
  bool direct = false;
  int64_t off = 0;            // bytes into the rank's arena
  std::vector<Rng> buf_box;   // the box the buffer holds (dense row-major)
  std::vector<Rng> box;       // the box the op uses (subset of buf_box)
  int dtype = TOFU_F32;
};

struct LOp {
  std::vector<Buf> in;
  Buf out;
  bool partial = false;
  bool skip = false;          // fused into the previous op
  bool fused_sgd = false;
  int fused_opt = -1;         // GEMM epilogue absorbs mom (this index) + sgd (index + 1)
  int64_t wt_off = -1;        // conv data gradient: arena offset of the transposed weight shard (K-major B)
  bool fused_next = false;    // LSTM cell: this launch also computes the next op (c+h, bwd_a+bwd_c)
  int cell_after = -1;        // gate GEMM: this launch also runs that (fused c+h) cell op, which reduces the
                              // GEMM's split-K partials itself (one kernel for reduction + cell)
  bool fused_loss_grad = false;  // sumsq: this launch also computes the next op, mse_grad of the same inputs
  int ep = 0;                 // element-wise epilogue of the output's consumers: 1 relu, 2 add, 4 mask
  int red_ep = 0;             // the reduce pieces apply the output's consumer (TOFU_PIECE_*)
  std::vector<int> absorbed;      // ops whose work this op's compute launch does (fused; their launches skip)
  std::vector<int> red_absorbed;  // ops whose work this op's reduce launch does
  Buf epi_add, epi_mask;      // its bf16 operands (the output's layout)
  std::vector<tofu_piece> fetch, reduce;
  std::vector<int> fetch_src, reduce_nremote;  // for the ledger
  bool remote_direct = false;  // the compute reads peer memory in place (fused fetch)
};

// Memory planner ("leveraging the existing memory planner"; TOFU_MEMPLAN=1): the transient
// tensors of a step (roles act / grad: activations, gradients, weight gradients) share arena space when their
// lifetimes are disjoint; inputs, weights, optimizer state and the loss keep their own.  A lifetime runs from
// the earliest op that may write the tensor — its producer, or an op whose launch absorbs the producer by
// fusion (R8: a producer of one of the producer's inputs, two levels up) — to its last reader.  Offsets are
// identical on every rank (shards of a tensor have the same size on every rank that owns one).  Off by
// default: the per-op parity tests read every tensor after the step.
bool memplan_enabled() {  // read at every layout (arena size, shard offsets and the executor must agree)
  const char* e = std::getenv("TOFU_MEMPLAN");
  return e && e[0] == '1';
}

bool transient(const Graph& g, int t) {
  const std::string& r = g.tensors[t].role;
  return r == "act" || r == "grad";
}

// [first op that may write t, last op that reads it] (op indices), for the transient tensors
std::vector<std::pair<int, int>> lifetimes(const Graph& g) {
  const int nt = (int)g.tensors.size(), no = (int)g.ops.size();
  std::vector<std::vector<int>> producers(nt);
  for (int o = 0; o < no; ++o) producers[g.ops[o].output].push_back(o);
  std::vector<std::pair<int, int>> life(nt, {INT32_MAX, -1});
  for (int o = 0; o < no; ++o) {
    const int t = g.ops[o].output;
    int start = o;
    for (int x : g.ops[o].inputs)
      for (int p : producers[x]) {
        start = std::min(start, p);
        for (int y : g.ops[p].inputs)
          for (int q : producers[y]) start = std::min(start, q);
      }
    if (o > 0) start = std::min(start, o - 1);  // (fused_next / loss pair: written by the previous op's launch)
    life[t].first = std::min(life[t].first, start);
    life[t].second = std::max(life[t].second, o);
    for (int x : g.ops[o].inputs) life[x].second = std::max(life[x].second, o);
  }
  for (auto& l : life)
    if (l.first == INT32_MAX) l = {0, std::max(l.second, 0)};
  return life;
}

Layout layout_rank(const Graph& g, const PlanSeq& p, int rank, std::vector<std::vector<LOp>>* lops_all = nullptr) {
  Layout L;
  const int nt = (int)g.tensors.size();
  auto dig = worker_digits(rank, p.factors);
  L.shard_off.assign(nt, -1);
  L.shard_box.assign(nt, {});
  std::map<int, int> alias_old;
  for (auto& pr : g.alias) alias_old[pr.first] = pr.second;
  std::set<int> aliased;
  for (auto& pr : g.alias) {
    aliased.insert(pr.first);
    aliased.insert(pr.second);
  }
  const bool plan_mem = memplan_enabled();
  int64_t off = 0;
  std::vector<int> packed;
  for (int t = 0; t < nt; ++t) {
    std::vector<Rng> box;
    bool own = owned_box(g, t, p.tdims[t], p.factors, dig, box);
    L.shard_box[t] = box;
    if (!own) continue;
    if (alias_old.count(t)) continue;  // stored in the old tensor's shard
    if (plan_mem && transient(g, t) && !aliased.count(t)) {
      packed.push_back(t);
      continue;
    }
    L.shard_off[t] = off;
    off = align_up(off + vol(box) * g.itemsize(t));
  }
  if (!packed.empty()) {
    // interval packing: in order of first write, each tensor at the lowest offset whose range no tensor of an
    // overlapping lifetime occupies
    const auto life = lifetimes(g);
    std::stable_sort(packed.begin(), packed.end(), [&](int a, int b) { return life[a].first < life[b].first; });
    struct Placed {
      int64_t lo, hi;
      int t;
    };
    std::vector<Placed> placed;
    const int64_t base = off;
    int64_t top = off;
    for (int t : packed) {
      const int64_t sz = align_up(vol(L.shard_box[t]) * g.itemsize(t));
      std::vector<std::pair<int64_t, int64_t>> busy;
      for (auto& q : placed)
        if (!(life[q.t].second < life[t].first || life[t].second < life[q.t].first)) busy.push_back({q.lo, q.hi});
      std::sort(busy.begin(), busy.end());
      int64_t at = base;
      for (auto& b : busy) {
        if (at + sz <= b.first) break;
        at = std::max(at, b.second);
      }
      placed.push_back({at, at + sz, t});
      L.shard_off[t] = at;
      top = std::max(top, at + sz);
    }
    off = align_up(top);
  }
  for (auto& kv : alias_old) {
    // chains resolve to the root storage
    int root = kv.second;
    while (alias_old.count(root)) root = alias_old[root];
    L.shard_off[kv.first] = L.shard_off[root];
  }
  L.staging_off = off;
  return L;
}

}  // namespace

struct Exec {
  const Graph* g = nullptr;
  Graph gcopy;
  PlanSeq plan;
  int k = 1;
  std::vector<int> local;           // local ranks
  std::vector<char*> arena;         // all k ranks (as addressable here)
  std::vector<void*> flags;         // all k ranks' epoch words (multi-process) or empty
  void* flags_dev = nullptr;        // device array of flag pointers
  std::vector<Layout> lay;          // all ranks
  std::vector<std::vector<LOp>> lops;  // [local index][op]
  std::set<int> unmat;              // tensors some rank never writes to HBM (fused intermediates, R8/R13)
  struct Launch {
    int kind;  // 0 fetch pieces, 1 compute, 2 reduce pieces, 3 barrier, 4 memset
    int op, li;
    int64_t piece_off, npieces, max_elems;
    int stream = 0;           // 0: the caller's (compute) stream, 1: the executor's comm stream
    std::vector<int> waits;   // launches on the other stream this one waits for (their events)
    bool rec = false;         // record this launch's event (a launch on the other stream waits for it)
    int64_t task_off = 0, ntasks = 0;  // fetch / reduce: tofu_piece_task range (tofu_pieces_tasks)
    int all_raw = 0;                   // 1: every task a plain copy (the copy kernel); 2: >= 4 sources
  };
  std::vector<Launch> launches;
  tofu_piece* pieces_dev = nullptr;
  tofu_piece_task* tasks_dev = nullptr;
  std::vector<tofu_piece_task> host_tasks;
  void* ws_dev = nullptr;  // split-K workspace shared by this executor's GEMMs (one stream)
  void* ew_ws = nullptr;   // the loss reduction's partials + ticket (tofu_elementwise_ws), zero between launches
  void* sk_dev = nullptr;  // stream-K workspace (partials + flags, zero-filled), shared likewise
  std::vector<tofu_piece> host_pieces;
  bool finalized = false;
  struct GemmLaunch {
    tofu_gemm_args a;
    alignas(64) CUtensorMap tm[TOFU_GEMM_TMAPS];
    int bn;
    tofu_operand_pieces pa, pb;  // piecewise operands (fused fetch), referenced by a.a_pieces / a.b_pieces
  };
  std::map<std::pair<int, int>, GemmLaunch> gemms;  // (op, li)
  struct ConvLaunch {
    tofu_conv_args a;
    alignas(64) CUtensorMap tm[5];
  };
  std::map<std::pair<int, int>, std::vector<ConvLaunch>> convs;  // (op, li) -> launches (4 phases: stride-2 dgrad)
  int64_t ledger_el = 0, ledger_bytes = 0;
  std::vector<int64_t> rank_in, rank_out;  // per rank: bytes it reads from peers / peers read from it
  int64_t n_kernels = 0;
  bool skip_comm = false;
  uint64_t jitter = 0;    // TOFU_JITTER: seed + 1 of the injected delays (0 = off)
  uint64_t jitter_step = 0;
  bool multi_process = false;
  // virtual ranks: 2 (default; same-box A/B, programmatic launch on: WResNet-152-4 k = 8 87.67 -> 86.89 ms, LSTM
  // and FC even) or 1 (TOFU_STREAMS=1); multi-process always 2
  int streams = 2;
  bool fuse = true;
  bool fuse_fetch = true;  // GEMM operands read in place from their owners' shards (TOFU_PFETCH=0: staged)
  // ... also 1x1 stride-1 convolutions' operands (TOFU_PFETCH_CONV=1).  Off by default: measured on 8 virtual
  // ranks of one B200 (WResNet-152-4, tools/kineto_step.py) 94.7 -> 97.5 ms per step although 171 of 425
  // staged fetch launches disappear: the fused-fetch fp32-partial GEMMs run 28 -> 41 us each
  bool fuse_fetch_conv = false;
  bool fuse_gate_cell = false;  // gate GEMM + LSTM cell in one launch (TOFU_FUSE_GATE_CELL=1; see the fusion pass)
  struct OpAcc {  // objects (tensor alias roots; staging buffers nt, nt + 1) an op's launches touch, all ranks
    bool any_fetch = false, any_reduce = false, fetch_remote = false;
    int stage = -1;
    std::vector<int> f_rreads;                    // fetch: reads (in peers' memory when remote) -> writes stage
    std::vector<int> c_reads, c_writes, c_rreads;  // compute (+ absorbed ops); c_rreads: read in place remotely
    std::vector<int> r_reads, r_writes, r_rreads;  // reduce (+ absorbed ops); r_rreads: peers' staging
  };
  std::vector<OpAcc> acc;
  cudaStream_t comm = nullptr;        // the second stream (fetch / reduce / barrier launches)
  std::vector<cudaEvent_t> events;    // per launch (recorded when a launch on the other stream waits for it)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::vector<char> remote_fetch, remote_reduce;  // per op, over all ranks
  std::vector<char> remote_direct;                 // per op: a compute launch reads peer memory (fused fetch)
  int timed_launch = -1;
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
};

namespace {

// A contraction def `reduce(Sum; K..; A[..] * B[..])` whose indices are single variables maps onto the
// tcgen05 GEMM: output dims = (M vars)(N vars), A = (M)(K) K-major or (K)(M) MN-major, B = (N)(K) K-major
// or (K)(N) MN-major; multi-variable groups are flattened (e.g. the LSTM gate dims (g, h)).
struct GemmForm {
  bool ok = false;
  int a_param = 0, b_param = 1;
  int nm = 0, nn = 0, nk = 0;
  bool a_mn = false, b_mn = false;  // MN-major operands
  int a_split = 0, b_split = 0;     // number of leading dims in the operand's first group
};

GemmForm gemm_form(const OpDef& d) {
  GemmForm f;
  if (!d.prod2 || d.accesses.size() != 2) return f;
  auto vars_of = [&](const Access& a, std::vector<int>& out) {
    for (size_t k = 0; k < a.idx.size(); ++k) {
      if (a.slice[k] || !a.idx[k].plain() || a.idx[k].coef.size() != 1 || a.idx[k].coef[0].second != 1 || a.idx[k].c != 0) return false;
      out.push_back(a.idx[k].coef[0].first);
    }
    return true;
  };
  std::vector<int> av, bv;
  if (!vars_of(d.accesses[0], av) || !vars_of(d.accesses[1], bv)) return f;
  std::vector<int> mv, nv, kv;
  for (int v = 0; v < d.n_out; ++v) {
    const bool ina = std::find(av.begin(), av.end(), v) != av.end();
    const bool inb = std::find(bv.begin(), bv.end(), v) != bv.end();
    if (ina == inb) return f;
    (ina ? mv : nv).push_back(v);
  }
  for (int v = d.n_out; v < (int)d.vars.size(); ++v) kv.push_back(v);
  // output order must be (M)(N)
  for (size_t k = 0; k < mv.size(); ++k)
    if (mv[k] != (int)k) return f;
  auto cat = [](std::vector<int> a, const std::vector<int>& b) {
    a.insert(a.end(), b.begin(), b.end());
    return a;
  };
  if (av == cat(mv, kv)) f.a_mn = false;
  else if (av == cat(kv, mv)) f.a_mn = true;
  else return f;
  if (bv == cat(nv, kv)) f.b_mn = false;
  else if (bv == cat(kv, nv)) f.b_mn = true;
  else return f;
  f.a_param = d.accesses[0].param;
  f.b_param = d.accesses[1].param;
  f.nm = (int)mv.size();
  f.nn = (int)nv.size();
  f.nk = (int)kv.size();
  f.a_split = f.a_mn ? f.nk : f.nm;
  f.b_split = f.b_mn ? f.nk : f.nn;
  f.ok = f.nm > 0 && f.nn > 0 && f.nk > 0;
  return f;
}

// View `box` inside the dense row-major buffer `buf` as a 2-D matrix [dims < split][dims >= split]:
// every dim of a group except its first must be fully covered so rows have a uniform pitch and each row
// is contiguous.  Outputs rows/cols, the row pitch and the element offset of the box origin.
bool flat2(const std::vector<Rng>& buf, const std::vector<Rng>& box, int split, int64_t& rows, int64_t& cols,
           int64_t& ld, int64_t& off) {
  const int n = (int)buf.size();
  if (split <= 0 || split >= n) return false;
  for (int d = 0; d < n; ++d) {
    if (d == 0 || d == split) continue;
    if (box[d].lo != buf[d].lo || box[d].hi != buf[d].hi) return false;
  }
  rows = cols = ld = 1;
  for (int d = 0; d < split; ++d) rows *= box[d].len();
  for (int d = split; d < n; ++d) {
    cols *= box[d].len();
    ld *= buf[d].len();
  }
  off = offset_in(buf, box);
  return true;
}

// Convolution defs (tofu_inputs.graphs.conv_defs, reading R11): recognised by name AND checked to be the
// canonical convolution by re-deriving its TDL from (kind, R, s, p) and comparing every access index.
struct ConvGeom {
  int kind = -1;  // 0 forward, 1 data gradient, 2 weight gradient
  int R = 0, s = 0, p = 0;
};

std::string conv_tdl(int kind, int R, int s, int p) {
  const std::string n = "k" + std::to_string(R) + "s" + std::to_string(s) + "p" + std::to_string(p);
  const std::string P = std::to_string(p);
  const std::string sy = s == 1 ? "y" : std::to_string(s) + "*y", sx = s == 1 ? "x" : std::to_string(s) + "*x";
  if (kind == 0)
    return "def conv_" + n + "(X(4), W(4)) -> lambda b, y, x, co: reduce(Sum; ky, kx, ci; X[b, " + sy + " + ky - " + P +
           ", " + sx + " + kx - " + P + ", ci] * W[co, ky, kx, ci])";
  if (kind == 2)
    return "def wconv_" + n + "(D(4), X(4)) -> lambda co, ky, kx, ci: reduce(Sum; b, y, x; D[b, y, x, co] * X[b, " + sy +
           " + ky - " + P + ", " + sx + " + kx - " + P + ", ci])";
  if (s == 1)
    return "def dconv_" + n + "(D(4), W(4)) -> lambda b, y, x, ci: reduce(Sum; ky, kx, co; D[b, y - ky + " + P +
           ", x - kx + " + P + ", co] * W[co, ky, kx, ci])";
  return "def dconv_" + n + "(D(4), W(4)) -> lambda b, y, x, ci: reduce(Sum; ty, tx, co; D[b, (y - 2*ty + " + P +
         ") / 2, (x - 2*tx + " + P + ") / 2, co] * W[co, (y + " + P + ") % 2 + 2*ty, (x + " + P + ") % 2 + 2*tx, ci])";
}

bool same_access(const Access& a, const Access& b) {
  if (a.param != b.param || a.idx.size() != b.idx.size()) return false;
  for (size_t k = 0; k < a.idx.size(); ++k) {
    const Affine &x = a.idx[k], &y = b.idx[k];
    if (x.coef != y.coef || x.c != y.c || x.terms.size() != y.terms.size()) return false;
    for (size_t q = 0; q < x.terms.size(); ++q) {
      const auto &u = x.terms[q], &v = y.terms[q];
      if (u.mod != v.mod || u.mult != v.mult || u.d != v.d || u.inner.coef != v.inner.coef || u.inner.c != v.inner.c)
        return false;
    }
  }
  return true;
}

ConvGeom conv_geom(const OpDef& d) {
  ConvGeom g;
  int kind = -1, R = 0, s = 0, p = 0;
  const char* nm = d.name.c_str();
  if (std::sscanf(nm, "conv_k%ds%dp%d", &R, &s, &p) == 3 && d.name.rfind("conv_", 0) == 0) kind = 0;
  else if (std::sscanf(nm, "dconv_k%ds%dp%d", &R, &s, &p) == 3) kind = 1;
  else if (std::sscanf(nm, "wconv_k%ds%dp%d", &R, &s, &p) == 3) kind = 2;
  if (kind < 0 || R < 1 || s < 1 || s > 2 || p < 0 || !d.prod2) return g;   // body: reduce(Sum; ..; A[..] * B[..])
  const OpDef ref = parse_tdl(conv_tdl(kind, R, s, p));
  if (ref.vars != d.vars || ref.n_out != d.n_out || ref.reducer != d.reducer ||
      ref.accesses.size() != d.accesses.size())
    return g;
  for (size_t q = 0; q < ref.accesses.size(); ++q)
    if (!same_access(ref.accesses[q], d.accesses[q])) return g;
  g.kind = kind;
  g.R = R;
  g.s = s;
  g.p = p;
  return g;
}

// A 1x1 stride-1 convolution's operands as the GEMM it runs on (conv1x1_gemm): A = param 0, the pixel-row
// operand [b, y, x][c] (MN-major for the weight gradient); B = param 1, the weight [co][1][1][ci] (MN-major for
// the data gradient) or, for the weight gradient, the activations [b, y, x][ci] (MN-major).  Lets the lowering
// read those operands in place from their owners' shards (fused fetch), as for GEMM defs.
GemmForm conv1x1_form(const ConvGeom& cg) {
  GemmForm f;
  if (cg.kind < 0 || cg.R != 1 || cg.s != 1 || cg.p != 0) return f;
  f.ok = true;
  f.a_param = 0;
  f.b_param = 1;
  f.a_split = 3;
  f.a_mn = cg.kind == 2;
  f.b_split = cg.kind == 2 ? 3 : 1;
  f.b_mn = cg.kind != 0;
  return f;
}

const char* kernel_kind(const OpDef& d) {
  static const std::set<std::string> ew = {"relu",  "relu_grad",  "mse_grad", "mom",  "sgd",     "mom3", "sgd3",
                                           "sumsq", "relu4",      "relu_grad4", "mom4", "sgd4", "add4", "addrelu"};
  static const std::set<std::string> lstm = {"cell_c", "cell_h", "cell_bwd_a", "cell_bwd_c"};
  static const std::set<std::string> win = {"maxpool", "maxpool_grad", "gap", "gap_grad"};
  // element-wise / cell / window kernels are bound by the def's canonical TDL (kernel_match.cpp), not its name
  if (gemm_form(d).ok) return "gemm";
  if (ew.count(d.kernel)) return "ew";
  if (lstm.count(d.kernel)) return "lstm";
  if (win.count(d.kernel)) return "window";
  if (conv_geom(d).kind >= 0) return "conv";
  return nullptr;
}
bool is_mom(const std::string& n) { return n == "mom" || n == "mom3" || n == "mom4"; }
bool is_sgd(const std::string& n) { return n == "sgd" || n == "sgd3" || n == "sgd4"; }

// box == buffer in dims [from, n)
bool full_from(const std::vector<Rng>& buf, const std::vector<Rng>& box, int from) {
  for (int d = from; d < (int)buf.size(); ++d)
    if (box[d].lo != buf[d].lo || box[d].hi != buf[d].hi) return false;
  return true;
}

// Can the conv kernel read operand `pi` (box inside buffer buf) in place?  (Staged operands are dense boxes.)
bool conv_operand_ok(const ConvGeom& cg, int pi, const std::vector<Rng>& buf, const std::vector<Rng>& box) {
  if (box.size() != 4) return false;
  const bool gather = (cg.kind == 2) ? pi == 1 : pi == 0;
  if (gather) return (box[3].lo - buf[3].lo) % 8 == 0 && buf[3].len() % 8 == 0 && box[3].len() % 8 == 0;
  if (cg.kind == 2) return full_from(buf, box, 1) || (box[1].lo == buf[1].lo && box[1].hi == buf[1].hi &&
                                                     box[2].lo == buf[2].lo && box[2].hi == buf[2].hi);
  // weights [co][ky][kx][ci]: all taps present; the forward's K columns (taps x ci) either come in whole
  // 64-channel blocks per tap or are contiguous (ci not a sub-range)
  if (box[1].lo != buf[1].lo || box[1].hi != buf[1].hi || box[2].lo != buf[2].lo || box[2].hi != buf[2].hi) return false;
  if (cg.kind == 0) return box[3].len() % 64 == 0 || (box[3].lo == buf[3].lo && box[3].hi == buf[3].hi);
  return true;
}

// lowering options from the environment (TOFU_FUSE=0: no fusion; TOFU_PFETCH=0: staged MultiFetch only)
void read_env_options(Exec& E) {
  if (const char* j = std::getenv("TOFU_JITTER")) E.jitter = std::strtoull(j, nullptr, 10) + 1;
  if (const char* f = std::getenv("TOFU_FUSE")) E.fuse = std::string(f) != "0";
  if (const char* f = std::getenv("TOFU_STREAMS")) E.streams = std::atoi(f) >= 2 ? 2 : 1;
  if (const char* f = std::getenv("TOFU_PFETCH")) E.fuse_fetch = std::string(f) != "0";
  if (const char* f = std::getenv("TOFU_PFETCH_CONV")) E.fuse_fetch_conv = std::string(f) == "1";
  if (const char* f = std::getenv("TOFU_FUSE_GATE_CELL")) E.fuse_gate_cell = std::string(f) == "1";
}

void lower(Exec& E) {
  const Graph& g = *E.g;
  const PlanSeq& p = E.plan;
  const int k = E.k;
  E.lay.resize(k);
  // staging sizes per rank: computed while lowering each rank
  std::vector<std::vector<LOp>> all(k, std::vector<LOp>(g.ops.size()));
  for (int r = 0; r < k; ++r) E.lay[r] = layout_rank(g, p, r);
  std::vector<int64_t> stage_need(k, 0);
  // Fused fetch (P:L862-877 MultiFetch, B200 form): a GEMM operand whose required region is not a view of
  // the rank's own shard is read in place by the GEMM's TMA producer from the shards of its owners (peer
  // HBM over NVLink), when the owners' pieces tile the region along ONE GEMM dimension in whole tiles and
  // each piece is a 2-D strided view of its owner's shard.  No staging copy, and the transfer overlaps the
  // tensor-core work tile by tile.  Otherwise the region is staged by a MultiFetch launch as before.
  // (an op whose output shares storage with the input is never read in place: a peer could overwrite it
  // before this rank's read completes)
  auto root_of = [&](int t) {
    std::map<int, int> al(g.alias.begin(), g.alias.end());
    while (al.count(t)) t = al[t];
    return t;
  };
  auto aliases = [&](int t, int u) { return root_of(t) == root_of(u); };
  auto try_pieces = [&](int t, bool is_a, const GemmForm& gf, Buf& b) -> bool {
    const int split = is_a ? gf.a_split : gf.b_split;
    const bool mn = is_a ? gf.a_mn : gf.b_mn;
    const int nd = (int)b.box.size();
    std::vector<std::pair<int, std::vector<Rng>>> parts;
    for (int s = 0; s < k; ++s) {
      if (E.lay[s].shard_off[t] < 0) continue;
      std::vector<Rng> x;
      if (nd == 0 || !inter(b.box, E.lay[s].shard_box[t], x)) continue;
      parts.push_back({s, x});
    }
    if (parts.empty() || (int)parts.size() > TOFU_MAX_PIECES) return false;
    int d = -1;  // the single dimension along which the pieces differ from the region
    for (auto& pr : parts)
      for (int e = 0; e < nd; ++e)
        if (pr.second[e].lo != b.box[e].lo || pr.second[e].hi != b.box[e].hi) {
          if (d >= 0 && d != e) return false;
          d = e;
        }
    if (d < 0) d = 0;  // one owner holds the whole region
    const int g0 = d < split ? 0 : split, g1 = d < split ? split : nd;
    for (int e = g0; e < d; ++e)
      if (b.box[e].len() != 1) return false;  // pieces must be contiguous ranges of the 2-D view
    int64_t inner = 1;
    for (int e = d + 1; e < g1; ++e) inner *= b.box[e].len();
    std::sort(parts.begin(), parts.end(),
              [d](const std::pair<int, std::vector<Rng>>& x, const std::pair<int, std::vector<Rng>>& y) {
                return x.second[d].lo < y.second[d].lo;
              });
    int64_t at = b.box[d].lo;
    for (auto& pr : parts) {
      if (pr.second[d].lo != at) return false;
      at = pr.second[d].hi + 1;
    }
    if (at != b.box[d].hi + 1) return false;
    // GEMM dimension of the cut: K-major operands are [M|N][K], MN-major [K][M|N]
    const bool kdim = (d < split) == mn;
    const int gran = kdim ? 64 : (is_a ? 128 : 256);
    std::vector<Buf::RPiece> rp;
    for (auto& pr : parts) {
      const int s = pr.first;
      int64_t r_, c_, ld_, off_;
      if (!flat2(E.lay[s].shard_box[t], pr.second, split, r_, c_, ld_, off_)) return false;
      const int64_t start = (pr.second[d].lo - b.box[d].lo) * inner;
      if (start % gran || ld_ % 8 || (off_ * g.itemsize(t)) % 16) return false;
      rp.push_back({s, E.lay[s].shard_off[t] + off_ * g.itemsize(t), ld_, (int)start});
    }
    b.rp = std::move(rp);
    b.rp_dim = kdim ? 1 : 0;
    return true;
  };
  for (int r = 0; r < k; ++r) {
    auto dig = worker_digits(r, p.factors);
    for (size_t o = 0; o < g.ops.size(); ++o) {
      const OpDef& d = g.def_of((int)o);
      const OpInfo& oi = g.ops[o];
      if (!kernel_kind(d))
        throw Error(TOFU_ERR_ARG, "no sub-operator kernel for def '" + d.name + "'");
      LOp& L = all[r][o];
      std::vector<Rng> ib;
      iter_box(g, (int)o, p.osplit[o], p.factors, dig, ib);
      for (int v : p.osplit[o])
        if (d.is_red(v)) L.partial = true;
      const std::string kind = kernel_kind(d);
      const GemmForm gf = gemm_form(d);
      int64_t soff = 0;
      for (size_t pi = 0; pi < d.params.size(); ++pi) {
        int t = oi.inputs[pi];
        Buf b;
        b.box = required_box(g, (int)o, (int)pi, ib);
        b.dtype = g.tensors[t].dtype;
        const auto& own = E.lay[r].shard_box[t];
        const bool owns = E.lay[r].shard_off[t] >= 0;
        bool usable = owns && (kind == "ew" ? same(own, b.box) : contains(own, b.box));
        if (usable && kind == "conv") usable = conv_operand_ok(conv_geom(d), (int)pi, own, b.box);
        if (usable && kind == "window") usable = b.box.size() < 4 || (b.box[3].lo - own[3].lo) % 8 == 0;
        if (usable && kind == "gemm") {
          int64_t r_, c_, ld_, off_;
          const int split = (int)pi == gf.a_param ? gf.a_split : gf.b_split;
          usable = flat2(own, b.box, split, r_, c_, ld_, off_);
        }
        if (usable) {
          b.direct = true;
          b.off = E.lay[r].shard_off[t];
          b.buf_box = own;
        } else if (E.fuse_fetch && !aliases(t, oi.output) &&
                   ((kind == "gemm" && gf.ok && try_pieces(t, (int)pi == gf.a_param, gf, b)) ||
                    (kind == "conv" && E.fuse_fetch_conv && pi < 2 && conv1x1_form(conv_geom(d)).ok &&
                     try_pieces(t, pi == 0, conv1x1_form(conv_geom(d)), b)))) {
          b.direct = false;  // read in place from the owners (b.rp); no staging
          b.off = -1;
          b.buf_box = b.box;
        } else {
          b.direct = false;
          b.off = soff;  // relative to staging, fixed up below
          b.buf_box = b.box;
          soff = align_up(soff + vol(b.box) * g.itemsize(t));
        }
        L.in.push_back(b);
      }
      Buf ob;
      ob.box = produced_box(g, (int)o, ib);
      const int t = oi.output;
      const bool owns = E.lay[r].shard_off[t] >= 0;
      const auto& oown = E.lay[r].shard_box[t];
      bool odirect = !L.partial && owns && (kind == "ew" ? same(oown, ob.box) : contains(oown, ob.box));
      if (odirect && kind == "gemm") {
        int64_t r_, c_, ld_, off_;
        odirect = flat2(oown, ob.box, gf.nm, r_, c_, ld_, off_);
      }
      if (odirect && kind == "conv") {
        const ConvGeom cg = conv_geom(d);
        odirect = cg.kind == 2 ? full_from(oown, ob.box, 1) : (ob.box[3].lo - oown[3].lo) % 8 == 0;
      }
      if (odirect && kind == "window") odirect = (ob.box.back().lo - oown.back().lo) % 8 == 0;
      if (odirect) {
        ob.direct = true;
        ob.off = E.lay[r].shard_off[t];
        ob.buf_box = oown;
        ob.dtype = g.tensors[t].dtype;
      } else {
        ob.direct = false;
        ob.dtype = L.partial ? TOFU_F32 : g.tensors[t].dtype;
        ob.off = soff;
        ob.buf_box = ob.box;
        soff = align_up(soff + vol(ob.box) * (ob.dtype == TOFU_BF16 ? 2 : 4));
      }
      L.out = ob;
      stage_need[r] = std::max(stage_need[r], soff);
    }
  }
  // two staging buffers, alternating op by op (parity of the op index): an op's fetch / partial outputs do not
  // overwrite the previous op's, so the next op's fetch can run (on the comm stream) while this op's compute
  // and reduce still read theirs (build_launches)
  for (int r = 0; r < k; ++r) {
    E.lay[r].staging_bytes = 2 * stage_need[r];
    E.lay[r].total = E.lay[r].staging_off + 2 * stage_need[r];
    for (size_t o = 0; o < all[r].size(); ++o) {
      LOp& L = all[r][o];
      const int64_t base = E.lay[r].staging_off + (int64_t)(o % 2) * stage_need[r];
      for (auto& b : L.in)
        if (!b.direct && b.rp.empty()) b.off += base;
      if (!L.out.direct) L.out.off += base;
    }
  }
  // ------------------------------------------------------------------ pieces
  auto ptr = [&](int r, int64_t off) -> char* { return E.arena.empty() ? nullptr : E.arena[r] + off; };
  auto fill_geom = [](tofu_piece& pc, const std::vector<Rng>& ext_box) {
    const int n = (int)ext_box.size();
    for (int d = 0; d < 4; ++d) pc.extent[d] = 1;
    for (int d = 0; d < n; ++d) pc.extent[4 - n + d] = ext_box[d].len();
  };
  auto set_strides = [](int64_t* dst, const std::vector<Rng>& buf) {
    auto s = strides_of(buf);
    const int n = (int)buf.size();
    for (int d = 0; d < 4; ++d) dst[d] = 0;
    for (int d = 0; d < n; ++d) dst[4 - n + d] = s[d];
  };
  E.ledger_el = E.ledger_bytes = 0;
  E.rank_in.assign(k, 0);
  E.rank_out.assign(k, 0);
  for (int r = 0; r < k; ++r)
    for (size_t o = 0; o < g.ops.size(); ++o) {
      LOp& L = all[r][o];
      const OpInfo& oi = g.ops[o];
      for (size_t pi = 0; pi < L.in.size(); ++pi) {
        Buf& b = L.in[pi];
        if (b.direct) continue;
        const int t = oi.inputs[pi];
        if (!b.rp.empty()) {  // fused fetch: the GEMM reads the pieces in place; the ledger counts them
          for (auto& q : b.rp) {
            L.fetch_src.push_back(q.src);
            if (q.src != r) {
              std::vector<Rng> x;
              inter(b.box, E.lay[q.src].shard_box[t], x);
              E.ledger_el += vol(x);
              E.ledger_bytes += vol(x) * g.itemsize(t);
              E.rank_in[r] += vol(x) * g.itemsize(t);
              E.rank_out[q.src] += vol(x) * g.itemsize(t);
              L.remote_direct = true;
            }
          }
          continue;
        }
        for (int s = 0; s < k; ++s) {
          if (E.lay[s].shard_off[t] < 0) continue;
          std::vector<Rng> x;
          const auto& own = E.lay[s].shard_box[t];
          if (!b.box.empty() && !inter(b.box, own, x)) continue;
          tofu_piece pc;
          std::memset(&pc, 0, sizeof pc);
          fill_geom(pc, b.box.empty() ? b.box : x);
          pc.dst = ptr(r, b.off) ? ptr(r, b.off) + offset_in(b.buf_box, x) * g.itemsize(t) : nullptr;
          set_strides(pc.dst_stride, b.buf_box);
          pc.dst_dtype = pc.src_dtype = g.tensors[t].dtype;
          pc.nsrc = 1;
          pc.src[0] = ptr(s, E.lay[s].shard_off[t]) ? ptr(s, E.lay[s].shard_off[t]) + offset_in(own, x) * g.itemsize(t)
                                                    : nullptr;
          set_strides(pc.src_stride, own);
          L.fetch.push_back(pc);
          L.fetch_src.push_back(s);
          if (s != r) {
            E.ledger_el += vol(x);
            E.ledger_bytes += vol(x) * g.itemsize(t);
            E.rank_in[r] += vol(x) * g.itemsize(t);
            E.rank_out[s] += vol(x) * g.itemsize(t);
          }
        }
      }
    }
  // reduce / scatter: owner r pulls from every non-direct producer c
  for (size_t o = 0; o < g.ops.size(); ++o) {
    const int t = g.ops[o].output;
    for (int r = 0; r < k; ++r) {
      if (E.lay[r].shard_off[t] < 0) continue;
      const auto& own = E.lay[r].shard_box[t];
      std::vector<int> contrib;
      for (int c = 0; c < k; ++c) {
        const Buf& ob = all[c][o].out;
        if (ob.direct) continue;
        std::vector<Rng> x;
        if (!ob.box.empty() && !inter(ob.box, own, x)) continue;
        contrib.push_back(c);
      }
      if (contrib.empty()) continue;
      // grid of breakpoints within own
      const int n = (int)own.size();
      std::vector<std::vector<int64_t>> cuts(n);
      for (int d = 0; d < n; ++d) {
        std::set<int64_t> cs = {own[d].lo, own[d].hi + 1};
        for (int c : contrib) {
          const auto& b = all[c][o].out.box;
          if (b[d].lo > own[d].lo && b[d].lo <= own[d].hi) cs.insert(b[d].lo);
          if (b[d].hi + 1 > own[d].lo && b[d].hi + 1 <= own[d].hi) cs.insert(b[d].hi + 1);
        }
        cuts[d].assign(cs.begin(), cs.end());
      }
      std::vector<int> ci(n, 0);
      while (true) {
        std::vector<Rng> cell(n);
        for (int d = 0; d < n; ++d) cell[d] = {cuts[d][ci[d]], cuts[d][ci[d] + 1] - 1};
        std::vector<int> srcs;
        for (int c : contrib)
          if (n == 0 || contains(all[c][o].out.box, cell)) srcs.push_back(c);
        if (!srcs.empty()) {
          if ((int)srcs.size() > TOFU_MAX_SRC) throw Error(TOFU_ERR_ARG, "more than 8 contributors to one element");
          tofu_piece pc;
          std::memset(&pc, 0, sizeof pc);
          fill_geom(pc, cell);
          const int64_t es = g.itemsize(t);
          pc.dst = ptr(r, E.lay[r].shard_off[t]) ? ptr(r, E.lay[r].shard_off[t]) + offset_in(own, cell) * es : nullptr;
          set_strides(pc.dst_stride, own);
          pc.dst_dtype = g.tensors[t].dtype;
          pc.nsrc = (int)srcs.size();
          const Buf& ob0 = all[srcs[0]][o].out;
          pc.src_dtype = ob0.dtype;
          set_strides(pc.src_stride, ob0.buf_box);
          int nrem = 0;
          for (size_t s = 0; s < srcs.size(); ++s) {
            const Buf& ob = all[srcs[s]][o].out;
            const int64_t ses = ob.dtype == TOFU_BF16 ? 2 : 4;
            pc.src[s] = ptr(srcs[s], ob.off) ? ptr(srcs[s], ob.off) + offset_in(ob.buf_box, cell) * ses : nullptr;
            if (srcs[s] != r) {
              ++nrem;
              E.ledger_el += vol(cell);
              E.ledger_bytes += vol(cell) * ses;
              E.rank_in[r] += vol(cell) * ses;
              E.rank_out[srcs[s]] += vol(cell) * ses;
            }
          }
          all[r][o].reduce.push_back(pc);
          all[r][o].reduce_nremote.push_back(nrem);
        }
        int d = n - 1;
        while (d >= 0 && ++ci[d] + 1 >= (int)cuts[d].size()) ci[d--] = 0;
        if (d < 0) break;
      }
    }
  }
  // fused momentum + SGD (consecutive element-wise optimizer ops share one partition)
  for (int r = 0; r < k; ++r)
    for (size_t o = 0; o + 1 < g.ops.size(); ++o) {
      const OpInfo &a = g.ops[o], &b = g.ops[o + 1];
      if (!is_mom(g.defs[a.def].kernel) || !is_sgd(g.defs[b.def].kernel) || b.inputs[1] != a.output) continue;
      LOp &La = all[r][o], &Lb = all[r][o + 1];
      bool ok = La.out.direct && Lb.out.direct && La.fetch.empty() && Lb.fetch.empty();
      for (auto& x : La.in) ok &= x.direct;
      for (auto& x : Lb.in) ok &= x.direct;
      ok &= La.in[0].off == La.out.off && Lb.in[0].off == Lb.out.off;  // in place (aliased state)
      if (ok) {
        La.fused_sgd = true;
        La.absorbed.push_back((int)o + 1);
        Lb.skip = true;
      }
    }
  // wgrad GEMM -> mom -> sgd: fold the optimizer into the GEMM epilogue (c_mode 3) when the gradient is
  // complete and local and read by nothing else; the gradient then never reaches HBM.
  if (E.fuse)
    for (int r = 0; r < k; ++r)
      for (size_t o = 0; o < g.ops.size(); ++o) {
        const OpInfo& a = g.ops[o];
        const char* kk = kernel_kind(g.defs[a.def]);
        if (!kk || !(std::string(kk) == "gemm" || (std::string(kk) == "conv" && conv_geom(g.defs[a.def]).kind == 2)))
          continue;
        int reader = -1, readers = 0;
        for (size_t x = 0; x < g.ops.size(); ++x)
          for (int t : g.ops[x].inputs)
            if (t == a.output) {
              ++readers;
              reader = (int)x;
            }
        if (readers != 1 || reader <= (int)o || reader + 1 >= (int)g.ops.size()) continue;
        const OpInfo &b = g.ops[reader], &c = g.ops[reader + 1];
        if (!is_mom(g.defs[b.def].kernel) || !all[r][reader].fused_sgd) continue;
        // moving mom+sgd up to the GEMM must not reorder any access to M / W
        std::set<int> state = {b.inputs[0], b.output, c.inputs[0], c.output};
        for (auto& pr : g.alias)
          if (state.count(pr.first) || state.count(pr.second)) {
            state.insert(pr.first);
            state.insert(pr.second);
          }
        bool clash = false;
        for (int x = (int)o + 1; x < reader; ++x) {
          for (int t : g.ops[x].inputs) clash |= state.count(t) > 0;
          clash |= state.count(g.ops[x].output) > 0;
        }
        LOp& La = all[r][o];
        if (clash || !La.out.direct || La.partial || La.out.dtype != TOFU_F32) continue;
        La.fused_opt = reader;
        E.unmat.insert(a.output);   // the weight gradient stays in TMEM / registers
        La.absorbed.push_back(reader);
        La.absorbed.push_back(reader + 1);
        all[r][reader].skip = true;
      }
  // LSTM: the two cell ops of one timestep read the same gate rows -> one kernel (one pass over GX / GH)
  if (E.fuse)
    for (int r = 0; r < k; ++r)
      for (size_t o = 0; o + 1 < g.ops.size(); ++o) {
        const std::string &na = g.defs[g.ops[o].def].kernel, &nb = g.defs[g.ops[o + 1].def].kernel;
        const bool fwd = na == "cell_c" && nb == "cell_h";
        const bool bwd = na == "cell_bwd_a" && nb == "cell_bwd_c";
        if (!fwd && !bwd) continue;
        LOp &La = all[r][o], &Lb = all[r][o + 1];
        if (La.skip || !La.out.direct || !Lb.out.direct || !Lb.fetch.empty()) continue;
        auto same_buf = [](const Buf& x, const Buf& y) { return x.off == y.off && same(x.box, y.box) && same(x.buf_box, y.buf_box); };
        // gate operands: both direct views of the same shard rows (the ops read different gate subsets; the
        // kernel addresses gates from the row base, so only rows and h must agree)
        auto same_rows = [](const Buf& x, const Buf& y) {
          return x.direct && y.direct && x.off == y.off && same(x.buf_box, y.buf_box) && x.box.size() == 3 &&
                 x.box[0].lo == y.box[0].lo && x.box[0].hi == y.box[0].hi && x.box[2].lo == y.box[2].lo &&
                 x.box[2].hi == y.box[2].hi;
        };
        bool ok = same_rows(La.in[0], Lb.in[0]) && same_rows(La.in[1], Lb.in[1]);
        if (fwd) ok &= g.ops[o + 1].inputs[2] == g.ops[o].output && same_buf(Lb.in[2], La.out);  // h reads this c
        if (bwd)
          for (int q = 0; q < 4; ++q) ok &= same_buf(La.in[3 + q], Lb.in[2 + q]);  // C, DU, DR, DN
        if (!ok) continue;
        La.fused_next = true;
        La.absorbed.push_back((int)o + 1);
        Lb.skip = true;
      }
  // LSTM forward: the gate GEMM of step t (GH_t = h_{t-1} Wh) and the fused cell pair reading GH_t (c_t, h_t):
  // one launch — when the GEMM splits K, the cell kernel sums the fp32 partial planes itself (in split order,
  // rounding GH to its dtype, storing GH and using it as stored), so the split-K reduction launch and the
  // cell launch become one kernel.  Off by default (TOFU_FUSE_GATE_CELL=1 turns it on): measured on 8 virtual
  // ranks (LSTM-6-4K, tools/kineto_step.py) the fused kernel (7.6 us with one element per thread, 9.0 us with
  // four) costs what the reduction (2.7 us) and the cell (5.6 us) cost apart: 49.0 vs 49.0 ms per step.
  if (E.fuse && E.fuse_gate_cell)
    for (int r = 0; r < k; ++r)
      for (size_t o = 0; o + 2 < g.ops.size(); ++o) {
        const OpDef& dg = g.defs[g.ops[o].def];
        if (!kernel_kind(dg) || std::string(kernel_kind(dg)) != "gemm" || g.defs[g.ops[o + 1].def].kernel != "cell_c")
          continue;
        LOp &La = all[r][o], &Lc = all[r][o + 1];
        if (La.skip || Lc.skip || !Lc.fused_next || !La.out.direct || La.partial || La.fused_opt >= 0 || La.ep ||
            La.red_ep || !La.reduce.empty() || La.out.dtype != TOFU_BF16 || La.out.box.size() != 3 ||
            !same(La.out.box, La.out.buf_box) || !Lc.fetch.empty() || !Lc.reduce.empty() ||
            g.ops[o + 1].inputs.size() < 2 || g.ops[o + 1].inputs[1] != g.ops[o].output)
          continue;
        bool ok = Lc.in.size() >= 3 && Lc.out.direct;
        for (auto& b : Lc.in) ok &= b.direct;
        const Buf& G = Lc.in[1];
        ok = ok && G.off == La.out.off && same(G.buf_box, La.out.buf_box) && G.box.size() == 3 &&
             G.box[0].lo == La.out.box[0].lo && G.box[0].hi == La.out.box[0].hi && G.box[2].lo == La.out.box[2].lo &&
             G.box[2].hi == La.out.box[2].hi && La.out.box[1].lo == 0 && Lc.out.box.size() == 2 &&
             Lc.out.box[0].len() == La.out.box[0].len() &&  // (c rows: the merged timestep storage's coordinates)
             Lc.out.box[1].lo == La.out.box[2].lo && Lc.out.box[1].hi == La.out.box[2].hi;
        if (!ok) continue;
        La.cell_after = (int)o + 1;
        La.absorbed.push_back((int)o + 1);
        La.absorbed.push_back((int)o + 2);
        Lc.skip = true;
      }
  // The loss and its gradient read the same (Y, T) shards: one pass computes both (sumsq + mse_grad, R8)
  if (E.fuse)
    for (int r = 0; r < k; ++r)
      for (size_t o = 0; o + 1 < g.ops.size(); ++o) {
        if (g.defs[g.ops[o].def].kernel != "sumsq" || g.defs[g.ops[o + 1].def].kernel != "mse_grad") continue;
        if (g.ops[o].inputs != g.ops[o + 1].inputs) continue;
        LOp &La = all[r][o], &Lb = all[r][o + 1];
        if (La.skip || Lb.skip || !Lb.out.direct || !Lb.fetch.empty() || !Lb.reduce.empty() || !La.fetch.empty())
          continue;
        auto same_buf = [](const Buf& x, const Buf& y) {
          return x.direct && y.direct && x.off == y.off && same(x.box, y.box) && same(x.buf_box, y.buf_box);
        };
        if (!same_buf(La.in[0], Lb.in[0]) || !same_buf(La.in[1], Lb.in[1]) || !same(Lb.out.box, Lb.in[0].box))
          continue;
        La.fused_loss_grad = true;
        La.absorbed.push_back((int)o + 1);
        Lb.skip = true;
      }
  // Element-wise consumers folded into their producer's epilogue (R8/R13): a GEMM / convolution whose bf16
  // output T is read only by one relu / addrelu / add / relu_grad(·, T) op (and an add's result only by one
  // relu_grad) writes that op's output directly; the other operands (produced earlier) are read by the
  // epilogue.  Every operand must be the rank's own shard of the same box (no communication moves).
  if (E.fuse) {
    std::vector<int> producer(g.tensors.size(), -1), nprod(g.tensors.size(), 0), nread(g.tensors.size(), 0);
    for (size_t o = 0; o < g.ops.size(); ++o) {
      producer[g.ops[o].output] = (int)o;
      ++nprod[g.ops[o].output];
      for (int t : g.ops[o].inputs) ++nread[t];
    }
    std::set<int> aliased;
    for (auto& pr : g.alias) {
      aliased.insert(pr.first);
      aliased.insert(pr.second);
    }
    auto consumer = [&](int t) {  // the single op reading t (after its producer), else -1
      if (nread[t] != 1 || nprod[t] != 1 || aliased.count(t)) return -1;
      for (size_t x = producer[t] + 1; x < g.ops.size(); ++x)
        for (int u : g.ops[x].inputs)
          if (u == t) return (int)x;
      return -1;
    };
    auto earlier = [&](int t, int o) { return nprod[t] == 0 || (nprod[t] == 1 && producer[t] < o); };
    for (int r = 0; r < k; ++r)
      for (size_t o = 0; o < g.ops.size(); ++o) {
        LOp& Lo = all[r][o];
        const OpDef& d = g.def_of((int)o);
        const char* kk = kernel_kind(d);
        if (!kk || Lo.skip || Lo.partial || Lo.fused_opt >= 0 || !Lo.reduce.empty() || Lo.out.dtype != TOFU_BF16)
          continue;
        const std::string kind = kk;
        if (kind == "conv") {
          const ConvGeom cg = conv_geom(d);
          if (!(cg.kind == 0 || (cg.kind == 1 && cg.s == 1))) continue;
          if (!(cg.R == 1 && cg.s == 1) && Lo.out.box.back().len() % 32) continue;  // gather-kernel epilogue chunks
        } else if (kind != "gemm") {
          continue;
        }
        const int t = g.ops[o].output;
        const int e = consumer(t);
        if (e < 0) continue;
        LOp& Le = all[r][e];
        const std::string& en = g.def_of(e).kernel;
        auto same_direct = [&](const Buf& b) { return b.direct && same(b.box, Lo.out.box) && same(b.buf_box, b.box); };
        bool ok = Le.fetch.empty() && Le.reduce.empty() && !Le.skip && same_direct(Le.out) && Le.out.dtype == TOFU_BF16;
        for (auto& b : Le.in) ok &= same_direct(b) && b.dtype == TOFU_BF16;
        if (!ok) continue;
        const auto& ins = g.ops[e].inputs;
        int ep = 0, add_i = -1, mask_i = -1;
        if ((en == "relu" || en == "relu4") && ins[0] == t) ep = 1;
        else if ((en == "addrelu" || en == "add4") && ins.size() == 2 && (ins[0] == t) != (ins[1] == t)) {
          add_i = ins[0] == t ? 1 : 0;
          ep = 2 | (en == "addrelu" ? 1 : 0);
        } else if ((en == "relu_grad" || en == "relu_grad4") && ins[1] == t && ins[0] != t) {
          mask_i = 0;
          ep = 4;
        }
        if (!ep || (add_i >= 0 && !earlier(ins[add_i], (int)o)) || (mask_i >= 0 && !earlier(ins[mask_i], (int)o)))
          continue;
        Buf out = Le.out;
        Buf mask;
        int e2 = -1;
        if (en == "add4") {  // gradient sum followed by its single relu_grad: fold the mask too
          const int t2 = g.ops[e].output, c2 = consumer(t2);
          if (c2 >= 0) {
            LOp& L2 = all[r][c2];
            const std::string& n2 = g.def_of(c2).kernel;
            bool ok2 = (n2 == "relu_grad" || n2 == "relu_grad4") && g.ops[c2].inputs[1] == t2 &&
                       g.ops[c2].inputs[0] != t2 && earlier(g.ops[c2].inputs[0], (int)o) && L2.fetch.empty() &&
                       L2.reduce.empty() && !L2.skip && same_direct(L2.out) && L2.out.dtype == TOFU_BF16;
            for (auto& b : L2.in) ok2 &= same_direct(b);
            if (ok2) {
              e2 = c2;
              ep |= 4;
              mask = L2.in[0];
              out = L2.out;
            }
          }
        }
        Lo.ep = ep;
        if (add_i >= 0) Lo.epi_add = Le.in[add_i];
        if (mask_i >= 0) Lo.epi_mask = Le.in[mask_i];
        if (e2 >= 0) {
          Lo.epi_mask = mask;
          all[r][e2].skip = true;
          Lo.absorbed.push_back(e2);
          E.unmat.insert(g.ops[e].output);   // the gradient sum before its mask
        }
        Lo.absorbed.push_back(e);
        E.unmat.insert(t);                   // the producer's own (pre-epilogue) output
        Lo.out = out;
        Le.skip = true;
      }
  }
  // Partition-n-reduce fused with the reduced tensor's element-wise consumer (P:L674-678 coalescing, R8): when
  // op o's output T is summed by reduce pieces (a split reduction) and T's single reader e is a relu,
  // relu_grad(·, T), add / addrelu or momentum(+SGD) op whose operands are all the rank's own shards of T's
  // box, the reduce pieces apply e while storing: T itself is never written, e's launch disappears (and, for the
  // optimizer, the separate fp32 gradient round trip).  Decided for all ranks at once (the launch sequence is
  // the same in every process).
  if (E.fuse) {
    std::vector<int> producer(g.tensors.size(), -1), nprod(g.tensors.size(), 0), nread(g.tensors.size(), 0);
    for (size_t o = 0; o < g.ops.size(); ++o) {
      producer[g.ops[o].output] = (int)o;
      ++nprod[g.ops[o].output];
      for (int t : g.ops[o].inputs) ++nread[t];
    }
    std::set<int> aliased;
    for (auto& pr : g.alias) {
      aliased.insert(pr.first);
      aliased.insert(pr.second);
    }
    auto earlier = [&](int t, int o) { return nprod[t] == 0 || (nprod[t] == 1 && producer[t] < o); };
    for (size_t o = 0; o < g.ops.size(); ++o) {
      const int t = g.ops[o].output;
      if (nread[t] != 1 || nprod[t] != 1 || aliased.count(t)) continue;
      int e = -1;
      for (size_t x = o + 1; x < g.ops.size() && e < 0; ++x)
        for (int u : g.ops[x].inputs)
          if (u == t) e = (int)x;
      if (e < 0) continue;
      const std::string& en = g.def_of(e).kernel;
      const auto& ins = g.ops[e].inputs;
      int ep = 0, aux_i = -1;
      if ((en == "relu" || en == "relu4") && ins[0] == t) ep = TOFU_PIECE_RELU;
      else if ((en == "relu_grad" || en == "relu_grad4") && ins[1] == t && ins[0] != t) {
        ep = TOFU_PIECE_MASK;
        aux_i = 0;
      } else if ((en == "add4" || en == "addrelu") && ins.size() == 2 && (ins[0] == t) != (ins[1] == t)) {
        ep = en == "add4" ? TOFU_PIECE_ADD : TOFU_PIECE_ADDRELU;
        aux_i = ins[0] == t ? 1 : 0;
      } else if (is_mom(en) && ins[1] == t && e + 1 < (int)g.ops.size()) {
        ep = TOFU_PIECE_MOM_SGD;
      }
      if (!ep || (aux_i >= 0 && !earlier(ins[aux_i], (int)o))) continue;
      if (ep == TOFU_PIECE_MOM_SGD) {  // moving mom + sgd up to o must not reorder any access to M / W
        const OpInfo &b = g.ops[e], &c = g.ops[e + 1];
        std::set<int> state = {b.inputs[0], b.output, c.inputs[0], c.output};
        for (auto& pr : g.alias)
          if (state.count(pr.first) || state.count(pr.second)) {
            state.insert(pr.first);
            state.insert(pr.second);
          }
        bool clash = false;
        for (int x = (int)o + 1; x < e; ++x) {
          for (int u : g.ops[x].inputs) clash |= state.count(u) > 0;
          clash |= state.count(g.ops[x].output) > 0;
        }
        if (clash) continue;
      }
      bool ok = true, any = false;
      for (int r = 0; r < k && ok; ++r) {
        LOp &Lo = all[r][o], &Le = all[r][e];
        if (E.lay[r].shard_off[t] < 0) {
          ok = Lo.reduce.empty();
          continue;
        }
        const auto& own = E.lay[r].shard_box[t];
        int64_t cov = 0;
        for (auto& pc : Lo.reduce) cov += pc.extent[0] * pc.extent[1] * pc.extent[2] * pc.extent[3];
        if (Lo.reduce.empty() || cov != vol(own)) {
          ok = false;
          break;
        }
        any = true;
        auto mine = [&](const Buf& b) { return b.direct && same(b.box, own) && same(b.buf_box, own); };
        ok = !Le.skip && Le.fetch.empty() && Le.reduce.empty() && mine(Le.out) && Lo.fused_opt < 0;
        for (auto& b : Le.in) ok = ok && (b.direct ? mine(b) : false) ;
        if (ep == TOFU_PIECE_MOM_SGD) {
          const LOp& Ls = all[r][e + 1];
          ok = ok && Le.fused_sgd && Ls.skip;
          for (auto& b : Ls.in) ok = ok && mine(b);
          ok = ok && mine(Ls.out) && Le.out.dtype == TOFU_F32;
        } else {
          ok = ok && Le.out.dtype == TOFU_BF16;
        }
      }
      if (!ok || !any) continue;
      const float s0 = ep == TOFU_PIECE_MOM_SGD ? (float)g.def_of(e).kconst.at(0) : 0.f;
      const float s1 = ep == TOFU_PIECE_MOM_SGD ? (float)g.def_of(e + 1).kconst.at(0) : 0.f;
      for (int r = 0; r < k; ++r) {
        if (E.lay[r].shard_off[t] < 0) continue;
        LOp &Lo = all[r][o], &Le = all[r][e];
        const auto& own = E.lay[r].shard_box[t];
        char* base = E.arena.empty() ? nullptr : E.arena[r];
        for (auto& pc : Lo.reduce) {
          // the piece's destination cell inside `own`: recover its element offset from the T destination
          const int64_t cell_off = base ? ((char*)pc.dst - (base + E.lay[r].shard_off[t])) / g.itemsize(t) : 0;
          pc.ep = ep;
          pc.s0 = s0;
          pc.s1 = s1;
          const Buf& outb = Le.out;  // relu / mask / add: e's output; mom: M_new = M (in place)
          pc.dst_dtype = outb.dtype;
          pc.dst = base ? base + outb.off + cell_off * (outb.dtype == TOFU_BF16 ? 2 : 4) : nullptr;
          if (aux_i >= 0) pc.aux0 = base ? base + Le.in[aux_i].off + cell_off * 2 : nullptr;
          if (ep == TOFU_PIECE_MOM_SGD) {
            const Buf& W = all[r][e + 1].in[0];
            pc.aux0 = base ? base + W.off + cell_off * 2 : nullptr;
          }
        }
        Lo.red_ep = ep;
        Lo.red_absorbed.push_back(e);
        if (ep == TOFU_PIECE_MOM_SGD) Lo.red_absorbed.push_back(e + 1);
        Le.skip = true;
        (void)own;
      }
      E.unmat.insert(t);
    }
  }
  // Conv data gradients read their weights K-major from an executor-owned transposed copy of the weight
  // shard (W[co][ky][kx][ci] -> WT[ci][ky][kx][co], refreshed right before the launch): the MN-major weight
  // operand runs ~30% slower on the tensor cores (profiles/r01b_summary.md).  Appended after the staging
  // region (persistent, one per op).  TOFU_WT=0 disables.
  // A weight fetched into staging (a batch-split layer's whole weight under a k-way plan) is transposed from the
  // staging copy into one scratch region per rank shared by all such launches (each transposes right before
  // its own convolution, on the compute stream): the 8-way WResNet data gradients otherwise ran MN-major.
  {
    const char* ev = std::getenv("TOFU_WT");
    const bool use_wt = !(ev && ev[0] == '0');
    for (int r = 0; r < k && use_wt; ++r) {
      std::vector<int> staged;
      int64_t scratch = 0;
      for (size_t o = 0; o < g.ops.size(); ++o) {
        const OpDef& d = g.def_of((int)o);
        const char* kk = kernel_kind(d);
        if (!kk || std::string(kk) != "conv") continue;
        const ConvGeom cg = conv_geom(d);
        LOp& L = all[r][o];
        if (cg.kind != 1 || L.skip || (cg.R == 1 && cg.s == 1)) continue;  // 1x1 stride-1: the GEMM path
        const Buf& W = L.in[1];
        const bool stg = !W.direct && W.rp.empty() && same(W.box, W.buf_box);
        if ((!W.direct && !stg) || W.buf_box.size() != 4 || W.box[1].lo != W.buf_box[1].lo ||
            W.box[1].hi != W.buf_box[1].hi || W.box[2].lo != W.buf_box[2].lo || W.box[2].hi != W.buf_box[2].hi)
          continue;
        const int64_t nch = W.box[0].len(), co_sh = W.buf_box[0].len();
        if (nch % 64 || co_sh % 8 || W.buf_box[3].len() % 8) continue;  // whole 64-channel K blocks per tap
        if (stg) {
          staged.push_back((int)o);
          scratch = std::max<int64_t>(scratch, vol(W.buf_box) * 2);
          continue;
        }
        L.wt_off = E.lay[r].total;
        E.lay[r].total = align_up(E.lay[r].total + vol(W.buf_box) * 2);
      }
      if (!staged.empty()) {
        const int64_t off = E.lay[r].total;
        E.lay[r].total = align_up(off + scratch);
        for (int o : staged) all[r][o].wt_off = off;
      }
    }
  }
  E.remote_fetch.assign(g.ops.size(), 0);
  E.remote_reduce.assign(g.ops.size(), 0);
  E.remote_direct.assign(g.ops.size(), 0);
  for (int r = 0; r < k; ++r)
    for (size_t o = 0; o < g.ops.size(); ++o) {
      for (int s : all[r][o].fetch_src) E.remote_fetch[o] |= s != r;
      E.remote_direct[o] |= all[r][o].remote_direct;
      for (int n : all[r][o].reduce_nremote) E.remote_reduce[o] |= n > 0;
    }
  // Global memory-access summary of every op's launches (union over ALL ranks, so every process derives the
  // same synchronisation): objects are tensor storages (alias roots) and the two staging buffers (kStage0 +
  // op parity).  rreads = objects some rank reads in a PEER's memory.
  {
    std::map<int, int> al(g.alias.begin(), g.alias.end());
    auto aroot = [&](int t) {
      while (al.count(t)) t = al[t];
      return t;
    };
    const int nt = (int)g.tensors.size();
    // tensors whose storage overlaps on some rank (the memory planner packs transient tensors of disjoint
    // lifetimes into the same bytes) are ONE object: a write to one waits for the readers of the other
    std::vector<int> uf(nt);
    for (int t = 0; t < nt; ++t) uf[t] = t;
    std::function<int(int)> find = [&](int x) { return uf[x] == x ? x : uf[x] = find(uf[x]); };
    for (int r = 0; r < k; ++r) {
      std::vector<std::tuple<int64_t, int64_t, int>> iv;
      for (int t = 0; t < nt; ++t)
        if (E.lay[r].shard_off[t] >= 0 && !al.count(t))
          iv.emplace_back(E.lay[r].shard_off[t], E.lay[r].shard_off[t] + vol(E.lay[r].shard_box[t]) * g.itemsize(t), t);
      std::sort(iv.begin(), iv.end());
      int64_t hi = -1;
      int grp = -1;
      for (auto& [lo, h, t] : iv) {
        if (grp >= 0 && lo < hi) uf[find(t)] = find(grp);
        else grp = t;
        if (lo >= hi) grp = t;
        hi = std::max(hi, h);
      }
    }
    auto root = [&](int t) { return find(aroot(t)); };
    E.acc.assign(g.ops.size(), {});
    for (size_t o = 0; o < g.ops.size(); ++o) {
      Exec::OpAcc& A = E.acc[o];
      const int S = nt + (int)(o % 2);
      std::set<int> fr, cr, cw, crr, rr, rw;
      bool rrem = false;
      for (int r = 0; r < k; ++r) {
        const LOp& L = all[r][o];
        A.any_fetch |= !L.fetch.empty();
        A.any_reduce |= !L.reduce.empty();
        for (size_t q = 0; q < L.fetch.size(); ++q)
          if (L.fetch_src[q] != r) A.fetch_remote = true;
        for (size_t pi = 0; pi < L.in.size(); ++pi) {
          const Buf& b = L.in[pi];
          const int t = root(g.ops[o].inputs[pi]);
          if (b.direct) {
            cr.insert(t);
          } else if (!b.rp.empty()) {
            cr.insert(t);
            for (auto& q : b.rp)
              if (q.src != r) crr.insert(t);
          } else {
            fr.insert(t);  // the fetch reads the owners' shards, writes staging
            cr.insert(S);
          }
        }
        cw.insert(L.out.direct ? root(g.ops[o].output) : S);
        if (!L.out.direct) cw.insert(root(g.ops[o].output));  // (conservative: the scatter / reduce writes it)
        for (int a : L.absorbed) {
          for (int t : g.ops[a].inputs) cr.insert(root(t));
          cw.insert(root(g.ops[a].output));
        }
        if (!L.reduce.empty()) {
          rr.insert(S);
          rw.insert(root(g.ops[o].output));
          for (int n : L.reduce_nremote) rrem |= n > 0;
          for (int a : L.red_absorbed) {
            for (int t : g.ops[a].inputs) rr.insert(root(t));
            rw.insert(root(g.ops[a].output));
          }
        }
      }
      A.f_rreads.assign(fr.begin(), fr.end());
      A.c_reads.assign(cr.begin(), cr.end());
      A.c_writes.assign(cw.begin(), cw.end());
      A.c_rreads.assign(crr.begin(), crr.end());
      A.r_reads.assign(rr.begin(), rr.end());
      A.r_writes.assign(rw.begin(), rw.end());
      if (rrem) A.r_rreads.push_back(S);
      A.stage = S;
    }
  }
  E.lops.clear();
  for (int r : E.local) E.lops.push_back(all[r]);
}

void build_launches(Exec& E) {
  const Graph& g = *E.g;
  std::vector<tofu_piece> host;
  E.launches.clear();
  const int nl = (int)E.local.size();
  const int nobj = (int)g.tensors.size() + 2;
  // Two streams: compute launches (and the loss memset) on the caller's stream, fetch / reduce / barrier
  // launches on the executor's comm stream, ordered by the data dependencies between them (the objects of
  // E.acc: last writer / readers since): a fetch runs as soon as its inputs exist and its staging buffer is
  // free, overlapping the previous op's compute (communication overlapped with computation).
  //
  // Multi-process synchronisation.  A device barrier (all ranks, comm stream) is inserted only where a hazard
  // between ranks exists, tracked over the same objects from the ALL-rank summaries (every process derives the
  // same barrier sequence): before a launch that reads an object in a peer's memory which some rank wrote since
  // the last barrier (RAW), and before a launch that writes an object some rank read remotely since the last
  // barrier (WAR).  A barrier waits for the local writers / readers of those objects and later launches that
  // touch them wait for it.  A final barrier closes the step.
  // pass 1 (all ranks alike): where the barriers go, and the objects each one orders
  std::map<std::pair<int, int>, std::vector<int>> bar_before;  // (op, phase 0 fetch / 1 compute / 2 reduce)
  if (E.multi_process) {
    std::set<int> w_since, rr_since;  // since the last barrier: objects written (any rank), read remotely
    auto step = [&](int o, int ph, const std::vector<int>& writes, const std::vector<int>& rreads) {
      bool hazard = false;
      for (int x : rreads) hazard |= w_since.count(x) > 0;
      for (int x : writes) hazard |= rr_since.count(x) > 0;
      if (hazard) {
        std::set<int> objs(w_since.begin(), w_since.end());
        objs.insert(rr_since.begin(), rr_since.end());
        bar_before[{o, ph}].assign(objs.begin(), objs.end());
        w_since.clear();
        rr_since.clear();
      }
      w_since.insert(writes.begin(), writes.end());
      rr_since.insert(rreads.begin(), rreads.end());
    };
    for (size_t o = 0; o < g.ops.size(); ++o) {
      const Exec::OpAcc& A = E.acc[o];
      if (A.any_fetch) step((int)o, 0, {A.stage}, A.fetch_remote ? A.f_rreads : std::vector<int>());
      step((int)o, 1, A.c_writes, A.c_rreads);
      if (A.any_reduce) step((int)o, 2, A.r_writes, A.r_rreads);
    }
  }
  // pass 2: this process's launches, each waiting for its data dependencies (last writer / readers since)
  std::vector<int> last_writer(nobj, -1);
  std::vector<std::vector<int>> readers(nobj);
  auto deps_of = [&](const std::vector<int>& reads, const std::vector<int>& writes) {
    std::set<int> deps;
    for (int x : reads)
      if (last_writer[x] >= 0) deps.insert(last_writer[x]);
    for (int x : writes) {
      if (last_writer[x] >= 0) deps.insert(last_writer[x]);
      for (int y : readers[x]) deps.insert(y);
    }
    return std::vector<int>(deps.begin(), deps.end());
  };
  int last_compute = -1;
  auto add = [&](Exec::Launch L, const std::vector<int>& reads, const std::vector<int>& writes) {
    const int li = (int)E.launches.size();
    L.waits = deps_of(reads, writes);
    // virtual ranks (no barriers, one GPU): one stream unless TOFU_STREAMS=2 — measured, the second stream
    // does not pay there (WResNet-152-4 k = 8: 100.3 ms one stream, 102.9-104.8 ms two: the copy kernels
    // compete with the convolutions for the same SMs / HBM, and a cross-stream event wait breaks the
    // programmatic-launch chain); with TOFU_STREAMS=2, a fetch / reduce that needs the compute launch just
    // before it stays on the compute stream
    if (!E.multi_process && L.stream == 1 &&
        (E.streams < 2 || (!L.waits.empty() && L.waits.back() == last_compute && last_compute == li - 1)))
      L.stream = 0;
    if (L.kind == 1 || L.kind == 4) last_compute = li;
    E.launches.push_back(L);
    for (int x : reads) readers[x].push_back(li);
    for (int x : writes) {
      last_writer[x] = li;
      readers[x].clear();
    }
  };
  // a barrier: after the local writers / readers of every object it orders, before any later launch
  // touching them (it reads and writes them all)
  auto barrier = [&](int o, const std::vector<int>& objs) {
    Exec::Launch B{3, o, -1, 0, 0, 0};
    B.stream = 1;
    add(B, objs, objs);
  };
  auto maybe_barrier = [&](int o, int ph) {
    auto it = bar_before.find({(int)o, ph});
    if (it != bar_before.end()) barrier(o, it->second);
  };
  for (size_t o = 0; o < g.ops.size(); ++o) {
    const Exec::OpAcc& A = E.acc[o];
    bool any_fetch = false;
    for (int li = 0; li < nl; ++li) any_fetch |= !E.lops[li][o].fetch.empty();
    maybe_barrier((int)o, 0);
    if (any_fetch) {
      Exec::Launch L{0, (int)o, -1, (int64_t)host.size(), 0, 0};
      L.stream = 1;
      for (int li = 0; li < nl; ++li)
        for (auto& pc : E.lops[li][o].fetch) {
          host.push_back(pc);
          L.max_elems = std::max(L.max_elems, pc.extent[0] * pc.extent[1] * pc.extent[2] * pc.extent[3]);
        }
      L.npieces = (int64_t)host.size() - L.piece_off;
      add(L, A.f_rreads, {A.stage});
    }
    maybe_barrier((int)o, 1);
    for (int li = 0; li < nl; ++li) {
      if (E.lops[li][o].skip) continue;
      if (g.defs[g.ops[o].def].kernel == "sumsq") add({4, (int)o, li, 0, 0, 0}, {}, A.c_writes);
      add({1, (int)o, li, 0, 0, 0}, A.c_reads, A.c_writes);
    }
    bool any_red = false;
    for (int li = 0; li < nl; ++li) any_red |= !E.lops[li][o].reduce.empty();
    maybe_barrier((int)o, 2);
    if (any_red) {
      Exec::Launch L{2, (int)o, -1, (int64_t)host.size(), 0, 0};
      L.stream = 1;
      for (int li = 0; li < nl; ++li)
        for (auto& pc : E.lops[li][o].reduce) {
          host.push_back(pc);
          L.max_elems = std::max(L.max_elems, pc.extent[0] * pc.extent[1] * pc.extent[2] * pc.extent[3]);
        }
      L.npieces = (int64_t)host.size() - L.piece_off;
      add(L, A.r_reads, A.r_writes);
    }
  }
  if (E.multi_process) {  // closes the step: orders every object
    std::vector<int> all_objs(nobj);
    for (int x = 0; x < nobj; ++x) all_objs[x] = x;
    barrier(-1, all_objs);
  }
  // keep only cross-stream waits (same-stream order is implicit), the latest one per stream suffices
  for (size_t i = 0; i < E.launches.size(); ++i) {
    auto& L = E.launches[i];
    int latest = -1;
    for (int j : L.waits)
      if (E.launches[j].stream != L.stream) latest = std::max(latest, j);
    L.waits.clear();
    if (latest >= 0) {
      L.waits.push_back(latest);
      E.launches[latest].rec = true;
    }
  }
  // piece tasks of every fetch / reduce launch (pieces normalised in place; task piece indices are
  // relative to the launch's first piece)
  E.host_tasks.clear();
  for (auto& L : E.launches) {
    if (L.kind != 0 && L.kind != 2) continue;
    int64_t nt = 0;
    int rc = tofu_pieces_tasks(host.data() + L.piece_off, (int)L.npieces, nullptr, 0, &nt);
    if (rc) throw Error(rc, "tofu_pieces_tasks failed");
    L.task_off = (int64_t)E.host_tasks.size();
    L.ntasks = nt;
    E.host_tasks.resize(L.task_off + nt);
    rc = tofu_pieces_tasks(host.data() + L.piece_off, (int)L.npieces, E.host_tasks.data() + L.task_off, nt, &nt);
    if (rc) throw Error(rc, "tofu_pieces_tasks failed");
    L.all_raw = 1;
    for (int64_t q = 0; q < nt; ++q) L.all_raw &= E.host_tasks[L.task_off + q].pad_ == 1;
    int maxsrc = 0;
    for (int64_t pq = L.piece_off; pq < L.piece_off + L.npieces; ++pq) maxsrc = std::max(maxsrc, host[pq].nsrc);
    if (!L.all_raw && maxsrc >= 4) L.all_raw = 2;  // many-source reduce kernel (tofu_pieces_run)
  }
  E.host_pieces = std::move(host);
  int64_t n = 0;
  for (auto& L : E.launches)
    if (L.kind != 4) ++n;
  E.n_kernels = n;
}

std::vector<tofu_conv_args> conv_args(Exec& E, int o, int li);

// fused fetch: a GEMM operand read in place from its owners' shards (piece 0 doubles as the shape reference)
void set_operand_pieces(const Exec& E, const Buf& X, tofu_operand_pieces& P, const void*& ptr, int& ld) {
  std::memset(&P, 0, sizeof P);
  P.n = (int)X.rp.size();
  P.dim = X.rp_dim;
  for (int i = 0; i < P.n; ++i) {
    P.start[i] = X.rp[i].start;
    P.ptr[i] = E.arena[X.rp[i].src] + X.rp[i].off;
    P.ld[i] = X.rp[i].ld;
  }
  ptr = P.ptr[0];
  ld = (int)P.ld[0];
}

// 1x1 stride-1 convolution as tofu_gemm_args (forward: pixels x ci . (co x ci)^T; data gradient:
// pixels x co . (co x ci); weight gradient: (pixels x co)^T . (pixels x ci)), optimizer fused as for GEMMs.
bool conv1x1_gemm(Exec& E, int o, int li, Exec::GemmLaunch& G) {
  const Graph& g = *E.g;
  const ConvGeom cg = conv_geom(g.def_of(o));
  if (cg.R != 1 || cg.s != 1 || cg.p != 0) return false;
  const int r = E.local[li];
  const LOp& L = E.lops[li][o];
  const Buf &P0 = L.in[0], &P1 = L.in[1], &O = L.out;
  int64_t r0, c0, ld0, off0, r1, c1, ld1, off1, ro, co, ldo, offo;
  const bool w_out = cg.kind == 2;
  // activations / gradients over pixels: [b, y, x][c] row blocks; weights [co][1][1][ci]: [co][ci]
  if (!flat2(P0.buf_box, P0.box, 3, r0, c0, ld0, off0)) return false;
  if (!flat2(P1.buf_box, P1.box, cg.kind == 2 ? 3 : 1, r1, c1, ld1, off1)) return false;
  if (!flat2(O.buf_box, O.box, w_out ? 1 : 3, ro, co, ldo, offo)) return false;
  std::memset(&G.a, 0, sizeof G.a);
  char* base = E.arena[r];
  G.a.A = base + P0.off + off0 * 2;
  G.a.lda = (int)ld0;
  G.a.B = base + P1.off + off1 * 2;
  G.a.ldb = (int)ld1;
  G.a.M = (int)ro;
  G.a.N = (int)co;
  if (cg.kind == 0) {        // A = X [pixels][ci] K-major, B = W [co][ci] K-major
    G.a.K = (int)c0;
  } else if (cg.kind == 1) { // A = dY [pixels][co] K-major, B = W [co][ci] MN-major
    G.a.K = (int)c0;
    G.a.b_mn_major = 1;
  } else {                   // A = dY [pixels][co] MN-major, B = X [pixels][ci] MN-major
    G.a.K = (int)r0;
    G.a.a_mn_major = 1;
    G.a.b_mn_major = 1;
  }
  if (!P0.rp.empty()) {  // operands read in place from their owners' shards (fused fetch, conv1x1_form)
    set_operand_pieces(E, P0, G.pa, G.a.A, G.a.lda);
    G.a.a_pieces = &G.pa;
  }
  if (!P1.rp.empty()) {
    set_operand_pieces(E, P1, G.pb, G.a.B, G.a.ldb);
    G.a.b_pieces = &G.pb;
  }
  const int64_t ec = O.dtype == TOFU_BF16 ? 2 : 4;
  G.a.C = base + O.off + offo * ec;
  G.a.ldc = (int)ldo;
  G.a.c_mode = O.dtype == TOFU_BF16 ? 0 : 1;
  if (L.ep) {
    G.a.ep = L.ep;
    if (L.ep & 2) G.a.aux_add = base + L.epi_add.off + offset_in(L.epi_add.buf_box, L.epi_add.box) * 2;
    if (L.ep & 4) G.a.aux_mask = base + L.epi_mask.off + offset_in(L.epi_mask.buf_box, L.epi_mask.box) * 2;
  }
  if (L.fused_opt >= 0) {
    const LOp& Lm = E.lops[li][L.fused_opt];
    const LOp& Ls = E.lops[li][L.fused_opt + 1];
    int64_t mr, mc, ldm, moff, wr, wc, ldw, woff;
    if (!flat2(Lm.in[0].buf_box, Lm.in[0].box, 1, mr, mc, ldm, moff) ||
        !flat2(Ls.in[0].buf_box, Ls.in[0].box, 1, wr, wc, ldw, woff) || mr != ro || mc != co)
      return false;
    auto at = [&](int op, const char*) {  // the mom / sgd def's constant (its TDL literal)
      return (float)g.defs[g.ops[op].def].kconst.at(0);
    };
    G.a.c_mode = 3;
    G.a.C = base + Lm.in[0].off + moff * 4;
    G.a.ldc = (int)ldm;
    G.a.D = base + Ls.in[0].off + woff * 2;
    G.a.ldd = (int)ldw;
    G.a.s0 = at(L.fused_opt, "mu");
    G.a.s1 = at(L.fused_opt + 1, "lr");
  }
  return true;
}

void finalize(Exec& E) {
  if (E.finalized) return;
  const Graph& g = *E.g;
  if (E.multi_process && !E.flags_dev) {
    if (cudaMalloc(&E.flags_dev, sizeof(void*) * E.k) != cudaSuccess) throw Error(TOFU_ERR_CUDA, "cudaMalloc flags");
    cudaMemcpy(E.flags_dev, E.flags.data(), sizeof(void*) * E.k, cudaMemcpyHostToDevice);
  }
  const auto& host = E.host_pieces;
  const int nl = (int)E.local.size();
  if (!host.empty()) {
    if (cudaMalloc(&E.pieces_dev, host.size() * sizeof(tofu_piece)) != cudaSuccess)
      throw Error(TOFU_ERR_CUDA, "cudaMalloc pieces");
    if (cudaMemcpy(E.pieces_dev, host.data(), host.size() * sizeof(tofu_piece), cudaMemcpyHostToDevice) != cudaSuccess)
      throw Error(TOFU_ERR_CUDA, "cudaMemcpy pieces");
  }
  if (!E.host_tasks.empty()) {
    const size_t nb = E.host_tasks.size() * sizeof(tofu_piece_task);
    if (cudaMalloc(&E.tasks_dev, nb) != cudaSuccess) throw Error(TOFU_ERR_CUDA, "cudaMalloc piece tasks");
    if (cudaMemcpy(E.tasks_dev, E.host_tasks.data(), nb, cudaMemcpyHostToDevice) != cudaSuccess)
      throw Error(TOFU_ERR_CUDA, "cudaMemcpy piece tasks");
  }
  if (!E.ew_ws) {
    const int64_t b = tofu_sumsq_workspace_bytes();
    if (cudaMalloc(&E.ew_ws, b) != cudaSuccess || cudaMemset(E.ew_ws, 0, b) != cudaSuccess)
      throw Error(TOFU_ERR_CUDA, "cudaMalloc loss workspace");
  }
  // stream-K workspace: launches run one at a time on the executor's stream, each leaves the flags zeroed
  if (!E.sk_dev) {
    const int64_t skb = tofu_sk_workspace_bytes();
    if (skb <= 0 || cudaMalloc(&E.sk_dev, skb) != cudaSuccess || cudaMemset(E.sk_dev, 0, skb) != cudaSuccess)
      throw Error(TOFU_ERR_CUDA, "cudaMalloc stream-K workspace");
  }
  // GEMM descriptors (pass 0 sizes the shared split-K workspace with a placeholder address, pass 1 encodes
  // the real descriptors)
  // k-block order alternated launch by launch over the same weight tensor (per rank, op order): a pass then
  // starts on the rows the previous pass read last, still in L2 — the LSTM's per-timestep recurrent GEMMs each
  // stream their whole Wh (134 MB at configs[2], L2 126 MB).  Keyed by the B operand's tensor (alias root), so
  // fused / staged fetch and one / two streams take the same orders (bitwise-equal tests).  TOFU_KREV=0: off.
  static const bool krev_on = [] {
    const char* e = std::getenv("TOFU_KREV");
    return !(e && e[0] == '0');
  }();
  std::map<int, int> alias_up(g.alias.begin(), g.alias.end());
  auto troot = [&](int t) {
    while (alias_up.count(t)) t = alias_up[t];
    return t;
  };
  for (int pass = 0; pass < 2; ++pass) {
  int64_t ws_need = 0;
  std::map<std::pair<int, int>, int> kdir;  // (local rank, B tensor root) -> the last launch's order
  auto next_dir = [&](int li, int t) {
    if (!krev_on) return 0;
    const auto key = std::make_pair(li, troot(t));
    const auto it = kdir.find(key);
    const int d = it == kdir.end() ? 0 : 1 - it->second;
    kdir[key] = d;
    return d;
  };
  for (int li = 0; li < nl; ++li) {
    const int r = E.local[li];
    for (size_t o = 0; o < g.ops.size(); ++o) {
      const OpDef& d = g.def_of((int)o);
      if (std::string(kernel_kind(d)) != "gemm") continue;
      LOp& L = E.lops[li][o];
      if (L.skip) continue;
      const GemmForm gf = gemm_form(d);
      const Buf &A = L.in[gf.a_param], &B = L.in[gf.b_param];
      int64_t ar, ac, lda, aoff, br, bc, ldb, boff, cr, cc, ldc, coff;
      if (!flat2(A.buf_box, A.box, gf.a_split, ar, ac, lda, aoff) ||
          !flat2(B.buf_box, B.box, gf.b_split, br, bc, ldb, boff) ||
          !flat2(L.out.buf_box, L.out.box, gf.nm, cr, cc, ldc, coff))
        throw Error(TOFU_ERR_ARG, "GEMM operand of op " + g.ops[o].name + " is not a 2-D view");
      Exec::GemmLaunch G;
      std::memset(&G.a, 0, sizeof G.a);
      G.a.M = (int)cr;
      G.a.N = (int)cc;
      G.a.K = (int)(gf.a_mn ? ar : ac);
      G.a.A = E.arena[r] + A.off + aoff * 2;
      G.a.lda = (int)lda;
      G.a.a_mn_major = gf.a_mn ? 1 : 0;
      G.a.B = E.arena[r] + B.off + boff * 2;
      G.a.ldb = (int)ldb;
      G.a.b_mn_major = gf.b_mn ? 1 : 0;
      auto set_pieces = [&](const Buf& X, tofu_operand_pieces& P, const void*& ptr, int& ld) {
        set_operand_pieces(E, X, P, ptr, ld);
      };
      if (!A.rp.empty()) {
        set_pieces(A, G.pa, G.a.A, G.a.lda);
        G.a.a_pieces = &G.pa;
      }
      if (!B.rp.empty()) {
        set_pieces(B, G.pb, G.a.B, G.a.ldb);
        G.a.b_pieces = &G.pb;
      }
      const int64_t ec = L.out.dtype == TOFU_BF16 ? 2 : 4;
      G.a.C = E.arena[r] + L.out.off + coff * ec;
      G.a.ldc = (int)ldc;
      G.a.c_mode = L.out.dtype == TOFU_BF16 ? 0 : 1;
      if (L.ep) {
        G.a.ep = L.ep;
        if (L.ep & 2) G.a.aux_add = E.arena[r] + L.epi_add.off + offset_in(L.epi_add.buf_box, L.epi_add.box) * 2;
        if (L.ep & 4) G.a.aux_mask = E.arena[r] + L.epi_mask.off + offset_in(L.epi_mask.buf_box, L.epi_mask.box) * 2;
      }
      if (L.fused_opt >= 0) {
        const LOp& Lm = E.lops[li][L.fused_opt];      // mom(M, G) -> M_new (in place)
        const LOp& Ls = E.lops[li][L.fused_opt + 1];  // sgd(W, M_new) -> W_new (in place)
        auto at = [&](int op, const char*) {  // the mom / sgd def's constant (its TDL literal)
          return (float)g.defs[g.ops[op].def].kconst.at(0);
        };
        int64_t mr, mc, ldm, moff, wr, wc, ldw, woff;
        if (!flat2(Lm.in[0].buf_box, Lm.in[0].box, gf.nm, mr, mc, ldm, moff) ||
            !flat2(Ls.in[0].buf_box, Ls.in[0].box, gf.nm, wr, wc, ldw, woff) || mr != cr || mc != cc)
          throw Error(TOFU_ERR_ARG, "fused optimizer operands of op " + g.ops[o].name + " do not match the GEMM");
        G.a.c_mode = 3;
        G.a.C = E.arena[r] + Lm.in[0].off + moff * 4;
        G.a.ldc = (int)ldm;
        G.a.D = E.arena[r] + Ls.in[0].off + woff * 2;
        G.a.ldd = (int)ldw;
        G.a.s0 = at(L.fused_opt, "mu");
        G.a.s1 = at(L.fused_opt + 1, "lr");
      }
      G.a.splits = 0;
      G.a.ws = pass == 0 ? reinterpret_cast<void*>(uintptr_t(1) << 20) : E.ws_dev;
      G.a.sk_ws = E.sk_dev;
      G.a.k_reverse = next_dir(li, g.ops[o].inputs[gf.b_param]);
      int rc = tofu_gemm_plan_tmaps(&G.a, G.tm, &G.bn);
      if (rc) throw Error(rc, "gemm tensor map for op " + g.ops[o].name + " (pitch/alignment)");
      ws_need = std::max<int64_t>(ws_need, tofu_gemm_workspace_bytes(&G.a));
      if (pass == 1) {
        Exec::GemmLaunch& S = E.gemms[{(int)o, li}];
        S = G;  // (the piece tables move with it: re-point the args at the stored copies)
        if (S.a.a_pieces) S.a.a_pieces = &S.pa;
        if (S.a.b_pieces) S.a.b_pieces = &S.pb;
      }
    }
  }
  for (int li = 0; li < nl; ++li)
    for (size_t o = 0; o < g.ops.size(); ++o) {
      const OpDef& d = g.def_of((int)o);
      if (std::string(kernel_kind(d)) != "conv" || E.lops[li][o].skip) continue;
      LOp& L = E.lops[li][o];
      {  // a 1x1 stride-1 convolution is a plain GEMM over pixel rows: the TMA-fed tcgen05 GEMM when every
         // operand is a row block of its buffer (else the gather kernel)
        Exec::GemmLaunch G;
        const bool fused = !L.in[0].rp.empty() || (L.in.size() > 1 && !L.in[1].rp.empty());
        if (conv1x1_gemm(E, (int)o, li, G)) {
          G.a.splits = 0;
          G.a.ws = pass == 0 ? reinterpret_cast<void*>(uintptr_t(1) << 20) : E.ws_dev;
          G.a.sk_ws = E.sk_dev;
          if (tofu_gemm_plan_tmaps(&G.a, G.tm, &G.bn) == TOFU_OK) {  // else: the convolution kernel below
            ws_need = std::max<int64_t>(ws_need, tofu_gemm_workspace_bytes(&G.a));
            if (pass == 1) {
              Exec::GemmLaunch& S = E.gemms[{(int)o, li}];
              S = G;  // (re-point the piece tables at the stored copies)
              if (S.a.a_pieces) S.a.a_pieces = &S.pa;
              if (S.a.b_pieces) S.a.b_pieces = &S.pb;
            }
            continue;
          }
        }
        // (the convolution kernel reads staged or owned operands only)
        if (fused) throw Error(TOFU_ERR_ARG, "fused-fetch 1x1 convolution " + g.ops[o].name + " has no GEMM form");
      }
      std::vector<Exec::ConvLaunch> cls;
      for (auto& a : conv_args(E, (int)o, li)) {
        Exec::ConvLaunch C;
        C.a = a;
        if (a.kind == 1 && L.fused_opt >= 0) {
          const int r = E.local[li];
          const LOp& Lm = E.lops[li][L.fused_opt];      // mom(M, G) -> M_new (in place)
          const LOp& Ls = E.lops[li][L.fused_opt + 1];  // sgd(W, M_new) -> W_new (in place)
          if (!full_from(Lm.in[0].buf_box, Lm.in[0].box, 1) || !full_from(Ls.in[0].buf_box, Ls.in[0].box, 1))
            throw Error(TOFU_ERR_ARG, "fused optimizer operands of op " + g.ops[o].name + " are not row blocks");
          C.a.c_mode = 3;
          C.a.C = E.arena[r] + Lm.in[0].off + offset_in(Lm.in[0].buf_box, Lm.in[0].box) * 4;
          C.a.ldc = strides_of(Lm.in[0].buf_box)[0];
          C.a.D = E.arena[r] + Ls.in[0].off + offset_in(Ls.in[0].buf_box, Ls.in[0].box) * 2;
          C.a.ldd = strides_of(Ls.in[0].buf_box)[0];
          auto at = [&](int op, const char*) {  // the mom / sgd def's constant (its TDL literal)
            return (float)g.defs[g.ops[op].def].kconst.at(0);
          };
          C.a.s0 = at(L.fused_opt, "mu");
          C.a.s1 = at(L.fused_opt + 1, "lr");
        }
        C.a.splits = 0;
        C.a.ws = pass == 0 ? reinterpret_cast<void*>(uintptr_t(1) << 20) : E.ws_dev;
        C.a.sk_ws = E.sk_dev;
        const int rc = tofu_conv_plan(&C.a, C.tm);
        if (rc) throw Error(rc, "conv descriptors for op " + g.ops[o].name + " (geometry/alignment)");
        ws_need = std::max<int64_t>(ws_need, tofu_conv_workspace_bytes(&C.a));
        cls.push_back(C);
      }
      if (pass == 1) E.convs[{(int)o, li}] = std::move(cls);
    }
  if (pass == 0 && ws_need > 0 && cudaMalloc(&E.ws_dev, ws_need) != cudaSuccess)
    throw Error(TOFU_ERR_CUDA, "cudaMalloc split-K workspace");
  }
  E.finalized = true;
}

bool lo_fused(const Exec& E, const Exec::Launch& L) { return E.lops[L.li][L.op].fused_sgd; }

// tofu_conv_args of one convolution sub-op (op o, local rank li) on its iteration box: the pixel grid, tap
// table and buffer geometry (DESIGN reading R11; include/tofu.h documents the fields).
std::vector<tofu_conv_args> conv_args(Exec& E, int o, int li) {
  const Graph& g = *E.g;
  const int r = E.local[li];
  const OpDef& d = g.def_of(o);
  const ConvGeom cg = conv_geom(d);
  const LOp& L = E.lops[li][o];
  std::vector<Rng> ib;
  iter_box(g, o, E.plan.osplit[o], E.plan.factors, worker_digits(r, E.plan.factors), ib);
  char* base = E.arena[r];
  auto es = [](int dt) { return (int64_t)(dt == TOFU_BF16 ? 2 : 4); };
  auto box_ptr = [&](const Buf& b) { return base + b.off + offset_in(b.buf_box, b.box) * es(b.dtype); };
  tofu_conv_args a;
  std::memset(&a, 0, sizeof a);
  const int R = cg.R, s = cg.s, p = cg.p;
  auto set_epilogue = [&](tofu_conv_args& x) {
    if (!L.ep) return;
    x.ep = L.ep;
    if (L.ep & 2) x.aux_add = box_ptr(L.epi_add);
    if (L.ep & 4) x.aux_mask = box_ptr(L.epi_mask);
  };
  // gathered source
  const Buf& S = L.in[cg.kind == 2 ? 1 : 0];
  auto st = strides_of(S.buf_box);
  a.S = base + S.off;
  a.s_sb = st[0];
  a.s_sy = st[1];
  a.s_sx = st[2];
  a.sH = (int)S.buf_box[1].len();
  a.sW = (int)S.buf_box[2].len();
  std::vector<tofu_conv_args> out;
  if (cg.kind == 0 || cg.kind == 2) {
    // pixels = output (forward) or reduce (weight gradient) box over (b, y, x); vars b,y,x at 0..2 (fwd) or 4..6
    const int vb = cg.kind == 0 ? 0 : 4, vky = cg.kind == 0 ? 4 : 1, vci = cg.kind == 0 ? 6 : 3;
    a.nb = (int)ib[vb].len();
    a.ngy = (int)ib[vb + 1].len();
    a.ngx = (int)ib[vb + 2].len();
    a.sb0 = (int)(ib[vb].lo - S.buf_box[0].lo);
    a.ay = a.ax = s;
    a.cy = (int)(s * ib[vb + 1].lo - p - S.buf_box[1].lo);
    a.cx = (int)(s * ib[vb + 2].lo - p - S.buf_box[2].lo);
    a.ntaps = 0;
    for (int64_t ky = ib[vky].lo; ky <= ib[vky].hi; ++ky)
      for (int64_t kx = ib[vky + 1].lo; kx <= ib[vky + 1].hi; ++kx) {
        a.tap_dy[a.ntaps] = (short)ky;
        a.tap_dx[a.ntaps] = (short)kx;
        a.tap_w[a.ntaps] = (short)(ky * R + kx);
        ++a.ntaps;
      }
    a.nch = (int)ib[vci].len();
    a.sc0 = (int)(ib[vci].lo - S.buf_box[3].lo);
    if (cg.kind == 0) {
      const Buf& W = L.in[1];
      a.kind = 0;
      a.n_out = (int)ib[3].len();
      a.Bp = box_ptr(W);
      a.ldb = strides_of(W.buf_box)[0];
      a.b_tap = (int)W.buf_box[3].len();
      a.b_rows = (int)W.box[0].len();
      a.b_cols = (int)(a.ldb - (W.box[3].lo - W.buf_box[3].lo));
      a.b_mn_major = 0;
      const Buf& O = L.out;
      auto os = strides_of(O.buf_box);
      a.C = box_ptr(O);
      a.c_sb = os[0];
      a.c_sy = os[1];
      a.c_sx = os[2];
      a.c_ys = a.c_xs = 1;
      a.c_mode = O.dtype == TOFU_F32 ? 1 : 0;
      set_epilogue(a);
      out.push_back(a);
    } else {
      const Buf& D = L.in[0];
      a.kind = 1;
      a.m_out = (int)ib[0].len();
      a.Ap = box_ptr(D);
      a.lda = D.buf_box[3].len();
      const Buf& O = L.out;
      a.C = box_ptr(O);
      a.ldc = strides_of(O.buf_box)[0];
      a.c_mode = 1;  // weight gradients are f32 (partials included)
      out.push_back(a);
    }
    return out;
  }
  // data gradient: rows = dX pixels (b, y, x); vars b,y,x,ci = 0..3, (ky|ty),(kx|tx) = 4,5, co = 6
  const Buf& W = L.in[1];
  const Buf& O = L.out;
  auto os = strides_of(O.buf_box);
  a.kind = 0;
  a.nb = (int)ib[0].len();
  a.sb0 = (int)(ib[0].lo - S.buf_box[0].lo);
  a.nch = (int)ib[6].len();
  a.sc0 = (int)(ib[6].lo - S.buf_box[3].lo);
  a.n_out = (int)ib[3].len();
  if (L.wt_off >= 0) {  // K-major from the transposed shard WT[ci][ky][kx][co]
    const int64_t co_sh = W.buf_box[0].len(), ci_sh = W.buf_box[3].len(), taps_sh = W.buf_box[1].len() * W.buf_box[2].len();
    a.ldb = taps_sh * co_sh;
    a.Bp = base + L.wt_off + ((W.box[3].lo - W.buf_box[3].lo) * a.ldb + (W.box[0].lo - W.buf_box[0].lo)) * 2;
    a.b_tap = (int)co_sh;
    a.b_rows = (int)W.box[3].len();
    a.b_cols = (int)(a.ldb - (W.box[0].lo - W.buf_box[0].lo));
    a.b_mn_major = 0;
    (void)ci_sh;
  } else {
    a.Bp = box_ptr(W);
    a.ldb = strides_of(W.buf_box)[0];
    a.b_tap = (int)W.buf_box[3].len();
    a.b_rows = (int)W.box[0].len();
    a.b_cols = (int)(a.ldb - (W.box[3].lo - W.buf_box[3].lo));
    a.b_mn_major = 1;
  }
  a.C = box_ptr(O);
  a.c_sb = os[0];
  a.c_sy = os[1];
  a.c_sx = os[2];
  a.c_mode = O.dtype == TOFU_F32 ? 1 : 0;
  a.ay = a.ax = 1;
  if (s == 1) {  // dX[y] = Σ D[y - ky + p] W[ky]
    a.ngy = (int)ib[1].len();
    a.ngx = (int)ib[2].len();
    a.cy = (int)(ib[1].lo + p - S.buf_box[1].lo);
    a.cx = (int)(ib[2].lo + p - S.buf_box[2].lo);
    a.c_ys = a.c_xs = 1;
    a.ntaps = 0;
    for (int64_t ky = ib[4].lo; ky <= ib[4].hi; ++ky)
      for (int64_t kx = ib[5].lo; kx <= ib[5].hi; ++kx) {
        a.tap_dy[a.ntaps] = (short)-ky;
        a.tap_dx[a.ntaps] = (short)-kx;
        a.tap_w[a.ntaps] = (short)(ky * R + kx);
        ++a.ntaps;
      }
    set_epilogue(a);
    out.push_back(a);
    return out;
  }
  // stride 2: one launch per sub-pixel phase (ry, rx); y = 2u + ry reads D[u + (ry+p)/2 - ty] through tap
  // ky = (ry+p)%2 + 2ty (< R), the dconv_k*s2 def's floor-division / remainder indices
  auto fdiv = [](int64_t v, int64_t q) { return v >= 0 ? v / q : -((-v + q - 1) / q); };
  for (int ry = 0; ry < 2; ++ry)
    for (int rx = 0; rx < 2; ++rx) {
      tofu_conv_args b = a;
      const int64_t ulo = fdiv(ib[1].lo - ry + 1, 2), uhi = fdiv(ib[1].hi - ry, 2);
      const int64_t vlo = fdiv(ib[2].lo - rx + 1, 2), vhi = fdiv(ib[2].hi - rx, 2);
      if (uhi < ulo || vhi < vlo) continue;
      b.ngy = (int)(uhi - ulo + 1);
      b.ngx = (int)(vhi - vlo + 1);
      b.cy = (int)(ulo + (ry + p) / 2 - S.buf_box[1].lo);
      b.cx = (int)(vlo + (rx + p) / 2 - S.buf_box[2].lo);
      b.c_ys = b.c_xs = 2;
      b.c_y0 = (int)(2 * ulo + ry - ib[1].lo);
      b.c_x0 = (int)(2 * vlo + rx - ib[2].lo);
      b.ntaps = 0;
      for (int64_t ty = ib[4].lo; ty <= ib[4].hi; ++ty)
        for (int64_t tx = ib[5].lo; tx <= ib[5].hi; ++tx) {
          const int64_t ky = (ry + p) % 2 + 2 * ty, kx = (rx + p) % 2 + 2 * tx;
          if (ky >= R || kx >= R) continue;
          b.tap_dy[b.ntaps] = (short)-ty;
          b.tap_dx[b.ntaps] = (short)-tx;
          b.tap_w[b.ntaps] = (short)(ky * R + kx);
          ++b.ntaps;
        }
      out.push_back(b);
    }
  return out;
}

// maxpool / maxpool_grad / gap / gap_grad on the op's iteration box (tofu_window_args in include/tofu.h)
int run_window(Exec& E, int o, int li, cudaStream_t st) {
  const Graph& g = *E.g;
  const int r = E.local[li];
  const LOp& L = E.lops[li][o];
  const std::string& dn = g.def_of(o).kernel;
  std::vector<Rng> ib;
  iter_box(g, o, E.plan.osplit[o], E.plan.factors, worker_digits(r, E.plan.factors), ib);
  char* base = E.arena[r];
  auto es = [](int dt) { return (int64_t)(dt == TOFU_BF16 ? 2 : 4); };
  // pointer to (box b lo, buffer row 0, buffer col 0, box c lo) of a 4-D buffer
  auto p4 = [&](const Buf& b) {
    auto s = strides_of(b.buf_box);
    return base + b.off + ((b.box[0].lo - b.buf_box[0].lo) * s[0] + (b.box[3].lo - b.buf_box[3].lo)) * es(b.dtype);
  };
  tofu_window_args a;
  std::memset(&a, 0, sizeof a);
  a.out_f32 = L.out.dtype == TOFU_F32;
  auto os = strides_of(L.out.buf_box);
  const int64_t oe = es(L.out.dtype);
  if (dn == "maxpool") {  // vars b, y, x, c | ky, kx
    const Buf& X = L.in[0];
    auto xs = strides_of(X.buf_box);
    a.nb = (int)ib[0].len(); a.C = (int)ib[3].len();
    a.H = (int)X.buf_box[1].len(); a.W = (int)X.buf_box[2].len();
    a.y0 = (int)X.buf_box[1].lo; a.x0 = (int)X.buf_box[2].lo;
    a.Ho = (int)ib[1].len(); a.Wo = (int)ib[2].len(); a.oy0 = (int)ib[1].lo; a.ox0 = (int)ib[2].lo;
    a.x_sb = xs[0]; a.x_sy = xs[1]; a.x_sx = xs[2];
    a.X = p4(X);
    a.o_sb = os[0]; a.o_sy = os[1]; a.o_sx = os[2];
    a.out = base + L.out.off + offset_in(L.out.buf_box, L.out.box) * oe;
    return tofu_maxpool(&a, st);
  }
  if (dn == "maxpool_grad") {  // vars b, y, x, c | ty, tx ; inputs X, Y, D, K
    const Buf &X = L.in[0], &Y = L.in[1], &D = L.in[2], &K = L.in[3];
    auto xs = strides_of(X.buf_box), ys = strides_of(Y.buf_box), ds = strides_of(D.buf_box), ks = strides_of(K.buf_box);
    if (Y.buf_box[1].lo != D.buf_box[1].lo || Y.buf_box[2].lo != D.buf_box[2].lo ||
        Y.buf_box[1].len() != D.buf_box[1].len() || Y.buf_box[2].len() != D.buf_box[2].len())
      throw Error(TOFU_ERR_ARG, "maxpool_grad: Y and dY regions differ");
    a.nb = (int)ib[0].len(); a.C = (int)ib[3].len();
    a.H = (int)ib[1].len(); a.W = (int)ib[2].len(); a.y0 = (int)ib[1].lo; a.x0 = (int)ib[2].lo;
    a.Ho = (int)Y.buf_box[1].len(); a.Wo = (int)Y.buf_box[2].len();
    a.oy0 = (int)Y.buf_box[1].lo; a.ox0 = (int)Y.buf_box[2].lo;
    a.x_sb = xs[0]; a.x_sy = xs[1]; a.x_sx = xs[2];
    a.y_sb = ys[0]; a.y_sy = ys[1]; a.y_sx = ys[2];
    a.d_sb = ds[0]; a.d_sy = ds[1]; a.d_sx = ds[2];
    a.k_sy = ks[0]; a.k_sx = ks[1];
    a.X = base + X.off + offset_in(X.buf_box, X.box) * 2;
    a.Y = p4(Y);
    a.dY = p4(D);
    // K[ky][kx][c]: pointer at (ky 0, kx 0, box c lo)
    a.K = base + K.off + ((0 - K.buf_box[0].lo) * ks[0] + (0 - K.buf_box[1].lo) * ks[1] + (K.box[2].lo - K.buf_box[2].lo)) * 2;
    if (K.buf_box[0].lo != 0 || K.buf_box[1].lo != 0 || K.buf_box[0].len() < 3 || K.buf_box[1].len() < 3)
      throw Error(TOFU_ERR_ARG, "maxpool_grad: mask region must hold all taps");
    a.ty0 = (int)ib[4].lo; a.ty1 = (int)ib[4].hi; a.tx0 = (int)ib[5].lo; a.tx1 = (int)ib[5].hi;
    a.o_sb = os[0]; a.o_sy = os[1]; a.o_sx = os[2];
    a.out = base + L.out.off + offset_in(L.out.buf_box, L.out.box) * oe;
    return tofu_maxpool_grad(&a, st);
  }
  if (dn == "gap") {  // vars b, c | y, x
    const Buf& X = L.in[0];
    auto xs = strides_of(X.buf_box);
    a.nb = (int)ib[0].len(); a.C = (int)ib[1].len();
    a.H = (int)ib[2].len(); a.W = (int)ib[3].len();
    a.x_sb = xs[0]; a.x_sy = xs[1]; a.x_sx = xs[2];
    a.X = base + X.off + offset_in(X.buf_box, X.box) * 2;
    a.o_sb = os[0];
    a.out = base + L.out.off + offset_in(L.out.buf_box, L.out.box) * oe;
    a.s = (float)g.def_of(o).kconst.at(0);   // the def's own constant (1/(H*W))
    return tofu_gap(&a, st);
  }
  // gap_grad: vars b, y, x, c ; input D[b, c]
  const Buf& D = L.in[0];
  auto ds = strides_of(D.buf_box);
  a.nb = (int)ib[0].len(); a.C = (int)ib[3].len();
  a.H = (int)ib[1].len(); a.W = (int)ib[2].len();
  a.y_sb = ds[0];
  a.dY = base + D.off + offset_in(D.buf_box, D.box) * 2;
  a.o_sb = os[0]; a.o_sy = os[1]; a.o_sx = os[2];
  a.out = base + L.out.off + offset_in(L.out.buf_box, L.out.box) * oe;
  a.s = (float)g.def_of(o).kconst.at(0);
  return tofu_gap_grad(&a, st);
}

// CUDA kernels one compute launch issues (split-K reductions, weight transposes and convolution phases included)
int64_t kernels_of(const Exec& E, int o, int li) {
  const std::string kind = kernel_kind(E.g->def_of(o));
  auto gemm_k = [](const tofu_gemm_args& a) -> int64_t {
    return a.M == 0 || a.N == 0 || a.K == 0 ? 0 : 1 + (a.splits > 1 ? 1 : 0);
  };
  if (kind == "gemm") {
    const auto& a = E.gemms.at({o, li}).a;
    // gate GEMM + cell: the cell kernel replaces the split-K reduction (or follows the unsplit GEMM)
    if (E.lops[li][o].cell_after >= 0) return a.M == 0 || a.N == 0 || a.K == 0 ? 1 : 2;
    return gemm_k(a);
  }
  if (kind == "conv") {
    auto git = E.gemms.find({o, li});
    if (git != E.gemms.end()) return gemm_k(git->second.a);
    int64_t n = E.lops[li][o].wt_off >= 0 ? 1 : 0;
    for (auto& C : E.convs.at({o, li})) {
      const auto& a = C.a;
      const int64_t pix = (int64_t)a.nb * a.ngy * a.ngx;
      const int64_t M = a.kind == 0 ? pix : a.m_out, N = a.kind == 0 ? a.n_out : (int64_t)a.ntaps * a.nch;
      if (M == 0 || N == 0) continue;
      n += 1 + (a.splits > 1 && !a.direct ? 1 : 0);
    }
    return n;
  }
  return 1;
}

// LSTM cell launch of op o (fused kinds included); gs: the gate GEMM whose split-K partial planes hold GH (the
// gate GEMM + cell fusion, LOp::cell_after), else NULL.
int run_lstm(Exec& E, int o, int li, cudaStream_t st, const tofu_gemm_args* gs) {
  const Graph& g = *E.g;
  const int r = E.local[li];
  LOp& L = E.lops[li][o];
  const OpInfo& oi = g.ops[o];
  const std::string& dn = g.defs[oi.def].kernel;
  char* base = E.arena[r];
  {
    // operand slots of the cell kernel: gx, gh, cp, c, du, dr, dn
    static const std::map<std::string, std::vector<int>> slots = {
        {"cell_c", {0, 1, 2}}, {"cell_h", {0, 1, 3}}, {"cell_bwd_a", {0, 1, 2, 3, 4, 5, 6}},
        {"cell_bwd_c", {0, 1, 3, 4, 5, 6}}};
    const void* ptrs[7] = {};
    int64_t lds[7] = {}, gss[7] = {};
    int dts[7] = {};
    const auto& sl = slots.at(dn);
    for (size_t pi = 0; pi < sl.size(); ++pi) {
      const Buf& b = L.in[pi];
      auto st_ = strides_of(b.buf_box);
      const int64_t es = b.dtype == TOFU_BF16 ? 2 : 4;
      // the kernel addresses gates by absolute index x (p[b*ld + x*gs + h]); the required box may start at
      // a later gate (e.g. cell_h reads only gate 3), so point at gate 0 of the box row
      const int64_t g_lo = b.buf_box.size() == 3 ? b.box[1].lo : 0;
      ptrs[sl[pi]] = base + b.off + (offset_in(b.buf_box, b.box) - (b.buf_box.size() == 3 ? g_lo * st_[1] : 0)) * es;
      lds[sl[pi]] = st_[0];
      gss[sl[pi]] = b.buf_box.size() == 3 ? st_[1] : 0;
      dts[sl[pi]] = b.dtype;
    }
    const Buf& ob = L.out;
    auto ost = strides_of(ob.buf_box);
    const int64_t oes = ob.dtype == TOFU_BF16 ? 2 : 4;
    const int64_t nb = ob.box[0].len(), nh = ob.box.back().len();
    const int g0 = ob.box.size() == 3 ? (int)ob.box[1].lo : 0, ng = ob.box.size() == 3 ? (int)ob.box[1].len() : 0;
    static const std::map<std::string, int> kinds = {{"cell_c", 0}, {"cell_h", 1}, {"cell_bwd_a", 2}, {"cell_bwd_c", 3}};
    int kind_id = kinds.at(dn);
    void* out2 = nullptr;
    int64_t out2_ld = 0;
    int out2_dt = TOFU_F32;
    if (L.fused_next) {
      const Buf& nb2 = E.lops[li][o + 1].out;
      auto st2 = strides_of(nb2.buf_box);
      out2 = base + nb2.off + offset_in(nb2.buf_box, nb2.box) * (nb2.dtype == TOFU_BF16 ? 2 : 4);
      out2_ld = st2[0];
      out2_dt = nb2.dtype;
      kind_id = kind_id == 0 ? 4 : 5;
    }
    if (gs) {  // GH from the gate GEMM's split-K planes ([splits][M][N] dense; N = gates x h of GH's box)
      // (the GEMM wrote GH's whole box, = its buffer: gate stride in a plane = the buffer's h extent; the
      // cell op's own GH box may name fewer gates, e.g. cell_c reads i, f, g)
      const int64_t M = gs->M, N = gs->N, wgs = L.in[1].buf_box[2].len();
      if (L.in[1].buf_box.size() != 3 || N != L.in[1].buf_box[1].len() * wgs || M != nb || nh > wgs)
        return TOFU_ERR_ARG;  // (the fusion pass admits only GEMMs whose output box is GH's buffer)
      return tofu_lstm_cell_splitk(kind_id, nb, nh, g0, ng, ptrs, lds, gss, dts,
                                   base + ob.off + offset_in(ob.buf_box, ob.box) * oes, ost[0],
                                   ob.box.size() == 3 ? ost[1] : 0, ob.dtype, out2, out2_ld, out2_dt,
                                   reinterpret_cast<const float*>(gs->ws), gs->splits, M * N, N, wgs, st);
    }
    return tofu_lstm_cell(kind_id, nb, nh, g0, ng, ptrs, lds, gss, dts,
                          base + ob.off + offset_in(ob.buf_box, ob.box) * oes, ost[0],
                          ob.box.size() == 3 ? ost[1] : 0, ob.dtype, out2, out2_ld, out2_dt, st);
    }
}

int run_compute(Exec& E, int o, int li, cudaStream_t st) {
  const Graph& g = *E.g;
  const int r = E.local[li];
  LOp& L = E.lops[li][o];
  const OpInfo& oi = g.ops[o];
  const std::string& dn = g.defs[oi.def].kernel;
  const OpDef& d = g.defs[oi.def];
  char* base = E.arena[r];
  const std::string kind = kernel_kind(d);
  if (kind == "gemm") {
    auto& G = E.gemms.at({o, li});
    if (L.cell_after < 0) return tofu_gemm_launch_planned(&G.a, G.tm, G.bn, st);
    // gate GEMM + cell: the partial planes stay in the workspace and the cell kernel reduces them
    tofu_gemm_args a = G.a;
    const bool split = a.splits > 1;
    a.defer_reduce = split ? 1 : 0;
    const int rc = tofu_gemm_launch_planned(&a, G.tm, G.bn, st);
    if (rc) {
      if (std::getenv("TOFU_DEBUG")) std::fprintf(stderr, "gate gemm: rc %d %s\n", rc, cudaGetErrorString(cudaGetLastError()));
      return rc;
    }
    return run_lstm(E, L.cell_after, li, st, split ? &G.a : nullptr);
  }
  if (kind == "conv") {
    auto git = E.gemms.find({o, li});
    if (git != E.gemms.end()) return tofu_gemm_launch_planned(&git->second.a, git->second.tm, git->second.bn, st);
    if (L.wt_off >= 0) {  // refresh the transposed weight shard (the weights may have been updated since)
      const Buf& W = L.in[1];
      const int rc = tofu_transpose_taps(base + W.off, base + L.wt_off, (int)W.buf_box[0].len(),
                                         (int)(W.buf_box[1].len() * W.buf_box[2].len()), (int)W.buf_box[3].len(), st);
      if (rc) return rc;
    }
    for (auto& C : E.convs.at({o, li})) {
      const int rc = tofu_conv_launch_planned(&C.a, C.tm, st);
      if (rc) return rc;
    }
    return TOFU_OK;
  }
  if (kind == "window") return run_window(E, o, li, st);
  if (kind == "lstm") return run_lstm(E, o, li, st, nullptr);
  const int64_t n = vol(L.out.box);
  void* y = base + L.out.off;
  const void* x0 = L.in.size() > 0 ? base + L.in[0].off : nullptr;
  const void* x1 = L.in.size() > 1 ? base + L.in[1].off : nullptr;
  // the kernel's constant: the real literal of the def's TDL (kernel_match.cpp)
  auto kc = [&](int op) { return (float)g.defs[g.ops[op].def].kconst.at(0); };
  if (dn == "relu" || dn == "relu4") return tofu_elementwise(TOFU_EW_RELU, n, y, x0, nullptr, nullptr, 0, 0, st);
  if (dn == "relu_grad" || dn == "relu_grad4") return tofu_elementwise(TOFU_EW_RELU_GRAD, n, y, x0, x1, nullptr, 0, 0, st);
  if (dn == "add4") return tofu_elementwise(TOFU_EW_ADD, n, y, x0, x1, nullptr, 0, 0, st);
  if (dn == "addrelu") return tofu_elementwise(TOFU_EW_ADDRELU, n, y, x0, x1, nullptr, 0, 0, st);
  if (dn == "mse_grad") return tofu_elementwise(TOFU_EW_MSE_GRAD, n, y, x0, x1, nullptr, kc(o), 0, st);
  if (dn == "sumsq") {
    const int64_t m = vol(L.in[0].box);
    if (L.fused_loss_grad) {  // + the next op (mse_grad of the same inputs) in the same pass
      const LOp& Ln = E.lops[li][o + 1];
      return tofu_elementwise_ws(TOFU_EW_SUMSQ_MSE_GRAD, m, y, x0, x1, base + Ln.out.off, kc(o), kc(o + 1), E.ew_ws,
                                 st);
    }
    return tofu_elementwise_ws(TOFU_EW_SUMSQ, m, y, x0, x1, nullptr, kc(o), 0, E.ew_ws, st);
  }
  if (is_mom(dn)) {
    if (L.fused_sgd) {
      const OpInfo& nx = g.ops[o + 1];
      LOp& Ln = E.lops[li][o + 1];
      (void)nx;
      return tofu_elementwise(TOFU_EW_SGD_MOM, n, nullptr, base + L.in[0].off, x1, base + Ln.in[0].off, kc(o),
                              kc(o + 1), st);
    }
    return tofu_elementwise(TOFU_EW_MOM, n, y, x0, x1, nullptr, kc(o), 0, st);
  }
  if (is_sgd(dn)) return tofu_elementwise(TOFU_EW_SGD, n, y, x0, x1, nullptr, kc(o), 0, st);
  return TOFU_ERR_ARG;
}

}  // namespace
}  // namespace tofu

struct tofu_exec {
  tofu::Exec e;
};

extern "C" int tofu_exec_arena_bytes(const tofu_graph* g, const tofu_plan* p, int rank, int64_t* bytes) {
  return tofu::guard([&]() {
    if (!g || !p || !bytes) throw tofu::Error(TOFU_ERR_ARG, "null argument");
    tofu::Exec E;
    E.g = &tofu::graph_of(g);
    E.plan = tofu::plan_of(p).seq;
    E.k = tofu::plan_of(p).k;
    if (rank < 0 || rank >= E.k) throw tofu::Error(TOFU_ERR_ARG, "rank out of range");
    E.local = {rank};
    tofu::read_env_options(E);  // the same lowering options as tofu_exec_create (staging sizes depend on them)
    tofu::lower(E);
    *bytes = E.lay[rank].total;
    return TOFU_OK;
  });
}

extern "C" int tofu_exec_shard(const tofu_graph* g, const tofu_plan* p, int rank, const char* tensor, int64_t* offset,
                               int64_t* box, int* rank_out) {
  return tofu::guard([&]() {
    const tofu::Graph& G = tofu::graph_of(g);
    auto it = G.tensor_ix.find(tensor ? tensor : "");
    if (it == G.tensor_ix.end()) throw tofu::Error(TOFU_ERR_ARG, "unknown tensor");
    const auto& plan = tofu::plan_of(p);
    if (rank < 0 || rank >= plan.k) throw tofu::Error(TOFU_ERR_ARG, "rank out of range");
    tofu::Layout L = tofu::layout_rank(G, plan.seq, rank);
    const int t = it->second;
    *offset = L.shard_off[t];
    *rank_out = (int)G.tensors[t].shape.size();
    for (size_t d = 0; d < L.shard_box[t].size() && d < 4; ++d) {
      box[2 * d] = L.shard_box[t][d].lo;
      box[2 * d + 1] = L.shard_box[t][d].hi;
    }
    return TOFU_OK;
  });
}

extern "C" int tofu_exec_create(const tofu_graph* g, const tofu_plan* p, int n_local, const int* local_ranks,
                                void* const* arena_dev, void* const* flags_dev, tofu_exec** out) {
  return tofu::guard([&]() {
    if (!g || !p || !out || n_local < 1 || !local_ranks || !arena_dev) throw tofu::Error(TOFU_ERR_ARG, "null argument");
    auto* h = new tofu_exec;
    tofu::Exec& E = h->e;
    try {
      E.gcopy = tofu::graph_of(g);
      E.g = &E.gcopy;
      E.plan = tofu::plan_of(p).seq;
      E.k = tofu::plan_of(p).k;
      for (int i = 0; i < n_local; ++i) {
        if (local_ranks[i] < 0 || local_ranks[i] >= E.k) throw tofu::Error(TOFU_ERR_ARG, "rank out of range");
        E.local.push_back(local_ranks[i]);
      }
      for (int r = 0; r < E.k; ++r) {
        if (!arena_dev[r] || (reinterpret_cast<uintptr_t>(arena_dev[r]) & 255))
          throw tofu::Error(TOFU_ERR_ALIGN, "arena pointers must be non-null and 256-byte aligned");
        E.arena.push_back(static_cast<char*>(arena_dev[r]));
      }
      E.multi_process = n_local < E.k;
      tofu::read_env_options(E);
      if (E.multi_process) {
        if (!flags_dev) throw tofu::Error(TOFU_ERR_ARG, "flags_dev required when not all ranks are local");
        for (int r = 0; r < E.k; ++r) E.flags.push_back(flags_dev[r]);
      }
      tofu::lower(E);
      tofu::build_launches(E);
    } catch (...) {
      if (E.pieces_dev) cudaFree(E.pieces_dev);
      if (E.tasks_dev) cudaFree(E.tasks_dev);
      if (E.flags_dev) cudaFree(E.flags_dev);
      delete h;
      throw;
    }
    *out = h;
    return TOFU_OK;
  });
}

extern "C" void tofu_exec_destroy(tofu_exec* h) {
  if (!h) return;
  if (h->e.pieces_dev) cudaFree(h->e.pieces_dev);
  if (h->e.tasks_dev) cudaFree(h->e.tasks_dev);
  for (auto ev : h->e.events)
    if (ev) cudaEventDestroy(ev);
  if (h->e.ev_fork) cudaEventDestroy(h->e.ev_fork);
  if (h->e.ev_join) cudaEventDestroy(h->e.ev_join);
  if (h->e.comm) cudaStreamDestroy(h->e.comm);
  if (h->e.flags_dev) cudaFree(h->e.flags_dev);
  if (h->e.ws_dev) cudaFree(h->e.ws_dev);
  if (h->e.sk_dev) cudaFree(h->e.sk_dev);
  if (h->e.ew_ws) cudaFree(h->e.ew_ws);
  delete h;
}

namespace tofu {
namespace {
int run_launch(Exec& E, const Exec::Launch& L, cudaStream_t st) {
  int rc = TOFU_OK;
  switch (L.kind) {
    case 0:
    case 2:
      if (!E.skip_comm) rc = tofu_pieces_run(E.pieces_dev + L.piece_off, E.tasks_dev + L.task_off, L.ntasks, L.all_raw, st);
      break;
    case 1:
      rc = run_compute(E, L.op, L.li, st);
      break;
    case 3:
      if (!E.skip_comm) rc = tofu_barrier_run(E.flags_dev, E.local[0], E.k, st);
      break;
    case 4: {
      const auto& out = E.lops[L.li][L.op].out;
      rc = cudaMemsetAsync(E.arena[E.local[L.li]] + out.off, 0, 4, st) == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
      break;
    }
  }
  if (rc)
    throw Error(rc, "launch failed at op " + (L.op >= 0 ? E.g->ops[L.op].name : std::string("end")) + ": " +
                        cudaGetErrorString(cudaGetLastError()));
  return rc;
}

// Launches [first, last): compute launches on st, comm launches on the executor's comm stream, forked from st
// at the start and joined back at the end (so st orders the whole range with the caller's work, and the
// pattern captures into a CUDA graph as a fork / join with the cross-stream waits as graph edges).
void run_range(Exec& E, int first, int last, cudaStream_t st) {
  finalize(E);
  if (!E.comm) {
    if (cudaStreamCreateWithFlags(&E.comm, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&E.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&E.ev_join, cudaEventDisableTiming) != cudaSuccess)
      throw Error(TOFU_ERR_CUDA, "comm stream / events");
    E.events.assign(E.launches.size(), nullptr);
    for (size_t i = 0; i < E.launches.size(); ++i)
      if (E.launches[i].rec && cudaEventCreateWithFlags(&E.events[i], cudaEventDisableTiming) != cudaSuccess)
        throw Error(TOFU_ERR_CUDA, "launch events");
  }
  bool any_comm = false;
  for (int i = first; i < last && !any_comm; ++i) any_comm = E.launches[i].stream == 1;
  auto chk = [](cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(TOFU_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  };
  if (any_comm) {
    chk(cudaEventRecord(E.ev_fork, st), "fork event");
    chk(cudaStreamWaitEvent(E.comm, E.ev_fork, 0), "fork wait");
  }
  for (int i = first; i < last; ++i) {
    const Exec::Launch& L = E.launches[i];
    cudaStream_t s = L.stream == 1 ? E.comm : st;
    for (int j : L.waits)
      if (j >= first) chk(cudaStreamWaitEvent(s, E.events[j], 0), "dependency wait");
    const bool timed = i == E.timed_launch && E.ev_start;
    // external event nodes when captured into a CUDA graph, so every replay re-times the launch
    // (the External flag is only valid while capturing; eager launches record plainly)
    unsigned evflags = cudaEventRecordDefault;
    if (timed) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(s, &cs);
      if (cs == cudaStreamCaptureStatusActive) evflags = cudaEventRecordExternal;
      chk(cudaEventRecordWithFlags(E.ev_start, s, evflags), "timing event");
    }
    if (E.jitter && L.kind != 3) {  // injected skew (tests): splitmix64 of (seed, rank, step, i)
      uint64_t z = E.jitter * 0x9E3779B97F4A7C15ull + (uint64_t)E.local[0] * 0xBF58476D1CE4E5B9ull +
                   E.jitter_step * 0x94D049BB133111EBull + (uint64_t)i;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      if ((z & 3) == 0) tofu_spin((int64_t)((z >> 8) % 200000), s);
    }
    run_launch(E, L, s);
    if (timed) chk(cudaEventRecordWithFlags(E.ev_stop, s, evflags), "timing event");
    if (L.rec) chk(cudaEventRecord(E.events[i], s), "launch event");
  }
  if (any_comm) {
    chk(cudaEventRecord(E.ev_join, E.comm), "join event");
    chk(cudaStreamWaitEvent(st, E.ev_join, 0), "join wait");
  }
}

std::string launch_desc(const Exec& E, int i) {
  const Graph& g = *E.g;
  const auto& L = E.launches[i];
  static const char* kinds[] = {"fetch", "compute", "reduce", "barrier", "memset"};
  std::string o = "{\"index\":" + std::to_string(i) + ",\"kind\":\"" + kinds[L.kind] + "\"";
  o += ",\"op\":" + (L.op >= 0 ? json_quote(g.ops[L.op].name) : std::string("null"));
  o += ",\"def\":" + (L.op >= 0 ? json_quote(g.defs[g.ops[L.op].def].name) : std::string("null"));
  o += ",\"rank\":" + std::to_string(L.li >= 0 ? E.local[L.li] : -1);
  o += ",\"stream\":" + std::to_string(L.stream);
  if (!L.waits.empty()) o += ",\"waits\":" + std::to_string(L.waits[0]);
  double flops = 0, bytes = 0;
  if (L.kind == 0 || L.kind == 2) {
    double rows = 0, row_bytes = 0, vec = 0, elems = 0;
    for (int64_t p = L.piece_off; p < L.piece_off + L.npieces; ++p) {
      const auto& pc = E.host_pieces[p];
      const double n = (double)pc.extent[0] * pc.extent[1] * pc.extent[2] * pc.extent[3];
      bytes += n * ((pc.src_dtype == TOFU_BF16 ? 2 : 4) * pc.nsrc + (pc.dst_dtype == TOFU_BF16 ? 2 : 4));
      if (pc.ep == TOFU_PIECE_MASK || pc.ep == TOFU_PIECE_ADD || pc.ep == TOFU_PIECE_ADDRELU) bytes += n * 2;
      if (pc.ep == TOFU_PIECE_MOM_SGD) bytes += n * (4 + 2 + 2);  // momentum read, weight read + written
      rows += (double)pc.extent[0] * pc.extent[1] * pc.extent[2];
      row_bytes += n * (pc.dst_dtype == TOFU_BF16 ? 2 : 4);
      vec += n * pc.pad_;
      elems += n;
    }
    // pieces, tasks, mean destination row length (bytes) and element-weighted mean vector width
    o += ",\"pieces\":" + std::to_string(L.npieces) + ",\"tasks\":" + std::to_string(L.ntasks) +
         ",\"row_bytes\":" + json_num(rows > 0 ? row_bytes / rows : 0) +
         ",\"vec\":" + json_num(elems > 0 ? vec / elems : 0);
    int maxsrc = 0;
    for (int64_t p = L.piece_off; p < L.piece_off + L.npieces; ++p) maxsrc = std::max(maxsrc, E.host_pieces[p].nsrc);
    o += ",\"max_src\":" + std::to_string(maxsrc) + ",\"piece_kernel\":\"" +
         (L.all_raw == 1 ? "copy" : L.all_raw == 2 ? "many_source" : "general") + "\"";
  } else if (L.kind == 1) {
    const LOp& lo = E.lops[L.li][L.op];
    const std::string& dn = g.defs[g.ops[L.op].def].name;
    const OpDef& dd = g.defs[g.ops[L.op].def];
    if (std::string(kernel_kind(dd)) == "gemm") {
      const GemmForm gf = gemm_form(dd);
      double M = 1, N = 1, K = 1;
      for (int v = 0; v < dd.n_out; ++v) (v < gf.nm ? M : N) *= (double)lo.out.box[v].len();
      const auto& ab = lo.in[gf.a_param].box;
      for (int q = 0; q < gf.nk; ++q) K *= (double)ab[gf.a_mn ? q : gf.nm + q].len();
      flops = 2 * M * N * K;
      bytes = 2 * (M * K + K * N) + M * N * (lo.fused_opt >= 0 ? (8 + 4) : (lo.out.dtype == TOFU_BF16 ? 2 : 4));
      o += ",\"mnk\":[" + json_num(M) + "," + json_num(N) + "," + json_num(K) + "]";
      auto git = E.gemms.find({L.op, L.li});
      if (git != E.gemms.end())
        o += ",\"splits\":" + std::to_string(git->second.a.splits) + ",\"bn\":" + std::to_string(git->second.bn);
      (void)dn;
    } else if (std::string(kernel_kind(dd)) == "conv") {
      // implicit GEMM: 2·M·N·K over the launches (the stride-2 data gradient's phases skip absent taps);
      // bytes: each operand region once + the output (fused optimizer: momentum and weight read + written)
      std::string shp;
      for (auto& a : conv_args(const_cast<Exec&>(E), L.op, L.li)) {
        const double pix = (double)a.nb * a.ngy * a.ngx, kn = (double)a.ntaps * a.nch;
        flops += a.kind == 0 ? 2 * pix * a.n_out * kn : 2 * (double)a.m_out * kn * pix;
        if (shp.empty())
          shp = a.kind == 0 ? "[" + json_num(pix) + "," + json_num(a.n_out) + "," + json_num(kn) + "]"
                            : "[" + json_num(a.m_out) + "," + json_num(kn) + "," + json_num(pix) + "]";
      }
      if (!shp.empty()) o += ",\"mnk\":" + shp;
      auto cit = E.convs.find({L.op, L.li});
      if (cit != E.convs.end() && !cit->second.empty()) o += ",\"splits\":" + std::to_string(cit->second[0].a.splits);
      auto git = E.gemms.find({L.op, L.li});
      if (git != E.gemms.end())
        o += ",\"splits\":" + std::to_string(git->second.a.splits) + ",\"bn\":" + std::to_string(git->second.bn);
      for (auto& b : lo.in) bytes += (double)vol(b.box) * (b.dtype == TOFU_BF16 ? 2 : 4);
      bytes += (double)vol(lo.out.box) * (lo.fused_opt >= 0 ? 12 : (lo.out.dtype == TOFU_BF16 ? 2 : 4));
    } else {
      const double n = (double)vol(lo.in[0].box);
      for (size_t k = 0; k < lo.in.size(); ++k) bytes += n * (lo.in[k].dtype == TOFU_BF16 ? 2 : 4);
      if (lo.fused_sgd) bytes += n * (4 + 2);  // m and w written back
      else if (dn != "sumsq") bytes += n * (lo.out.dtype == TOFU_BF16 ? 2 : 4);
      if (lo.fused_sgd) bytes += n * 2;       // w read
      if (lo.fused_loss_grad) bytes += n * 2;  // the loss gradient written (bf16)
    }
    bytes += (double)vol(lo.out.box) * 2 * (((lo.ep >> 1) & 1) + ((lo.ep >> 2) & 1));  // epilogue operands
  }
  o += ",\"flops\":" + json_num(flops) + ",\"bytes\":" + json_num(bytes);
  if (L.kind == 1 && !g.defs[g.ops[L.op].def].kernel.empty()) {  // the kernel bound by the def's TDL body
    const OpDef& kd = g.defs[g.ops[L.op].def];
    o += ",\"kernel\":" + json_quote(kd.kernel) + ",\"kconst\":[";
    for (size_t q = 0; q < kd.kconst.size(); ++q) o += (q ? "," : "") + json_num(kd.kconst[q]);
    o += "]";
  }
  if (L.kind == 2 && L.op >= 0 && !E.lops.empty()) {
    static const char* red_names[] = {"", "reduce+relu", "reduce+mask", "reduce+mom+sgd", "reduce+add", "reduce+addrelu"};
    int rep = 0;
    for (auto& lops : E.lops) rep = std::max(rep, lops[L.op].red_ep);
    if (rep) o += std::string(",\"fused\":\"") + red_names[rep] + "\"";
  }
  if (L.kind == 1 && lo_fused(E, L)) o += ",\"fused\":\"mom+sgd\"";
  if (L.kind == 1 && E.lops[L.li][L.op].fused_opt >= 0) o += ",\"fused\":\"gemm+mom+sgd\"";
  if (L.kind == 1 && E.lops[L.li][L.op].fused_next) o += ",\"fused\":\"lstm-cell-pair\"";
  if (L.kind == 1 && E.lops[L.li][L.op].cell_after >= 0) o += ",\"fused\":\"gemm+lstm-cell\"";
  if (L.kind == 1 && E.lops[L.li][L.op].fused_loss_grad) o += ",\"fused\":\"loss+loss_grad\"";
  if (L.kind == 1 && E.lops[L.li][L.op].wt_off >= 0) {
    o += ",\"weights\":\"transposed\"";
    if (!E.lops[L.li][L.op].in[1].direct) o += ",\"weights_from\":\"staging\"";  // (fetched; shared scratch)
  }
  if (L.kind == 1) {
    int np = 0;
    for (auto& b : E.lops[L.li][L.op].in) np += !b.rp.empty();
    if (np) o += ",\"inplace_remote_operands\":" + std::to_string(np);
  }
  if (L.kind == 1 && E.lops[L.li][L.op].ep) {
    const int ep = E.lops[L.li][L.op].ep;
    o += std::string(",\"fused\":\"epilogue") + (ep & 2 ? "+add" : "") + (ep & 1 ? "+relu" : "") + (ep & 4 ? "+mask" : "") + "\"";
  }
  return o + "}";
}
}  // namespace
}  // namespace tofu

extern "C" int tofu_execute(tofu_exec* h, void* stream) {
  return tofu::guard([&]() {
    if (!h) throw tofu::Error(TOFU_ERR_ARG, "null exec");
    tofu::run_range(h->e, 0, (int)h->e.launches.size(), reinterpret_cast<cudaStream_t>(stream));
    ++h->e.jitter_step;
    return TOFU_OK;
  });
}

extern "C" int tofu_execute_range(tofu_exec* h, int first, int last, void* stream) {
  return tofu::guard([&]() {
    if (!h || first < 0 || last > (int)h->e.launches.size() || first > last)
      throw tofu::Error(TOFU_ERR_ARG, "bad launch range");
    tofu::run_range(h->e, first, last, reinterpret_cast<cudaStream_t>(stream));
    return TOFU_OK;
  });
}

extern "C" int tofu_exec_num_launches(const tofu_exec* h, int* n) {
  if (!h || !n) return tofu::fail(TOFU_ERR_ARG, "null argument");
  *n = (int)h->e.launches.size();
  return TOFU_OK;
}

extern "C" int tofu_exec_launch_desc(const tofu_exec* h, int index, char* out, size_t cap, size_t* len) {
  return tofu::guard([&]() {
    if (!h || index < 0 || index >= (int)h->e.launches.size()) throw tofu::Error(TOFU_ERR_ARG, "bad launch index");
    return tofu::write_out(tofu::launch_desc(h->e, index), out, cap, len);
  });
}

extern "C" int tofu_exec_rank_bytes(const tofu_exec* h, int rank, int64_t* in_bytes, int64_t* out_bytes) {
  if (!h || rank < 0 || rank >= (int)h->e.rank_in.size()) return tofu::fail(TOFU_ERR_ARG, "bad rank");
  if (in_bytes) *in_bytes = h->e.skip_comm ? 0 : h->e.rank_in[rank];
  if (out_bytes) *out_bytes = h->e.skip_comm ? 0 : h->e.rank_out[rank];
  return TOFU_OK;
}

extern "C" int tofu_exec_unmaterialized(const tofu_exec* h, char* out, size_t cap, size_t* len) {
  return tofu::guard([&]() {
    if (!h) throw tofu::Error(TOFU_ERR_ARG, "null exec");
    std::string o = "[";
    for (int t : h->e.unmat) o += (o.size() > 1 ? "," : "") + tofu::json_quote(h->e.g->tensors[t].name);
    return tofu::write_out(o + "]", out, cap, len);
  });
}

extern "C" int tofu_exec_time_launch(tofu_exec* h, int index, void* ev_start, void* ev_stop) {
  if (!h) return tofu::fail(TOFU_ERR_ARG, "null exec");
  h->e.timed_launch = index;
  h->e.ev_start = reinterpret_cast<cudaEvent_t>(ev_start);
  h->e.ev_stop = reinterpret_cast<cudaEvent_t>(ev_stop);
  return TOFU_OK;
}

extern "C" int tofu_exec_ledger(const tofu_exec* h, int64_t* elements, int64_t* bytes) {
  if (!h) return tofu::fail(TOFU_ERR_ARG, "null exec");
  if (elements) *elements = h->e.skip_comm ? 0 : h->e.ledger_el;
  if (bytes) *bytes = h->e.skip_comm ? 0 : h->e.ledger_bytes;
  return TOFU_OK;
}

extern "C" int tofu_exec_launch_count(const tofu_exec* h, int64_t* launches) {
  if (!h || !launches) return tofu::fail(TOFU_ERR_ARG, "null argument");
  return tofu::guard([&]() {
    tofu::Exec& E = const_cast<tofu_exec*>(h)->e;
    // the descriptors decide the kernels per compute launch (split-K reductions, ...); without a device
    // (host-only lowering checks) every compute launch counts as one kernel
    bool ready = E.finalized;
    if (!ready) {
      try {
        tofu::finalize(E);
        ready = true;
      } catch (const tofu::Error&) {
        cudaGetLastError();
      }
    }
    int64_t n = 0;
    for (auto& L : E.launches) {
      if (L.kind == 4) continue;  // cudaMemsetAsync, not a kernel of ours
      if (E.skip_comm && (L.kind == 0 || L.kind == 2 || L.kind == 3)) continue;
      n += L.kind == 1 && ready ? tofu::kernels_of(E, L.op, L.li) : 1;
    }
    *launches = n;
    return TOFU_OK;
  });
}

extern "C" int tofu_exec_set_skip_comm(tofu_exec* h, int skip) {
  if (!h) return tofu::fail(TOFU_ERR_ARG, "null exec");
  h->e.skip_comm = skip != 0;
  return TOFU_OK;
}
