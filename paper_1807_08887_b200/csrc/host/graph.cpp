// Graph model, coarsening and the exact communication cost of a plan.
//   Coarsening, §5.1: element-wise op inputs/outputs unioned; tensors/ops with a
//   shared "merge" key (unrolled timesteps) unioned; in-place aliases unioned.  Forward /
//   backward groups impose no equality (members may differ).
//   Cost, P:L587 + Lemma proof P:L1618-1625 under the direct-transfer reading:
//   Σ_workers |Req \ Own| over inputs + |Prod \ Own| for the output (fp32 wire for partials).
#include "graph.h"

#include <algorithm>
#include <functional>
#include <numeric>
#include <set>

#include "common.h"
#include "json.h"

namespace tofu {

Graph graph_from_json(const std::string& text) {
  Json j = json_parse(text);
  Graph g;
  for (auto& kv : j.at("defs").obj) {
    OpDef d = parse_tdl(kv.second.as_str());
    match_kernel(d);
    if (d.name != kv.first) throw Error(TOFU_ERR_PARSE, "def key " + kv.first + " != def name " + d.name);
    g.def_ix[d.name] = (int)g.defs.size();
    g.defs.push_back(std::move(d));
  }
  std::vector<std::string> names;
  for (auto& kv : j.at("tensors").obj) names.push_back(kv.first);
  std::sort(names.begin(), names.end());
  for (auto& n : names) {
    const Json& t = j.at("tensors").at(n);
    TensorInfo ti;
    ti.name = n;
    for (auto& x : t.at("shape").arr) {
      if (x.as_int() <= 0) throw Error(TOFU_ERR_PARSE, "tensor " + n + ": non-positive dim");
      ti.shape.push_back(x.as_int());
    }
    if (auto* dt = t.get("dtype")) ti.dtype = dt->as_str() == "bf16" ? TOFU_BF16 : TOFU_F32;
    if (auto* r = t.get("role"); r && !r->is_null()) ti.role = r->as_str();
    if (auto* m = t.get("merge"); m && !m->is_null()) ti.merge = m->kind == Json::Str ? m->str : json_num(m->num);
    g.tensor_ix[n] = (int)g.tensors.size();
    g.tensors.push_back(ti);
  }
  auto tid = [&](const std::string& n) {
    auto it = g.tensor_ix.find(n);
    if (it == g.tensor_ix.end()) throw Error(TOFU_ERR_PARSE, "unknown tensor " + n);
    return it->second;
  };
  std::map<int, std::vector<std::vector<Rng>>> produced;
  for (auto& o : j.at("ops").arr) {
    OpInfo oi;
    oi.name = o.at("name").as_str();
    auto dit = g.def_ix.find(o.at("def").as_str());
    if (dit == g.def_ix.end()) throw Error(TOFU_ERR_PARSE, "UnknownOperator " + o.at("def").as_str());
    oi.def = dit->second;
    const OpDef& d = g.defs[oi.def];
    for (auto& x : o.at("inputs").arr) oi.inputs.push_back(tid(x.as_str()));
    oi.output = tid(o.at("output").as_str());
    if (oi.inputs.size() != d.params.size()) throw Error(TOFU_ERR_PARSE, "ShapeMismatch " + oi.name + ": arity");
    for (size_t p = 0; p < oi.inputs.size(); ++p)
      if ((int)g.tensors[oi.inputs[p]].shape.size() != d.ranks[p])
        throw Error(TOFU_ERR_PARSE, "ShapeMismatch " + oi.name + ": rank of " + g.tensors[oi.inputs[p]].name);
    const auto& oshape = g.tensors[oi.output].shape;
    if ((int)oshape.size() != d.n_out) throw Error(TOFU_ERR_PARSE, "ShapeMismatch " + oi.name + ": output rank");
    if (auto* m = o.get("merge"); m && !m->is_null()) oi.merge = m->kind == Json::Str ? m->str : json_num(m->num);
    if (auto* a = o.get("attrs"); a && a->kind == Json::Obj)
      for (auto& kv : a->obj)
        if (kv.second.kind == Json::Num) oi.attrs[kv.first] = kv.second.num;
    // offsets
    oi.in_off.resize(oi.inputs.size());
    const Json* offs = o.get("offsets");
    for (size_t p = 0; p < oi.inputs.size(); ++p) {
      oi.in_off[p].assign(g.tensors[oi.inputs[p]].shape.size(), 0);
      if (offs && offs->kind == Json::Arr && p < offs->arr.size() && offs->arr[p].kind == Json::Arr)
        for (size_t dd = 0; dd < offs->arr[p].arr.size() && dd < oi.in_off[p].size(); ++dd)
          oi.in_off[p][dd] = offs->arr[p].arr[dd].as_int();
    }
    oi.out_off.assign(oshape.size(), 0);
    if (auto* oo = o.get("out_offset"); oo && oo->kind == Json::Arr)
      for (size_t dd = 0; dd < oo->arr.size() && dd < oi.out_off.size(); ++dd) oi.out_off[dd] = oo->arr[dd].as_int();
    std::vector<std::vector<int64_t>> ins;
    for (int t : oi.inputs) ins.push_back(g.tensors[t].shape);
    // var extents: inferred from shapes, overridden by explicit "ranges" (views)
    std::map<std::string, int64_t> over;
    if (auto* rg = o.get("ranges"); rg && rg->kind == Json::Obj)
      for (auto& kv : rg->obj) over[kv.first] = kv.second.as_int();
    std::vector<int64_t> oshape_it(oshape);
    for (int v = 0; v < d.n_out; ++v)
      if (over.count(d.vars[v])) oshape_it[v] = over[d.vars[v]];
    std::vector<int64_t> given(d.vars.size(), -1);
    for (size_t v = 0; v < d.vars.size(); ++v)
      if (over.count(d.vars[v])) given[v] = over[d.vars[v]];
    oi.R = var_extents(d, ins, oshape_it, given);
    for (size_t v = 0; v < d.vars.size(); ++v)
      if (over.count(d.vars[v])) oi.R[v] = over[d.vars[v]];
    // output view inside the tensor and disjoint from other producers' views
    std::vector<Rng> obox;
    for (int v = 0; v < d.n_out; ++v) {
      obox.push_back({oi.out_off[v], oi.out_off[v] + oi.R[v] - 1});
      if (obox.back().lo < 0 || obox.back().hi >= oshape[v])
        throw Error(TOFU_ERR_PARSE, "ShapeMismatch " + oi.name + ": output view out of range");
    }
    for (auto& other : produced[oi.output]) {
      bool overlap = true;
      for (size_t dd = 0; dd < obox.size(); ++dd)
        overlap &= obox[dd].lo <= other[dd].hi && other[dd].lo <= obox[dd].hi;
      if (overlap) throw Error(TOFU_ERR_PARSE, "tensor " + g.tensors[oi.output].name + " produced twice");
    }
    produced[oi.output].push_back(obox);
    // accesses may leave their tensor: zero padding (reading R11), nothing to check
    g.ops.push_back(oi);
  }
  if (auto* al = j.get("alias"); al && al->kind == Json::Obj)
    for (auto& kv : al->obj) g.alias.emplace_back(tid(kv.first), tid(kv.second.as_str()));

  // ------------------------------------------------------------------ coarsening (union-find)
  const int nt = (int)g.tensors.size();
  std::vector<int> parent(nt);
  std::iota(parent.begin(), parent.end(), 0);
  std::function<int(int)> find = [&](int x) {
    while (parent[x] != x) x = parent[x] = parent[parent[x]];
    return x;
  };
  auto unite = [&](int a, int b) {
    a = find(a);
    b = find(b);
    if (a != b) {
      // keep the lexicographically smaller name as root (matches the oracle's ordering-independent classes)
      if (g.tensors[a].name < g.tensors[b].name) parent[b] = a;
      else parent[a] = b;
    }
  };
  for (auto& o : g.ops)
    if (g.defs[o.def].cls == "ElementWise" && !o.has_offsets())
      for (int t : o.inputs) unite(t, o.output);
  for (auto& pr : g.alias) unite(pr.first, pr.second);
  std::map<std::string, std::vector<int>> bykey;
  for (int t = 0; t < nt; ++t)
    if (!g.tensors[t].merge.empty()) bykey[g.tensors[t].merge].push_back(t);
  for (auto& kv : bykey)
    for (size_t k = 1; k < kv.second.size(); ++k) unite(kv.second[0], kv.second[k]);
  // class ids in order of first appearance (op inputs then output, then remaining tensors by name)
  std::vector<int> order, cid(nt, -1);
  auto see = [&](int t) {
    int r = find(t);
    if (cid[r] < 0) {
      cid[r] = (int)order.size();
      order.push_back(r);
    }
  };
  for (auto& o : g.ops) {
    for (int t : o.inputs) see(t);
    see(o.output);
  }
  for (int t = 0; t < nt; ++t) see(t);
  g.tclass.assign(nt, 0);
  g.classes.assign(order.size(), {});
  for (int t = 0; t < nt; ++t) {
    g.tclass[t] = cid[find(t)];
    g.classes[g.tclass[t]].push_back(t);  // tensors are stored sorted by name
  }
  for (auto& ms : g.classes) {
    size_t r = g.tensors[ms[0]].shape.size();
    for (int t : ms)
      if (g.tensors[t].shape.size() != r) throw Error(TOFU_ERR_PARSE, "tensor class mixes ranks");
  }
  std::map<std::string, int> okey;
  g.oclass.assign(g.ops.size(), 0);
  for (size_t o = 0; o < g.ops.size(); ++o) {
    const std::string& k = g.ops[o].merge;
    int c;
    if (!k.empty() && okey.count(k)) c = okey[k];
    else {
      c = (int)g.op_classes.size();
      g.op_classes.push_back({});
      if (!k.empty()) okey[k] = c;
    }
    g.op_classes[c].push_back((int)o);
    g.oclass[o] = c;
  }
  for (auto& ms : g.op_classes)
    for (int o : ms)
      if (g.ops[o].def != g.ops[ms[0]].def) throw Error(TOFU_ERR_PARSE, "merged ops have different defs");
  return g;
}

// ---------------------------------------------------------------------------------- boxes
std::vector<int> worker_digits(int w, const std::vector<int>& factors) {
  std::vector<int> d(factors.size());
  for (int i = (int)factors.size() - 1; i >= 0; --i) {
    d[i] = w % factors[i];
    w /= factors[i];
  }
  return d;
}

Rng nested_range(int64_t n, const std::vector<std::pair<int, int>>& splits) {
  int64_t lo = 0, size = n;
  for (auto& s : splits) {
    size /= s.first;
    lo += s.second * size;
  }
  return {lo, lo + size - 1};
}

bool owned_box(const Graph& g, int t, const std::vector<int>& tdims, const std::vector<int>& factors,
               const std::vector<int>& dig, std::vector<Rng>& box) {
  const auto& shape = g.tensors[t].shape;
  box.clear();
  if (shape.empty()) {
    for (int x : dig)
      if (x) return false;
    return true;
  }
  for (size_t d = 0; d < shape.size(); ++d) {
    std::vector<std::pair<int, int>> sp;
    for (size_t i = 0; i < factors.size(); ++i)
      if (tdims[i] == (int)d) sp.emplace_back(factors[i], dig[i]);
    box.push_back(nested_range(shape[d], sp));
  }
  return true;
}

void iter_box(const Graph& g, int op, const std::vector<int>& oseq, const std::vector<int>& factors,
              const std::vector<int>& dig, std::vector<Rng>& box) {
  const auto& R = g.ops[op].R;
  box.clear();
  for (size_t v = 0; v < R.size(); ++v) {
    std::vector<std::pair<int, int>> sp;
    for (size_t i = 0; i < factors.size(); ++i)
      if (oseq[i] == (int)v) sp.emplace_back(factors[i], dig[i]);
    box.push_back(nested_range(R[v], sp));
  }
}

std::vector<Rng> required_box(const Graph& g, int op, int param, const std::vector<Rng>& ib) {
  const OpDef& d = g.def_of(op);
  const auto& shape = g.tensors[g.ops[op].inputs[param]].shape;
  std::vector<Rng> req(shape.size(), Rng{INT64_MAX, INT64_MIN});
  for (auto& a : d.accesses) {
    if (a.param != param) continue;
    for (size_t dim = 0; dim < a.idx.size(); ++dim) {
      int64_t lo, hi;
      if (a.slice[dim]) {
        lo = 0;
        hi = shape[dim] - 1;
      } else {
        a.idx[dim].hull(ib, g.ops[op].in_off[param][dim], lo, hi);
      }
      req[dim].lo = std::min(req[dim].lo, lo);
      req[dim].hi = std::max(req[dim].hi, hi);
    }
  }
  // the hull ∩ the tensor: elements outside it read as zero and are never moved (reading R11)
  for (size_t dim = 0; dim < req.size(); ++dim) {
    req[dim].lo = std::max<int64_t>(req[dim].lo, 0);
    req[dim].hi = std::min<int64_t>(req[dim].hi, shape[dim] - 1);
  }
  return req;
}

std::vector<Rng> produced_box(const Graph& g, int op, const std::vector<Rng>& ib) {
  const OpDef& d = g.def_of(op);
  std::vector<Rng> b;
  for (int v = 0; v < d.n_out; ++v) b.push_back({ib[v].lo + g.ops[op].out_off[v], ib[v].hi + g.ops[op].out_off[v]});
  return b;
}

static int64_t vol(const std::vector<Rng>& b) {
  int64_t p = 1;
  for (auto& r : b) p *= r.len();
  return p;
}
static int64_t inter_vol(const std::vector<Rng>& a, const std::vector<Rng>& b) {
  int64_t p = 1;
  for (size_t i = 0; i < a.size(); ++i) p *= Rng{std::max(a[i].lo, b[i].lo), std::min(a[i].hi, b[i].hi)}.len();
  return p;
}

OpCost op_cost(const Graph& g, int op, const PlanSeq& p) {
  const OpDef& d = g.def_of(op);
  const OpInfo& o = g.ops[op];
  const auto& seq = p.osplit[op];
  int nw = 1;
  for (int k : p.factors) nw *= k;
  bool partial = false;
  for (int v : seq)
    if (d.is_red(v)) partial = true;
  OpCost c;
  std::vector<Rng> ib, own, prod;
  for (int w = 0; w < nw; ++w) {
    auto dig = worker_digits(w, p.factors);
    iter_box(g, op, seq, p.factors, dig, ib);
    for (size_t pi = 0; pi < d.params.size(); ++pi) {
      // every param is accessed at least once in valid defs; unaccessed params move nothing
      bool used = false;
      for (auto& a : d.accesses) used |= a.param == (int)pi;
      if (!used) continue;
      int t = o.inputs[pi];
      auto req = required_box(g, op, (int)pi, ib);
      int64_t n = vol(req);
      int64_t loc = owned_box(g, t, p.tdims[t], p.factors, dig, own) ? inter_vol(req, own) : 0;
      c.fetch += n - loc;
      c.bytes += (n - loc) * g.itemsize(t);
    }
    prod = produced_box(g, op, ib);
    int64_t n = vol(prod);
    int64_t loc = owned_box(g, o.output, p.tdims[o.output], p.factors, dig, own) ? inter_vol(prod, own) : 0;
    c.out += n - loc;
    c.bytes += (n - loc) * (partial ? 4 : g.itemsize(o.output));
  }
  c.elements = c.fetch + c.out;
  return c;
}

OpCost plan_cost(const Graph& g, const PlanSeq& p) {
  OpCost tot;
  for (size_t o = 0; o < g.ops.size(); ++o) {
    OpCost c = op_cost(g, (int)o, p);
    tot.elements += c.elements;
    tot.bytes += c.bytes;
    tot.fetch += c.fetch;
    tot.out += c.out;
  }
  return tot;
}

}  // namespace tofu

struct tofu_graph {
  tofu::Graph g;
};

extern "C" int tofu_graph_create(const char* graph_json, tofu_graph** out) {
  return tofu::guard([&]() {
    if (!graph_json || !out) throw tofu::Error(TOFU_ERR_ARG, "null argument");
    auto* h = new tofu_graph{tofu::graph_from_json(graph_json)};
    *out = h;
    return TOFU_OK;
  });
}
extern "C" void tofu_graph_destroy(tofu_graph* g) { delete g; }

namespace tofu {
const Graph& graph_of(const tofu_graph* h) { return h->g; }
}  // namespace tofu
