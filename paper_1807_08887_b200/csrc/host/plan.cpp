// tofu_plan: recursive partitioning (§5.2) with the per-step DP over the coarsened graph
// (P:L340-349).  One step = exact min-sum variable elimination over tensor-class and op-class
// variables (on a chain this is the chain DP; the per-group brute force of P:L655-658 is the factor table
// of each op class).  All co-optimal step plans are enumerated and carried forward as a frontier
// (DESIGN.md §R4), k = k1·…·km with ki non-increasing primes.  search = 1 runs the same
// elimination over sequence-valued variables (all steps jointly: exact, small graphs only).
#include <algorithm>
#include <chrono>
#include <functional>
#include <map>
#include <numeric>
#include <set>
#include <string>
#include <unordered_map>
#include <cstdlib>
#include <exception>
#include <thread>

#include "common.h"
#include "graph.h"
#include "json.h"
#include "plan.h"

namespace tofu {
namespace {

std::vector<int> factorize(int k) {
  std::vector<int> f;
  for (int p = 2; (int64_t)p * p <= k; ++p)
    while (k % p == 0) {
      f.push_back(p);
      k /= p;
    }
  if (k > 1) f.push_back(k);
  std::sort(f.rbegin(), f.rend());
  return f;
}

// ------------------------------------------------------------------------------ variable elimination
struct Factor {
  std::vector<int> scope;       // sorted var ids
  std::vector<int64_t> table;   // row-major over scope domain sizes
};

struct VE {
  std::vector<int> dsize;
  std::vector<Factor> factors;
  struct Trace {
    int x;
    std::vector<int> scope;
    std::vector<int64_t> comb;
    std::vector<int64_t> st;  // strides of scope
  };
  std::vector<Trace> trace;

  static std::vector<int64_t> strides(const std::vector<int>& scope, const std::vector<int>& dsize) {
    std::vector<int64_t> s(scope.size());
    int64_t acc = 1;
    for (int i = (int)scope.size() - 1; i >= 0; --i) {
      s[i] = acc;
      acc *= dsize[scope[i]];
    }
    return s;
  }

  // order: elimination order to follow (computed by the min-degree rule when empty and written back; it
  // depends only on the factor scopes and domain sizes, so frontier prefixes with equal domains share it)
  int64_t run(int cap, std::vector<std::vector<int>>& sols, std::vector<int>& order) {
    // min-degree greedy order (ties -> smallest var id), with var -> factor adjacency kept incrementally
    std::vector<Factor> active = factors;
    std::vector<char> alive(active.size(), 1);
    const int nv = (int)dsize.size();
    std::vector<std::set<int>> adj(nv);  // var -> ids of alive factors containing it
    for (size_t f = 0; f < active.size(); ++f)
      for (int y : active[f].scope) adj[y].insert((int)f);
    std::set<int> remaining;
    for (int v = 0; v < nv; ++v) remaining.insert(v);
    const bool given = (int)order.size() == nv;
    if (!given) order.clear();
    while (!remaining.empty()) {
      int bx = -1;
      if (given) {
        bx = order[nv - (int)remaining.size()];
      } else {
        double bw = 0;
        for (int x : remaining) {
          std::set<int> nb;
          for (int f : adj[x]) nb.insert(active[f].scope.begin(), active[f].scope.end());
          double w = 1;
          for (int y : nb) w *= dsize[y];
          if (bx < 0 || w < bw) {
            bx = x;
            bw = w;
          }
        }
        order.push_back(bx);
      }
      int x = bx;
      std::vector<int> tids(adj[x].begin(), adj[x].end());
      std::set<int> sc;
      for (int f : tids) sc.insert(active[f].scope.begin(), active[f].scope.end());
      sc.insert(x);
      std::vector<int> scope(sc.begin(), sc.end());
      int64_t n = 1;
      for (int y : scope) n *= dsize[y];
      std::vector<int64_t> comb(n, 0);
      std::vector<int> idx(scope.size());
      for (int fi : tids) {
        const Factor& f = active[fi];
        auto fst = strides(f.scope, dsize);
        std::vector<int> pos(f.scope.size());
        for (size_t a = 0; a < f.scope.size(); ++a)
          pos[a] = (int)(std::find(scope.begin(), scope.end(), f.scope[a]) - scope.begin());
        for (int64_t e = 0; e < n; ++e) {
          int64_t r = e, off = 0;
          for (int a = (int)scope.size() - 1; a >= 0; --a) {
            idx[a] = (int)(r % dsize[scope[a]]);
            r /= dsize[scope[a]];
          }
          for (size_t a = 0; a < f.scope.size(); ++a) off += idx[pos[a]] * fst[a];
          comb[e] += f.table[off];
        }
      }
      std::vector<int> mscope;
      for (int y : scope)
        if (y != x) mscope.push_back(y);
      auto mst = strides(mscope, dsize);
      int64_t mn = 1;
      for (int y : mscope) mn *= dsize[y];
      std::vector<int64_t> msg(mn, INT64_MAX);
      int xpos = (int)(std::find(scope.begin(), scope.end(), x) - scope.begin());
      for (int64_t e = 0; e < n; ++e) {
        int64_t r = e, off = 0;
        for (int a = (int)scope.size() - 1; a >= 0; --a) {
          idx[a] = (int)(r % dsize[scope[a]]);
          r /= dsize[scope[a]];
        }
        int b = 0;
        for (int a = 0; a < (int)scope.size(); ++a)
          if (a != xpos) off += idx[a] * mst[b++];
        msg[off] = std::min(msg[off], comb[e]);
      }
      trace.push_back({x, scope, std::move(comb), strides(scope, dsize)});
      for (int fi : tids) {
        alive[fi] = 0;
        for (int y : active[fi].scope) adj[y].erase(fi);
      }
      const int nid = (int)active.size();
      active.push_back({mscope, std::move(msg)});
      alive.push_back(1);
      for (int y : mscope) adj[y].insert(nid);
      remaining.erase(x);
    }
    std::vector<Factor> rest;
    for (size_t f = 0; f < active.size(); ++f)
      if (alive[f]) rest.push_back(std::move(active[f]));
    active.swap(rest);
    int64_t total = 0;
    for (auto& f : active) total += f.table.at(0);
    // enumerate co-optimal assignments (DFS in reverse elimination order)
    std::vector<int> assign(dsize.size(), -1);
    std::function<void(int)> dfs = [&](int i) {
      if ((int)sols.size() >= cap) return;
      if (i < 0) {
        sols.push_back(assign);
        return;
      }
      auto& tr = trace[i];
      const auto& st = tr.st;
      int64_t base = 0;
      int64_t xs = 0;
      for (size_t a = 0; a < tr.scope.size(); ++a) {
        if (tr.scope[a] == tr.x) xs = st[a];
        else base += assign[tr.scope[a]] * st[a];
      }
      int64_t m = INT64_MAX;
      for (int v = 0; v < dsize[tr.x]; ++v) m = std::min(m, tr.comb[base + v * xs]);
      for (int v = 0; v < dsize[tr.x]; ++v)
        if (tr.comb[base + v * xs] == m) {
          assign[tr.x] = v;
          dfs(i - 1);
          assign[tr.x] = -1;
        }
    };
    dfs((int)trace.size() - 1);
    return total;
  }
};

int64_t extent_after(int64_t n, const std::vector<int>& seq, int axis, const std::vector<int>& factors) {
  for (size_t i = 0; i < seq.size(); ++i)
    if (seq[i] == axis) n /= factors[i];
  return n;
}

std::vector<int> tensor_domain(const Graph& g, int cls, const PlanSeq& pre, int k) {
  const auto& ms = g.classes[cls];
  size_t rank = g.tensors[ms[0]].shape.size();
  if (rank == 0) return {-1};
  std::vector<int> dom;
  for (size_t d = 0; d < rank; ++d) {
    bool ok = true;
    for (int t : ms)
      if (extent_after(g.tensors[t].shape[d], pre.tdims[t], (int)d, pre.factors) % k) ok = false;
    if (ok) dom.push_back((int)d);
  }
  return dom;
}

std::vector<int> op_domain(const Graph& g, int ocls, const PlanSeq& pre, int k) {
  const auto& ms = g.op_classes[ocls];
  std::vector<int> dom;
  for (int v : g.def_of(ms[0]).split_vars()) {
    bool ok = true;
    for (int o : ms)
      if (extent_after(g.ops[o].R[v], pre.osplit[o], v, pre.factors) % k) ok = false;
    if (ok) dom.push_back(v);
  }
  return dom;
}

// canonical key (matches oracle.search.canon_key): per tensor class the dim sequence of its first member
// (None = -1), then per op class the index of each step's var in split_vars().
std::vector<int> canon_key(const Graph& g, const PlanSeq& p) {
  std::vector<int> key;
  for (auto& ms : g.classes)
    for (int d : p.tdims[ms[0]]) key.push_back(d);
  for (auto& ms : g.op_classes) {
    const OpDef& d = g.def_of(ms[0]);
    for (int v : p.osplit[ms[0]]) {
      if (!d.opaque) {  // split_vars() is 0..n-1: the index is the var itself
        key.push_back(v);
      } else {
        const auto& sv = d.opaque_free;
        key.push_back((int)(std::find(sv.begin(), sv.end(), v) - sv.begin()));
      }
    }
  }
  return key;
}

struct StepResult {
  int64_t cost;
  std::vector<PlanSeq> plans;
  bool truncated;
};

// Memo of per-op costs: an op's cost depends only on its own split sequence and the dim sequences of its
// tensors, which repeat across frontier prefixes and across factor-table entries.
struct CostMemo {
  std::unordered_map<std::string, int64_t> m;
  std::string key;  // reused buffer: op id (4 bytes), then one byte per factor / var / dim (all < 128)
  int64_t get(const Graph& g, int o, const PlanSeq& p) {
    key.assign(reinterpret_cast<const char*>(&o), sizeof o);
    for (int f : p.factors) key.push_back((char)f);
    for (int v : p.osplit[o]) key.push_back((char)v);
    for (int t : g.ops[o].inputs)
      for (int d : p.tdims[t]) key.push_back((char)d);
    for (int d : p.tdims[g.ops[o].output]) key.push_back((char)d);
    auto it = m.find(key);
    if (it != m.end()) return it->second;
    int64_t c = op_cost(g, o, p).elements;
    m.emplace(key, c);
    return c;
  }
};

using OrderCache = std::map<std::vector<int>, std::vector<int>>;  // domain sizes -> elimination order
// An op class's factor table depends on the prefix only through its members' own split sequences and their
// tensors' dim sequences (and the step's domains): frontier prefixes share most tables.
using TableCache = std::unordered_map<std::string, std::vector<int64_t>>;

StepResult step_search(const Graph& g, const PlanSeq& pre, int k, int cap, CostMemo& memo, OrderCache& oc,
                       TableCache& tc) {
  const int nT = (int)g.classes.size(), nO = (int)g.op_classes.size();
  std::vector<std::vector<int>> dom(nT + nO);
  for (int c = 0; c < nT; ++c) {
    dom[c] = tensor_domain(g, c, pre, k);
    if (dom[c].empty()) throw Error(TOFU_ERR_PLAN, "no divisible dim for tensor class of " + g.tensors[g.classes[c][0]].name);
  }
  for (int c = 0; c < nO; ++c) {
    dom[nT + c] = op_domain(g, c, pre, k);
    if (dom[nT + c].empty()) throw Error(TOFU_ERR_PLAN, "no divisible var for op " + g.ops[g.op_classes[c][0]].name);
  }
  VE ve;
  for (auto& d : dom) ve.dsize.push_back((int)d.size());
  PlanSeq cur = pre;
  cur.factors.push_back(k);
  for (auto& s : cur.tdims) s.push_back(-1);
  for (auto& s : cur.osplit) s.push_back(-1);
  for (int oc = 0; oc < nO; ++oc) {
    std::set<int> tcs;
    for (int o : g.op_classes[oc]) {
      for (int t : g.ops[o].inputs) tcs.insert(g.tclass[t]);
      tcs.insert(g.tclass[g.ops[o].output]);
    }
    Factor f;
    f.scope.assign(tcs.begin(), tcs.end());
    f.scope.push_back(nT + oc);
    int64_t n = 1;
    for (int x : f.scope) n *= ve.dsize[x];
    std::string tkey;
    tkey.append(reinterpret_cast<const char*>(&oc), sizeof oc);
    tkey.push_back((char)k);
    for (int fct : pre.factors) tkey.push_back((char)fct);
    for (int x : f.scope) {
      tkey.push_back((char)0x7f);
      for (int dv : dom[x]) tkey.push_back((char)dv);
    }
    for (int o : g.op_classes[oc]) {
      tkey.push_back((char)0x7e);
      for (int v : pre.osplit[o]) tkey.push_back((char)v);
      for (int t : g.ops[o].inputs)
        for (int d : pre.tdims[t]) tkey.push_back((char)d);
      for (int d : pre.tdims[g.ops[o].output]) tkey.push_back((char)d);
    }
    auto hit = tc.find(tkey);
    if (hit != tc.end()) {
      f.table = hit->second;
      ve.factors.push_back(std::move(f));
      continue;
    }
    f.table.assign(n, 0);
    std::vector<int> idx(f.scope.size());
    for (int64_t e = 0; e < n; ++e) {
      int64_t r = e;
      for (int a = (int)f.scope.size() - 1; a >= 0; --a) {
        idx[a] = (int)(r % ve.dsize[f.scope[a]]);
        r /= ve.dsize[f.scope[a]];
      }
      const int v = dom[nT + oc][idx.back()];
      int64_t val = 0;
      for (int o : g.op_classes[oc]) {
        for (size_t a = 0; a + 1 < f.scope.size(); ++a) {
          const int d = dom[f.scope[a]][idx[a]];
          for (int t : g.classes[f.scope[a]]) cur.tdims[t].back() = d;
        }
        cur.osplit[o].back() = v;
        val += memo.get(g, o, cur);
      }
      f.table[e] = val;
    }
    tc.emplace(std::move(tkey), f.table);
    ve.factors.push_back(std::move(f));
  }
  std::vector<std::vector<int>> sols;
  StepResult res;
  std::vector<int>& order = oc[ve.dsize];
  res.cost = ve.run(cap, sols, order);
  res.truncated = (int)sols.size() >= cap;
  for (auto& s : sols) {
    PlanSeq p = cur;
    for (size_t t = 0; t < g.tensors.size(); ++t) p.tdims[t].back() = dom[g.tclass[t]][s[g.tclass[t]]];
    for (size_t o = 0; o < g.ops.size(); ++o) p.osplit[o].back() = dom[nT + g.oclass[o]][s[nT + g.oclass[o]]];
    res.plans.push_back(std::move(p));
  }
  std::vector<std::pair<std::vector<int>, size_t>> keyed;
  for (size_t i = 0; i < res.plans.size(); ++i) keyed.emplace_back(canon_key(g, res.plans[i]), i);
  std::sort(keyed.begin(), keyed.end());
  std::vector<PlanSeq> sorted;
  sorted.reserve(keyed.size());
  for (auto& kv : keyed) sorted.push_back(std::move(res.plans[kv.second]));
  res.plans.swap(sorted);
  return res;
}

}  // namespace

static PlanResult make_plan_mode(const Graph& g, int k, int frontier_cap, int solution_cap, int search) {
  auto t0 = std::chrono::steady_clock::now();
  PlanResult r;
  r.k = k;
  PlanSeq empty;
  empty.tdims.assign(g.tensors.size(), {});
  empty.osplit.assign(g.ops.size(), {});
  std::vector<int> factors = factorize(k);
  if (k == 1) {
    r.seq = empty;
  } else if (search == 0) {
    std::vector<PlanSeq> frontier = {empty};
    // the frontier's prefixes are searched in parallel (host threads, each with its own caches: the caches
    // never change a value), and their results combined in frontier order — the same plan as sequentially
    const int nthreads = [] {
      const char* e = std::getenv("TOFU_PLAN_THREADS");
      const int hw = (int)std::thread::hardware_concurrency();
      return std::max(1, e ? std::atoi(e) : std::min(hw > 0 ? hw : 1, 16));
    }();
    std::vector<CostMemo> memo(nthreads);
    std::vector<OrderCache> ocache(nthreads);
    std::vector<TableCache> tcache(nthreads);
    for (int ki : factors) {
      int64_t best = INT64_MAX;
      std::vector<PlanSeq> cands;
      std::vector<StepResult> res(frontier.size());
      std::vector<std::exception_ptr> err(nthreads);
      auto work = [&](int tid) {
        try {
          for (size_t i = tid; i < frontier.size(); i += nthreads)
            res[i] = step_search(g, frontier[i], ki, solution_cap, memo[tid], ocache[tid], tcache[tid]);
        } catch (...) {
          err[tid] = std::current_exception();
        }
      };
      const int nt = std::min<int>(nthreads, (int)frontier.size());
      std::vector<std::thread> pool;
      for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
      work(0);
      for (auto& th : pool) th.join();
      for (auto& e : err)
        if (e) std::rethrow_exception(e);
      for (auto& s : res) {
        r.truncated |= s.truncated;
        if (s.cost < best) {
          best = s.cost;
          cands = std::move(s.plans);
        } else if (s.cost == best) {
          for (auto& p : s.plans) cands.push_back(std::move(p));
        }
      }
      std::map<std::vector<int>, PlanSeq> uniq;
      for (auto& p : cands) uniq.emplace(canon_key(g, p), std::move(p));
      frontier.clear();
      for (auto& kv : uniq) {
        if ((int)frontier.size() >= frontier_cap) {
          r.truncated = true;
          break;
        }
        frontier.push_back(std::move(kv.second));
      }
    }
    r.seq = frontier.front();
  } else {
    // flat exact search: VE over sequences of all steps
    const int nT = (int)g.classes.size(), nO = (int)g.op_classes.size();
    const int m = (int)factors.size();
    std::vector<std::vector<std::vector<int>>> dom(nT + nO);
    for (int c = 0; c < nT + nO; ++c) {
      bool is_t = c < nT;
      int rank = is_t ? (int)g.tensors[g.classes[c][0]].shape.size() : 0;
      std::vector<int> axes = is_t ? std::vector<int>() : g.def_of(g.op_classes[c - nT][0]).split_vars();
      if (is_t)
        for (int d = 0; d < rank; ++d) axes.push_back(d);
      if (is_t && rank == 0) {
        dom[c].push_back(std::vector<int>(m, -1));
        continue;
      }
      std::vector<int> seq(m, 0);
      std::function<void(int)> rec = [&](int i) {
        if (i == m) {
          bool ok = true;
          const auto& members = is_t ? g.classes[c] : g.op_classes[c - nT];
          for (int x : members)
            for (int a : axes) {
              int64_t n = is_t ? g.tensors[x].shape[a] : g.ops[x].R[a];
              for (int s = 0; s < m && ok; ++s)
                if (seq[s] == a) {
                  if (n % factors[s]) ok = false;
                  n /= factors[s];
                }
            }
          if (ok) dom[c].push_back(seq);
          return;
        }
        for (int a : axes) {
          seq[i] = a;
          rec(i + 1);
        }
      };
      rec(0);
      if (dom[c].empty()) throw Error(TOFU_ERR_PLAN, "flat search: no divisible sequence");
    }
    VE ve;
    for (auto& d : dom) ve.dsize.push_back((int)d.size());
    PlanSeq cur = empty;
    cur.factors = factors;
    for (auto& s : cur.tdims) s.assign(m, -1);
    for (auto& s : cur.osplit) s.assign(m, -1);
    for (int oc = 0; oc < nO; ++oc) {
      std::set<int> tcs;
      for (int o : g.op_classes[oc]) {
        for (int t : g.ops[o].inputs) tcs.insert(g.tclass[t]);
        tcs.insert(g.tclass[g.ops[o].output]);
      }
      Factor f;
      f.scope.assign(tcs.begin(), tcs.end());
      f.scope.push_back(nT + oc);
      int64_t n = 1;
      for (int x : f.scope) n *= ve.dsize[x];
      f.table.assign(n, 0);
      std::vector<int> idx(f.scope.size());
      for (int64_t e = 0; e < n; ++e) {
        int64_t rr = e;
        for (int a = (int)f.scope.size() - 1; a >= 0; --a) {
          idx[a] = (int)(rr % ve.dsize[f.scope[a]]);
          rr /= ve.dsize[f.scope[a]];
        }
        int64_t val = 0;
        for (int o : g.op_classes[oc]) {
          for (size_t a = 0; a + 1 < f.scope.size(); ++a)
            for (int t : g.classes[f.scope[a]]) cur.tdims[t] = dom[f.scope[a]][idx[a]];
          cur.osplit[o] = dom[nT + oc][idx.back()];
          val += op_cost(g, o, cur).elements;
        }
        f.table[e] = val;
      }
      ve.factors.push_back(std::move(f));
    }
    std::vector<std::vector<int>> sols;
    std::vector<int> order;
    ve.run(1, sols, order);
    PlanSeq p = cur;
    for (size_t t = 0; t < g.tensors.size(); ++t) p.tdims[t] = dom[g.tclass[t]][sols[0][g.tclass[t]]];
    for (size_t o = 0; o < g.ops.size(); ++o) p.osplit[o] = dom[nT + g.oclass[o]][sols[0][nT + g.oclass[o]]];
    r.seq = p;
  }
  OpCost c = plan_cost(g, r.seq);
  r.cost = c.elements;
  r.bytes = c.bytes;
  int64_t prev = 0;
  for (size_t i = 1; i <= r.seq.factors.size(); ++i) {
    PlanSeq pre;
    pre.factors.assign(r.seq.factors.begin(), r.seq.factors.begin() + i);
    for (auto& s : r.seq.tdims) pre.tdims.emplace_back(s.begin(), s.begin() + i);
    for (auto& s : r.seq.osplit) pre.osplit.emplace_back(s.begin(), s.begin() + i);
    int64_t ci = plan_cost(g, pre).elements;
    r.deltas.push_back(ci - prev);
    prev = ci;
  }
  r.search_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return r;
}

// Σ over op classes of the flat search's factor-table cells (product of the sequence-domain sizes of the
// class's tensor classes and its own): the size test of search = 2 (matches oracle.search.flat_cells).
static int64_t flat_cells(const Graph& g, const std::vector<int>& factors) {
  const int nT = (int)g.classes.size(), nO = (int)g.op_classes.size();
  const int m = (int)factors.size();
  std::vector<int64_t> dsize(nT + nO, 0);
  for (int c = 0; c < nT + nO; ++c) {
    bool is_t = c < nT;
    int rank = is_t ? (int)g.tensors[g.classes[c][0]].shape.size() : 0;
    std::vector<int> axes = is_t ? std::vector<int>() : g.def_of(g.op_classes[c - nT][0]).split_vars();
    if (is_t)
      for (int d = 0; d < rank; ++d) axes.push_back(d);
    if (is_t && rank == 0) {
      dsize[c] = 1;
      continue;
    }
    std::vector<int> seq(m, 0);
    std::function<void(int)> rec = [&](int i) {
      if (i == m) {
        const auto& members = is_t ? g.classes[c] : g.op_classes[c - nT];
        for (int x : members)
          for (int a : axes) {
            int64_t n = is_t ? g.tensors[x].shape[a] : g.ops[x].R[a];
            for (int st = 0; st < m; ++st)
              if (seq[st] == a) {
                if (n % factors[st]) return;
                n /= factors[st];
              }
          }
        ++dsize[c];
        return;
      }
      for (int a : axes) {
        seq[i] = a;
        rec(i + 1);
      }
    };
    rec(0);
  }
  int64_t tot = 0;
  for (int oc = 0; oc < nO; ++oc) {
    std::set<int> tcs;
    for (int o : g.op_classes[oc]) {
      for (int t : g.ops[o].inputs) tcs.insert(g.tclass[t]);
      tcs.insert(g.tclass[g.ops[o].output]);
    }
    int64_t n = dsize[nT + oc];
    for (int c : tcs) n = std::min<int64_t>(n * dsize[c], INT64_C(1) << 40);
    tot = std::min<int64_t>(tot + n, INT64_C(1) << 40);
  }
  return tot;
}

PlanResult make_plan(const Graph& g, int k, int frontier_cap, int solution_cap, int search) {
  if (search != 2) {
    PlanResult r = make_plan_mode(g, k, frontier_cap, solution_cap, search);
    r.search = search == 1 ? "flat" : "recursive";
    return r;
  }
  // auto (reading R4): the recursion; on graphs whose exact joint search is cheap, that search too,
  // keeping its plan only when strictly cheaper (the recursion is not always optimal under R3)
  auto t0 = std::chrono::steady_clock::now();
  PlanResult r = make_plan_mode(g, k, frontier_cap, solution_cap, 0);
  r.search = "recursive";
  if (k > 1 && flat_cells(g, factorize(k)) <= kFlatAutoCells) {
    PlanResult f = make_plan_mode(g, k, frontier_cap, solution_cap, 1);
    if (f.cost < r.cost) {
      f.truncated = r.truncated;
      r = f;
      r.search = "flat";
    }
  }
  r.search_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return r;
}

std::string plan_json(const Graph& g, const PlanResult& r) {
  std::string o = "{\"k\":" + std::to_string(r.k) + ",\"factors\":[";
  for (size_t i = 0; i < r.seq.factors.size(); ++i) o += (i ? "," : "") + std::to_string(r.seq.factors[i]);
  o += "],\"tdims\":{";
  for (size_t t = 0; t < g.tensors.size(); ++t) {
    o += (t ? "," : "") + json_quote(g.tensors[t].name) + ":[";
    for (size_t i = 0; i < r.seq.tdims[t].size(); ++i)
      o += (i ? "," : "") + (r.seq.tdims[t][i] < 0 ? std::string("null") : std::to_string(r.seq.tdims[t][i]));
    o += "]";
  }
  o += "},\"osplit\":{";
  for (size_t op = 0; op < g.ops.size(); ++op) {
    o += (op ? "," : "") + json_quote(g.ops[op].name) + ":[";
    for (size_t i = 0; i < r.seq.osplit[op].size(); ++i)
      o += (i ? "," : "") + json_quote(g.def_of((int)op).vars[r.seq.osplit[op][i]]);
    o += "]";
  }
  o += "},\"cost\":" + std::to_string(r.cost) + ",\"bytes\":" + std::to_string(r.bytes) + ",\"deltas\":[";
  for (size_t i = 0; i < r.deltas.size(); ++i) o += (i ? "," : "") + std::to_string(r.deltas[i]);
  o += "],\"frontier_truncated\":" + std::string(r.truncated ? "true" : "false") +
       ",\"search\":" + json_quote(r.search) + ",\"search_ms\":" + json_num(r.search_ms) + "}";
  return o;
}

}  // namespace tofu

struct tofu_plan {
  tofu::Graph g;
  tofu::PlanResult r;
};

namespace tofu {
const PlanResult& plan_of(const tofu_plan* p) { return p->r; }
}

extern "C" int tofu_plan_create(const tofu_graph* g, int k, const tofu_plan_options* opts, tofu_plan** out) {
  return tofu::guard([&]() {
    if (!g || !out || k < 1) throw tofu::Error(TOFU_ERR_ARG, "bad argument");
    int fc = 64, sc = 256, search = 2;
    if (opts) {
      if (opts->frontier_cap > 0) fc = opts->frontier_cap;
      if (opts->solution_cap > 0) sc = opts->solution_cap;
      search = opts->search;
    }
    auto* h = new tofu_plan{tofu::graph_of(g), tofu::make_plan(tofu::graph_of(g), k, fc, sc, search)};
    *out = h;
    return TOFU_OK;
  });
}
extern "C" void tofu_plan_destroy(tofu_plan* p) { delete p; }
extern "C" int tofu_plan_cost(const tofu_plan* p, int64_t* elements, int64_t* bytes) {
  if (!p) return tofu::fail(TOFU_ERR_ARG, "null plan");
  if (elements) *elements = p->r.cost;
  if (bytes) *bytes = p->r.bytes;
  return TOFU_OK;
}

extern "C" int tofu_plan_json(const tofu_plan* p, char* out, size_t cap, size_t* len) {
  return tofu::guard([&]() {
    if (!p) throw tofu::Error(TOFU_ERR_ARG, "null plan");
    return tofu::write_out(tofu::plan_json(p->g, p->r), out, cap, len);
  });
}
