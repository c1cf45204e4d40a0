// TDL parser + symbolic interval analysis for tofu_describe_op.
//   P:L380-409 §4.1 (tensor-as-a-lambda, reducers Sum/Max/Min/Prod, opaque functions P:L411-423)
//   P:L491-530 §4.2 (Eq. 1 symbolic intervals, Fig. int-arith; product/comparison of intervals rejected)
//   P:L532-561 §4.2 (Case-1: split an output var -> concat; Case-2: split a reduce var -> reduce)
//   Assumption #1: a var may index only one dim of each input tensor.
#include "tdl.h"

#include <algorithm>
#include <cctype>
#include <map>
#include <numeric>
#include <set>

#include "common.h"
#include "json.h"

namespace tofu {

namespace {

[[noreturn]] void perr(const std::string& kind, const std::string& msg) {
  throw Error(TOFU_ERR_PARSE, kind + ": " + msg);
}

struct Tok {
  int kind;  // 0 num, 1 id, 2 sym, 3 eof
  std::string s;
  size_t pos;
};

std::vector<Tok> lex(const std::string& src) {
  std::vector<Tok> t;
  size_t i = 0, n = src.size();
  while (true) {
    while (i < n && std::isspace((unsigned char)src[i])) ++i;
    if (i >= n) break;
    char c = src[i];
    size_t st = i;
    if (std::isdigit((unsigned char)c)) {
      while (i < n && std::isdigit((unsigned char)src[i])) ++i;
      if (i < n && src[i] == '.') {
        ++i;
        while (i < n && std::isdigit((unsigned char)src[i])) ++i;
      }
      t.push_back({0, src.substr(st, i - st), st});
    } else if (std::isalpha((unsigned char)c) || c == '_') {
      while (i < n && (std::isalnum((unsigned char)src[i]) || src[i] == '_')) ++i;
      t.push_back({1, src.substr(st, i - st), st});
    } else {
      static const char* two[] = {"->", ">=", "<=", "=="};
      bool done = false;
      for (auto s2 : two)
        if (src.compare(i, 2, s2) == 0) {
          t.push_back({2, s2, st});
          i += 2;
          done = true;
          break;
        }
      if (done) continue;
      if (std::string("-+*/%()[],:;<>").find(c) == std::string::npos)
        perr("Syntax", "bad character at " + std::to_string(i));
      t.push_back({2, std::string(1, c), st});
      ++i;
    }
  }
  t.push_back({3, "", n});
  return t;
}

const std::set<std::string> kReducers = {"Sum", "Max", "Min", "Prod"};
const std::map<std::string, int> kFuncs = {{"max", 2}, {"min", 2}, {"exp", 1}, {"tanh", 1},
                                            {"sigmoid", 1}, {"select", 3}, {"sqrt", 1}};

struct Parser {
  std::vector<Tok> t;
  size_t i = 0;
  OpDef d;
  std::map<std::string, int> var_ix;
  std::map<std::string, int> par_ix;

  const Tok& peek() { return t[i]; }
  Tok next() { return t[i++]; }
  bool accept(const std::string& s) {
    if (t[i].kind != 3 && t[i].s == s && t[i].kind != 0) {
      ++i;
      return true;
    }
    return false;
  }
  void expect(const std::string& s) {
    Tok k = next();
    if (k.s != s) perr("Syntax", "expected '" + s + "' at " + std::to_string(k.pos) + ", got '" + k.s + "'");
  }
  std::string ident() {
    Tok k = next();
    if (k.kind != 1) perr("Syntax", "expected identifier at " + std::to_string(k.pos));
    return k.s;
  }

  // index := term (('+'|'-') term)* ; term := int ['*' var] | var ['*' int] | [int '*'] '(' lin ')' ('/'|'%') int
  Affine affine(bool inner = false) {
    std::map<int, int64_t> co;
    int64_t c = 0;
    int64_t sign = 1;
    Affine a;
    if (accept("-")) sign = -1;
    else accept("+");
    while (true) {
      Tok k = next();
      int64_t mult = 0;
      if (k.kind == 0 && peek().s == "*" && i + 1 < t.size() && t[i + 1].s == "(") {
        if (k.s.find('.') != std::string::npos) perr("NonAffineIndex", "non-integer constant in index");
        mult = std::stoll(k.s);
        ++i;
        k = next();
      }
      if (k.kind == 2 && k.s == "(") {
        if (inner) perr("NonAffineIndex", "nested index division");
        Affine in = affine(true);
        expect(")");
        Tok op = next();
        if (op.s != "/" && op.s != "%") perr("NonAffineIndex", "parenthesised index term needs / or %");
        Tok dv = next();
        if (dv.kind != 0 || dv.s.find('.') != std::string::npos || std::stoll(dv.s) <= 0)
          perr("NonAffineIndex", "index division by a positive integer constant only");
        Affine::Term term;
        term.mod = op.s == "%";
        term.mult = sign * (mult ? mult : 1);
        term.d = std::stoll(dv.s);
        term.inner.coef = in.coef;
        term.inner.c = in.c;
        a.terms.push_back(term);
      } else if (mult) {
        perr("Syntax", "bad index term at " + std::to_string(k.pos));
      } else if (k.kind == 0) {
        if (k.s.find('.') != std::string::npos) perr("NonAffineIndex", "non-integer constant in index");
        int64_t n = std::stoll(k.s);
        if (accept("*")) {
          std::string v = ident();
          auto it = var_ix.find(v);
          if (it == var_ix.end()) perr("UnknownVar", v);
          co[it->second] += sign * n;
        } else {
          c += sign * n;
        }
      } else if (k.kind == 1) {
        auto it = var_ix.find(k.s);
        if (it == var_ix.end()) perr("UnknownVar", k.s);
        if (accept("*")) {
          Tok m = next();
          if (m.kind != 0) perr("NonAffineIndex", "product of index variables");
          co[it->second] += sign * std::stoll(m.s);
        } else {
          co[it->second] += sign;
        }
      } else {
        perr("Syntax", "bad index term at " + std::to_string(k.pos));
      }
      const std::string& nx = peek().s;
      if (nx == "+") { ++i; sign = 1; }
      else if (nx == "-") { ++i; sign = -1; }
      else if (inner ? nx == ")" : (nx == "," || nx == "]")) break;
      else if (nx == "*" || nx == "/" || nx == "%") perr("NonAffineIndex", "non-affine index expression");
      else perr("Syntax", "unexpected '" + nx + "' in index");
    }
    for (auto& kv : co)
      if (kv.second) a.coef.push_back(kv);
    a.c = c;
    return a;
  }

  Access access(const std::string& name, bool allow_slice) {
    auto it = par_ix.find(name);
    if (it == par_ix.end()) perr("UndeclaredTensor", name);
    expect("[");
    Access a;
    a.param = it->second;
    while (true) {
      if (allow_slice && peek().s == ":") {
        ++i;
        a.idx.push_back(Affine{});
        a.slice.push_back(1);
      } else {
        a.idx.push_back(affine());
        a.slice.push_back(0);
      }
      if (accept("]")) break;
      expect(",");
    }
    if ((int)a.idx.size() != d.ranks[a.param])
      perr("RankMismatch", name + " has rank " + std::to_string(d.ranks[a.param]) + ", indexed with " +
                               std::to_string(a.idx.size()));
    return a;
  }

  void primary() {
    Tok k = next();
    if (k.kind == 0) return;
    if (k.s == "(") {
      expr();
      expect(")");
      return;
    }
    if (k.s == "-") {
      primary();
      return;
    }
    if (k.kind == 1) {
      if (kReducers.count(k.s) || k.s == "reduce") perr("NestedReduce", "reduce only allowed at top level");
      if (peek().s == "[") {
        d.accesses.push_back(access(k.s, false));
        return;
      }
      if (peek().s == "(") {
        auto f = kFuncs.find(k.s);
        if (f == kFuncs.end()) perr("Syntax", "unknown function " + k.s);
        ++i;
        int n = 1;
        expr();
        while (accept(",")) {
          expr();
          ++n;
        }
        expect(")");
        if (n != f->second) perr("Syntax", k.s + " takes " + std::to_string(f->second) + " args");
        return;
      }
      if (var_ix.count(k.s)) return;
      if (par_ix.count(k.s)) perr("RankMismatch", "tensor " + k.s + " used without index");
      perr("UnknownVar", k.s);
    }
    perr("Syntax", "unexpected '" + k.s + "' at " + std::to_string(k.pos));
  }
  void term() {
    primary();
    while (peek().s == "*" || peek().s == "/") {
      ++i;
      primary();
    }
  }
  void arith() {
    term();
    while (peek().s == "+" || peek().s == "-") {
      ++i;
      term();
    }
  }
  void expr() {
    arith();
    const std::string& s = peek().s;
    if (s == ">" || s == "<" || s == ">=" || s == "<=" || s == "==") {
      ++i;
      arith();
    }
  }

  OpDef run() {
    if (ident() != "def") perr("Syntax", "expected 'def'");
    d.name = ident();
    expect("(");
    if (!accept(")")) {
      while (true) {
        std::string p = ident();
        expect("(");
        Tok r = next();
        if (r.kind != 0) perr("Syntax", "expected rank");
        expect(")");
        if (par_ix.count(p)) perr("Syntax", "duplicate parameter");
        par_ix[p] = (int)d.params.size();
        d.params.push_back(p);
        d.ranks.push_back(std::stoi(r.s));
        if (accept(")")) break;
        expect(",");
      }
    }
    expect("->");
    if (ident() != "lambda") perr("Syntax", "expected lambda");
    if (!accept(":")) {
      while (true) {
        std::string v = ident();
        var_ix[v] = (int)d.vars.size();
        d.vars.push_back(v);
        if (accept(":")) break;
        expect(",");
      }
    }
    d.n_out = (int)d.vars.size();
    if (peek().s == "reduce") {
      ++i;
      expect("(");
      d.reducer = ident();
      if (!kReducers.count(d.reducer)) perr("Syntax", "unknown reducer " + d.reducer);
      expect(";");
      while (true) {
        std::string v = ident();
        if (var_ix.count(v)) perr("Syntax", "reduce vars overlap output vars");
        var_ix[v] = (int)d.vars.size();
        d.vars.push_back(v);
        if (accept(";")) break;
        expect(",");
      }
      const size_t body0 = i;
      expr();
      const size_t body1 = i;
      expect(")");
      // contraction form: ID [ ... ] * ID [ ... ] at bracket depth 0 with nothing else
      if (d.reducer == "Sum" && d.accesses.size() == 2) {
        int depth = 0, stars = 0, others = 0;
        for (size_t q = body0; q < body1; ++q) {
          const std::string& x = t[q].s;
          if (x == "[") ++depth;
          else if (x == "]") --depth;
          else if (depth == 0 && t[q].kind == 2) {
            if (x == "*") ++stars;
            else ++others;
          } else if (depth == 0 && t[q].kind == 0) ++others;
        }
        d.prod2 = stars == 1 && others == 0 && t[body0].kind == 1 && d.accesses[0].param != d.accesses[1].param;
      }
    } else if (peek().s == "opaque") {
      ++i;
      expect("(");
      ident();
      expect(";");
      std::string tn = ident();
      Access a = access(tn, true);
      expect(")");
      expect("[");
      while (true) {
        ident();
        if (accept("]")) break;
        expect(",");
      }
      d.opaque = true;
      for (size_t k = 0; k < a.idx.size(); ++k)
        if (!a.slice[k] && a.idx[k].plain() && a.idx[k].coef.size() == 1 && a.idx[k].coef[0].second == 1 &&
            a.idx[k].c == 0)
          d.opaque_free.push_back(a.idx[k].coef[0].first);
      d.accesses.push_back(a);
    } else {
      expr();
    }
    if (peek().kind != 3) perr("Syntax", "trailing input at " + std::to_string(peek().pos));
    // validation: Assumption #1 and reduce vars must index something
    std::set<int> used;
    for (auto& a : d.accesses) {
      std::map<int, size_t> seen;
      for (size_t dim = 0; dim < a.idx.size(); ++dim) {
        if (a.slice[dim]) continue;
        for (int v : a.idx[dim].vars()) {
          used.insert(v);
          auto it = seen.find(v);
          if (it != seen.end() && it->second != dim)
            perr("AssumptionViolation", d.vars[v] + " indexes two dims of " + d.params[a.param]);
          seen[v] = dim;
        }
      }
    }
    for (int v = d.n_out; v < (int)d.vars.size(); ++v)
      if (!used.count(v)) perr("Syntax", "reduce var " + d.vars[v] + " indexes no input");
    // classification
    if (d.opaque) d.cls = "OpaqueBatched";
    else if (!d.reducer.empty()) d.cls = "Reduction";
    else {
      bool ew = !d.accesses.empty();
      for (auto& a : d.accesses) {
        if ((int)a.idx.size() != d.n_out) { ew = false; break; }
        for (int k = 0; k < d.n_out; ++k)
          if (!a.idx[k].identity_of(k)) ew = false;
      }
      d.cls = ew ? "ElementWise" : "General";
    }
    return d;
  }
};

// exact rationals for the symbolic analysis
struct Q {
  int64_t n = 0, d = 1;
  Q() = default;
  Q(int64_t a, int64_t b = 1) : n(a), d(b) { norm(); }
  void norm() {
    if (d < 0) { n = -n; d = -d; }
    int64_t g = std::gcd(n < 0 ? -n : n, d);
    if (g > 1) { n /= g; d /= g; }
  }
  Q operator+(const Q& o) const { return Q(n * o.d + o.n * d, d * o.d); }
  Q operator*(const Q& o) const { return Q(n * o.n, d * o.d); }
};
std::string qj(const Q& q) { return "[" + std::to_string(q.n) + "," + std::to_string(q.d) + "]"; }

}  // namespace

std::vector<int> OpDef::split_vars() const {
  if (opaque) return opaque_free;
  std::vector<int> v(vars.size());
  std::iota(v.begin(), v.end(), 0);
  return v;
}

OpDef parse_tdl(const std::string& src) {
  Parser p;
  p.t = lex(src);
  OpDef d = p.run();
  d.src = src;
  return d;
}

// Canonical token text of a def: the def's own name dropped, parameter names -> P<i>, index variables ->
// V<i> (output vars, then reduce vars), real-valued literals (with a '.') -> '#' with their values appended
// to `consts` in order of appearance; integer literals (ranks, gate indices, strides, 0 / 1) stay literal.
// Two defs with the same canonical text compute the same function of their operands up to the constants.
std::string canonical_def(const OpDef& d, std::vector<double>& consts) {
  consts.clear();
  std::map<std::string, int> par, var;
  for (size_t i = 0; i < d.params.size(); ++i) par[d.params[i]] = (int)i;
  for (size_t i = 0; i < d.vars.size(); ++i) var[d.vars[i]] = (int)i;
  std::vector<Tok> t = lex(d.src);
  std::string o;
  for (size_t i = 0; i < t.size(); ++i) {
    const Tok& x = t[i];
    if (x.kind == 3) break;
    if (i == 1 && x.kind == 1) continue;  // the def's name
    std::string w = x.s;
    if (x.kind == 1 && par.count(x.s)) w = "P" + std::to_string(par[x.s]);
    else if (x.kind == 1 && var.count(x.s)) w = "V" + std::to_string(var[x.s]);
    else if (x.kind == 0 && x.s.find('.') != std::string::npos) {
      consts.push_back(std::stod(x.s));
      w = "#";
    }
    o += (o.empty() ? "" : " ") + w;
  }
  return o;
}

int64_t Lin::eval(const int64_t* env) const {
  int64_t x = c;
  for (auto& kv : coef) x += kv.second * env[kv.first];
  return x;
}

int64_t Affine::eval(const int64_t* env) const {
  int64_t x = Lin::eval(env);
  for (auto& t : terms) {
    const int64_t in = t.inner.eval(env);
    x += t.mult * (t.mod ? floormod(in, t.d) : floordiv(in, t.d));
  }
  return x;
}

static void lin_hull(const Lin& l, const std::vector<Rng>& box, int64_t& lo, int64_t& hi) {
  lo = hi = l.c;
  for (auto& kv : l.coef) {
    const int64_t x = kv.second * box[kv.first].lo, y = kv.second * box[kv.first].hi;
    lo += std::min(x, y);
    hi += std::max(x, y);
  }
}

void Affine::hull(const std::vector<Rng>& box, int64_t off, int64_t& lo, int64_t& hi) const {
  lin_hull(*this, box, lo, hi);
  lo += off;
  hi += off;
  for (auto& t : terms) {
    int64_t il, ih, tl, th;
    lin_hull(t.inner, box, il, ih);
    if (!t.mod) {
      tl = floordiv(il, t.d);
      th = floordiv(ih, t.d);
    } else if (ih - il + 1 >= t.d || floordiv(il, t.d) != floordiv(ih, t.d)) {
      tl = 0;
      th = t.d - 1;
    } else {
      tl = floormod(il, t.d);
      th = floormod(ih, t.d);
    }
    lo += std::min(t.mult * tl, t.mult * th);
    hi += std::max(t.mult * tl, t.mult * th);
  }
}

std::vector<int> Affine::vars() const {
  std::vector<int> v;
  for (auto& kv : coef) v.push_back(kv.first);
  for (auto& t : terms)
    for (auto& kv : t.inner.coef)
      if (std::find(v.begin(), v.end(), kv.first) == v.end()) v.push_back(kv.first);
  return v;
}

std::vector<int64_t> var_extents(const OpDef& d, const std::vector<std::vector<int64_t>>& in_shapes,
                                 const std::vector<int64_t>& out_shape, const std::vector<int64_t>& given) {
  std::vector<int64_t> R(d.vars.size(), -1);
  for (int v = 0; v < d.n_out; ++v) R[v] = out_shape.at(v);
  for (int v = d.n_out; v < (int)d.vars.size(); ++v) {
    if (v < (int)given.size() && given[v] >= 0) {
      R[v] = given[v];
      continue;
    }
    for (auto& a : d.accesses) {
      for (size_t dim = 0; dim < a.idx.size() && R[v] < 0; ++dim)
        if (!a.slice[dim] && a.idx[dim].identity_of(v)) R[v] = in_shapes.at(a.param).at(dim);
      if (R[v] >= 0) break;
    }
    if (R[v] < 0) throw Error(TOFU_ERR_PARSE, "UnknownVar: cannot infer range of reduce var " + d.vars[v]);
  }
  return R;
}

std::string describe_json(const OpDef& d, int ways) {
  std::string o = "{\"name\":" + json_quote(d.name) + ",\"params\":[";
  for (size_t p = 0; p < d.params.size(); ++p)
    o += (p ? "," : "") + std::string("[") + json_quote(d.params[p]) + "," + std::to_string(d.ranks[p]) + "]";
  o += "],\"out_vars\":[";
  for (int v = 0; v < d.n_out; ++v) o += (v ? "," : "") + json_quote(d.vars[v]);
  o += "],\"red_vars\":[";
  for (int v = d.n_out; v < (int)d.vars.size(); ++v) o += (v > d.n_out ? "," : "") + json_quote(d.vars[v]);
  o += "],\"reducer\":" + (d.reducer.empty() ? std::string("null") : json_quote(d.reducer));
  o += ",\"class\":" + json_quote(d.cls) + ",\"split_vars\":[";
  auto sv = d.split_vars();
  for (size_t k = 0; k < sv.size(); ++k) o += (k ? "," : "") + json_quote(d.vars[sv[k]]);
  o += "],\"accesses\":[";
  for (size_t ai = 0; ai < d.accesses.size(); ++ai) {
    auto& a = d.accesses[ai];
    o += (ai ? "," : "") + std::string("{\"tensor\":") + json_quote(d.params[a.param]) + ",\"index\":[";
    for (size_t dim = 0; dim < a.idx.size(); ++dim) {
      o += dim ? "," : "";
      if (a.slice[dim]) { o += "null"; continue; }
      o += "{\"coef\":{";
      for (size_t k = 0; k < a.idx[dim].coef.size(); ++k)
        o += (k ? "," : "") + json_quote(d.vars[a.idx[dim].coef[k].first]) + ":" +
             std::to_string(a.idx[dim].coef[k].second);
      o += "},\"const\":" + std::to_string(a.idx[dim].c);
      if (!a.idx[dim].terms.empty()) {
        o += ",\"terms\":[";
        for (size_t q = 0; q < a.idx[dim].terms.size(); ++q) {
          const auto& tm = a.idx[dim].terms[q];
          o += (q ? "," : "") + std::string("{\"kind\":") + (tm.mod ? "\"mod\"" : "\"div\"") +
               ",\"mult\":" + std::to_string(tm.mult) + ",\"d\":" + std::to_string(tm.d) + ",\"coef\":{";
          for (size_t r = 0; r < tm.inner.coef.size(); ++r)
            o += (r ? "," : "") + json_quote(d.vars[tm.inner.coef[r].first]) + ":" +
                 std::to_string(tm.inner.coef[r].second);
          o += "},\"const\":" + std::to_string(tm.inner.c) + "}";
        }
        o += "]";
      }
      o += "}";
    }
    o += "]}";
  }
  o += "],\"strategies\":[";
  // Symbolic interval of each access dim for worker j: vars init ZV[l=j/s,u=(j+1)/s] (split var) or ZV[u=1].
  for (size_t k = 0; k < sv.size(); ++k) {
    int v = sv[k];
    o += (k ? "," : "") + std::string("{\"var\":") + json_quote(d.vars[v]) + ",\"kind\":" +
         (d.is_red(v) ? "\"Reduce\"" : "\"Concat\"") + ",\"regions\":[";
    for (int j = 0; j < ways; ++j) {
      o += (j ? "," : "") + std::string("[");
      for (size_t ai = 0; ai < d.accesses.size(); ++ai) {
        auto& a = d.accesses[ai];
        o += (ai ? "," : "") + std::string("{\"tensor\":") + json_quote(d.params[a.param]) + ",\"dims\":[";
        for (size_t dim = 0; dim < a.idx.size(); ++dim) {
          o += dim ? "," : "";
          if (a.slice[dim]) { o += "null"; continue; }
          // Fig. int-arith: each var's ZV interval times its (rational) coefficient, summed; a remainder
          // term contributes the constant interval [min(0, mult(d-1)), max(0, mult(d-1))] (reading R11)
          std::map<int, Q> lo, hi;
          Q clo(a.idx[dim].c), chi(a.idx[dim].c);
          auto add_lin = [&](const Lin& l, Q q) {
            for (auto& kv : l.coef) {
              Q co = Q(kv.second) * q;
              Q lv = kv.first == v ? Q(j, ways) : Q(0), uv = kv.first == v ? Q(j + 1, ways) : Q(1);
              const bool neg = co.n < 0;
              lo[kv.first] = lo[kv.first] + co * (neg ? uv : lv);
              hi[kv.first] = hi[kv.first] + co * (neg ? lv : uv);
            }
          };
          add_lin(a.idx[dim], Q(1));
          for (auto& tm : a.idx[dim].terms) {
            if (!tm.mod) {
              add_lin(tm.inner, Q(tm.mult, tm.d));
              clo = clo + Q(tm.inner.c) * Q(tm.mult, tm.d);
              chi = chi + Q(tm.inner.c) * Q(tm.mult, tm.d);
            } else {
              const int64_t e = tm.mult * (tm.d - 1);
              clo = clo + Q(std::min<int64_t>(0, e));
              chi = chi + Q(std::max<int64_t>(0, e));
            }
          }
          auto dump = [&](std::map<int, Q>& m) {
            std::string s = "{";
            bool first = true;
            for (auto& kv : m) {
              if (kv.second.n == 0) continue;
              s += (first ? "" : ",") + json_quote(d.vars[kv.first]) + ":" + qj(kv.second);
              first = false;
            }
            return s + "}";
          };
          auto qs = [](const Q& q) { return q.d == 1 ? std::to_string(q.n) : qj(q); };
          o += "{\"lo\":" + dump(lo) + ",\"c_lo\":" + qs(clo) + ",\"hi\":" + dump(hi) + ",\"c_hi\":" + qs(chi) + "}";
        }
        o += "]}";
      }
      o += "]";
    }
    o += "]}";
  }
  o += "]}";
  return o;
}

}  // namespace tofu

extern "C" int tofu_describe_op(const char* tdl, int ways, char* out, size_t cap, size_t* len) {
  return tofu::guard([&]() {
    if (!tdl || ways < 2) throw tofu::Error(TOFU_ERR_ARG, "tdl must be non-null and ways >= 2");
    tofu::OpDef d = tofu::parse_tdl(tdl);
    return tofu::write_out(tofu::describe_json(d, ways), out, cap, len);
  });
}
