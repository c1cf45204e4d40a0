// TDL operator descriptions (§4.1) — host parser and access analysis.
#pragma once
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace tofu {

// Closed integer range [lo, hi] (empty when hi < lo).
struct Rng {
  int64_t lo, hi;
  int64_t len() const { return hi >= lo ? hi - lo + 1 : 0; }
};

// Σ coef[v]·var_v + c, integer coefficients.
struct Lin {
  std::vector<std::pair<int, int64_t>> coef;  // (var index, coefficient), sorted by var index, non-zero
  int64_t c = 0;
  int64_t eval(const int64_t* env) const;
};

// Index expression: Σ coef[v]·var_v + c (Eq. 1 admits affine intervals), plus quasi-affine
// terms mult·⌊inner / d⌋ and mult·(inner mod d) (reading R11: the I / k of Fig. int-arith, P:L510-522,
// taken as integer division of an index, and its remainder) used by strided-convolution gradients.
struct Affine : Lin {
  struct Term {
    bool mod = false;
    int64_t mult = 1, d = 1;
    Lin inner;
  };
  std::vector<Term> terms;
  bool identity_of(int v) const {
    return coef.size() == 1 && coef[0].first == v && coef[0].second == 1 && c == 0 && terms.empty();
  }
  bool plain() const { return terms.empty(); }
  int64_t eval(const int64_t* env) const;
  // closed range over a var box: the linear part exactly, each term bounded on its own
  void hull(const std::vector<Rng>& box, int64_t off, int64_t& lo, int64_t& hi) const;
  std::vector<int> vars() const;  // every var the index mentions
};

inline int64_t floordiv(int64_t a, int64_t d) { return a >= 0 ? a / d : -((-a + d - 1) / d); }
inline int64_t floormod(int64_t a, int64_t d) { return a - d * floordiv(a, d); }

struct Access {
  int param = 0;                 // index into OpDef::params
  std::vector<Affine> idx;       // one per dim
  std::vector<char> slice;       // ':' inside an opaque call (whole dim)
};

struct OpDef {
  std::string name;
  std::vector<std::string> params;
  std::vector<int> ranks;
  std::vector<std::string> vars;  // output vars, then reduce vars
  int n_out = 0;
  std::string reducer;            // "" if none
  bool opaque = false;
  std::vector<int> opaque_free;   // pass-through batch vars of an opaque op
  std::vector<Access> accesses;
  std::string cls;                // ElementWise | Reduction | OpaqueBatched | General
  bool prod2 = false;             // body is exactly `reduce(Sum; ..; A[..] * B[..])` (a contraction)
  std::string src;                // the def's TDL text
  std::string kernel;             // element-wise / cell / window kernel whose canonical TDL this def matches, or ""
  std::vector<double> kconst;     // that kernel's constants, read from the def's text (in order of appearance)

  int n_red() const { return (int)vars.size() - n_out; }
  bool is_red(int v) const { return v >= n_out; }
  std::vector<int> split_vars() const;  // Case-1 output vars + Case-2 reduce vars
};

// Throws Error(TOFU_ERR_PARSE, "<Kind>: message").
OpDef parse_tdl(const std::string& src);

// Canonical text of a def (names -> positions, real literals -> '#' collected in consts); see tdl.cpp.
std::string canonical_def(const OpDef& d, std::vector<double>& consts);

// Bind d to the element-wise / cell / window kernel whose canonical TDL it matches (kernel_match.cpp):
// sets d.kernel ("" when none) and d.kconst.
void match_kernel(OpDef& d);

// Extent of every var given input and output shapes (reduce vars from the first dim they index alone).
// `given` (may be empty) holds explicit extents (-1 = infer) for vars no dim determines.
std::vector<int64_t> var_extents(const OpDef& d, const std::vector<std::vector<int64_t>>& in_shapes,
                                 const std::vector<int64_t>& out_shape, const std::vector<int64_t>& given = {});

// JSON analysis for tofu_describe_op.
std::string describe_json(const OpDef& d, int ways);

}  // namespace tofu
