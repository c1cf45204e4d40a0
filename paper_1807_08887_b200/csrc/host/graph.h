// Dataflow graph, coarsening (§5.1) and the direct-transfer cost model.
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "tdl.h"
#include "tofu.h"

namespace tofu {

struct TensorInfo {
  std::string name;
  std::vector<int64_t> shape;
  int dtype = TOFU_F32;
  std::string role;
  std::string merge;  // "" = none
};

struct OpInfo {
  std::string name;
  int def = 0;
  std::vector<int> inputs;  // tensor ids, one per def param
  int output = 0;
  std::string merge;
  std::map<std::string, double> attrs;
  std::vector<int64_t> R;  // extent of every def var
  // output views: constant offsets added to each input's access indices and to the
  // output index, so an op reads / writes a slice (e.g. one timestep) of a tensor
  std::vector<std::vector<int64_t>> in_off;  // [param][dim]
  std::vector<int64_t> out_off;              // [dim]
  bool has_offsets() const {
    for (auto& v : in_off)
      for (auto x : v)
        if (x) return true;
    for (auto x : out_off)
      if (x) return true;
    return false;
  }
};

struct Graph {
  std::vector<OpDef> defs;
  std::map<std::string, int> def_ix;
  std::vector<TensorInfo> tensors;
  std::map<std::string, int> tensor_ix;
  std::vector<OpInfo> ops;
  std::vector<std::pair<int, int>> alias;  // (new, old)
  // coarsening
  std::vector<int> tclass;                 // tensor -> class
  std::vector<std::vector<int>> classes;   // class -> tensors (sorted by name)
  std::vector<int> oclass;                 // op -> op class
  std::vector<std::vector<int>> op_classes;

  const OpDef& def_of(int op) const { return defs[ops[op].def]; }
  int64_t itemsize(int t) const { return tensors[t].dtype == TOFU_BF16 ? 2 : 4; }
};

Graph graph_from_json(const std::string& text);

// A (prefix of a) k-way plan: per tensor a dim per step (-1 for rank-0), per op a var per step.
struct PlanSeq {
  std::vector<int> factors;
  std::vector<std::vector<int>> tdims;  // [tensor][step]
  std::vector<std::vector<int>> osplit;  // [op][step]
};

// Closed range of the part selected by (k_i, digit_i) nested splits of an extent-n axis.
Rng nested_range(int64_t n, const std::vector<std::pair<int, int>>& splits);
std::vector<int> worker_digits(int w, const std::vector<int>& factors);

// Box of worker `dig` of a tensor (nullopt-like: empty vector + owned=false for non-owner of rank-0).
bool owned_box(const Graph& g, int t, const std::vector<int>& tdims, const std::vector<int>& factors,
               const std::vector<int>& dig, std::vector<Rng>& box);
void iter_box(const Graph& g, int op, const std::vector<int>& oseq, const std::vector<int>& factors,
              const std::vector<int>& dig, std::vector<Rng>& box);
// Required hull of every access of input param p over an iteration box (input offsets applied).
std::vector<Rng> required_box(const Graph& g, int op, int param, const std::vector<Rng>& ibox);
// Produced output box of an iteration box (output offset applied).
std::vector<Rng> produced_box(const Graph& g, int op, const std::vector<Rng>& ibox);

struct OpCost {
  int64_t elements = 0, bytes = 0, fetch = 0, out = 0;
};
OpCost op_cost(const Graph& g, int op, const PlanSeq& p);
OpCost plan_cost(const Graph& g, const PlanSeq& p);

}  // namespace tofu
