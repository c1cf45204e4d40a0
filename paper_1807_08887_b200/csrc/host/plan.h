// Plan result shared by plan.cpp (search) and exec.cpp (lowering).
#pragma once
#include <string>
#include <vector>

#include "graph.h"

struct tofu_graph;
struct tofu_plan;

namespace tofu {

struct PlanResult {
  int k = 1;
  PlanSeq seq;
  int64_t cost = 0, bytes = 0;
  std::vector<int64_t> deltas;
  bool truncated = false;
  double search_ms = 0;
  std::string search = "recursive";   // the search that produced seq: "recursive" | "flat"
};

constexpr int64_t kFlatAutoCells = INT64_C(1) << 20;   // search = 2: flat search when flat_cells <= this

PlanResult make_plan(const Graph& g, int k, int frontier_cap, int solution_cap, int search);
std::string plan_json(const Graph& g, const PlanResult& r);
const PlanResult& plan_of(const tofu_plan* p);
const Graph& graph_of(const tofu_graph* h);

}  // namespace tofu
