// Plan types and plan_from_placement — proj/include/helio/placement.hpp:47-83.
// (The MILP planner itself stays out of scope.)
#pragma once

#include <string>
#include <vector>

#include "helio/flow_graph.hpp"

namespace helio {

enum class MilpStatus { kOptimal, kFeasible, kInfeasible, kUnbounded, kNoIncumbent };

struct PlanEdge {
  std::string src, dst;
  double flow = 0;
  int exec_start = 0, exec_end = 0;
};

struct PlacementPlan {
  std::string method;
  Placement placement;
  std::vector<PlanEdge> edges;  // positive-flow edges only
  double objective = 0;
  bool allow_partial = true;
  MilpStatus status = MilpStatus::kOptimal;
  double best_bound = 0;
  long nodes_explored = 0;
  long nodes_to_best = 0;
  std::vector<std::string> warnings;
};

PlacementPlan plan_from_placement(const ClusterSpec& c, const Placement& p, bool allow_partial,
                                  const std::string& method);

}  // namespace helio
